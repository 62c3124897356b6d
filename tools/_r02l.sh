python tools/sweep.py run --variants nofree_r,nofree0,fw2,fw2r --workloads C5,C3,C4 --reps 2 --tag r02l 2>&1 | tail -24
timeout 900 python -m pytest tests/test_gpu_scan_own.py tests/test_gpu_multi.py -q -x > gpurun_out/r02l_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02l_pytest.log
