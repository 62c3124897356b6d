python tools/sweep.py run --variants r1,acq0,free --workloads C5,C3,C4 --reps 2 --tag r02g 2>&1 | tail -18
timeout 600 python -m pytest tests/test_gpu_scan_own.py -q -x > gpurun_out/r02g_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02g_pytest.log
