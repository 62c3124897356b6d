python tools/sweep.py run --variants r1,acq0,acq2,relax --workloads C5,C3 --reps 2 --tag r02d 2>&1 | tail -20
timeout 600 python -m pytest tests/test_gpu_scan_own.py tests/test_gpu_features.py -q -x > gpurun_out/r02d_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02d_pytest.log
python bench.py --no-cpu > gpurun_out/r02d_bench.log 2>&1; tail -c 600 gpurun_out/r02d_bench.log
