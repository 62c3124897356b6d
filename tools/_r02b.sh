set -x
timeout 1500 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_window.py tests/test_gpu_features.py tests/test_gpu_scan_own.py -q -x --durations=25 > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
python bench.py --no-cpu --no-e2e > gpurun_out/r02b_bench.log 2>&1
tail -3 gpurun_out/r02b_pytest.log
