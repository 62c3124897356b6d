mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_features.py tests/test_gpu_parity.py -q -x --timeout=600 -k "features or c1_all or edge or window or long_run or overflow" > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu6.log
