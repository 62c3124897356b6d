mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_features.py -q -x --timeout=900 > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu10.log
