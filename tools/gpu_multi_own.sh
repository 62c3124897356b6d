mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q --timeout=600 -k packet_owned > gpurun_out/multi_own.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/multi_own.log
