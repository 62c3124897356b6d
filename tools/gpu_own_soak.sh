mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan_own.py -x -q --timeout=600 -k many_slices > gpurun_out/own_soak.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/own_soak.log
