mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -k "mod_p or keys or c1_all or full_size" > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu11.log
