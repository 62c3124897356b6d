mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --maxfail=8 --timeout=600 --durations=20 -k "not full_size and not multi and not c2_all" > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"
tail -80 gpurun_out/pytest_gpu3.log
