mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --maxfail=6 --durations=15 > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
tail -60 gpurun_out/pytest_gpu2.log
