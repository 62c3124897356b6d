mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 --durations=12 > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"
tail -22 gpurun_out/pytest_gpu5.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench6.log 2>&1; echo "bench rc=$?"
