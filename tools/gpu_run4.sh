mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -k "not full_size and not c2_all" > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu4.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/bench4.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench4.log
