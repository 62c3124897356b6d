mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -k "large_atv or c1_all" > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu7.log
timeout 600 python bench.py --workload PAPER --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_paper.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench_paper.log | cut -c1-1500
