mkdir -p gpurun_out
for w in C5 C4 C3 PAPER; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -k "large_atv or backbone or long_run or window" > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu8.log
