mkdir -p gpurun_out
for w in C1 C2 C3 C4 C5 PAPER; do
  timeout 900 python bench.py --workload $w --steps 30 --warmup 5 > gpurun_out/benchall_$w.log 2>&1; echo "$w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.log
