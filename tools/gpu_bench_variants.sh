mkdir -p gpurun_out
for w in C1 C2 C3 C4 C5; do
  for v in 1 2; do
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant $v > gpurun_out/var_${w}_$v.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/var_${w}_$v.log').read().strip().splitlines()[-1]); print('$w v$v', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4), 'end_ms', round(d['end_slice_ms'],4))" 2>&1 | tail -1
  done
done
