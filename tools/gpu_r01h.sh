mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/h_pytest.log
for w in C5 C3 C4; do
  for v in 3 2; do
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant $v > gpurun_out/h_${w}_$v.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/h_${w}_$v.log').read().strip().splitlines()[-1]); print('$w v$v', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4), 'end_ms', round(d['end_slice_ms'],4))" 2>&1 | tail -1
  done
done
