mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 > gpurun_out/rest1_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rest1_pytest.log
for w in C5 C3 C4 C2; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/rest1_$w.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/rest1_$w.log').read().strip().splitlines()[-1]); print('$w', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4), 'end', round(d['end_slice_ms'],4), d['end_slice_breakdown_ms'])" 2>&1 | tail -1
done
