mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scan_own.py -x -q --timeout=300 > gpurun_out/own1_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/own1_pytest.log
for v in 3 2; do
  timeout 300 python bench.py --workload C5 --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant $v > gpurun_out/own1_C5_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/own1_C5_$v.log').read().strip().splitlines()[-1]); print('C5 v$v', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4), 'end_ms', round(d['end_slice_ms'],4))" 2>&1 | tail -1
done
ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu --scan-variant 3 2>&1 | grep "k_scan_own" | tail -2
ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu --scan-variant 2 2>&1 | grep "k_scan_bin" | tail -2
