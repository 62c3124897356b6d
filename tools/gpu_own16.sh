mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan_own.py -x -q --timeout=300 > gpurun_out/own16_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/own16_pytest.log
for r in 1 2; do
timeout 300 python bench.py --workload C5 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/o16_C5.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/o16_C5.log').read().strip().splitlines()[-1]); print('C5', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))"
done
ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | grep "^k_scan_own" | tail -1
timeout 300 python bench.py --workload C5 --steps 10 --warmup 3 --no-cpu > gpurun_out/o16_e2e.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/o16_e2e.log').read().strip().splitlines()[-1]); print('C5 e2e', d['e2e'])"
