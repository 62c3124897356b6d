mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan_own.py -x -q --timeout=300 > gpurun_out/own7_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/own7_pytest.log
ASSE_SCAN_OWN_GENERIC=1 timeout 900 python -m pytest tests/test_gpu_scan_own.py -x -q --timeout=300 -k "C3 or ragged or mod_p" > gpurun_out/own7g_pytest.log 2>&1; echo "pytest generic rc=$?"; tail -2 gpurun_out/own7g_pytest.log
for w in C5 C3 C4; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/o7_$w.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/o7_$w.log').read().strip().splitlines()[-1]); print('$w', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4), d['roofline']['kernel'])" 2>&1 | tail -1
done
ASSE_SCAN_OWN_GENERIC=1 timeout 300 python bench.py --workload C5 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/o7g_C5.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/o7g_C5.log').read().strip().splitlines()[-1]); print('C5 generic', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))"
ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | grep "^k_scan_own" | tail -1
