for rep in 1 2; do for nx in 0 1; do for w in C5 C3 C4; do
  if [ $nx = 0 ]; then export ASSE_SCAN_NO_NX=1; else unset ASSE_SCAN_NO_NX; fi
  python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > /tmp/b.log 2>&1; python -c "import json;l=[x for x in open('/tmp/b.log') if x.startswith('{')][-1];d=json.loads(l);print('nx $nx $w', round(d['roofline']['avg_launch_ms'],4), round(d['value'],2))" || tail -3 /tmp/b.log
done; done; done
unset ASSE_SCAN_NO_NX
timeout 900 python -m pytest tests/test_gpu_scan_own.py tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
