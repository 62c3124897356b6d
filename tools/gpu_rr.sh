for rr in 2 1 0; do
  export ASSE_SCAN_RR=$rr
  echo "RR=$rr dbg ok: $(python tools/dbg_bin.py 2>&1 | grep -c 'rc 0')/12"
  timeout 100 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('RR=$rr', d['value'], d['roofline']['avg_launch_ms'])"
  ASSE_SCAN_PROF=1 timeout 100 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --scan-variant 2 2>&1 | grep "k_scan_bin n=100000000" | tail -1 | sed "s/- 0\/0; //g"
done
unset ASSE_SCAN_RR
timeout 300 python -m pytest tests/test_gpu_scan_bin.py -x -q 2>&1 | tail -2
