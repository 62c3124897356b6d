for w in C3 C4 C2; do for rr in 0 1 2; do
  ASSE_SCAN_RR=$rr timeout 200 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w RR=$rr', round(d['value'],2), 'scan', round(d['roofline']['avg_launch_ms'],4), d['roofline']['kernel'])"
done; done
