mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
for v in def nowait; do
  cp tools/variants/libasse_$v.so $L
  ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | grep "^k_scan_own" | tail -1 | cut -c1-330
  timeout 300 python bench.py --workload C5 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/sw_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))"
done
cp /tmp/libasse_orig.so $L
