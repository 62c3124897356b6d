# timing upper bounds (variants nocopy/nores give wrong results by construction)
mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
for v in base nocopy nores both; do
  cp tools/variants/libasse_$v.so $L
  ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu --scan-variant 3 > gpurun_out/x_$v.log 2>&1
  grep "^k_scan_own" gpurun_out/x_$v.log | tail -1 | cut -c1-330
  python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/x_$v.log').read().splitlines() if l.startswith('{')][-1]); print('$v', 'scan_ms', round(d['roofline']['avg_launch_ms'],4))"
done
cp /tmp/libasse_orig.so $L
