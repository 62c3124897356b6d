mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
one() {
  cp tools/variants/libasse_$1.so $L
  timeout 300 python bench.py --workload $2 --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 3 > gpurun_out/sw_$1_$2.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2.log').read().strip().splitlines()[-1]); print('$1 $2', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1
}
for r in 1 2; do for v in def c4 b12 c4nb4 nb4; do one $v C5; done; done
cp /tmp/libasse_orig.so $L
