# sweep k_scan_own build variants (tools/variants/libasse_*.so) and tiles on C5
mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
one() {  # name tile workload
  cp tools/variants/libasse_$1.so $L
  if [ "$2" = "-" ]; then unset ASSE_SCAN_TILE; else export ASSE_SCAN_TILE=$2; fi
  timeout 300 python bench.py --workload $3 --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 3 > gpurun_out/sw_$1_$2_$3.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2_$3.log').read().strip().splitlines()[-1]); print('$1 tile=$2 $3', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1
}
for v in b16c8u2 b16c10u2 b16c8u4 b16c12u2 b12c8u2; do one $v - C5; done
for t in 1536 2304; do one b12c12u2 $t C5; one b12c8u2 $t C5; done
for t in 1792 2560; do one b16c8u2 $t C5; one b16c10u2 $t C5; done
for w in C3 C4; do one b16c8u2 - $w; one b16c10u2 - $w; done
cp /tmp/libasse_orig.so $L
