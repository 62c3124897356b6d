mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
one() {  # name tile workload
  cp tools/variants/libasse_$1.so $L
  if [ "$2" = "-" ]; then unset ASSE_SCAN_TILE; else export ASSE_SCAN_TILE=$2; fi
  timeout 300 python bench.py --workload $3 --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 3 > gpurun_out/sw_$1_$2_$3.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2_$3.log').read().strip().splitlines()[-1]); print('$1 tile=$2 $3', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1
}
for r in 1 2; do one def - C5; one b20x2 2560 C5; one b20x1 2560 C5; one b18x2 2304 C5; one b20x2 - C5; done
unset ASSE_SCAN_TILE
cp /tmp/libasse_orig.so $L
