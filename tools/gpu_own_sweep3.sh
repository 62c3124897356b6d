mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
cp tools/variants/libasse_s1.so $L
timeout 600 python -m pytest tests/test_gpu_scan_own.py -x -q --timeout=300 > gpurun_out/own4_pytest.log 2>&1; echo "pytest(s1) rc=$?"; tail -2 gpurun_out/own4_pytest.log
one() {  # name tile workload
  cp tools/variants/libasse_$1.so $L
  if [ "$2" = "-" ]; then unset ASSE_SCAN_TILE; else export ASSE_SCAN_TILE=$2; fi
  timeout 300 python bench.py --workload $3 --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 3 > gpurun_out/sw_$1_$2_$3.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2_$3.log').read().strip().splitlines()[-1]); print('$1 tile=$2 $3', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1
}
for rep in 1 2; do for v in e2 s0 s1 s1p3 s1p8; do one $v - C5; done; done
for v in s0 s1 s1p3; do one $v - C3; one $v - C4; done
cp /tmp/libasse_orig.so $L
