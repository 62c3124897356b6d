mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scan_own.py -x -q --timeout=300 > gpurun_out/own6_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/own6_pytest.log
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
one() {  # name tile workload
  cp tools/variants/libasse_$1.so $L
  if [ "$2" = "-" ]; then unset ASSE_SCAN_TILE; else export ASSE_SCAN_TILE=$2; fi
  timeout 300 python bench.py --workload $3 --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 3 > gpurun_out/sw_$1_$2_$3.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2_$3.log').read().strip().splitlines()[-1]); print('$1 tile=$2 $3', round(d['value'],2), 'Gpps scan_ms', round(d['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1
}
for v in r4 r8 r12 r16; do one $v - C5; done
for v in r4 r8 r12 r16; do one $v - C3; done
cp /tmp/libasse_orig.so $L
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k_scan_own -c 2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --distinct 2 > gpurun_out/ncu_dram_r8.log 2>&1; grep -E "dram__|duration|hit_rate" gpurun_out/ncu_dram_r8.log | tail -4
