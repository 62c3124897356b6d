mkdir -p gpurun_out
ASSE_SCAN_PROF=1 timeout 300 python bench.py --steps 4 --warmup 1 --no-e2e --no-cpu --scan-variant 2 > gpurun_out/bin3_bench2.log 2>&1; echo "bench2 rc=$?"; grep k_scan_bin gpurun_out/bin3_bench2.log | tail -3
