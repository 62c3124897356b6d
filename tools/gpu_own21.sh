mkdir -p gpurun_out
ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | grep "^k_scan_own" | tail -1
