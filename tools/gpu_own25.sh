mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
cp tools/variants/libasse_offwait.so $L
ASSE_SCAN_PROF=1 timeout 300 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | grep "^k_scan_own" | tail -1 | cut -c1-300
cp /tmp/libasse_orig.so $L
