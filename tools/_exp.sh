python tools/sweep.py run --variants cur,ng2,ng4 --workloads C5,C3,C4 --reps 2 --tag r02o 2>&1 | tail -18
ASSE_LIB=tools/variants/libasse_ng2.so timeout 600 python -m pytest tests/test_gpu_scan_own.py -q -x 2>&1 | tail -2
