python tools/sweep.py run --variants r1,acq0,sig,sigrr1 --workloads C5,C3,C4 --reps 2 --tag r02e 2>&1 | tail -24
ASSE_LIB=tools/variants/libasse_sigrr1.so timeout 600 python -m pytest tests/test_gpu_scan_own.py -q -x > gpurun_out/r02e_rr1.log 2>&1; echo "rr1 pytest rc=$?"; tail -2 gpurun_out/r02e_rr1.log
timeout 600 python -m pytest tests/test_gpu_scan_own.py tests/test_gpu_scan_bin.py -q -x > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02e_pytest.log
