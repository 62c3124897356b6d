mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_scan_bin.py -x -q --timeout=280 -k "C1 or C3" > gpurun_out/bin1_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/bin1_pytest.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 2 > gpurun_out/bin1_bench2.log 2>&1; echo "bench2 rc=$?"; tail -c 1500 gpurun_out/bin1_bench2.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 1 > gpurun_out/bin1_bench1.log 2>&1; echo "bench1 rc=$?"; tail -c 600 gpurun_out/bin1_bench1.log
