mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/full_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/full_pytest.log
timeout 600 python bench.py > gpurun_out/full_bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/full_bench.log
