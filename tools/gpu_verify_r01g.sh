mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/g_smoke.log
timeout 600 python bench.py > gpurun_out/g_bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/g_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g_ref.log 2>&1; echo "ref rc=$?"; tail -c 800 gpurun_out/g_ref.log
