mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/val_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/val_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/val_pytest.log
timeout 600 python bench.py > gpurun_out/val_bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/val_bench.log
