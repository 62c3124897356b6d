set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "keys or c1_all or edge or order or overflow or state or window or generator" > gpurun_out/pytest_gpu1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu1.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench1.log
