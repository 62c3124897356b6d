set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x --durations=40 > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_pytest.log
python bench.py > gpurun_out/r02a_bench.log 2>&1
tail -3 gpurun_out/r02a_pytest.log
