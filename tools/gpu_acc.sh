mkdir -p gpurun_out
free -g | head -2
ASSE_ACCURACY_OUT=gpurun_out/accuracy_r01.json timeout 1500 python -m pytest tests/test_gpu_accuracy.py -q -x --timeout=1200 --durations=5 > gpurun_out/pytest_acc.log 2>&1; echo "rc=$?"
tail -12 gpurun_out/pytest_acc.log
