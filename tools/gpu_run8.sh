mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -q -x --timeout=600 -k "c1_all or c2_all or features or overflow or edge or state" > gpurun_out/pytest_gpu9.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu9.log
for w in C1 C2; do timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu > gpurun_out/benchall_$w.log 2>&1; echo "$w rc=$?"; done
