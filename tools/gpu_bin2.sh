mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_scan_bin.py -x -q --timeout=280 > gpurun_out/bin15_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/bin15_pytest.log
timeout 100 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --scan-variant 2 > gpurun_out/bin15_bench2.log 2>&1; echo "bench2 rc=$?"; python - <<'P'
import json
for f in ["gpurun_out/bin15_bench2.log"]:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, "value", d["value"], "scan ms", d["roofline"]["avg_launch_ms"], "end", d["end_slice_ms"])
P
ASSE_SCAN_PROF=1 timeout 100 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --scan-variant 2 2>&1 | grep k_scan_bin | tail -1
