mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin_smoke.log
timeout 600 python bench.py > gpurun_out/fin_bench.log 2>&1; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/fin_bench.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'], d['e2e']['value'], d['e2e']['frac_of_h2d'], d['clocks'], d['gpu_launches'])"
timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.log 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/fin_ref.log
