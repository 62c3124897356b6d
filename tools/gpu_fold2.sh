mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
one() {
  cp tools/variants/libasse_$1.so $L
  timeout 300 python bench.py --workload $2 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/sw_$1_$2.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2.log').read().strip().splitlines()[-1]); print('$1 $2', round(d['value'],2), 'Gpps fold_ms', round(d['kernels']['k_fold']['avg_launch_ms'],4), 'frac', round(d['kernels']['k_fold']['frac'],3))" 2>&1 | tail -1
}
for r in 1 2; do for v in u2 u1; do one $v C4; done; done
cp tools/variants/libasse_u1.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py -k C4 -x -q --timeout=300 > gpurun_out/fold1_pytest.log 2>&1; echo "pytest(u1) rc=$?"; tail -1 gpurun_out/fold1_pytest.log
cp /tmp/libasse_orig.so $L
