#!/bin/bash
# The standard measurement run on the GPU box (one gpurun call):
#   gpurun -- 'bash tools/gpu_measure.sh r02a [quick]'
# pytest -m gpu, smoke, bench on every workload, the reference arm, and the ncu evidence:
# a launch list of the default bench and one --set full capture of the hot kernels, each
# only after the same command exited 0 without ncu. Outputs land in gpurun_out/<tag>_*;
# tools/ncu_summary.py turns them into profiles/<tag>_* here.
TAG=${1:?tag}; MODE=${2:-full}
mkdir -p gpurun_out
O=gpurun_out/$TAG
if [ "$MODE" != "quick" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --durations=30 > ${O}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 ${O}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 ${O}_smoke.log
fi
for w in C5 C1 C2 C3 C4 PAPER; do
  timeout 900 python bench.py --workload $w --steps 30 --warmup 5 --slice-log ${O}_slices_$w.jsonl > ${O}_bench_$w.log 2>&1; echo "$w rc=$?"
done
if [ "$MODE" != "quick" ]; then
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > ${O}_bench_ref.log 2>&1; echo "ref rc=$?"
fi
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
$CMD > ${O}_prof_plain.log 2>&1 && echo plain-ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv $CMD > ${O}_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan_own|k_fold|k_restore" -s 3 -c 3 -o ${O}_prof $CMD > ${O}_ncu_full.log 2>&1; echo "full rc=$?"
