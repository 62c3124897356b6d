mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/p_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/p_smoke.log
for w in C5 C1 C2 C3 C4 PAPER; do
  timeout 900 python bench.py --workload $w --steps 30 --warmup 5 > gpurun_out/benchall_p_$w.log 2>&1; echo "$w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_p.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
$CMD > gpurun_out/prof_plain_p.log 2>&1 && echo plain-ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01p.csv $CMD > gpurun_out/ncu_launch_p.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan_own|k_fold|k_restore" -s 3 -c 3 -o gpurun_out/prof_r01p $CMD > gpurun_out/ncu_full_p.log 2>&1; echo "full rc=$?"
