mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
ASSE_SCAN_PROF=1 $CMD 2>&1 | grep "^k_scan_own" | tail -1
$CMD > gpurun_out/prof_plain_g.log 2>&1 && echo plain-ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01g.csv $CMD > gpurun_out/ncu_launch_g.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan_own|k_fold|k_restore" -s 3 -c 3 -o gpurun_out/prof_r01g $CMD > gpurun_out/ncu_full_g.log 2>&1; echo "full rc=$?"
tail -2 gpurun_out/ncu_full_g.log
