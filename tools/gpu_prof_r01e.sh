mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
$CMD > gpurun_out/prof_plain_e.log 2>&1 && echo plain-ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01e.csv $CMD > gpurun_out/ncu_launch_e.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_fold|k_restore|k_nat_est" -s 4 -c 4 -o gpurun_out/prof_r01e $CMD > gpurun_out/ncu_full_e.log 2>&1; echo "full rc=$?"
tail -2 gpurun_out/ncu_full_e.log
