mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
$CMD > gpurun_out/prof_plain3.log 2>&1 && echo plain-ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01c.csv $CMD > gpurun_out/ncu_launch3.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_fold|k_restore|k_nat_est|k_rank_sort|k_sort_small" -s 6 -c 6 -o gpurun_out/prof_r01c $CMD > gpurun_out/ncu_full3.log 2>&1; echo "full rc=$?"
