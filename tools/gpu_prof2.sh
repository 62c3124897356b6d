mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
$CMD > gpurun_out/prof_plain2.log 2>&1 && echo plain-ok && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_launch2.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_fold|k_restore|k_nat_est" -s 4 -c 4 -o gpurun_out/prof_r01b $CMD > gpurun_out/ncu_full2.log 2>&1; echo "full rc=$?"
timeout 900 python bench.py --steps 40 --warmup 5 > gpurun_out/bench5.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench5.log
./tools/l2bench > gpurun_out/l2bench_r01.txt 2>&1
