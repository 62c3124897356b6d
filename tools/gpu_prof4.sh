mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
$CMD > gpurun_out/prof_plain4.log 2>&1 && echo plain-ok && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fold" -s 2 -c 1 -o gpurun_out/prof_fold4 $CMD > gpurun_out/ncu_fold4.log 2>&1; echo "full rc=$?"
