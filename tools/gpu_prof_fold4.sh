mkdir -p gpurun_out
CMD="python bench.py --workload C4 --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
$CMD > gpurun_out/pf4_plain.log 2>&1 && echo plain-ok && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fold" -s 3 -c 1 -o gpurun_out/prof_fold4 $CMD > gpurun_out/ncu_fold4.log 2>&1; echo "ncu rc=$?"
