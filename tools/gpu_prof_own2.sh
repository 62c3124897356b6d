mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --distinct 4"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan_own" -s 1 -c 1 -o gpurun_out/prof_r01i $CMD > gpurun_out/ncu_full_i.log 2>&1; echo "full rc=$?"
