mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --distinct 2 --scan-variant 2"
$CMD > gpurun_out/profbin18_plain.log 2>&1 && echo plain-ok && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_bin" -s 1 -c 1 -o gpurun_out/prof_bin18 $CMD > gpurun_out/ncu_bin18.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_bin18.log
