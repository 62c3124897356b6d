mkdir -p gpurun_out
python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1 && echo plain-ok && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/memcheck_r01.log 2>&1; echo "memcheck rc=$?"
tail -15 gpurun_out/memcheck_r01.log
