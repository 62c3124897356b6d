mkdir -p gpurun_out
timeout 300 python tools/sanitize_run.py > gpurun_out/san_plain_own.log 2>&1 && echo plain-ok; tail -2 gpurun_out/san_plain_own.log
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/memcheck_r01l.log 2>&1; echo "memcheck rc=$?"
tail -6 gpurun_out/memcheck_r01l.log
