mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/check_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/check_pytest.log
python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1 && echo plain-ok && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/memcheck_r01c.log 2>&1; echo "memcheck rc=$?"
tail -6 gpurun_out/memcheck_r01c.log
