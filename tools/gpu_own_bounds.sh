# k_scan_own parity tests with device bounds asserts (ASSE_OWN_DEBUG_BOUNDS=1); compute-sanitizer
# is not available on the GPU pool
mkdir -p gpurun_out
L=paper_1807_01527_b200/libasse.so
cp $L /tmp/libasse_orig.so
cp tools/variants/libasse_bounds.so $L
timeout 1200 python -m pytest tests/test_gpu_scan_own.py tests/test_gpu_multi.py -x -q --timeout=600 -k "owned or packet_owned" > gpurun_out/own_bounds.log 2>&1; echo "pytest(bounds) rc=$?"; tail -2 gpurun_out/own_bounds.log
timeout 300 python tools/sanitize_run.py > gpurun_out/own_bounds_san.log 2>&1; echo "sanitize_run(bounds) rc=$?"; tail -1 gpurun_out/own_bounds_san.log
cp /tmp/libasse_orig.so $L
