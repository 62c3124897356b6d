mkdir -p gpurun_out
timeout 600 cuda-gdb -batch -ex run -ex bt --args python -m pytest tests/test_gpu_multi.py -x -q -k "C1" > gpurun_out/gdb.log 2>&1
tail -40 gpurun_out/gdb.log
