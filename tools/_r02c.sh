python tools/sweep.py run --variants acq0,acq1,acq1rel1,chk --workloads C5,C3 --reps 2 --tag r02c 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_window.py -q -x --durations=5 -k "c4_shape or c5" > gpurun_out/r02c_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r02c_pytest.log
