for w in gsweep c4 c5 c1c3; do timeout 1500 python tools/accuracy.py $w > gpurun_out/r02f_acc_$w.log 2>&1; echo "$w rc=$?"; tail -8 gpurun_out/r02f_acc_$w.log; done
