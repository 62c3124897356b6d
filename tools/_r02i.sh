python tools/sweep.py run --variants r1,r1new,free0,free0rel1 --workloads C5,C3 --reps 2 --tag r02i 2>&1 | tail -16
