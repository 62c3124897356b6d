python tools/sweep.py run --variants r1,free0,free4 --workloads C5,C3,C4 --reps 2 --tag r02h 2>&1 | tail -18
