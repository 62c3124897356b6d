python tools/sweep.py run --variants r1,free0,fr64,fr256,fr1024,fr256r --workloads C5,C3 --reps 2 --tag r02j 2>&1 | tail -24
