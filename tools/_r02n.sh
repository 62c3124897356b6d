python tools/sweep.py run --variants nofree_r,fw2,fw2m,fw3m,fw3r --workloads C5,C3 --reps 2 --tag r02n 2>&1 | tail -20
