python tools/sweep.py run --variants nofree_r,fw2,fw2a4,fw2rel1,fw2a4rel1,fw2r --workloads C5 --reps 2 --tag r02m 2>&1 | tail -12
