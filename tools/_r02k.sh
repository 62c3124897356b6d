python tools/sweep.py run --variants r1,nofree_r,nofree0,fr256,fr256r --workloads C5 --reps 2 --tag r02k 2>&1 | tail -10
