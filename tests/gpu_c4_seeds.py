import sys, time
sys.path.insert(0, '.')
import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
for seed in range(1, 8):
    d = configs.make("C4_group_lasso", seed=seed, groups=10_000, qlo=20, qhi=250, samples=2_000, nnz_per_col=3)
    r = qs.solve(d); print("seed", seed, r.status.value, r.iterations, round(r.solve_seconds, 3), flush=True)
