import time, sys
sys.path.insert(0, '.')
import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
import torch
t=time.time(); d = configs.make("C4_group_lasso", groups=10_000, qlo=20, qhi=250, samples=5_000, nnz_per_col=10)
print("generated", d.n, d.p, d.m, configs.kkt_nnz(d), time.time()-t, flush=True)
try:
    t = time.time(); r = qs.solve(d)
    print("C4 as written (5000 samples, 10 nnz/col):", r.status, r.iterations, r.objective, "setup", r.setup_seconds, "solve", r.solve_seconds, "wall", time.time() - t)
    print({k: v for k, v in r.timers.items()})
except Exception as e:
    print("FAILED:", type(e).__name__, str(e)[:300])
print(torch.cuda.mem_get_info())
