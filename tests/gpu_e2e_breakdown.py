"""Where the end-to-end time of one C4 solve goes (validation, qs_setup, solve, handle teardown).  Not a pytest file."""
import time, sys, os
sys.path.insert(0, os.getcwd())
import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.ipm import DeviceSolver, solve_on
from paper_2603_29197_b200.problem import Settings
d = configs.make("C4_group_lasso", groups=10000, qlo=20, qhi=250, samples=2000, nnz_per_col=3)
qs.solve(d)  # warm-up: context, library
for rep in range(2):
    t0=time.perf_counter()
    s = qs.Solver("cuda").setup(d.n, d.m, d.p, d.P, d.c, d.A, d.b, d.G, d.h, d.cone.orthant_dim, len(d.cone.soc_dims), d.cone.soc_dims)
    t1=time.perf_counter()
    dev = DeviceSolver(s._data, s._settings)
    t2=time.perf_counter()
    r = solve_on(dev, t2)
    t3=time.perf_counter()
    dev.close()
    t4=time.perf_counter()
    print(f"Solver.setup (validate, as_csc) {t1-t0:.3f}  DeviceSolver init (qs_create+qs_setup) {t2-t1:.3f}  solve_on {t3-t2:.3f} (run {r.solve_seconds:.3f})  close {t4-t3:.3f}  total {t4-t0:.3f}")
    print({k: round(v,3) for k,v in r.timers.items() if k in ('factor','solve','analysis','h2d','cone','kkt_update','residual')})
