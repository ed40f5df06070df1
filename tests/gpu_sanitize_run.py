"""Small solves that exercise every device code path (blocked fronts, cluster solves, DMMA updates, leaf fronts,
extend-add bands, both scatter variants, all three row-product modes, pattern reuse), for compute-sanitizer:
    compute-sanitizer --tool memcheck python tests/gpu_sanitize_run.py
Not a pytest file."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
from util import load_golden, problem_from_golden


def run(d, **kw):
    r = qs.Solver("cuda").setup(d.n, d.m, d.p, d.P, d.c, d.A, d.b, d.G, d.h, d.cone.orthant_dim,
                                len(d.cone.soc_dims), d.cone.soc_dims, **kw).solve()
    print(r.status.value, r.iterations, f"{r.objective:.9g}", flush=True)
    return r


cases = [
    problem_from_golden(load_golden("portfolio_4")),
    problem_from_golden(load_golden("tv_denoising_8")),
    configs.group_lasso(groups=80, qlo=20, qhi=250, samples=300, nnz_per_col=3, seed=1),   # banded root, blocked fronts
    configs.group_lasso(groups=30, qlo=20, qhi=120, samples=20, nnz_per_col=3, seed=2),    # CTA-per-row products
    configs.portfolio(assets=800, factors=30, sector=40, seed=3),
    configs.mpc(horizon=12, nx=6, nu=2, seed=4),
    configs.random_qp(n=300, p=60, m=500, seed=5),
]
for d in cases:
    run(d)
os.environ["QS_WTW_STAGED"] = "1"
run(cases[2])
del os.environ["QS_WTW_STAGED"]
os.environ["QS_NO_GRAPH"] = "1"
os.environ["QS_LDL_LOCKSTEP"] = "1"
run(cases[2])
del os.environ["QS_NO_GRAPH"], os.environ["QS_LDL_LOCKSTEP"]
run(cases[4], ruiz_iters=5)
s = qs.Solver("cuda")
d = cases[5]
s.setup(d.n, d.m, d.p, d.P, d.c, d.A, d.b, d.G, d.h, d.cone.orthant_dim, len(d.cone.soc_dims), d.cone.soc_dims)
s.solve()
s.update(c=d.c * 1.1, h=d.h * 1.05)
print(s.solve().status.value)
s.close()
print("sanitize run complete")

# batched small-problem mode (every kernel with gridDim.z > 1, the arena allocator, copy_if / broadcast)
from paper_2603_29197_b200.batched import solve_batched

import dataclasses

base = configs.group_lasso(groups=12, qlo=20, qhi=90, samples=40, nnz_per_col=3, seed=7)  # blocked fronts, SOCs
batches = {"mpc": [configs.mpc(horizon=12, nx=6, nu=2, seed=s) for s in range(5)],
           "group_lasso": [dataclasses.replace(base, c=base.c * (1.0 + 0.1 * s), b=base.b * (1.0 + 0.05 * s)) for s in range(4)]}
for fam, probs in batches.items():
    res = solve_batched(probs)
    print("batched", fam, [r.status.value for r in res], [r.iterations for r in res], flush=True)
print("sanitize run (batched) complete")
