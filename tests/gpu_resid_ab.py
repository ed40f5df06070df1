"""A/B of the residual kernels on the real C4 matrices (not a pytest file): QS_RESID_MLP=0|1 python tests/gpu_resid_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.ipm import DeviceSolver

name = sys.argv[1] if len(sys.argv) > 1 else "C4_group_lasso"
kw = dict(C4_group_lasso=dict(groups=10_000, qlo=20, qhi=250, samples=2_000, nnz_per_col=3),
          C3_portfolio=dict(assets=100_000, factors=100, sector=100), C2_lasso=dict(features=100_000, samples=5_000))[name]
d = configs.make(name, **kw)
dev = DeviceSolver(d)
status, iters, _ = dev.run()
nnz = 2 * d.P.nnz + 2 * d.A.nnz + 2 * d.G.nnz
alg = 12 * nnz + 8 * (3 * d.n + 2 * d.p + 4 * d.m)
for kid, label in ((7, "residuals"), (14, "kkt_residual"), (1, "scatter")):
    w, c = dev.time_kernel(kid, 20) * 1e3, dev.time_kernel(kid, 10, cold=True) * 1e3
    extra = f"  alg {alg / 1e6:.1f} MB -> {alg / c / 1e3:.0f} GB/s cold = {alg / c / 1e3 / 6552:.3f} of peak" if kid == 7 else ""
    print(f"{name} QS_RESID_MLP={os.environ.get('QS_RESID_MLP', '1')} {label}: warm {w:.1f} us cold {c:.1f} us{extra}  ({status.value}, {iters} it)")
dev.close()
