"""Kernel microbenchmark on the C4 cone layout (10^4 SOCs, q ~ U{20..250}):
CUDA-event timing of each hot-path kernel on the handle's stream, reported as
algorithmic bytes / time vs the measured HBM peak.  Not a pytest file."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main(nsoc=10000, qlo=20, qhi=250, l=0, reps=20):
    from paper_2603_29197_b200.ipm import DeviceSolver
    from paper_2603_29197_b200.problem import ConeSpec, ProblemData, Settings
    from paper_2603_29197_b200.sparse import SparseMatrixCSC, empty_csc
    from util import random_interior_point

    rng = np.random.default_rng(0)
    q = rng.integers(qlo, qhi + 1, nsoc)
    m = int(l + q.sum())
    n = m
    # G = -I (group-lasso epigraph structure), no equalities: the factor is trivial, the cone path is not
    G = SparseMatrixCSC(m, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), -np.ones(n))
    P = SparseMatrixCSC(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))
    cone = ConeSpec(l, tuple(int(v) for v in q))
    d = ProblemData(n=n, m=m, p=0, P=P, c=rng.standard_normal(n), A=empty_csc(0, n), b=np.zeros(0), G=G,
                    h=random_interior_point(cone, rng), cone=cone)
    dev = DeviceSolver(d, Settings())
    S = int(l + (q * (q + 1) // 2).sum())
    dev.set_iterate(rng.standard_normal(n), None, random_interior_point(cone, rng), random_interior_point(cone, rng))
    dev.compute_residuals()
    dev.ipm_step()  # populates every buffer with a consistent state
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6650.0
    N = n + m
    kernels = [  # id, name, algorithmic bytes of the logical ops the kernel covers
        (0, "nt_scaling+lam_sq+pred_rhs", 40 * m + 8 * (l + nsoc) + 64 * m),
        (3, "nt_scaling+lam_sq (alone)", 40 * m + 8 * (l + nsoc)),
        (1, "neg_wtw_scatter(direct)", 8 * S + 8 * (m + nsoc)),
        (2, "neg_wtw_scatter(map)", 8 * S + 8 * (m + nsoc)),
        (4, "post_solve(pred)+mu_aff", 80 * m + 32 * m),
        (5, "post_solve(corr)", 80 * m),
        (6, "dcomp+corr_rhs", 80 * m + 64 * m),
        (15, "update_iterate", 24 * n + 48 * m),
        (7, "residuals(5 spmv+norms)", 12 * (2 * n + 2 * m) + 8 * (3 * n + 4 * m)),
        (8, "apply_w", 24 * m),
        (9, "jordan_product", 24 * m),
        (10, "jordan_divide", 24 * m),
        (11, "max_step", 16 * m),
    ]
    out = {"nsoc": nsoc, "m": m, "S": S, "peak_gbs": peak, "kernels": {}}
    print(f"{'kernel':32s} {'warm us':>9s} {'cold us':>9s} {'alg MB':>9s} {'warm GB/s':>10s} {'cold GB/s':>10s}  warm%  cold%"
          "   (warm = back to back, operands may sit in L2; cold = L2 flushed before every launch)")
    for kid, name, nbytes in kernels:
        ms = dev.time_kernel(kid, reps)
        msc = dev.time_kernel(kid, max(reps // 2, 1), cold=True)
        gbs, gbc = nbytes / (ms * 1e-3) / 1e9, nbytes / (msc * 1e-3) / 1e9
        out["kernels"][name] = {"us": ms * 1e3, "cold_us": msc * 1e3, "alg_bytes": nbytes, "gbs": gbs, "frac": gbs / peak,
                                "cold_gbs": gbc, "cold_frac": gbc / peak}
        print(f"{name:32s} {ms*1e3:9.1f} {msc*1e3:9.1f} {nbytes/1e6:9.1f} {gbs:10.1f} {gbc:10.1f} {gbs/peak:6.1%} {gbc/peak:6.1%}")
    print(json.dumps(out))
    dev.close()


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
