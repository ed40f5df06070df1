"""Offline CPU run of the oracle (= the reference's algorithm, bitwise pinned) on a FULL-SIZE benchmark configuration.

TEST INFRASTRUCTURE.  Takes minutes to hours; run once in the build container, the result is committed as
tests/golden/full_<workload>.npz = {status, iterations, objective, per-iteration mu, final residual norms, CPU
seconds, L nnz, host description}.  The GPU tests (tests/test_gpu_fullsize.py) regenerate the same seeded instance
(paper_2603_29197_b200/configs.py) and assert iteration count +-1 and objective / residuals to 1e-6 against it.

    python tools/oracle_fullsize.py C4_group_lasso [--perm-cache /tmp/c4_perm.npy] [--time-limit 36000]
"""
import argparse
import json
import os
import platform
import sys
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from bench import LADDERS, WORKLOADS
    from oracle import qsocp_oracle as orc
    from paper_2603_29197_b200 import configs

    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=sorted(WORKLOADS))
    ap.add_argument("--perm-cache", default=None)
    ap.add_argument("--time-limit", type=float, default=48 * 3600.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--rung", default=None, help="a rung of bench.LADDERS[workload] (e.g. 1/10) instead of the full size; "
                                                 "written to tests/golden/ladder_<workload>_<rung>.npz")
    ap.add_argument("--product-perm", action="store_true",
                    help="take the fill-reducing permutation from the product's host ordering (cone-block AMD) instead "
                         "of the reference's AMD, whose cost grows like size^2.5 on dense SOC blocks (117 s at 1/10 "
                         "of C4); the numerics (KKT, LDL', refinement, IPM) stay the oracle's.  Recorded in the file.")
    args = ap.parse_args()
    key, full_kw = WORKLOADS[args.workload][:2]
    if args.rung:
        full_kw = dict(LADDERS[args.workload])[args.rung]
    t0 = time.time()
    d = configs.make(key, **full_kw)
    print(f"generated {args.workload} {full_kw}: n={d.n} p={d.p} m={d.m} in {time.time()-t0:.1f}s", flush=True)
    dd = SimpleNamespace(n=d.n, m=d.m, p=d.p, P=orc._csc(d.P), A=orc._csc(d.A), G=orc._csc(d.G), c=orc._vec(d.c),
                         b=orc._vec(d.b), h=orc._vec(d.h), cone=d.cone)
    perm = None
    t_amd = 0.0
    if args.perm_cache and os.path.exists(args.perm_cache):
        perm = np.load(args.perm_cache)
        print("ordering loaded from", args.perm_cache, flush=True)
    elif args.product_perm:
        import paper_2603_29197_b200 as qs  # noqa: F401  (host C++ ordering only; no GPU involved)
        from paper_2603_29197_b200 import ordering as pord
        from paper_2603_29197_b200.kkt import assemble_kkt as product_assemble

        t = time.time()
        kk = product_assemble(d)
        dims = np.asarray(d.cone.soc_dims, np.int64)
        starts = np.ascontiguousarray(d.n + d.p + d.cone.orthant_dim + np.concatenate([[0], np.cumsum(dims)[:-1]]),
                                      dtype=np.int64) if dims.size else None
        perm, stats = pord.analyze(kk.matrix.cols, kk.matrix.col_pointers, kk.matrix.row_indices, "amd",
                                   clique_starts=starts, clique_sizes=dims if dims.size else None)
        t_amd = time.time() - t
        print(f"product ordering (cone-block AMD, host C++): {t_amd:.1f}s, predicted L nnz {stats['L_nnz']:.3g}", flush=True)
        if args.perm_cache:
            np.save(args.perm_cache, perm)
        del kk
    else:
        t = time.time()
        K = orc.assemble_kkt(dd).matrix
        print(f"KKT assembled: nnz {int(K.col_pointers[-1])} in {time.time()-t:.1f}s", flush=True)
        t = time.time()
        perm = orc.default_perm(K)
        t_amd = time.time() - t
        print(f"reference AMD: {t_amd:.1f}s", flush=True)
        if args.perm_cache:
            np.save(args.perm_cache, perm)
        del K
    mus, stamps = [], []

    def hook(it):
        mus.append(it.mu)
        stamps.append(time.time())
        print(f"  iterate {len(mus)-1}: mu {it.mu:.6e}  t+{stamps[-1]-t0:.0f}s", flush=True)

    st = orc.OracleSettings(time_limit_seconds=args.time_limit)
    res = orc.solve(d, st, perm=perm, hook=hook)
    r = orc.compute_residuals(dd, orc.Iterate(res.x, res.y, res.z, res.s, 0.0))
    host = {"cores_available": len(os.sched_getaffinity(0)), "threads_used": 1, "machine": platform.machine(), "cpu": ""}
    try:
        host["cpu"] = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")][0]
    except (OSError, IndexError):
        pass
    name = f"ladder_{args.workload}_{args.rung.replace('/', 'of')}.npz" if args.rung else f"full_{args.workload}.npz"
    out = args.out or os.path.join(ROOT, "tests", "golden", name)
    np.savez_compressed(
        out, workload=np.array(args.workload), config=np.array(json.dumps(full_kw)), status=np.array(res.status),
        iterations=np.array(res.iterations), objective=np.array(res.objective), trace_mu=np.array(mus),
        iterate_stamps=np.array(stamps) - t0, norm_r_dual=np.array(orc._inf(r.r_dual)),
        norm_r_eq=np.array(orc._inf(r.r_eq)), norm_r_cone=np.array(orc._inf(r.r_cone)), gap=np.array(r.gap),
        norms=np.array([r.norm_Px, r.norm_Aty, r.norm_Gtz, r.norm_c, r.norm_Ax, r.norm_b, r.norm_Gx, r.norm_h]),
        x_head=res.x[:64].copy(), x_norm=np.array(float(np.linalg.norm(res.x))),
        s_norm=np.array(float(np.linalg.norm(res.s))), z_norm=np.array(float(np.linalg.norm(res.z))),
        setup_seconds=np.array(res.setup_seconds + t_amd), solve_seconds=np.array(res.solve_seconds),
        amd_seconds=np.array(t_amd), timers=np.array(json.dumps(res.timers)), host=np.array(json.dumps(host)),
        factor_count=np.array(res.factor_count), solve_count=np.array(res.solve_count),
        ordering=np.array("product cone-block AMD (permutation handed to the oracle)" if args.product_perm
                          else "reference AMD (oracle restatement)"))
    print(f"{args.workload}: {res.status} in {res.iterations} iterations, objective {res.objective:.12g}, "
          f"setup {res.setup_seconds + t_amd:.1f}s solve {res.solve_seconds:.1f}s -> {out}", flush=True)


if __name__ == "__main__":
    main()
