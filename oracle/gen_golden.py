"""Generate tests/golden/*.npz by running the UNMODIFIED reference (qsocp).

TEST INFRASTRUCTURE.  Runs only in the build container, where /root/reference
exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden.py

The fixtures are committed, so the GPU box (which has no /root/reference) can
check both the oracle and the CUDA path against numbers the reference itself
produced.  Every array in a fixture is an input to, or an output of, a
reference function named in the key.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("QSOCP_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import qsocp  # noqa: E402
from qsocp import ConeSpec, ProblemData, Settings, csc_from_triplets  # noqa: E402
from qsocp import cones as rc  # noqa: E402
from qsocp import ipm as ripm  # noqa: E402
from qsocp import kkt as rkkt  # noqa: E402
from qsocp.bench.generators import Family, GeneratorConfig, generate_problem  # noqa: E402
from qsocp.cones import ScalingMode  # noqa: E402
from qsocp.linsys import make_backend  # noqa: E402
from qsocp.sparse import empty_csc, spmv, spmv_sym_upper  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def random_interior_point(cone, rng):  # same recipe as pkg/tests/conftest.py:57-66
    u = rng.standard_normal(cone.total_dim)
    l = cone.orthant_dim
    u[:l] = np.abs(u[:l]) + 0.1
    off = l
    for q in cone.soc_dims:
        tail = u[off + 1: off + q]
        u[off] = np.linalg.norm(tail) + abs(rng.standard_normal()) + 0.1
        off += q
    return u


def pack_problem(d: ProblemData, prefix=""):
    out = {prefix + "dims": np.array([d.n, d.m, d.p, d.cone.orthant_dim], dtype=np.int64),
           prefix + "soc_dims": np.asarray(d.cone.soc_dims, dtype=np.int64),
           prefix + "c": d.c, prefix + "b": d.b, prefix + "h": d.h}
    for name in "PAG":
        M = getattr(d, name)
        out[f"{prefix}{name}_shape"] = np.array([M.rows, M.cols], dtype=np.int64)
        out[f"{prefix}{name}_p"] = M.col_pointers
        out[f"{prefix}{name}_i"] = M.row_indices
        out[f"{prefix}{name}_x"] = M.values
    return out


CONES = [
    ConeSpec(5, ()),
    ConeSpec(0, (1,)),
    ConeSpec(0, (2,)),
    ConeSpec(0, (3, 3, 3, 3)),
    ConeSpec(3, (1, 2, 5)),
    ConeSpec(7, (4, 1, 9, 33, 2)),
    ConeSpec(0, (64, 65, 31, 32, 33)),
    ConeSpec(17, tuple([5] * 40)),
    ConeSpec(2, (120, 7, 400)),
]


def gen_cones():
    g = {}
    g["n_cases"] = np.array(len(CONES))
    for ci, cone in enumerate(CONES):
        rng = np.random.default_rng(1000 + ci)
        s = random_interior_point(cone, rng)
        z = random_interior_point(cone, rng)
        u = rng.standard_normal(cone.total_dim)
        v = rng.standard_normal(cone.total_dim)
        sc = rc.compute_nt_scaling(s, z, cone)
        k = f"c{ci}_"
        g[k + "l"] = np.array(cone.orthant_dim)
        g[k + "q"] = np.asarray(cone.soc_dims, dtype=np.int64)
        g[k + "s"], g[k + "z"], g[k + "u"], g[k + "v"] = s, z, u, v
        g[k + "w"], g[k + "eta"], g[k + "wbar"], g[k + "lam"] = sc.w_orthant, sc.soc_eta, sc.soc_wbar, sc.lam
        g[k + "Wu"] = rc.apply_scaling(sc, u, ScalingMode.MULTIPLY)
        g[k + "Winvu"] = rc.apply_scaling(sc, u, ScalingMode.MULTIPLY_INVERSE)
        g[k + "uv"] = rc.jordan_product(u, v, cone)
        g[k + "lam_div_v"] = rc.jordan_divide(sc.lam, v, cone)
        g[k + "step_s_u"] = np.array(rc.max_step_to_boundary(s, u, cone))
        g[k + "step_z_v"] = np.array(rc.max_step_to_boundary(z, v, cone))
        g[k + "step_s_s"] = np.array(rc.max_step_to_boundary(s, s, cone))  # unbounded sentinel
        g[k + "viol_u"] = np.array(rc.interior_violation(u, cone))
        g[k + "viol_s"] = np.array(rc.interior_violation(s, cone))
        g[k + "shift_u"] = rc.bring_to_interior(u, cone)
        g[k + "mu"] = np.array(rc.compute_mu(s, z, cone))
        # slot values of -W'W in the reference's slot order
        views = rc.cone_views(cone)
        cnt = [rkkt.scaling_slot_count(vw) for vw in views]
        off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        soc_starts = off[(1 if cone.orthant_dim else 0):-1] if cone.soc_dims else np.zeros(0, np.int64)
        slots = np.empty(int(off[-1]))
        rc.neg_wtw_values(sc, np.asarray(soc_starts, dtype=np.int64), slots)
        g[k + "slots"] = slots
    # hand cases pinned by pkg/tests/test_cones.py (max-step branches)
    cone = ConeSpec(0, (3,))
    uu = np.array([2.0, 0.5, -0.25])
    dirs = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.0],
                     [-1.0, 1.0, 0.0], [0.0, 0.0, 0.0], [-3.0, 0.1, 0.2], [1.0, -1.0, 1e-9]])
    g["hand_u"], g["hand_dirs"] = uu, dirs
    g["hand_steps"] = np.array([rc.max_step_to_boundary(uu, d, cone) for d in dirs])
    np.savez_compressed(os.path.join(OUT, "cones.npz"), **g)


def small_problems():
    """(name, ProblemData) list: analytic fixtures, the five reference
    families at desk size, and random feasible mixed-cone problems."""
    out = []
    out.append(("tiny_qp", ProblemData(
        n=1, m=1, p=0, P=csc_from_triplets(1, 1, [(0, 0, 1.0)]), c=np.array([1.0]),
        A=empty_csc(0, 1), b=np.zeros(0), G=csc_from_triplets(1, 1, [(0, 0, -1.0)]),
        h=np.array([-1.0]), cone=ConeSpec(1))))
    out.append(("soc_slice", ProblemData(
        n=3, m=3, p=1, P=empty_csc(3, 3), c=np.array([0.0, 1.0, 0.0]),
        A=csc_from_triplets(1, 3, [(0, 0, 1.0)]), b=np.array([1.0]),
        G=csc_from_triplets(3, 3, [(i, i, -1.0) for i in range(3)]), h=np.zeros(3),
        cone=ConeSpec(0, (3,)))))
    out.append(("two_asset", ProblemData(
        n=2, m=2, p=1, P=csc_from_triplets(2, 2, [(0, 0, 0.2), (1, 1, 0.4)]),
        c=np.array([-0.1, -0.2]), A=csc_from_triplets(1, 2, [(0, 0, 1.0), (0, 1, 1.0)]),
        b=np.array([1.0]), G=csc_from_triplets(2, 2, [(0, 0, -1.0), (1, 1, -1.0)]),
        h=np.zeros(2), cone=ConeSpec(2))))
    for fam, size in ((Family.HUBER, 20), (Family.PORTFOLIO, 4), (Family.MULTI_PERIOD_PORTFOLIO, 2),
                      (Family.GROUP_LASSO, 3), (Family.TV_DENOISING, 8)):
        kw = {"assets": 30} if fam is Family.MULTI_PERIOD_PORTFOLIO else {}
        out.append((f"{fam.value}_{size}", generate_problem(GeneratorConfig(fam, size, seed=0, **kw))))
    for seed in range(6):
        out.append((f"random_{seed}", random_feasible(np.random.default_rng(7000 + seed))))
    return out


def random_feasible(rng):  # recipe of pkg/tests/conftest.py:69-104 with a few larger cones
    n = int(rng.integers(3, 14))
    p = int(rng.integers(0, 3))
    l = int(rng.integers(0, 6))
    nsoc = int(rng.integers(0, 4))
    qs = tuple(int(rng.integers(1, 7)) for _ in range(nsoc))
    if l + sum(qs) == 0:
        l = 1
    cone = ConeSpec(l, qs)
    m = cone.total_dim
    M = rng.standard_normal((n, n))
    Pd = M.T @ M + 0.1 * np.eye(n)
    P = csc_from_triplets(n, n, [(i, j, Pd[i, j]) for i in range(n) for j in range(i, n)])
    A = csc_from_triplets(p, n, [(i, j, float(rng.standard_normal())) for i in range(p) for j in range(n)]) \
        if p else empty_csc(0, n)
    dens = rng.random((m, n)) < 0.6
    G = csc_from_triplets(m, n, [(i, j, float(rng.standard_normal())) for i in range(m) for j in range(n)
                                 if dens[i, j] or j == i % n])
    x0 = rng.standard_normal(n)
    s0 = random_interior_point(cone, rng)
    return qsocp.validate_problem(ProblemData(n=n, m=m, p=p, P=P, c=rng.standard_normal(n), A=A, b=spmv(A, x0),
                                              G=G, h=spmv(G, x0) + s0, cone=cone))


def gen_problems():
    names = []
    for name, d in small_problems():
        g = pack_problem(d)
        # KKT pattern + index maps (kkt.py:55-135): must be reproduced bit for bit
        kkt = rkkt.assemble_kkt(d)
        g["K_p"], g["K_i"], g["K_x"] = kkt.matrix.col_pointers, kkt.matrix.row_indices, kkt.matrix.values
        g["nt_entry_positions"] = kkt.nt_entry_positions
        g["nt_slot_offsets"] = kkt.nt_slot_offsets
        g["soc_slot_starts"] = kkt.soc_slot_starts
        # SpMV family (sparse.py:119-150)
        rng = np.random.default_rng(5)
        xv, yv, zv = rng.standard_normal(d.n), rng.standard_normal(d.p), rng.standard_normal(d.m)
        g["spmv_x"], g["spmv_y"], g["spmv_z"] = xv, yv, zv
        g["Px"] = spmv_sym_upper(d.P, xv)
        g["Ax"], g["Gx"] = spmv(d.A, xv), spmv(d.G, xv)
        g["Aty"], g["Gtz"] = spmv(d.A, yv, transpose=True), spmv(d.G, zv, transpose=True)
        kv = rng.standard_normal(d.n + d.p + d.m)
        g["kkt_vec"], g["K_times_vec"] = kv, spmv_sym_upper(kkt.matrix, kv)
        # full solve with trace (ipm.py:238-312)
        trace = []
        res = qsocp.solve(d, Settings(), backend_name="builtin",
                          iterate_hook=lambda it: trace.append((it.x.copy(), it.y.copy(), it.z.copy(), it.s.copy(), it.mu)))
        g["status"] = np.array(res.status.value)
        g["iterations"] = np.array(res.iterations)
        g["objective"] = np.array(res.objective)
        g["factor_count"], g["solve_count"] = np.array(res.factor_count), np.array(res.solve_count)
        g["x"], g["y"], g["z"], g["s"] = res.x, res.y, res.z, res.s
        g["trace_mu"] = np.array([t[4] for t in trace])
        g["init_x"], g["init_y"], g["init_z"], g["init_s"] = trace[0][:4]
        if len(trace) > 1:
            g["it1_x"], g["it1_y"], g["it1_z"], g["it1_s"] = trace[1][:4]
        # one instrumented ipm_step from the initial iterate (ipm.py:159-235)
        kkt2 = rkkt.assemble_kkt(d)
        be = make_backend("builtin")
        be.initialize(kkt2, Settings())
        g["amd_perm"] = np.asarray(be.symbolic.perm.forward, dtype=np.int64)  # _amd.py via sparse.py:205-222
        it0 = ripm.initialize_iterate(d, kkt2, be)
        r0 = ripm.compute_residuals(d, it0)
        g["res0_r_dual"], g["res0_r_eq"], g["res0_r_cone"] = r0.r_dual, r0.r_eq, r0.r_cone
        g["res0_scalars"] = np.array([r0.gap, r0.objective_primal, r0.norm_Px, r0.norm_Aty, r0.norm_Gtz, r0.norm_c,
                                      r0.norm_Ax, r0.norm_b, r0.norm_Gx, r0.norm_h])
        nxt, info = ripm.ipm_step(d, kkt2, be, it0, Settings(), res=r0)
        g["step0_info"] = np.array([info.alpha, info.alpha_affine, info.sigma, info.mu_affine, nxt.mu])
        np.savez_compressed(os.path.join(OUT, f"problem_{name}.npz"), **g)
        names.append(name)
        print(f"{name}: n={d.n} p={d.p} m={d.m} K nnz={kkt.matrix.nnz} iters={res.iterations} "
              f"status={res.status.value} obj={res.objective:.12g}")
    with open(os.path.join(OUT, "problems.txt"), "w") as f:
        f.write("\n".join(names) + "\n")


def gen_problem_file():
    """A QOCOPROB 1 text file written by the reference's own save_problem (fileio.py:62-64): the reader of
    paper_2603_29197_b200/fileio.py must load it to the same arrays, and its writer must produce the same text."""
    from qsocp.fileio import save_problem

    d = dict(small_problems())["portfolio_4"]
    save_problem(d, os.path.join(OUT, "portfolio_4.qocoprob"))


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    gen_cones()
    gen_problems()
    gen_problem_file()
    print("reference version", qsocp.__version__)
