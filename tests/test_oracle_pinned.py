"""Pins the CPU oracle (oracle/) to the reference.

Two anchors: (1) tests/golden/*.npz -- outputs of the unmodified reference,
produced by oracle/gen_golden.py; (2) when /root/reference is present (the
build container), a direct function-by-function comparison with the imported
reference on fresh seeded inputs.  Integer/index results must be bit-exact;
elementwise float results are compared bitwise as well (the oracle is compiled
without FMA contraction so the operation sequence is the reference's).
"""

import os
import sys

import numpy as np
import pytest

from util import GOLDEN, golden_problem_names, load_golden, problem_from_golden
from paper_2603_29197_b200.problem import ConeSpec

REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF_SRC)


def _cone_cases():
    g = dict(np.load(os.path.join(GOLDEN, "cones.npz")))
    for ci in range(int(g["n_cases"])):
        k = f"c{ci}_"
        cone = ConeSpec(int(g[k + "l"]), tuple(int(q) for q in g[k + "q"]))
        yield ci, cone, {key[len(k):]: v for key, v in g.items() if key.startswith(k)}


@pytest.mark.parametrize("ci,cone,c", list(_cone_cases()), ids=lambda v: str(v) if isinstance(v, int) else "")
def test_cone_ops_match_reference_golden(oracle, ci, cone, c):
    sc = oracle.compute_nt_scaling(c["s"], c["z"], cone)
    assert np.array_equal(sc.w_orthant, c["w"])
    assert np.array_equal(sc.soc_eta, c["eta"])
    assert np.array_equal(sc.soc_wbar, c["wbar"])
    assert np.array_equal(sc.lam, c["lam"])
    assert np.array_equal(oracle.apply_scaling(sc, c["u"]), c["Wu"])
    assert np.array_equal(oracle.apply_scaling(sc, c["u"], inverse=True), c["Winvu"])
    assert np.array_equal(oracle.jordan_product(c["u"], c["v"], cone), c["uv"])
    assert np.array_equal(oracle.jordan_divide(sc.lam, c["v"], cone), c["lam_div_v"])
    assert oracle.max_step_to_boundary(c["s"], c["u"], cone) == float(c["step_s_u"])
    assert oracle.max_step_to_boundary(c["z"], c["v"], cone) == float(c["step_z_v"])
    assert oracle.max_step_to_boundary(c["s"], c["s"], cone) == float(c["step_s_s"]) == oracle.STEP_UNBOUNDED
    assert oracle.interior_violation(c["u"], cone) == float(c["viol_u"])
    assert oracle.interior_violation(c["s"], cone) == float(c["viol_s"])
    assert np.array_equal(oracle.bring_to_interior(c["u"], cone), c["shift_u"])
    assert oracle.compute_mu(c["s"], c["z"], cone) == float(c["mu"])
    starts, dims = oracle.soc_layout(cone)
    cnt = ([cone.orthant_dim] if cone.orthant_dim else []) + [int(d * (d + 1) // 2) for d in dims]
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    soc_starts = off[(1 if cone.orthant_dim else 0):-1] if dims.size else np.zeros(0, np.int64)
    slots = np.empty(int(off[-1]))
    oracle.neg_wtw_values(sc, soc_starts, slots)
    assert np.array_equal(slots, c["slots"])


def test_max_step_hand_cases(oracle):
    g = dict(np.load(os.path.join(GOLDEN, "cones.npz")))
    cone = ConeSpec(0, (3,))
    got = [oracle.max_step_to_boundary(g["hand_u"], d, cone) for d in g["hand_dirs"]]
    assert got == list(g["hand_steps"])


@pytest.mark.parametrize("name", golden_problem_names())
def test_kkt_and_spmv_match_reference_golden(oracle, name):
    g = load_golden(name)
    d = problem_from_golden(g)
    kkt = oracle.assemble_kkt(d)
    for got, key in ((kkt.matrix.col_pointers, "K_p"), (kkt.matrix.row_indices, "K_i"),
                     (kkt.nt_entry_positions, "nt_entry_positions"), (kkt.nt_slot_offsets, "nt_slot_offsets"),
                     (kkt.soc_slot_starts, "soc_slot_starts")):
        assert got.dtype == np.int64 and np.array_equal(got, g[key]), key
    assert np.array_equal(kkt.matrix.values, g["K_x"])
    x, y, z = g["spmv_x"], g["spmv_y"], g["spmv_z"]
    assert np.array_equal(oracle.spmv_sym_upper(d.P, x), g["Px"])
    assert np.array_equal(oracle.spmv(d.A, x), g["Ax"])
    assert np.array_equal(oracle.spmv(d.G, x), g["Gx"])
    assert np.array_equal(oracle.spmv(d.A, y, True), g["Aty"])
    assert np.array_equal(oracle.spmv(d.G, z, True), g["Gtz"])
    assert np.array_equal(oracle.spmv_sym_upper(kkt.matrix, g["kkt_vec"]), g["K_times_vec"])


@pytest.mark.parametrize("name", golden_problem_names())
def test_ordering_matches_reference_golden(oracle, name):
    """The oracle's AMD (oracle/qsocp_oracle_amd.c) returns the reference's permutation element by
    element, whatever the heap capacity (a full heap is compacted to its live keys)."""
    g = load_golden(name)
    K = oracle.assemble_kkt(problem_from_golden(g)).matrix
    for cap in (None, 8):
        perm = oracle.amd_order(K.cols, K.col_pointers, K.row_indices, heap_words=cap)
        assert perm.dtype == np.int64 and np.array_equal(perm, g["amd_perm"])


@pytest.mark.parametrize("name", golden_problem_names())
def test_solve_matches_reference_golden(oracle, name):
    """End to end, no argument handed over: same ordering, same factorisation, same arithmetic as the
    reference, so the result is the reference's bit for bit."""
    g = load_golden(name)
    d = problem_from_golden(g)
    mus = []
    res = oracle.solve(d, hook=lambda it: mus.append(it.mu))
    assert res.status == str(g["status"])
    assert res.iterations == int(g["iterations"])
    assert res.factor_count == int(g["factor_count"]) and res.solve_count == int(g["solve_count"])
    assert res.objective == float(g["objective"])
    assert np.array_equal(np.asarray(mus), g["trace_mu"])
    for k in "xyzs":
        assert np.array_equal(getattr(res, k), g[k]), k


def test_oracle_never_touches_the_product_library(oracle):
    """The checker must be independent of what it checks: solving with the oracle maps neither
    libqsocp_cuda.so (fresh interpreter; the data classes of the problem come from the package, its
    native library must stay unloaded)."""
    import subprocess

    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from util import load_golden, problem_from_golden\n"
            "from oracle import qsocp_oracle as o\n"
            "r = o.solve(problem_from_golden(load_golden('portfolio_4')))\n"
            "assert r.status == 'Solved'\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libqsocp_cuda' not in maps, 'oracle mapped the product library'\n"
            % (os.path.dirname(GOLDEN), os.path.dirname(os.path.dirname(GOLDEN))))
    subprocess.run([sys.executable, "-c", code], check=True)


@pytest.mark.skipif(not HAVE_REF, reason="reference tree not present on this machine")
def test_direct_against_imported_reference(oracle):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF_SRC)
    try:
        import qsocp
        from qsocp import cones as rc
        from qsocp import ipm as ripm
        from qsocp import kkt as rkkt
        from qsocp.linsys import make_backend
    finally:
        sys.path.remove(REF_SRC)
    from util import random_interior_point

    rng = np.random.default_rng(42)
    for trial in range(25):
        l = int(rng.integers(0, 9))
        qs = tuple(int(q) for q in rng.integers(1, 40, int(rng.integers(0, 7))))
        if l + sum(qs) == 0:
            l = 2
        cone = ConeSpec(l, qs)
        rcone = qsocp.ConeSpec(l, qs)
        s, z = random_interior_point(cone, rng), random_interior_point(cone, rng)
        u, v = rng.standard_normal(cone.total_dim), rng.standard_normal(cone.total_dim)
        a, b = oracle.compute_nt_scaling(s, z, cone), rc.compute_nt_scaling(s, z, rcone)
        for f in ("w_orthant", "soc_eta", "soc_wbar", "lam"):
            assert np.array_equal(getattr(a, f), getattr(b, f))
        assert np.array_equal(oracle.apply_scaling(a, u), rc.apply_scaling(b, u, rc.ScalingMode.MULTIPLY))
        assert np.array_equal(oracle.apply_scaling(a, u, True), rc.apply_scaling(b, u, rc.ScalingMode.MULTIPLY_INVERSE))
        assert np.array_equal(oracle.jordan_product(u, v, cone), rc.jordan_product(u, v, rcone))
        assert np.array_equal(oracle.jordan_divide(a.lam, v, cone), rc.jordan_divide(b.lam, v, rcone))
        assert oracle.max_step_to_boundary(s, u, cone) == rc.max_step_to_boundary(s, u, rcone)
        assert oracle.interior_violation(u, cone) == rc.interior_violation(u, rcone)
    # ordering: the reference's amd_order on fresh patterns (random QP, group lasso with dense SOC blocks, MPC chain)
    from qsocp import _amd
    from paper_2603_29197_b200 import configs

    for d in (configs.random_qp(n=300, p=60, m=500, density=0.03, seed=3), configs.group_lasso(groups=24, samples=30, seed=1),
              configs.mpc(horizon=12, seed=5), configs.portfolio(assets=400, factors=8, sector=20, seed=2)):
        K = oracle.assemble_kkt(d).matrix
        want = _amd.amd_order(K.cols, K.col_pointers, K.row_indices)
        assert np.array_equal(oracle.amd_order(K.cols, K.col_pointers, K.row_indices), want)
        assert np.array_equal(oracle.amd_order(K.cols, K.col_pointers, K.row_indices, heap_words=1), want)
    # the reference's own LDL with the reference's AMD permutation handed to the oracle: bitwise trace
    for name in ("huber_20", "tv_denoising_8", "random_1", "group_lasso_3"):
        g = load_golden(name)
        d = problem_from_golden(g)
        rd = qsocp.ProblemData(n=d.n, m=d.m, p=d.p, c=d.c, b=d.b, h=d.h, cone=qsocp.ConeSpec(d.cone.orthant_dim, d.cone.soc_dims),
                               **{k: qsocp.SparseMatrixCSC(M.rows, M.cols, M.col_pointers, M.row_indices, M.values)
                                  for k, M in (("P", d.P), ("A", d.A), ("G", d.G))})
        kk = rkkt.assemble_kkt(rd)
        be = make_backend("builtin")
        be.initialize(kk, qsocp.Settings())
        perm = be.symbolic.perm.forward
        res = oracle.solve(d, perm=np.asarray(perm))
        ref = qsocp.solve(rd)
        own = oracle.solve(d)  # the oracle's own ordering is the same permutation
        assert own.objective == ref.objective and np.array_equal(own.x, ref.x)
        assert res.iterations == ref.iterations
        assert res.objective == ref.objective
        for k in "xyzs":
            assert np.array_equal(getattr(res, k), getattr(ref, k))
