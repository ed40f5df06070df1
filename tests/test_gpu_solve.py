"""End-to-end parity of Solver(algebra='cuda') with the reference (golden
fixtures) and the CPU oracle, plus the backend contract and status paths.

North-star tolerances: iteration count within +-1, objective and residuals to
a relative 1e-6.
"""

import numpy as np
import pytest

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200.cones import identity_scaling
from paper_2603_29197_b200.ipm import DeviceSolver, check_termination
from paper_2603_29197_b200.kkt import assemble_kkt
from paper_2603_29197_b200.linsys import make_backend
from paper_2603_29197_b200.problem import Settings, SolveStatus
from util import golden_problem_names, load_golden, problem_from_golden

pytestmark = pytest.mark.gpu


def run(d, **kw):
    return qs.Solver("cuda").setup(d.n, d.m, d.p, d.P, d.c, d.A, d.b, d.G, d.h, d.cone.orthant_dim,
                                   len(d.cone.soc_dims), d.cone.soc_dims, **kw).solve()


@pytest.mark.parametrize("name", golden_problem_names())
def test_solve_matches_reference(oracle, name):
    g = load_golden(name)
    d = problem_from_golden(g)
    res = run(d)
    assert res.status.value == str(g["status"]) == "Solved"
    assert abs(res.iterations - int(g["iterations"])) <= 1
    obj = float(g["objective"])
    assert abs(res.objective - obj) <= 1e-6 * max(1.0, abs(obj))
    assert res.factor_count == res.iterations + 1 and res.solve_count == 2 * res.iterations + 2  # test_ipm.py:239-243
    for k in "xyzs":
        ref = g[k]
        assert np.max(np.abs(getattr(res, k) - ref), initial=0.0) <= 1e-5 * max(1.0, np.max(np.abs(ref), initial=0.0)), k
    # the GPU solution satisfies the reference's own termination test when its residuals are recomputed by the oracle
    it = oracle.Iterate(res.x, res.y, res.z, res.s, 0.0)
    r = oracle.compute_residuals(oracle.SimpleNamespace(
        n=d.n, m=d.m, p=d.p, P=oracle._csc(d.P), A=oracle._csc(d.A), G=oracle._csc(d.G), c=d.c, b=d.b, h=d.h,
        cone=d.cone), it)
    loose = oracle.OracleSettings(eps_abs=1.000001e-7, eps_rel=1.000001e-7)
    assert oracle.check_termination(r, it, loose)
    assert oracle.interior_violation(res.s, d.cone) < 0 and oracle.interior_violation(res.z, d.cone) < 0


@pytest.mark.parametrize("name", ["huber_20", "random_0", "tv_denoising_8", "group_lasso_3"])
def test_initial_iterate_first_residuals_and_first_step(name):
    g = load_golden(name)
    d = problem_from_golden(g)
    dev = DeviceSolver(d, Settings())
    mu0 = dev.initialize_iterate()
    it = dev.iterate()
    for k in "xyzs":
        ref = g["init_" + k]
        assert np.allclose(getattr(it, k), ref, rtol=1e-7, atol=1e-7 * np.max(np.abs(ref), initial=1.0)), k
    assert abs(mu0 - g["trace_mu"][0]) <= 1e-7 * abs(g["trace_mu"][0])
    r = dev.compute_residuals()
    gap, obj, nPx, nAty, nGtz, nc, nAx, nb, nGx, nh = g["res0_scalars"]
    for got, ref in ((r.gap, gap), (r.objective, obj), (r.norm_Px, nPx), (r.norm_Aty, nAty), (r.norm_Gtz, nGtz),
                     (r.norm_c, nc), (r.norm_Ax, nAx), (r.norm_b, nb), (r.norm_Gx, nGx), (r.norm_h, nh),
                     (r.norm_r_dual, np.max(np.abs(g["res0_r_dual"]), initial=0.0)),
                     (r.norm_r_cone, np.max(np.abs(g["res0_r_cone"]), initial=0.0))):
        assert abs(got - ref) <= 1e-6 * max(1.0, abs(ref))
    info = dev.ipm_step()
    alpha, alpha_aff, sigma, mu_aff, mu1 = g["step0_info"]
    assert abs(info.alpha - alpha) <= 1e-6 and abs(info.alpha_affine - alpha_aff) <= 1e-6
    assert abs(info.sigma - sigma) <= 1e-5 and abs(info.mu - mu1) <= 1e-6 * max(1.0, abs(mu1))
    dev.close()


def test_backend_contract(oracle):
    """LinsysBackend lifecycle and numerics (linsys.py:24-108, test_kkt.py:128-168)."""
    g = load_golden("random_1")
    d = problem_from_golden(g)
    kkt = assemble_kkt(d)
    be = make_backend("cuda")
    with pytest.raises(RuntimeError):
        be.factor()
    be.initialize(kkt, Settings())
    with pytest.raises(RuntimeError):
        be.initialize(kkt, Settings())
    with pytest.raises(RuntimeError):
        be.solve(np.zeros(kkt.dim))
    be.update(identity_scaling(d.cone))
    be.factor()
    rhs = np.random.default_rng(0).standard_normal(kkt.dim)
    x = be.solve(rhs)
    assert (be.n_factor, be.n_solve) == (1, 1)
    K = kkt.matrix.to_dense_symmetric()
    assert np.max(np.abs(K @ x - rhs)) <= 1e-9 * (1 + np.max(np.abs(rhs)))
    # update with a real scaling: device K values equal the oracle's, and the solve follows
    from util import random_interior_point

    rng = np.random.default_rng(1)
    sc = oracle.compute_nt_scaling(random_interior_point(d.cone, rng), random_interior_point(d.cone, rng), d.cone)
    be.update(sc)
    ref = oracle.assemble_kkt(d)
    oracle.write_scaling(ref, sc)
    assert np.allclose(be.kkt_values(), ref.matrix.values, rtol=1e-12, atol=0)
    be.factor()
    x = be.solve(rhs)
    Kd = np.zeros((kkt.dim, kkt.dim))
    cols = np.repeat(np.arange(kkt.dim), np.diff(ref.matrix.col_pointers))
    Kd[ref.matrix.row_indices, cols] = ref.matrix.values
    Kd = Kd + Kd.T - np.diag(np.diag(Kd))
    assert np.max(np.abs(Kd @ x - rhs)) <= 1e-8 * (1 + np.max(np.abs(rhs)))
    be.close()
    with pytest.raises(ValueError):
        make_backend("builtin")


def test_statuses():
    g = load_golden("huber_20")
    d = problem_from_golden(g)
    assert run(d, max_iters=2).status is SolveStatus.MAX_ITERS  # test_ipm.py:245-252
    assert run(d, time_limit_seconds=1e-9).status is SolveStatus.TIME_LIMIT
    bad = problem_from_golden(g)
    bad.c = bad.c.copy()
    bad.c[0] = np.nan
    assert run(bad).status is SolveStatus.NUMERICAL_ERROR  # test_ipm.py:290-294


def test_orderings_and_literal_refinement_agree():
    g = load_golden("portfolio_4")
    d = problem_from_golden(g)
    a = qs.solve(d, ordering="amd")
    b = qs.solve(d, ordering="natural")
    assert a.status is b.status is SolveStatus.SOLVED and abs(a.iterations - b.iterations) <= 1
    assert abs(a.objective - b.objective) <= 1e-7 * max(1.0, abs(a.objective))
    dev = DeviceSolver(d, Settings(), kkt_literal=True)
    st, iters, it = dev.run()
    dev.close()
    assert st is SolveStatus.SOLVED and abs(iters - int(g["iterations"])) <= 1


def test_deterministic_trace():
    """Two runs give bitwise-identical iterates (test_ipm.py:217-226): every
    reduction has a fixed order and there are no atomics on the path."""
    d = problem_from_golden(load_golden("tv_denoising_8"))
    a, b = run(d), run(d)
    for k in "xyzs":
        assert np.array_equal(getattr(a, k), getattr(b, k))
    assert a.objective == b.objective and a.iterations == b.iterations


@pytest.mark.parametrize("name", ["portfolio_4", "group_lasso_3", "tv_denoising_8", "random_3", "soc_slice",
                                  "cfg:group_lasso", "cfg:portfolio"])
@pytest.mark.parametrize("staged", [False, True])
def test_in_solver_scaling_update_matches_oracle(oracle, name, staged, monkeypatch):
    """The resident path's KKT update (whole-column staged bulk stores, kkt_kernels.cu) leaves exactly the
    reference's write_scaling result in K.values (kkt.py:146-150) and touches nothing else."""
    if name == "cfg:group_lasso":  # ~45 output tiles of mixed parity, cones of 20..250
        from paper_2603_29197_b200 import configs

        d = configs.group_lasso(groups=40, qlo=20, qhi=250, samples=200, nnz_per_col=3, seed=3)
    elif name == "cfg:portfolio":  # orthant block + SOCs, G rows of different lengths
        from paper_2603_29197_b200 import configs

        d = configs.portfolio(assets=600, factors=20, sector=50, seed=1)
    else:
        d = problem_from_golden(load_golden(name))
    if staged:
        monkeypatch.setenv("QS_WTW_STAGED", "1")  # shared-memory staging + TMA bulk stores instead of streaming
    dev = DeviceSolver(d, Settings())
    dev.initialize_iterate()
    dev.compute_residuals()
    dev.ipm_step()  # NT scaling of the initial iterate -> K.values
    sc = dev.scaling()
    got = dev.kkt()
    ref = oracle.assemble_kkt(d)
    oracle.write_scaling(ref, oracle.Scaling(d.cone, sc.w_orthant, sc.soc_eta, sc.soc_wbar, sc.lam))
    assert np.array_equal(got.matrix.col_pointers, ref.matrix.col_pointers)
    assert np.array_equal(got.matrix.row_indices, ref.matrix.row_indices)
    assert np.allclose(got.matrix.values, ref.matrix.values, rtol=1e-12, atol=0)
    mask = np.ones(got.matrix.values.size, bool)
    mask[got.nt_entry_positions] = False
    assert np.array_equal(got.matrix.values[mask], ref.matrix.values[mask])  # P, A', G' entries bit-identical
    dev.close()


@pytest.mark.parametrize("name", golden_problem_names() + ["cfg:group_lasso", "cfg:portfolio", "cfg:mpc"])
def test_device_assembled_kkt_is_bit_exact(name, monkeypatch):
    """KKT assembly on the device (qsk_kkt_fill) reproduces assemble_kkt (kkt.py:55-135) bit for bit: column
    pointers, row indices, initial values and the slot -> position map; so does the host-assembly alternative."""
    from paper_2603_29197_b200 import configs

    if name == "cfg:group_lasso":
        d = configs.group_lasso(groups=40, qlo=20, qhi=250, samples=200, nnz_per_col=3, seed=3)
    elif name == "cfg:portfolio":
        d = configs.portfolio(assets=600, factors=20, sector=50, seed=1)
    elif name == "cfg:mpc":
        d = configs.mpc(horizon=10, nx=6, nu=2, seed=2)
    else:
        d = problem_from_golden(load_golden(name))
    ref = assemble_kkt(d)  # host C++ assembly, itself pinned bitwise to the reference (tests/test_host.py)
    for host in (False, True):
        if host:
            monkeypatch.setenv("QS_HOST_ASSEMBLY", "1")
        dev = DeviceSolver(d, Settings())
        got = dev.kkt()
        assert np.array_equal(got.matrix.col_pointers, ref.matrix.col_pointers)
        assert np.array_equal(got.matrix.row_indices, ref.matrix.row_indices)
        assert np.array_equal(got.matrix.values, ref.matrix.values)
        assert np.array_equal(np.signbit(got.matrix.values), np.signbit(ref.matrix.values))
        assert np.array_equal(got.nt_entry_positions, ref.nt_entry_positions)
        dev.close()


def test_solve_with_long_design_rows_matches_oracle(oracle):
    """A group-lasso instance whose equality rows hold ~800 entries each: the residual and refinement kernels take
    their CTA-per-row path; iterations and objective must still match the CPU oracle."""
    from paper_2603_29197_b200 import configs

    d = configs.group_lasso(groups=40, qlo=20, qhi=250, samples=20, nnz_per_col=3, seed=5)
    assert d.A.nnz / d.p >= 512
    res = run(d)
    ref = oracle.solve(d)
    assert res.status.value == ref.status == "Solved"
    assert abs(res.iterations - ref.iterations) <= 1
    assert abs(res.objective - ref.objective) <= 1e-6 * max(1.0, abs(ref.objective))


def test_update_values_reuses_the_pattern_and_matches_a_fresh_solve():
    """Solver.update (qs_update_values): same pattern, new numbers; the re-solve on the kept handle is bitwise the
    solve of a fresh handle on the same numbers, and a different pattern is refused."""
    import dataclasses

    from paper_2603_29197_b200.errors import BadSparseStructure
    from paper_2603_29197_b200.sparse import SparseMatrixCSC

    d = problem_from_golden(load_golden("portfolio_4"))
    s = qs.Solver("cuda").setup(d.n, d.m, d.p, d.P, d.c, d.A, d.b, d.G, d.h, d.cone.orthant_dim,
                                len(d.cone.soc_dims), d.cone.soc_dims)
    first = s.solve()
    assert first.status is SolveStatus.SOLVED

    def scaled(M, f):
        return SparseMatrixCSC(M.rows, M.cols, M.col_pointers, M.row_indices, M.values * f)

    d2 = dataclasses.replace(d, P=scaled(d.P, 1.5), c=d.c * 0.9, h=d.h + 0.05 * np.abs(d.h), G=scaled(d.G, 1.0))
    second = s.update(P=d2.P, c=d2.c, G=d2.G, h=d2.h).solve()
    fresh = run(d2)
    assert second.status is fresh.status is SolveStatus.SOLVED
    assert second.iterations == fresh.iterations and second.objective == fresh.objective
    for k in "xyzs":
        assert np.array_equal(getattr(second, k), getattr(fresh, k)), k
    assert second.factor_count == second.iterations + 1 and second.solve_count == 2 * second.iterations + 2
    # back to the original numbers: the original solution, bit for bit
    third = s.update(P=d.P, c=d.c, G=d.G, h=d.h).solve()
    for k in "xyzs":
        assert np.array_equal(getattr(third, k), getattr(first, k)), k
    # a different pattern is not an update
    bad = SparseMatrixCSC(d.G.rows, d.G.cols, d.G.col_pointers, d.G.row_indices[::-1].copy(), d.G.values)
    if not np.array_equal(bad.row_indices, d.G.row_indices):
        with pytest.raises(BadSparseStructure):
            s.update(G=bad)
    s.close()


def test_batch_with_pattern_reuse_matches_independent_solves():
    from paper_2603_29197_b200 import configs
    from paper_2603_29197_b200.batch import pattern_reuse_solver, solve_batch

    probs = [configs.mpc(horizon=10, nx=6, nu=2, seed=i) for i in range(6)]
    a, _ = solve_batch(lambda i: probs[i], len(probs), Settings())
    b, _ = solve_batch(lambda i: probs[i], len(probs), Settings(), solve_fn=pattern_reuse_solver(), workers=2)
    for ra, rb in zip(a, b):
        assert ra.index == rb.index and ra.status == rb.status == "Solved"
        assert ra.iterations == rb.iterations and ra.objective == rb.objective


def test_linear_system_calls_replay_captured_graphs():
    """On the handle's own (non-default) stream every factor / solve after the first of its kind is a CUDA-graph
    replay (qs_get_graph_stats); QS_NO_GRAPH is the only path to direct launch sequences."""
    from paper_2603_29197_b200.ipm import DeviceSolver

    d = problem_from_golden(load_golden("portfolio_4"))
    dev = DeviceSolver(d)
    try:
        status, iters, _ = dev.run()
        st = dev.graph_stats()
        f, s, _ = dev.counters()
        assert status is SolveStatus.SOLVED
        assert st["direct_launch_sequences"] == 0 and st["graph_replays"] >= f + s
    finally:
        dev.close()


def test_a_failed_step_leaves_the_last_good_iterate():
    """The reference builds the next iterate and raises BEFORE it replaces the current one (ipm.py:219-235), so a
    NumericalError / NotInterior result carries the last good iterate.  Here the step writes to shadow buffers that are
    swapped in only when no flag was raised."""
    from paper_2603_29197_b200.errors import NotInterior, NumericalError

    d = problem_from_golden(load_golden("portfolio_4"))
    dev = DeviceSolver(d)
    try:
        dev.initialize_iterate()
        dev.compute_residuals()
        dev.ipm_step()
        good = dev.iterate()
        # (1) a point outside the cone: the step raises NotInterior and must not touch the iterate
        s_bad = good.s.copy()
        s_bad[0] = -1.0
        dev.set_iterate(s=s_bad)
        with pytest.raises(NotInterior):
            dev.ipm_step()
        after = dev.iterate()
        assert np.array_equal(after.x, good.x) and np.array_equal(after.z, good.z) and np.array_equal(after.s, s_bad)
        # (2) a non-finite direction (NaN right-hand side through y): NumericalError, iterate untouched
        dev.set_iterate(s=good.s)
        y_bad = good.y.copy()
        y_bad[0] = np.nan
        dev.set_iterate(y=y_bad)
        with pytest.raises(NumericalError):
            dev.compute_residuals()
        with pytest.raises(NumericalError):
            dev.ipm_step()
        after = dev.iterate()
        assert np.array_equal(after.x, good.x) and np.array_equal(after.z, good.z) and np.array_equal(after.s, good.s)
        # and the driver reports NUMERICAL_ERROR for such data instead of raising (ipm.py:292-293)
        bad = problem_from_golden(load_golden("portfolio_4"))
        bad.b = bad.b.copy()
        bad.b[0] = np.inf
        res = qs.solve(bad)
        assert res.status is SolveStatus.NUMERICAL_ERROR
    finally:
        dev.close()


def test_bench_line_carries_the_contract_keys():
    """bench.py on the smallest workload: one JSON line with the keys the driver and DESIGN section 7 rely on."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", "C5_mpc", "--steps", "2", "--warmup",
                          "1", "--e2e-steps", "1", "--batch-count", "24", "--cpu-budget", "5"], capture_output=True,
                         text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks",
                "ladder", "batch", "hot_path", "graphs"):
        assert key in line, key
    assert line["metric"] == "ipm_solve_seconds" and line["dtype"] == "f64" and line["higher_is_better"] is False
    assert line["gpu_launches"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert set(line["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] == 1
    rung = line["ladder"][0]
    assert rung["cpu"]["source"].startswith("measured") and rung["iterations_equal"] and rung["objective_rel_diff"] < 1e-6
    assert line["batch"]["instances"] == 24 and line["batch"]["not_solved"] == 0 and "lockstep" in line["batch"]["mode"]
    assert line["graphs"]["direct_launch_sequences"] == 0
