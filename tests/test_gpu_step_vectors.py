"""Vector-level parity of the FUSED per-iteration kernels (the ones qs_step launches) against the reference's
ipm_step intermediates (pkg/src/qsocp/ipm.py:180-234), through the C ABI entry points qs_predictor_rhs,
qs_corrector_rhs, qs_post_solve and qs_update_iterate on caller-owned device vectors.

Expected values: (1) the oracle's cone functions composed exactly as ipm_step composes them, on seeded cone layouts
that include dimension-1 cones and a cone longer than 2048 (CTA-per-cone, chunked path); (2) the `trace` of real
oracle solves (rhs_a, rhs_c, d_comp, ds_a, dz_a, ds, dz, step info, next iterate) at every iteration.

Tolerance rtol 1e-12 of the vector's scale: same elementwise arithmetic (no FMA contraction), only the per-cone
reductions are summed in another order.  Step lengths: 1e-10 relative (quotients of reduced quantities).
"""

import numpy as np
import pytest

from paper_2603_29197_b200.cones import DeviceCones
from paper_2603_29197_b200.problem import ConeSpec
from util import golden_problem_names, load_golden, problem_from_golden, random_interior_point

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def close(a, b, rtol=RTOL):
    a, b = np.asarray(a), np.asarray(b)
    return np.allclose(a, b, rtol=rtol, atol=rtol * np.max(np.abs(b), initial=1.0))


def rel(a, b):
    return abs(a - b) <= 1e-10 * max(abs(b), 1e-300)


LAYOUTS = {
    "orthant-only": ConeSpec(257, ()),
    "dim-1 cones": ConeSpec(3, (1, 1, 5, 1, 2, 1)),
    "small mixed": ConeSpec(40, tuple(int(q) for q in np.random.default_rng(1).integers(1, 40, 200))),
    "C4-like": ConeSpec(0, tuple(int(q) for q in np.random.default_rng(2).integers(20, 251, 300))),
    "one cone > 2048": ConeSpec(5, (3, 2500, 17, 1)),
    "big only": ConeSpec(0, (4097, 2049)),
}


@pytest.mark.parametrize("name", list(LAYOUTS))
@pytest.mark.parametrize("big", [0, 64], ids=["default-threshold", "block-per-cone>64"])
def test_fused_step_kernels_vs_oracle_composition(oracle, name, big):
    """One whole predictor-corrector step assembled from the oracle's unit functions (ipm.py:180-234) with a
    stand-in for the linear solves (random dz), against the four fused kernels."""
    cone = LAYOUTS[name]
    rng = np.random.default_rng(list(LAYOUTS).index(name))
    m, deg = cone.total_dim, cone.orthant_dim + len(cone.soc_dims)
    s, z = random_interior_point(cone, rng), random_interior_point(cone, rng)
    r_cone = rng.standard_normal(m)
    dc = DeviceCones(cone, big_threshold=big)
    # ---- predictor RHS
    sc = oracle.compute_nt_scaling(s, z, cone)
    lam_sq = oracle.jordan_product(sc.lam, sc.lam, cone)
    d_a = oracle.jordan_divide(sc.lam, -lam_sq, cone)
    rhs_a = -r_cone - oracle.apply_scaling(sc, d_a)
    got_sc, got_lsq, got_d, got_rhs = dc.predictor_rhs(s, z, r_cone)
    assert close(got_sc.w_orthant, sc.w_orthant) and close(got_sc.soc_eta, sc.soc_eta)
    assert close(got_sc.soc_wbar, sc.soc_wbar) and close(got_sc.lam, sc.lam)
    assert close(got_lsq, lam_sq) and close(got_d, d_a) and close(got_rhs, rhs_a)
    # ---- predictor post-solve (dz_a stands for the solve's third block; scaled so the steps are finite and < 1 often)
    dz_a = rng.standard_normal(m) * 0.7
    wdz_a = oracle.apply_scaling(sc, dz_a)
    ds_a = oracle.apply_scaling(sc, d_a - wdz_a)
    step_s = oracle.max_step_to_boundary(s, ds_a, cone)
    step_z = oracle.max_step_to_boundary(z, dz_a, cone)
    alpha_aff = min(1.0, step_s, step_z)
    mu_aff = max(0.0, float(np.dot(s + alpha_aff * ds_a, z + alpha_aff * dz_a)) / deg)
    mu = oracle.compute_mu(s, z, cone)
    sigma = min(1.0, max(0.0, (mu_aff / mu) ** 3))
    g_wdz, g_ds, info = dc.post_solve(sc, d_a, dz_a, s, z, corrector=False)
    assert close(g_wdz, wdz_a) and close(g_ds, ds_a)
    assert rel(info["step_s"], step_s) and rel(info["step_z"], step_z) and rel(info["alpha_aff"], alpha_aff)
    assert abs(info["mu"] - mu) <= 1e-13 * mu and abs(info["mu_aff"] - mu_aff) <= 1e-9 * max(mu, mu_aff)
    assert abs(info["sigma"] - sigma) <= 1e-8 * max(sigma, 1e-3) and info["flags"] == 0
    # ---- corrector RHS with the ORACLE's sigma and mu (so the comparison is of the kernel, not of the scalar chain)
    winv_ds = oracle.apply_scaling(sc, ds_a, inverse=True)
    d_comp = sigma * mu * oracle.cone_identity(cone) - lam_sq - oracle.jordan_product(winv_ds, wdz_a, cone)
    d_c = oracle.jordan_divide(sc.lam, d_comp, cone)
    rhs_c = -r_cone - oracle.apply_scaling(sc, d_c)
    g_dc, g_d, g_rhs = dc.corrector_rhs(sc, lam_sq, ds_a, wdz_a, r_cone, sigma, mu)
    assert close(g_dc, d_comp) and close(g_d, d_c) and close(g_rhs, rhs_c)
    # ---- corrector post-solve + iterate update
    dz = rng.standard_normal(m) * 0.5
    ds = oracle.apply_scaling(sc, d_c - oracle.apply_scaling(sc, dz))
    st_s, st_z = oracle.max_step_to_boundary(s, ds, cone), oracle.max_step_to_boundary(z, dz, cone)
    alpha = min(1.0, 0.99 * min(st_s, st_z))
    _, g_ds2, info2 = dc.post_solve(sc, d_c, dz, s, z, corrector=True, step_fraction=0.99)
    assert close(g_ds2, ds) and rel(info2["step_s"], st_s) and rel(info2["step_z"], st_z) and rel(info2["alpha"], alpha)
    n, p = 37, 11
    x, y, dx, dy = (rng.standard_normal(k) for k in (n, p, n, p))
    xo, yo, zo, so, mu2, flags = dc.update_iterate(x, y, z, s, np.concatenate([dx, dy, dz]), ds, alpha)
    # the update is elementwise: bitwise equal to NumPy's a + alpha * b
    assert np.array_equal(xo, x + alpha * dx) and np.array_equal(yo, y + alpha * dy)
    assert np.array_equal(zo, z + alpha * dz) and np.array_equal(so, s + alpha * ds)
    mu_ref = oracle.compute_mu(s + alpha * ds, z + alpha * dz, cone)
    assert abs(mu2 - mu_ref) <= 1e-12 * float(np.abs(s + alpha * ds) @ np.abs(z + alpha * dz)) / deg and flags == 0
    dc.close()


def test_update_iterate_flags_a_non_finite_iterate():
    cone = ConeSpec(4, (3,))
    dc = DeviceCones(cone)
    s = z = np.array([1.0, 1.0, 1.0, 1.0, 2.0, 0.5, 0.5])
    sol = np.zeros(2 + 1 + 7)
    sol[0] = np.inf
    *_, flags = dc.update_iterate(np.zeros(2), np.zeros(1), z, s, sol, np.zeros(7), 0.5)
    assert flags & 2  # NONFINITE (ipm.py:231-233)
    dc.close()


@pytest.mark.parametrize("name", [n for n in golden_problem_names() if n in
                                  ("portfolio_4", "group_lasso_3", "tv_denoising_8", "soc_slice", "random_3", "huber_20")])
def test_fused_step_kernels_vs_reference_trace(oracle, name):
    """Every iteration of a real solve: the oracle's trace (the reference's ipm_step intermediates, bitwise pinned)
    against the fused kernels fed with the oracle's inputs of that iteration."""
    g = load_golden(name)
    d = problem_from_golden(g)
    trace, iterates = [], []
    ref = oracle.solve(d, trace=trace, hook=lambda it: iterates.append((it.x.copy(), it.y.copy(), it.z.copy(), it.s.copy(), it.mu)))
    assert ref.status == "Solved" and len(trace) == ref.iterations and len(iterates) == ref.iterations + 1
    cone = d.cone
    n, p = d.n, d.p
    dc = DeviceCones(cone)
    for k, t in enumerate(trace):
        x, y, z, s, mu = iterates[k]
        rhs_a, rhs_c = t["rhs_a"], t["rhs_c"]
        sc = t["scaling"]
        # r_cone from the predictor RHS: rhs_a[n+p:] = -r_cone - W (lam \ -lam_sq)
        d_a = oracle.jordan_divide(sc.lam, -t["lam_sq"], cone)
        r_cone = -(rhs_a[n + p:] + oracle.apply_scaling(sc, d_a))
        # Near the optimum the cones sit on their boundary: s0^2 - |s1|^2 cancels and |wbar| grows, so a different
        # summation order moves the results by eps x (condition of the NT scaling), not by eps.  kappa = that
        # condition at this iterate (1 at the first iterations: the test is tight there, honest later).
        kappa = 1.0 + float(np.max(np.abs(sc.soc_wbar), initial=0.0)) ** 2
        for v in (s, z):
            for k0, q in zip(np.cumsum([cone.orthant_dim, *cone.soc_dims[:-1]]) if cone.soc_dims else [], cone.soc_dims):
                head, tail = v[k0], v[k0 + 1:k0 + q]
                kappa = max(kappa, head * head / max(head * head - float(tail @ tail), 1e-300))
        tol = min(1e-12 * kappa, 1e-6)
        g_sc, g_lsq, g_d, g_rhs = dc.predictor_rhs(s, z, r_cone)
        assert close(g_sc.lam, sc.lam, tol) and close(g_sc.soc_wbar, sc.soc_wbar, tol) and close(g_lsq, t["lam_sq"], tol)
        assert close(g_rhs, rhs_a[n + p:], 10 * tol)  # r_cone itself was recovered through one rounding
        wdz_a, g_ds_a, info = dc.post_solve(sc, d_a, t["dz_a"], s, z, corrector=False)
        assert close(g_ds_a, t["ds_a"], 10 * tol)
        assert abs(info["alpha_aff"] - t["info"].alpha_affine) <= max(1e-10, 10 * tol) * t["info"].alpha_affine
        assert abs(info["mu_aff"] - t["info"].mu_affine) <= max(1e-9, 10 * tol) * max(mu, t["info"].mu_affine)
        assert abs(info["sigma"] - t["info"].sigma) <= max(1e-7, 100 * tol) * max(t["info"].sigma, 1e-3)
        g_dc, g_d, g_rhs_c = dc.corrector_rhs(sc, t["lam_sq"], t["ds_a"], oracle.apply_scaling(sc, t["dz_a"]), r_cone,
                                              t["info"].sigma, mu)
        assert close(g_dc, t["d_comp"], 10 * tol) and close(g_rhs_c, rhs_c[n + p:], 100 * tol)
        _, g_ds, info2 = dc.post_solve(sc, oracle.jordan_divide(sc.lam, t["d_comp"], cone), t["dz"], s, z, corrector=True)
        assert close(g_ds, t["ds"], 100 * tol)
        assert abs(info2["alpha"] - t["info"].alpha) <= max(1e-10, 100 * tol) * t["info"].alpha
        if k == 0:
            assert tol <= 1e-9, "the first iterate is well inside the cone: tight tolerance expected"
        xo, yo, zo, so, mu2, flags = dc.update_iterate(x, y, z, s, np.concatenate([t["dx"], t["dy"], t["dz"]]), t["ds"],
                                                       t["info"].alpha)
        nx, ny, nz, ns, nmu = iterates[k + 1]
        assert np.array_equal(xo, nx) and np.array_equal(yo, ny) and np.array_equal(zo, nz) and np.array_equal(so, ns)
        # s'z over second-order cones cancels (elementwise products of both signs): the tolerance is relative to
        # sum |s_i z_i|, the magnitude the two summation orders actually add up
        assert abs(mu2 - nmu) <= 1e-12 * float(np.abs(ns) @ np.abs(nz)) / (cone.orthant_dim + len(cone.soc_dims))
        assert flags == 0
    dc.close()
