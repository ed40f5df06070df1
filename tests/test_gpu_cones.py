"""GPU parity of every cone kernel against the reference's golden outputs and
the CPU oracle, through the C ABI (DeviceCones -> libqsocp_cuda.so).

Tolerance: the elementwise arithmetic is the reference's (compiled without FMA
contraction); only the per-cone reductions are summed in a different order, so
results agree to a few ulp of the reduced quantities: rtol 1e-12 (+ atol
1e-12 * scale where a value is a difference of reduced terms).  max_step and
violation use min/max, which are order independent.
"""

import os

import numpy as np
import pytest

from paper_2603_29197_b200.cones import DeviceCones, ScalingMode, slot_layout
from paper_2603_29197_b200.errors import NotInterior
from paper_2603_29197_b200.problem import ConeSpec
from util import GOLDEN, random_interior_point

pytestmark = pytest.mark.gpu
RTOL = 1e-12


def close(a, b, scale=None):
    a, b = np.asarray(a), np.asarray(b)
    sc = np.max(np.abs(b), initial=1.0) if scale is None else scale
    return np.allclose(a, b, rtol=RTOL, atol=RTOL * sc)


def cone_cases():
    g = dict(np.load(os.path.join(GOLDEN, "cones.npz")))
    for ci in range(int(g["n_cases"])):
        k = f"c{ci}_"
        cone = ConeSpec(int(g[k + "l"]), tuple(int(q) for q in g[k + "q"]))
        yield ci, cone, {key[len(k):]: v for key, v in g.items() if key.startswith(k)}


@pytest.mark.parametrize("big", [0, 8], ids=["lane-groups", "block-per-cone>8"])
@pytest.mark.parametrize("ci,cone,c", list(cone_cases()), ids=lambda v: str(v) if isinstance(v, int) else "")
def test_cone_ops_vs_reference_golden(ci, cone, c, big):
    dc = DeviceCones(cone, big_threshold=big)
    sc, lam_sq = dc.compute_nt_scaling(c["s"], c["z"], with_lam_sq=True)
    assert close(sc.w_orthant, c["w"]) and close(sc.soc_eta, c["eta"])
    assert close(sc.soc_wbar, c["wbar"]) and close(sc.lam, c["lam"])
    assert close(dc.apply_scaling(sc, c["u"]), c["Wu"])
    assert close(dc.apply_scaling(sc, c["u"], ScalingMode.MULTIPLY_INVERSE), c["Winvu"])
    assert close(dc.jordan_product(c["u"], c["v"]), c["uv"])
    assert close(dc.jordan_divide(sc.lam, c["v"]), c["lam_div_v"])
    for a, b, key in ((c["s"], c["u"], "step_s_u"), (c["z"], c["v"], "step_z_v"), (c["s"], c["s"], "step_s_s")):
        got, ref = dc.max_step_to_boundary(a, b), float(c[key])
        assert got == ref or abs(got - ref) <= 1e-12 * abs(ref), key
    assert abs(dc.interior_violation(c["u"]) - float(c["viol_u"])) <= 1e-12 * max(1.0, abs(float(c["viol_u"])))
    assert close(dc.bring_to_interior(c["u"]), c["shift_u"])
    assert abs(dc.compute_mu(c["s"], c["z"]) - float(c["mu"])) <= 1e-13 * abs(float(c["mu"]))
    assert close(dc.neg_wtw_values(sc), c["slots"])
    dc.close()


def test_max_step_hand_cases_exact():
    g = dict(np.load(os.path.join(GOLDEN, "cones.npz")))
    dc = DeviceCones(ConeSpec(0, (3,)))
    got = [dc.max_step_to_boundary(g["hand_u"], d) for d in g["hand_dirs"]]
    for a, b in zip(got, g["hand_steps"]):
        if b == np.finfo(np.float64).max:
            assert a == b  # the STEP_UNBOUNDED sentinel (DBL_MAX), bit for bit
        elif b > 1e15:
            # a = du0^2 - |du1|^2 cancels catastrophically here (1 - 1 - 1e-18): the reference's sequential
            # subtraction keeps -1e-18 and returns 5e18, the tree sum gets exactly 0 and returns "unbounded";
            # either way the step is astronomically larger than the alpha <= 1 the IPM takes
            assert a > 1e15
        else:
            assert abs(a - b) <= 1e-14 * abs(b)  # tail sums are associated differently: a few ulp


@pytest.mark.parametrize("seed", range(4))
def test_random_cones_vs_oracle(oracle, seed):
    rng = np.random.default_rng(100 + seed)
    l = int(rng.integers(0, 300))
    qs = tuple(int(q) for q in rng.integers(1, [4, 40, 300, 3000][seed], int(rng.integers(1, 60))))
    cone = ConeSpec(l, qs)
    dc = DeviceCones(cone, big_threshold=1024)
    s, z = random_interior_point(cone, rng), random_interior_point(cone, rng)
    u, v = rng.standard_normal(cone.total_dim), rng.standard_normal(cone.total_dim)
    ref = oracle.compute_nt_scaling(s, z, cone)
    sc, lam_sq = dc.compute_nt_scaling(s, z, with_lam_sq=True)
    assert close(sc.soc_wbar, ref.soc_wbar) and close(sc.lam, ref.lam) and close(sc.soc_eta, ref.soc_eta)
    assert close(lam_sq, oracle.jordan_product(ref.lam, ref.lam, cone))
    # invariants pinned by the reference's tests (test_cones.py:169-186): lam = W z = W^-1 s, lam.lam = s.z
    assert close(dc.apply_scaling(sc, z), sc.lam) and close(dc.apply_scaling(sc, s, ScalingMode.MULTIPLY_INVERSE), sc.lam)
    assert abs(np.dot(sc.lam, sc.lam) - np.dot(s, z)) <= 1e-10 * abs(np.dot(s, z))
    assert close(dc.apply_scaling(ref, u), oracle.apply_scaling(ref, u))
    assert close(dc.jordan_divide(ref.lam, v), oracle.jordan_divide(ref.lam, v, cone))
    got, want = dc.max_step_to_boundary(s, u), oracle.max_step_to_boundary(s, u, cone)
    assert abs(got - want) <= 1e-10 * abs(want)
    off, starts = slot_layout(cone)
    want = np.empty(int(off[-1]))
    oracle.neg_wtw_values(ref, starts, want)
    assert close(dc.neg_wtw_values(ref), want)
    dc.close()


def test_not_interior_is_reported():
    cone = ConeSpec(2, (3,))
    dc = DeviceCones(cone)
    good = np.array([1.0, 1.0, 2.0, 0.5, 0.5])
    with pytest.raises(NotInterior):
        dc.compute_nt_scaling(np.array([1.0, -1.0, 2.0, 0.5, 0.5]), good)
    with pytest.raises(NotInterior):
        dc.compute_nt_scaling(good, np.array([1.0, 1.0, 1.0, 1.0, 1.0]))  # |tail| > head
    with pytest.raises(NotInterior):
        dc.max_step_to_boundary(np.array([1.0, 1.0, 1.0, 1.0, 0.0]), good)  # on the boundary
    assert dc.max_step_to_boundary(good, good) == np.finfo(np.float64).max


def test_scaling_round_trip_and_commutativity():
    rng = np.random.default_rng(9)
    cone = ConeSpec(33, (1, 2, 17, 64, 129))
    dc = DeviceCones(cone)
    s, z = random_interior_point(cone, rng), random_interior_point(cone, rng)
    u, v = rng.standard_normal(cone.total_dim), rng.standard_normal(cone.total_dim)
    sc = dc.compute_nt_scaling(s, z)
    back = dc.apply_scaling(sc, dc.apply_scaling(sc, u), ScalingMode.MULTIPLY_INVERSE)
    assert np.allclose(back, u, rtol=0, atol=1e-11 * np.max(np.abs(u)))  # test_cones.py:209-217
    assert np.array_equal(dc.jordan_product(u, v), dc.jordan_product(v, u))  # test_cones.py:120-129
    assert close(dc.jordan_product(sc.lam, dc.jordan_divide(sc.lam, v)), v, scale=np.max(np.abs(v)) * 1e2)
