"""The synthetic BASELINE configurations: deterministic, valid, solvable (CPU,
small variants, oracle) and -- on the GPU -- solved to the same answer."""

import numpy as np
import pytest

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.kkt import assemble_kkt

NAMES = sorted(configs.CONFIGS)


@pytest.mark.parametrize("name", NAMES)
def test_small_variant_is_deterministic_and_solvable(oracle, name):
    a, b = configs.make(name, small=True), configs.make(name, small=True)
    for M in "PAG":
        assert np.array_equal(getattr(a, M).values, getattr(b, M).values)
        assert np.array_equal(getattr(a, M).row_indices, getattr(b, M).row_indices)
    assert np.array_equal(a.c, b.c) and np.array_equal(a.h, b.h)
    assert assemble_kkt(a).matrix.nnz == configs.kkt_nnz(a)
    res = oracle.solve(a)
    assert res.status == "Solved" and res.iterations <= 30
    other = configs.make(name, small=True, seed=1)
    assert not (other.c.shape == a.c.shape and np.array_equal(other.c, a.c) and np.array_equal(other.h, a.h)
                and np.array_equal(other.G.values, a.G.values) and np.array_equal(other.b, a.b))


def test_full_size_shapes_match_baseline_configs():
    d = configs.make("C1_random_qp")
    assert (d.n, d.p, d.m, d.cone.orthant_dim) == (2000, 500, 4000, 4000)
    d = configs.make("C5_mpc")
    assert (d.p, d.cone.orthant_dim, d.cone.soc_dims) == (600, 1200, (5,) * 50)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_oracle_on_small_variants(oracle, name):
    d = configs.make(name, small=True)
    ref = oracle.solve(d)
    res = qs.solve(d)
    assert res.status.value == ref.status == "Solved"
    assert abs(res.iterations - ref.iterations) <= 1
    assert abs(res.objective - ref.objective) <= 1e-6 * max(1.0, abs(ref.objective))
    for k in "xs":
        a, b = getattr(res, k), getattr(ref, k)
        assert np.max(np.abs(a - b)) <= 1e-5 * max(1.0, np.max(np.abs(b)))


@pytest.mark.gpu
def test_gpu_c1_full_size_properties(oracle):
    """BASELINE configs[0] at full size (the oracle needs ~a minute for it, so the
    check is by properties): the reference's own termination test passes on the
    GPU iterate and the primal/dual objectives agree."""
    d = configs.make("C1_random_qp")
    res = qs.solve(d)
    assert res.status.value == "Solved" and res.factor_count == res.iterations + 1
    it = oracle.Iterate(res.x, res.y, res.z, res.s, 0.0)
    dd = oracle.SimpleNamespace(n=d.n, m=d.m, p=d.p, P=oracle._csc(d.P), A=oracle._csc(d.A), G=oracle._csc(d.G),
                                c=d.c, b=d.b, h=d.h, cone=d.cone)
    r = oracle.compute_residuals(dd, it)
    assert oracle.check_termination(r, it, oracle.OracleSettings(eps_abs=1.000001e-7, eps_rel=1.000001e-7))
    Px = oracle.spmv_sym_upper(dd.P, res.x)
    dual = -0.5 * float(res.x @ Px) - float(d.b @ res.y) - float(d.h @ res.z)
    assert abs(res.objective - dual) <= 1e-5 * max(1.0, abs(res.objective))  # test_ipm.py:228-237


@pytest.mark.gpu
def test_gpu_batch_of_mpc_instances():
    from paper_2603_29197_b200.batch import solve_batch

    recs, wall = solve_batch(lambda i: configs.make("C5_mpc", small=True, seed=i), 4)
    assert [r.index for r in recs] == [0, 1, 2, 3] and all(r.status == "Solved" for r in recs)
