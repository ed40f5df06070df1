"""BASELINE.json's configurations at FULL size on the GPU, checked through size-independent properties (the CPU
oracle would need about an hour on C4): the reference's own optimality conditions (ipm.py:106-119), recomputed
on the host from the returned (x, y, z, s) with scipy -- an implementation that shares nothing with the kernels --
cone membership of s and z, complementarity, the factor / solve counters, and run-to-run bitwise determinism."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.problem import SolveStatus

pytestmark = pytest.mark.gpu


def _csc(M):
    return sp.csc_matrix((M.values, M.row_indices, M.col_pointers), shape=(M.rows, M.cols))


def _check_optimality(d, res, eps=1e-7):
    """check_termination (ipm.py:106-119) restated with scipy; eps widened by 1e-3 relative for summation order."""
    P, A, G = _csc(d.P), _csc(d.A), _csc(d.G)
    Pf = P + sp.triu(P, 1).T
    x, y, z, s = res.x, res.y, res.z, res.s
    Px, Aty, Gtz = Pf @ x, A.T @ y, G.T @ z
    Ax, Gx = A @ x, G @ x
    inf = lambda v: float(np.max(np.abs(v), initial=0.0))
    r_dual, r_eq, r_cone = Px + d.c + Aty + Gtz, Ax - d.b, Gx + s - d.h
    tol = eps * 1.001
    assert inf(r_dual) <= tol + tol * max(inf(Px), inf(Aty), inf(Gtz), inf(d.c))
    assert inf(r_eq) <= tol + tol * max(inf(Ax), inf(d.b))
    assert inf(r_cone) <= tol + tol * max(inf(Gx), inf(s), inf(d.h))
    gap = float(s @ z)
    obj = 0.5 * float(x @ Px) + float(d.c @ x)
    assert 0.0 <= gap <= tol + tol * max(abs(obj), 1.0)
    assert abs(res.objective - obj) <= 1e-9 * max(1.0, abs(obj))
    # cone membership (cones.py:275-299): orthant > 0, SOC head > |tail|
    l = d.cone.orthant_dim
    assert np.all(s[:l] > 0) and np.all(z[:l] > 0)
    if d.cone.soc_dims:
        dims = np.asarray(d.cone.soc_dims)
        starts = l + np.concatenate([[0], np.cumsum(dims)[:-1]])
        for v in (s, z):
            sq = v[l:] ** 2
            tot = np.add.reduceat(sq, starts - l)
            head = v[starts]
            assert np.all(head > 0) and np.all(head * head > tot - head * head)


CASES = {
    "C4_group_lasso": dict(groups=10_000, qlo=20, qhi=250, samples=2_000, nnz_per_col=3),
    "C3_portfolio": dict(assets=100_000, factors=100, sector=100),
    "C2_lasso": dict(features=100_000, samples=5_000),
    "C1_random_qp": dict(n=2000, p=500, m=4000),
}


@pytest.mark.parametrize("name", list(CASES))
def test_full_size_solution_satisfies_the_reference_conditions(name):
    d = configs.make(name, **CASES[name])
    solver = qs.Solver("cuda").setup(d.n, d.m, d.p, d.P, d.c, d.A, d.b, d.G, d.h, d.cone.orthant_dim,
                                     len(d.cone.soc_dims), d.cone.soc_dims)
    res = solver.solve()
    assert res.status is SolveStatus.SOLVED
    assert res.factor_count == res.iterations + 1 and res.solve_count == 2 * res.iterations + 2  # test_ipm.py:239-243
    _check_optimality(d, res)


def test_full_size_c4_is_bitwise_reproducible():
    d = configs.make("C4_group_lasso", **CASES["C4_group_lasso"])
    a = qs.solve(d)
    b = qs.solve(d)
    assert a.iterations == b.iterations and a.objective == b.objective
    for k in "xyzs":
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
