"""Ruiz equilibration (not a reference feature -> "parity unpinned"):
the CUDA kernels against the oracle's independent NumPy restatement, and the
equilibrated solve against the plain one."""

import numpy as np
import pytest

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200.ipm import DeviceSolver
from paper_2603_29197_b200.problem import Settings, SolveStatus
from util import load_golden, problem_from_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["portfolio_4", "group_lasso_3", "huber_20", "random_1", "tv_denoising_8"])
def test_ruiz_scalings_and_solution(oracle, name):
    g = load_golden(name)
    d = problem_from_golden(g)
    dev = DeviceSolver(d, Settings(ruiz_iters=10))
    D, E, F = dev.ruiz_scalings()
    rD, rE, rF = oracle.ruiz_scalings(d, 10)
    assert np.allclose(D, rD, rtol=1e-12) and np.allclose(E, rE, rtol=1e-12) and np.allclose(F, rF, rtol=1e-12)
    starts, dims = oracle.soc_layout(d.cone)
    for o, q in zip(starts, dims):
        assert np.all(F[o:o + q] == F[o])  # one scalar per second-order cone
    status, iters, it = dev.run()
    dev.close()
    assert status is SolveStatus.SOLVED and iters <= int(g["iterations"]) + 5
    obj = float(g["objective"])
    P = d.P
    cols = P.column_of_entry()
    w = np.where(P.row_indices == cols, 0.5, 1.0)
    got = float(np.dot(w * P.values * it.x[P.row_indices], it.x[cols]) + d.c @ it.x)
    assert abs(got - obj) <= 1e-5 * max(1.0, abs(obj))
    # the un-scaled iterate is feasible for the ORIGINAL problem to the solver's tolerance class
    r_eq = oracle.spmv(oracle._csc(d.A), it.x) - d.b
    r_cone = oracle.spmv(oracle._csc(d.G), it.x) + it.s - d.h
    assert np.max(np.abs(r_eq), initial=0.0) <= 1e-5 * (1 + np.max(np.abs(d.b), initial=0.0))
    assert np.max(np.abs(r_cone)) <= 1e-5 * (1 + np.max(np.abs(d.h), initial=0.0) + np.max(np.abs(it.s)))
    assert oracle.interior_violation(it.s, d.cone) < 0 and oracle.interior_violation(it.z, d.cone) < 0


def test_ruiz_off_is_the_default_and_changes_nothing():
    d = problem_from_golden(load_golden("random_0"))
    a = qs.solve(d)
    b = qs.solve(d, Settings(ruiz_iters=0))
    assert np.array_equal(a.x, b.x) and a.iterations == b.iterations
