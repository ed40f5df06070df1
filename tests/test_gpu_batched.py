"""Batched small-problem mode (qs_batch_*) through the C ABI: every instance of a lockstep batch must
come out exactly as its stand-alone solve (same kernels, same reduction order => bitwise), which is itself checked
against the oracle elsewhere; here additionally against the oracle directly on a few instances."""

import numpy as np
import pytest

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.batched import BatchSolver, solve_batched
from paper_2603_29197_b200.errors import BadSparseStructure
from paper_2603_29197_b200.problem import SolveStatus

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.status is b.status and a.iterations == b.iterations, (a.status, b.status, a.iterations, b.iterations)
    for k in "xyzs":
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.objective == b.objective


@pytest.mark.parametrize("small,count", [(True, 7), (False, 12)])
def test_batch_equals_stand_alone_solves_bitwise(small, count):
    probs = [configs.make("C5_mpc", small=small, seed=i) for i in range(count)]
    got = solve_batched(probs)
    assert len(got) == count
    iters = set()
    for d, r in zip(probs, got):
        ref = qs.solve(d)
        assert ref.status is SolveStatus.SOLVED
        _same(r, ref)
        assert r.factor_count == r.iterations + 1 and r.solve_count == 2 * r.iterations + 2
        iters.add(r.iterations)
    assert got[0].timers["batch_size"] == count


def test_batch_matches_the_oracle(oracle):
    probs = [configs.make("C5_mpc", small=True, seed=100 + i) for i in range(5)]
    for d, r in zip(probs, solve_batched(probs)):
        ref = oracle.solve(d)
        assert r.status is SolveStatus.SOLVED and ref.status == "Solved"
        assert abs(r.iterations - ref.iterations) <= 1
        assert abs(r.objective - ref.objective) <= 1e-6 * max(1.0, abs(ref.objective))
        if r.iterations == ref.iterations:
            assert np.max(np.abs(r.x - ref.x)) <= 1e-5 * max(1.0, np.max(np.abs(ref.x)))


def test_instances_finish_at_different_iterations_and_keep_their_iterate():
    """Different right-hand sides => different iteration counts inside ONE batch: an instance that has converged is
    frozen while the others go on."""
    import dataclasses

    base = [configs.make("C5_mpc", small=True, seed=i) for i in range(6)]
    probs = [dataclasses.replace(d, b=d.b * (1.0 + 30.0 * (i % 3)), c=d.c * (1.0 + 5.0 * (i % 2))) for i, d in enumerate(base)]
    got = solve_batched(probs)
    refs = [qs.solve(d) for d in probs]
    for r, ref in zip(got, refs):
        _same(r, ref)
    assert len({r.iterations for r in refs}) > 1, "the test needs instances with different iteration counts"


def test_partial_batches_slot_reuse_and_chunks():
    probs = [configs.make("C5_mpc", small=True, seed=i) for i in range(9)]
    refs = [qs.solve(d) for d in probs]
    with BatchSolver(probs[0], 4) as bs:
        out = bs.solve(probs[:4]) + bs.solve(probs[4:8]) + bs.solve(probs[8:])  # last call fills 1 of 4 slots
        st = bs.stats()
    for r, ref in zip(out, refs):
        _same(r, ref)
    assert st["gpu_launches"] > 0 and st["slot_bytes"] < 32 * 2**20
    for r, ref in zip(solve_batched(probs, max_batch=4), refs):  # chunked driver
        _same(r, ref)


def test_one_bad_instance_does_not_disturb_the_others():
    import dataclasses

    probs = [configs.make("C5_mpc", small=True, seed=i) for i in range(4)]
    c = probs[2].c.copy()
    c[0] = np.nan
    probs[2] = dataclasses.replace(probs[2], c=c)
    got = solve_batched(probs)
    assert got[2].status is SolveStatus.NUMERICAL_ERROR
    for i in (0, 1, 3):
        _same(got[i], qs.solve(probs[i]))


def test_pattern_mismatch_is_rejected():
    a = configs.make("C5_mpc", small=True, seed=0)
    b = configs.make("C4_group_lasso", small=True, seed=0)
    with BatchSolver(a, 2) as bs:
        with pytest.raises(BadSparseStructure):
            bs.solve([a, b])


def test_solve_shard_picks_the_lockstep_mode_and_falls_back_for_mixed_patterns():
    from paper_2603_29197_b200.batch import solve_shard

    probs = [configs.make("C5_mpc", small=True, seed=i) for i in range(5)]
    recs, mode = solve_shard(probs, device=0)
    assert "lockstep" in mode and [r.index for r in recs] == list(range(5))
    assert all(r.status == "Solved" for r in recs)
    refs = [qs.solve(d) for d in probs]
    assert [r.iterations for r in recs] == [r.iterations for r in refs]
    assert [r.objective for r in recs] == [r.objective for r in refs]
    mixed = probs[:2] + [configs.make("C4_group_lasso", small=True, seed=0)]
    recs, mode = solve_shard(mixed, device=0, workers=2)
    assert "in flight" in mode and all(r.status == "Solved" for r in recs)


@pytest.mark.parametrize("family", ["C4_group_lasso", "C3_portfolio", "C2_lasso", "C1_random_qp"])
def test_batch_of_other_families_exercises_every_front_path(family):
    """Same pattern, different numbers, for the families whose factorisation uses leaf fronts, blocked fronts, DMMA
    Schur updates and the clustered root solves: every batched launch path against the stand-alone solve, bitwise."""
    import dataclasses

    base = configs.make(family, small=True, seed=3)
    rng = np.random.default_rng(5)
    # the cost vector only: feasibility (b = A x0, h = G x0 + s0) stays as generated
    probs = [base] + [dataclasses.replace(base, c=base.c * (1.0 + 0.2 * rng.random(base.c.size))) for _ in range(3)]
    got = solve_batched(probs)
    for d, r in zip(probs, got):
        ref = qs.solve(d)
        assert ref.status is SolveStatus.SOLVED, family
        _same(r, ref)
