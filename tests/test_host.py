"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
the host KKT assembly is bit-exact against the reference's golden fixtures, the
symbolic analysis is structurally valid, and the API boundary validates like
the reference."""

import os
import re
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import _lib, errors
from paper_2603_29197_b200.kkt import assemble_kkt
from paper_2603_29197_b200.problem import ConeSpec, ProblemData, Settings, validate_problem
from paper_2603_29197_b200.sparse import SparseMatrixCSC, as_csc, csc_from_triplets, empty_csc
from util import golden_problem_names, load_golden, problem_from_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "qsocp_cuda.h")).read()
    declared = set(re.findall(r"\b(qs_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in qsocp_cuda.h but not exported"
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    assert lib.qs_version() >= 100


@pytest.mark.parametrize("name", golden_problem_names())
def test_kkt_assembly_bit_exact(name):
    g = load_golden(name)
    k = assemble_kkt(problem_from_golden(g))
    for got, key in ((k.matrix.col_pointers, "K_p"), (k.matrix.row_indices, "K_i"),
                     (k.nt_entry_positions, "nt_entry_positions"), (k.nt_slot_offsets, "nt_slot_offsets"),
                     (k.soc_slot_starts, "soc_slot_starts")):
        assert got.dtype == np.int64 and np.array_equal(got, g[key]), key
    assert np.array_equal(k.matrix.values, g["K_x"])


def test_kkt_assembly_matches_oracle_on_random_mixed_cones(oracle):
    rng = np.random.default_rng(3)
    for _ in range(20):
        n, p = int(rng.integers(1, 30)), int(rng.integers(0, 8))
        l = int(rng.integers(0, 6))
        qsz = tuple(int(v) for v in rng.integers(1, 9, int(rng.integers(0, 5))))
        if l + sum(qsz) == 0:
            l = 1
        m = l + sum(qsz)

        def rnd(r, c, dens, upper=False):
            mask = rng.random((r, c)) < dens
            if upper:
                mask = np.triu(mask)
            rr, cc = np.nonzero(mask)
            v = rng.standard_normal(rr.size)
            v[rng.random(rr.size) < 0.1] = 0.0  # explicit zeros must be kept
            return csc_from_triplets(r, c, (rr, cc, v))

        d = ProblemData(n=n, m=m, p=p, P=rnd(n, n, 0.3, True), c=rng.standard_normal(n), A=rnd(p, n, 0.4),
                        b=rng.standard_normal(p), G=rnd(m, n, 0.3), h=rng.standard_normal(m), cone=ConeSpec(l, qsz))
        a, b = assemble_kkt(d), oracle.assemble_kkt(d)
        assert np.array_equal(a.matrix.col_pointers, b.matrix.col_pointers)
        assert np.array_equal(a.matrix.row_indices, b.matrix.row_indices)
        assert np.array_equal(a.matrix.values, b.matrix.values)
        assert np.array_equal(a.nt_entry_positions, b.nt_entry_positions)
        assert np.array_equal(a.nt_slot_offsets, b.nt_slot_offsets)
        assert np.array_equal(a.soc_slot_starts, b.soc_slot_starts)


def _symbolic(kkt, ordering, cone=None, user_perm=None):
    lib = _lib.load()
    K = kkt.matrix
    N = K.cols
    perm, stats = np.empty(N, np.int64), np.zeros(6)
    if cone is not None and cone.soc_dims:
        dims = np.asarray(cone.soc_dims, np.int64)
        starts = kkt.n + kkt.p + cone.orthant_dim + np.concatenate([[0], np.cumsum(dims)[:-1]])
        starts = np.ascontiguousarray(starts, dtype=np.int64)
        nc = dims.size
    else:
        dims = starts = None
        nc = 0
    up = _lib.i64(user_perm) if user_perm is not None else None
    rc = lib.qs_symbolic_stats(N, _lib.ptr(K.col_pointers), _lib.ptr(K.row_indices), ordering, _lib.ptr(up), nc,
                               _lib.ptr(starts), _lib.ptr(dims), _lib.ptr(perm), _lib.ptr(stats))
    assert rc == 0, lib.qs_global_error()
    return perm, dict(zip(("nsup", "nlevels", "lnz", "flops", "max_nr", "max_ns"), stats))


@pytest.mark.parametrize("name", golden_problem_names())
def test_symbolic_analysis_is_valid_and_counts_match_oracle(oracle, name, monkeypatch):
    monkeypatch.setenv("QS_RELAX", "0")  # exact supernodes: no padded zeros in the count
    g = load_golden(name)
    d = problem_from_golden(g)
    kkt = assemble_kkt(d)
    N = kkt.dim
    for ordering in (0, 1):
        for cone in (None, d.cone):  # with and without the clique (star) compression
            perm, st = _symbolic(kkt, ordering, cone)
            assert np.array_equal(np.sort(perm), np.arange(N)), "not a permutation"
            # entries of L (diagonal included) must equal the simplicial count for the same order
            sym = oracle.symbolic_factor(oracle._csc(kkt.matrix), perm)
            assert int(st["lnz"]) == sym.Li.size + N, (ordering, cone is not None)
            assert 1 <= st["nsup"] <= N and st["max_nr"] <= N


@pytest.mark.parametrize("name", ["portfolio_4", "group_lasso_3", "tv_denoising_8", "soc_slice", "random_3"])
def test_compact_pattern_gives_the_same_analysis(name):
    """qs_setup hands the analysis the KKT pattern WITHOUT the off-diagonal entries of the dense SOC blocks (they
    are implied by the clique ranges; the device writes them, host_setup.cpp: hs_kkt_pattern).  Ordering, supernodes
    and fill must not depend on whether those entries are spelled out."""
    d = problem_from_golden(load_golden(name))
    kkt = assemble_kkt(d)
    K = kkt.matrix
    base = kkt.n + kkt.p + d.cone.orthant_dim
    block_of = np.full(K.cols, -1, np.int64)
    o = base
    for k, q in enumerate(d.cone.soc_dims):
        block_of[o:o + q] = k
        o += q
    cols = np.repeat(np.arange(K.cols), np.diff(K.col_pointers))
    rows = K.row_indices
    keep = ~((block_of[rows] >= 0) & (block_of[rows] == block_of[cols]) & (rows != cols))
    cp = np.concatenate([[0], np.cumsum(np.bincount(cols[keep], minlength=K.cols))]).astype(np.int64)
    compact = SimpleNamespace(matrix=SimpleNamespace(cols=K.cols, col_pointers=cp,
                                                     row_indices=np.ascontiguousarray(rows[keep])),
                              n=kkt.n, p=kkt.p, m=kkt.m)
    for ordering in (0, 1):
        pa, sa = _symbolic(kkt, ordering, d.cone)
        pb, sb = _symbolic(compact, ordering, d.cone)
        assert np.array_equal(pa, pb) and sa == sb, ordering


def test_relaxed_amalgamation_pads_but_never_loses_entries(monkeypatch):
    d = problem_from_golden(load_golden("group_lasso_3"))
    kkt = assemble_kkt(d)
    monkeypatch.setenv("QS_RELAX", "0")
    _, exact = _symbolic(kkt, 1, d.cone)
    monkeypatch.setenv("QS_RELAX", "0.4")
    _, relaxed = _symbolic(kkt, 1, d.cone)
    assert relaxed["nsup"] <= exact["nsup"] and relaxed["lnz"] >= exact["lnz"]
    assert relaxed["lnz"] <= 2.0 * exact["lnz"]


def test_amd_reduces_fill_on_an_arrow_matrix():
    n = 200
    r = np.concatenate([np.zeros(n, np.int64), np.arange(n)])
    c = np.concatenate([np.arange(n), np.arange(n)])
    K = csc_from_triplets(n, n, (np.minimum(r, c), np.maximum(r, c), np.ones(2 * n)))

    KK = SimpleNamespace(matrix=K, n=n, p=0, m=0)
    _, nat = _symbolic(KK, 0)
    _, amd = _symbolic(KK, 1)
    assert nat["lnz"] == n * (n + 1) // 2  # arrow pointing the wrong way fills completely
    assert amd["lnz"] == 2 * n - 1


def test_amd_quality_on_grid_laplacian():
    k = 30
    idx = np.arange(k * k).reshape(k, k)
    r = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel(), idx.ravel()])
    c = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel(), idx.ravel()])
    K = csc_from_triplets(k * k, k * k, (np.minimum(r, c), np.maximum(r, c), np.ones(r.size)))

    KK = SimpleNamespace(matrix=K, n=k * k, p=0, m=0)
    _, nat = _symbolic(KK, 0)
    _, amd = _symbolic(KK, 1)
    assert amd["lnz"] < 0.5 * nat["lnz"], (amd["lnz"], nat["lnz"])


def test_validation_errors_match_reference_types():
    P1 = csc_from_triplets(1, 1, [(0, 0, 1.0)])
    G1 = csc_from_triplets(1, 1, [(0, 0, -1.0)])
    ok = dict(n=1, m=1, p=0, P=P1, c=np.ones(1), A=empty_csc(0, 1), b=np.zeros(0), G=G1, h=np.ones(1), cone=ConeSpec(1))
    validate_problem(ProblemData(**ok))
    with pytest.raises(errors.EmptyCone):
        validate_problem(ProblemData(**{**ok, "m": 0, "G": empty_csc(0, 1), "h": np.zeros(0), "cone": ConeSpec(0)}))
    with pytest.raises(errors.ConeMismatch):
        validate_problem(ProblemData(**{**ok, "cone": ConeSpec(2)}))
    with pytest.raises(errors.DimensionMismatch):
        validate_problem(ProblemData(**{**ok, "c": np.ones(2)}))
    bad = SparseMatrixCSC(2, 2, np.array([0, 1, 2]), np.array([1, 1]), np.ones(2))  # (1,0) is below the diagonal
    with pytest.raises(errors.BadSparseStructure):
        validate_problem(ProblemData(n=2, m=1, p=0, P=bad, c=np.ones(2), A=empty_csc(0, 2), b=np.zeros(0),
                                     G=csc_from_triplets(1, 2, [(0, 0, 1.0)]), h=np.ones(1), cone=ConeSpec(1)))
    with pytest.raises(ValueError):
        Settings(eps_abs=0.0)
    with pytest.raises(ValueError):
        Settings(step_fraction=1.0)


def test_api_surface_and_no_cpu_fallback():
    assert set(qs.BACKENDS) == {"cuda"}
    with pytest.raises(ValueError):
        qs.Solver(algebra="builtin")  # the reference's CPU backends are not shipped: no fallback
    with pytest.raises(errors.NotSetUp):
        qs.Solver("cuda").solve()
    s = qs.Solver("cuda").setup(1, 1, 0, [[1.0]], [1.0], None, [], [[-1.0]], [-1.0], 1, 0, ())
    if _lib.load().qs_device_count() == 0:
        with pytest.raises(errors.CudaUnavailable):
            s.solve()
        # the batched mode and the sharded batch driver fail as loudly: nothing solves on the CPU
        from paper_2603_29197_b200 import configs
        from paper_2603_29197_b200.batch import solve_shard
        from paper_2603_29197_b200.batched import solve_batched

        probs = [configs.make("C5_mpc", small=True, seed=i) for i in range(2)]
        with pytest.raises(errors.CudaUnavailable):
            solve_batched(probs)
        with pytest.raises(errors.CudaUnavailable):
            solve_shard(probs, device=0)


def test_as_csc_accepts_dense_scipy_and_none():
    import scipy.sparse as sp

    M = np.array([[1.0, 0.0], [2.0, 3.0]])
    a, b = as_csc(M, 2, 2), as_csc(sp.csr_matrix(M), 2, 2)
    assert np.array_equal(a.to_dense(), M) and np.array_equal(b.to_dense(), M)
    assert as_csc(None, 0, 3).nnz == 0
