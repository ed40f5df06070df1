"""Seeded, sparse-native generators for the five BASELINE.json configurations
 and scaled-down variants of each.

The reference's own generators (pkg/src/qsocp/bench/generators.py) draw dense
`rows x cols` masks and cannot reach these sizes; the formulations below follow
them (group lasso: generators.py:286-342) but build every matrix directly in
CSC.  Each generator is a pure function of its arguments (NumPy
`default_rng(seed)`), so the oracle, the reference and the GPU path consume
bit-identical arrays.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .problem import ConeSpec, ProblemData, validate_problem
from .sparse import SparseMatrixCSC


def _to_csc(M, rows, cols) -> SparseMatrixCSC:
    M = sp.csc_matrix(M, shape=(rows, cols))
    M.sort_indices()
    return SparseMatrixCSC(rows, cols, M.indptr.astype(np.int64), M.indices.astype(np.int64),
                           M.data.astype(np.float64))


def _fixed_nnz_columns(rng, rows, cols, k):
    """rows x cols matrix with exactly k distinct N(0,1) entries per column."""
    k = min(k, rows)
    gaps = rng.integers(1, max(rows // k, 1) + 1, size=(cols, k))
    idx = (rng.integers(0, rows, size=(cols, 1)) + np.cumsum(gaps, axis=1)) % rows
    idx.sort(axis=1)
    vals = rng.standard_normal((cols, k))
    return sp.csc_matrix((vals.ravel(), idx.ravel(), np.arange(0, cols * k + 1, k)), shape=(rows, cols))


def _interior(cone: ConeSpec, rng, lo=0.1, hi=1.1):
    u = rng.standard_normal(cone.total_dim)
    l = cone.orthant_dim
    u[:l] = rng.uniform(lo, hi, l)
    dims = np.asarray(cone.soc_dims, dtype=np.int64)
    if dims.size:
        starts = l + np.concatenate([[0], np.cumsum(dims)[:-1]])
        sq = u * u
        sq[:l] = 0.0
        sq[starts] = 0.0
        u[starts] = np.sqrt(np.add.reduceat(sq, starts)) + rng.uniform(lo, hi, dims.size)
    return u


def random_qp(n=2000, p=500, m=4000, density=0.01, seed=0) -> ProblemData:
    """C1: random sparse QP with orthant cones (the reference's CPU test scale)."""
    rng = np.random.default_rng(seed)
    rs = np.random.RandomState(seed)
    M = sp.random(n, n, density=density / 2, random_state=rs, data_rvs=rs.standard_normal, format="csc")
    P = sp.triu(M.T @ M + 0.01 * sp.identity(n), format="csc")
    A = sp.random(p, n, density=density, random_state=rs, data_rvs=rs.standard_normal, format="csc")
    G = sp.random(m, n, density=density, random_state=rs, data_rvs=rs.standard_normal, format="csc")
    cone = ConeSpec(m)
    x0, s0 = rng.standard_normal(n), _interior(cone, rng)
    return validate_problem(ProblemData(n=n, m=m, p=p, P=_to_csc(P, n, n), c=rng.standard_normal(n),
                                        A=_to_csc(A, p, n), b=A @ x0, G=_to_csc(G, m, n), h=G @ x0 + s0, cone=cone))


def lasso(features=100_000, samples=20_000, nnz_per_col=10, seed=0) -> ProblemData:
    """C2: min |r|^2 + lam 1't  s.t.  X beta - r = y,  -t <= beta <= t   over (beta, r, t)."""
    rng = np.random.default_rng(seed)
    nf, ns = features, samples
    X = _fixed_nnz_columns(rng, ns, nf, nnz_per_col)
    beta = np.where(rng.random(nf) < 0.01, rng.standard_normal(nf), 0.0)
    y = X @ beta + 0.1 * rng.standard_normal(ns)
    lam = 0.1 * float(np.max(np.abs(X.T @ y)))
    n = 2 * nf + ns
    I_f, I_s = sp.identity(nf, format="csc"), sp.identity(ns, format="csc")
    P = sp.block_diag([sp.csc_matrix((nf, nf)), 2.0 * I_s, sp.csc_matrix((nf, nf))], format="csc")
    A = sp.hstack([X, -I_s, sp.csc_matrix((ns, nf))], format="csc")
    G = sp.vstack([sp.hstack([I_f, sp.csc_matrix((nf, ns)), -I_f]),
                   sp.hstack([-I_f, sp.csc_matrix((nf, ns)), -I_f])], format="csc")
    c = np.concatenate([np.zeros(nf + ns), np.full(nf, lam)])
    m = 2 * nf
    return validate_problem(ProblemData(n=n, m=m, p=ns, P=_to_csc(P, n, n), c=c, A=_to_csc(A, ns, n), b=y,
                                        G=_to_csc(G, m, n), h=np.zeros(m), cone=ConeSpec(m)))


def portfolio(assets=100_000, factors=100, sector=100, gamma=1.0, seed=0) -> ProblemData:
    """C3: factor-model portfolio with per-sector risk cones.
    min -mu'x + gamma (t_f^2 + sum_g t_g^2)  s.t.  y = F'x, 1'x = 1, x >= 0,
    (t_f, y) in SOC(k+1), (t_g, D_g^(1/2) x_g) in SOC(sector+1)   over (x, y, t_f, t_g)."""
    rng = np.random.default_rng(seed)
    na, k = assets, factors
    ng = na // sector
    na = ng * sector
    F = _fixed_nnz_columns(rng, na, k, max(na // 10, 1)) * 0.1  # assets x factors, 10 % dense
    D = rng.uniform(0.05, 1.0, na)
    mu = rng.uniform(0.0, 0.1, na)
    n = na + k + 1 + ng
    ox, oy, otf, otg = 0, na, na + k, na + k + 1
    P = sp.diags(np.concatenate([np.zeros(na + k), np.full(1 + ng, 2.0 * gamma)]), format="csc")
    c = np.concatenate([-mu, np.zeros(k + 1 + ng)])
    A = sp.vstack([sp.hstack([F.T, -sp.identity(k), sp.csc_matrix((k, 1 + ng))]),
                   sp.hstack([np.ones((1, na)), sp.csc_matrix((1, k + 1 + ng))])], format="csc")
    b = np.concatenate([np.zeros(k), [1.0]])
    # G x + s = h with h = 0: s = -G x
    rows, cols, vals = [np.arange(na)], [ox + np.arange(na)], [-np.ones(na)]          # x >= 0
    r0 = na
    rows += [np.array([r0]), r0 + 1 + np.arange(k)]                                      # (t_f, y)
    cols += [np.array([otf]), oy + np.arange(k)]
    vals += [np.array([-1.0]), -np.ones(k)]
    r0 += k + 1
    g = np.arange(ng)
    head = r0 + g * (sector + 1)
    rows += [head, (head[:, None] + 1 + np.arange(sector)[None, :]).ravel()]            # (t_g, D^(1/2) x_g)
    cols += [otg + g, ox + np.arange(na)]
    vals += [-np.ones(ng), -np.sqrt(D)]
    m = na + (k + 1) + ng * (sector + 1)
    G = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(m, n))
    cone = ConeSpec(na, (k + 1,) + (sector + 1,) * ng)
    return validate_problem(ProblemData(n=n, m=m, p=k + 1, P=_to_csc(P, n, n), c=c, A=_to_csc(A, k + 1, n), b=b,
                                        G=_to_csc(G, m, n), h=np.zeros(m), cone=cone))


def group_lasso(groups=10_000, qlo=20, qhi=250, samples=5_000, nnz_per_col=10, seed=0) -> ProblemData:
    """C4: min r.r + lam sum t_k  s.t.  X beta - r = y, (t_k, beta_k) in SOC(q_k)   over (beta, r, t);
    the reference's epigraph form (generators.py:286-342) with group sizes q_k - 1, q_k ~ U{qlo..qhi}."""
    rng = np.random.default_rng(seed)
    q = rng.integers(qlo, qhi + 1, groups)
    gs = q - 1
    nf, ns = int(gs.sum()), samples
    X = _fixed_nnz_columns(rng, ns, nf, nnz_per_col)
    active = np.repeat(rng.random(groups) < 0.5, gs)
    beta = np.where(active, rng.standard_normal(nf), 0.0)
    y = X @ beta + 0.1 * rng.standard_normal(ns)
    lam = 0.1 * float(np.max(np.abs(X.T @ y)))
    n = nf + ns + groups
    r_off, t_off = nf, nf + ns
    P = sp.diags(np.concatenate([np.zeros(nf), np.full(ns, 2.0), np.zeros(groups)]), format="csc")
    c = np.concatenate([np.zeros(nf + ns), np.full(groups, lam)])
    A = sp.hstack([X, -sp.identity(ns), sp.csc_matrix((ns, groups))], format="csc")
    starts = np.concatenate([[0], np.cumsum(q)[:-1]])
    tail_rows = np.arange(int(q.sum()))
    tail_rows = np.delete(tail_rows, starts)  # every conic row that is not a head, in order
    m = int(q.sum())
    G = sp.csc_matrix((-np.ones(groups + nf), (np.concatenate([starts, tail_rows]),
                                              np.concatenate([t_off + np.arange(groups), np.arange(nf)]))),
                      shape=(m, n))
    cone = ConeSpec(0, tuple(int(v) for v in q))
    return validate_problem(ProblemData(n=n, m=m, p=ns, P=_to_csc(P, n, n), c=c, A=_to_csc(A, ns, n), b=y,
                                        G=_to_csc(G, m, n), h=np.zeros(m), cone=cone))


def mpc(horizon=50, nx=12, nu=4, seed=0) -> ProblemData:
    """C5 instance: min sum x_t'x_t + 0.1 u_t'u_t  s.t.  x_{t+1} = A x_t + B u_t, |x_t|_inf <= 5, |u_t|_2 <= 1."""
    rng = np.random.default_rng(seed)
    T = horizon
    Ad = rng.standard_normal((nx, nx))
    Ad *= 0.95 / np.max(np.abs(np.linalg.eigvals(Ad)))
    Bd = rng.standard_normal((nx, nu)) / np.sqrt(nx)
    xinit = rng.standard_normal(nx)
    n = T * nx + T * nu  # (x_1..x_T, u_0..u_{T-1})
    ox, ou = 0, T * nx
    P = sp.diags(np.concatenate([np.full(T * nx, 2.0), np.full(T * nu, 0.2)]), format="csc")
    # x_{t+1} - A x_t - B u_t = 0   (x_0 = xinit moves to the right-hand side)
    Ax = sp.identity(T * nx) - sp.kron(sp.diags([np.ones(T - 1)], [-1]), Ad)
    A = sp.hstack([Ax, -sp.kron(sp.identity(T), Bd)], format="csc")
    b = np.concatenate([Ad @ xinit, np.zeros((T - 1) * nx)])
    Ix = sp.identity(T * nx)
    box = sp.vstack([sp.hstack([Ix, sp.csc_matrix((T * nx, T * nu))]),
                     sp.hstack([-Ix, sp.csc_matrix((T * nx, T * nu))])])
    rows = (np.arange(T)[:, None] * (nu + 1) + 1 + np.arange(nu)[None, :]).ravel()
    soc = sp.csc_matrix((-np.ones(T * nu), (rows, ou + np.arange(T * nu))), shape=(T * (nu + 1), n))
    G = sp.vstack([box, soc], format="csc")
    hs = np.zeros(T * (nu + 1))
    hs[:: nu + 1] = 1.0
    h = np.concatenate([np.full(2 * T * nx, 5.0), hs])
    m = 2 * T * nx + T * (nu + 1)
    cone = ConeSpec(2 * T * nx, (nu + 1,) * T)
    return validate_problem(ProblemData(n=n, m=m, p=T * nx, P=_to_csc(P, n, n), c=np.zeros(n), A=_to_csc(A, T * nx, n),
                                        b=b, G=_to_csc(G, m, n), h=h, cone=cone))


# name -> (generator, kwargs at BASELINE size, kwargs of the small CI variant)
CONFIGS = {
    "C1_random_qp": (random_qp, dict(n=2000, p=500, m=4000), dict(n=200, p=50, m=400, density=0.05)),
    "C2_lasso": (lasso, dict(features=100_000, samples=20_000), dict(features=2000, samples=400)),
    "C3_portfolio": (portfolio, dict(assets=100_000, factors=100, sector=100), dict(assets=2000, factors=10, sector=20)),
    "C4_group_lasso": (group_lasso, dict(groups=10_000, qlo=20, qhi=250, samples=5_000),
                       dict(groups=60, qlo=3, qhi=40, samples=150)),
    "C5_mpc": (mpc, dict(horizon=50, nx=12, nu=4), dict(horizon=8, nx=4, nu=2)),
}


def make(name: str, small: bool = False, seed: int = 0, **override) -> ProblemData:
    gen, full, tiny = CONFIGS[name]
    kw = dict(tiny if small else full)
    kw.update(override)
    return gen(seed=seed, **kw)


def kkt_nnz(d: ProblemData) -> int:
    """Stored entries of the upper-triangular KKT matrix (kkt.py:55-135)."""
    diag_missing = d.n - int(np.count_nonzero(d.P.row_indices == d.P.column_of_entry()))
    blocks = d.cone.orthant_dim + sum(q * (q + 1) // 2 for q in d.cone.soc_dims)
    return d.P.nnz + diag_missing + d.A.nnz + d.p + d.G.nnz + blocks
