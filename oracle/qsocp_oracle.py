"""ORACLE -- TEST INFRASTRUCTURE ONLY (never imported by the product package).

CPU restatement of the reference interior-point solver (`qsocp`, Python +
numba) used as the parity checker for the CUDA path and as the timed
``cpu_baseline`` ("port") in bench.py.  Numeric loops live in
``qsocp_oracle.c`` (plain C, compiled by ``oracle/Makefile`` without FMA
contraction); this file is the NumPy driver around them and follows the
reference function by function -- every function cites the reference lines it
restates (paths relative to /root/reference/pkg/src/qsocp/).

Parity status: PINNED -- see tests/test_oracle_pinned.py (direct comparison
with the imported reference when /root/reference exists) and tests/golden/
(fixtures produced by the reference through oracle/gen_golden.py).

The oracle is self-contained: it never imports the product package nor loads
libqsocp_cuda.so.  The fill-reducing ordering is the reference's own AMD
(`_amd.py`), restated in ``qsocp_oracle_amd.c`` and pinned element by element
against the reference's permutation, so ``solve(data)`` with no arguments is
the reference's ``solve(data)`` bit for bit.  A permutation can still be
handed in (``perm=``) -- e.g. an ordering computed elsewhere and stored in a
problem file -- which changes fill and rounding only, never the algorithm.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
STEP_UNBOUNDED = float(np.finfo(np.float64).max)  # _cone_kernels.py:13
DYN_REG_EPS = 1e-14  # ldl.py:18
REFINE_STOP_TOL = 1e-12  # ldl.py:19
TINY_STEP = 1e-10  # ipm.py:24
MAX_CONSECUTIVE_STALLS = 3  # ipm.py:25

_i64 = np.int64
_f64 = np.float64


_SRC = ("qsocp_oracle.c", "qsocp_oracle_amd.c")


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in _SRC]
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(f) for f in srcs):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", _SO, *srcs, "-lm"]
        )
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.orc_soc_max_step.restype = ctypes.c_double
        L.orc_soc_violation.restype = ctypes.c_double
        L.orc_ldl_factor.restype = ctypes.c_int64
        L.orc_amd_kernel.restype = ctypes.c_int64
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _c64(v):
    return ctypes.c_int64(int(v))


def _vec(a):
    return np.ascontiguousarray(a, dtype=_f64)


# ------------------------------------------------------------------ cones ----
def soc_layout(cone):
    """(starts, dims) of the SOC blocks inside a flat conic vector (cones.py:52-58)."""
    dims = np.asarray(cone.soc_dims, dtype=_i64)
    starts = np.zeros(dims.size, dtype=_i64)
    if dims.size:
        starts[0] = cone.orthant_dim
        starts[1:] = cone.orthant_dim + np.cumsum(dims)[:-1]
    return starts, dims


def cone_degree(cone) -> int:  # cones.py:61-63
    return cone.orthant_dim + len(cone.soc_dims)


def cone_identity(cone) -> np.ndarray:  # cones.py:66-71
    e = np.zeros(cone.orthant_dim + int(sum(cone.soc_dims)))
    e[: cone.orthant_dim] = 1.0
    e[soc_layout(cone)[0]] = 1.0
    return e


@dataclass
class Scaling:  # cones.py:120-143
    cone: object
    w_orthant: np.ndarray
    soc_eta: np.ndarray
    soc_wbar: np.ndarray
    lam: np.ndarray


class NotInterior(ValueError):
    pass


class NumericalError(ArithmeticError):
    pass


def identity_scaling(cone) -> Scaling:  # cones.py:146-156
    e = cone_identity(cone)
    wbar = e.copy()
    wbar[: cone.orthant_dim] = 0.0
    return Scaling(cone, np.ones(cone.orthant_dim), np.ones(len(cone.soc_dims)), wbar, e)


def compute_nt_scaling(s, z, cone) -> Scaling:  # cones.py:159-184
    s, z = _vec(s), _vec(z)
    l, m = cone.orthant_dim, s.size
    sc = Scaling(cone, np.empty(l), np.empty(len(cone.soc_dims)), np.zeros(m), np.empty(m))
    if l:
        so, zo = s[:l], z[:l]
        if np.any(so <= 0.0) or np.any(zo <= 0.0):
            raise NotInterior("orthant coordinate not strictly positive")
        sc.w_orthant[:] = np.sqrt(so / zo)
        sc.lam[:l] = np.sqrt(so * zo)
    starts, dims = soc_layout(cone)
    if dims.size:
        flag = lib().orc_soc_nt_scaling(_p(s), _p(z), _p(starts), _p(dims), _c64(dims.size),
                                        _p(sc.soc_eta), _p(sc.soc_wbar), _p(sc.lam))
        if flag:
            raise NotInterior("point on or outside a second-order cone")
    return sc


def apply_scaling(sc: Scaling, u, inverse: bool = False) -> np.ndarray:  # cones.py:192-212
    u = _vec(u)
    l = sc.cone.orthant_dim
    out = np.empty_like(u)
    if l:
        out[:l] = u[:l] / sc.w_orthant if inverse else u[:l] * sc.w_orthant
    starts, dims = soc_layout(sc.cone)
    if dims.size:
        lib().orc_soc_apply_w(_p(sc.soc_eta), _p(sc.soc_wbar), _p(starts), _p(dims),
                              _c64(dims.size), _p(u), _p(out), ctypes.c_int(int(inverse)))
    return out


def jordan_product(u, v, cone) -> np.ndarray:  # cones.py:215-228
    u, v = _vec(u), _vec(v)
    l = cone.orthant_dim
    out = np.empty(u.size)
    if l:
        out[:l] = u[:l] * v[:l]
    starts, dims = soc_layout(cone)
    if dims.size:
        lib().orc_soc_jordan(_p(u), _p(v), _p(out), _p(starts), _p(dims), _c64(dims.size))
    return out


def jordan_divide(lam, v, cone) -> np.ndarray:  # cones.py:231-244
    lam, v = _vec(lam), _vec(v)
    l = cone.orthant_dim
    out = np.empty(lam.size)
    if l:
        out[:l] = v[:l] / lam[:l]
    starts, dims = soc_layout(cone)
    if dims.size:
        lib().orc_soc_jordan_div(_p(lam), _p(v), _p(out), _p(starts), _p(dims), _c64(dims.size))
    return out


def interior_violation(u, cone) -> float:  # cones.py:275-290
    u = _vec(u)
    worst = -np.inf
    if cone.orthant_dim:
        worst = float(-np.min(u[: cone.orthant_dim]))
    starts, dims = soc_layout(cone)
    if dims.size:
        v = lib().orc_soc_violation(_p(u), _p(starts), _p(dims), _c64(dims.size))
        if v > worst:
            worst = v
    return worst


def max_step_to_boundary(u, du, cone) -> float:  # cones.py:247-272
    u, du = _vec(u), _vec(du)
    if not interior_violation(u, cone) < 0.0:  # check_interior, cones.py:297-299
        raise NotInterior("point is not strictly inside the cone")
    l = cone.orthant_dim
    best = STEP_UNBOUNDED
    if l:
        uo, do = u[:l], du[:l]
        neg = do < 0.0
        if np.any(neg):
            best = float(np.min(-uo[neg] / do[neg]))
    starts, dims = soc_layout(cone)
    if dims.size:
        st = lib().orc_soc_max_step(_p(u), _p(du), _p(starts), _p(dims), _c64(dims.size))
        if st < best:
            best = st
    return best


def bring_to_interior(u, cone) -> np.ndarray:  # cones.py:302-311
    alpha = interior_violation(u, cone)
    if alpha < 0.0:
        return np.array(u, dtype=_f64)
    return u + (1.0 + alpha) * cone_identity(cone)


def compute_mu(s, z, cone) -> float:  # cones.py:314-316
    return float(np.dot(s, z)) / cone_degree(cone)


def neg_wtw_values(sc: Scaling, slot_starts_soc, out) -> None:  # cones.py:319-336
    l = sc.cone.orthant_dim
    if l:
        out[:l] = -(sc.w_orthant * sc.w_orthant)
    starts, dims = soc_layout(sc.cone)
    if dims.size:
        ss = np.ascontiguousarray(slot_starts_soc, dtype=_i64)
        lib().orc_soc_neg_wtw(_p(sc.soc_eta), _p(sc.soc_wbar), _p(starts), _p(dims),
                              _c64(dims.size), _p(ss), _p(out))


# ----------------------------------------------------------------- sparse ----
def _csc(M):
    return SimpleNamespace(
        rows=M.rows, cols=M.cols,
        col_pointers=np.ascontiguousarray(M.col_pointers, dtype=_i64),
        row_indices=np.ascontiguousarray(M.row_indices, dtype=_i64),
        values=np.ascontiguousarray(M.values, dtype=_f64),
    )


def csc_from_triplets(rows, cols, r, c, v):
    """sparse.py:83-116 (lexsort by (col,row), stable; duplicates summed in
    input order; explicit zeros kept)."""
    r = np.asarray(r, dtype=_i64)
    c = np.asarray(c, dtype=_i64)
    v = np.asarray(v, dtype=_f64)
    order = np.lexsort((r, c))
    r, c, v = r[order], c[order], v[order]
    if r.size:
        keep = np.ones(r.size, dtype=bool)
        keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        vals = np.zeros(int(keep.sum()))
        np.add.at(vals, np.cumsum(keep) - 1, v)
        r, c = r[keep], c[keep]
    else:
        vals = v
    ptr = np.zeros(cols + 1, dtype=_i64)
    np.add.at(ptr, c + 1, 1)
    np.cumsum(ptr, out=ptr)
    return SimpleNamespace(rows=rows, cols=cols, col_pointers=ptr, row_indices=r, values=vals)


def spmv(M, x, transpose=False) -> np.ndarray:  # sparse.py:119-140
    x = _vec(x)
    out = np.zeros(M.cols if transpose else M.rows)
    fn = lib().orc_csc_matvec_t if transpose else lib().orc_csc_matvec
    fn(_c64(M.cols), _p(M.col_pointers), _p(M.row_indices), _p(M.values), _p(x), _p(out))
    return out


def spmv_sym_upper(M, x) -> np.ndarray:  # sparse.py:143-150
    x = _vec(x)
    out = np.zeros(M.rows)
    lib().orc_csc_sym_upper_matvec(_c64(M.cols), _p(M.col_pointers), _p(M.row_indices),
                                   _p(M.values), _p(x), _p(out))
    return out


def symmetric_permute(K, fwd):  # sparse.py:180-208
    n = K.cols
    inv = np.empty(n, dtype=_i64)
    inv[fwd] = np.arange(n, dtype=_i64)
    src_col = np.repeat(np.arange(n, dtype=_i64), np.diff(K.col_pointers))
    nr, nc = inv[K.row_indices], inv[src_col]
    lo, hi = np.minimum(nr, nc), np.maximum(nr, nc)
    order = np.lexsort((lo, hi))
    emap = np.empty(order.size, dtype=_i64)
    emap[order] = np.arange(order.size, dtype=_i64)
    ptr = np.zeros(n + 1, dtype=_i64)
    np.add.at(ptr, hi + 1, 1)
    np.cumsum(ptr, out=ptr)
    return SimpleNamespace(rows=n, cols=n, col_pointers=ptr,
                           row_indices=np.ascontiguousarray(lo[order]),
                           values=K.values[order]), emap


# -------------------------------------------------------------------- kkt ----
@dataclass
class KKT:  # kkt.py:26-39
    matrix: object
    nt_entry_positions: np.ndarray
    nt_slot_offsets: np.ndarray
    soc_slot_starts: np.ndarray
    n: int
    p: int
    m: int


def _block_pattern(n, p, cone):
    """(rows, cols, identity values) of the scaling block in slot order
    (kkt.py:84-99 pattern, kkt.py:113-125 slot order: orthant diagonal, then per
    SOC the packed upper triangle column by column)."""
    l = cone.orthant_dim
    starts, dims = soc_layout(cone)
    base = n + p
    rr = [base + np.arange(l, dtype=_i64)]
    cc = [base + np.arange(l, dtype=_i64)]
    vv = [np.full(l, -1.0)]
    for o, d in zip(starts.tolist(), dims.tolist()):
        jj = np.repeat(np.arange(d, dtype=_i64), np.arange(1, d + 1))
        first = np.cumsum(np.arange(d, dtype=_i64))  # slot of (0, j)
        ii = np.arange(jj.size, dtype=_i64) - first[jj]
        rr.append(base + o + ii)
        cc.append(base + o + jj)
        vv.append(np.where(ii == jj, -1.0, 0.0))
    return np.concatenate(rr), np.concatenate(cc), np.concatenate(vv)


def assemble_kkt(data) -> KKT:  # kkt.py:55-135
    n, p, m = data.n, data.p, data.m
    P, A, G = _csc(data.P), _csc(data.A), _csc(data.G)
    colsP = np.repeat(np.arange(n, dtype=_i64), np.diff(P.col_pointers))
    colsA = np.repeat(np.arange(n, dtype=_i64), np.diff(A.col_pointers))
    colsG = np.repeat(np.arange(n, dtype=_i64), np.diff(G.col_pointers))
    dnp = np.arange(n + p, dtype=_i64)
    br, bc, bv = _block_pattern(n, p, data.cone)
    rows = np.concatenate([P.row_indices, dnp, colsA, colsG, br])
    cols = np.concatenate([colsP, dnp, A.row_indices + n, G.row_indices + n + p, bc])
    vals = np.concatenate([P.values, np.zeros(n + p), A.values, G.values, bv])
    K = csc_from_triplets(n + p + m, n + p + m, rows, cols, vals)
    pos = np.empty(br.size, dtype=_i64)
    rc = lib().orc_entry_positions(_p(K.col_pointers), _p(K.row_indices), _c64(br.size),
                                   _p(np.ascontiguousarray(br)), _p(np.ascontiguousarray(bc)), _p(pos))
    if rc:
        raise RuntimeError("scaling entry missing from the assembled pattern")
    l = data.cone.orthant_dim
    _, dims = soc_layout(data.cone)
    counts = ([l] if l > 0 else []) + [d * (d + 1) // 2 for d in dims.tolist()]
    offsets = np.zeros(len(counts) + 1, dtype=_i64)
    np.cumsum(np.asarray(counts, dtype=_i64), out=offsets[1:])
    soc_starts = offsets[(1 if l > 0 else 0):-1].copy() if dims.size else np.zeros(0, dtype=_i64)
    return KKT(K, pos, offsets, soc_starts, n, p, m)


def write_scaling(kkt: KKT, sc: Scaling) -> None:  # kkt.py:146-150
    slots = np.empty(kkt.nt_entry_positions.size)
    neg_wtw_values(sc, kkt.soc_slot_starts, slots)
    kkt.matrix.values[kkt.nt_entry_positions] = slots


# -------------------------------------------------------------------- ldl ----
def amd_order(n, col_ptr, row_idx, heap_words=None) -> np.ndarray:  # _amd.py:393-419
    """AMD permutation of a symmetric pattern given by its upper triangle: builds
    A + A' without the diagonal (rows of every column in the order the reference's
    stable argsort leaves them) and runs the C restatement of `_amd_kernel`."""
    if n == 0:
        return np.empty(0, dtype=_i64)
    col_ptr = np.asarray(col_ptr, dtype=_i64)
    cols = np.repeat(np.arange(n, dtype=_i64), np.diff(col_ptr))
    rows = np.asarray(row_idx, dtype=_i64)
    off = rows != cols
    rows, cols = rows[off], cols[off]
    counts = np.bincount(rows, minlength=n) + np.bincount(cols, minlength=n)
    cnz = int(counts.sum())
    nzmax = cnz + cnz // 5 + 8 * n + 16
    Cp = np.zeros(n + 2, dtype=_i64)
    np.cumsum(counts, out=Cp[1:n + 1])
    Ci = np.empty(nzmax, dtype=_i64)
    rr = np.concatenate([rows, cols])
    cc = np.concatenate([cols, rows])
    del rows, cols
    Ci[:cnz] = rr[np.argsort(cc, kind="stable")]
    del rr, cc
    # the reference's heap has 4*cnz+4n+64 words; the pivot sequence does not depend on the capacity
    # (a full heap is compacted to its live keys), so very large patterns may use less memory
    cap = max(4 * cnz + 4 * n + 64, 1024) if heap_words is None else max(int(heap_words), 2 * n + 64)
    heap = np.empty(cap, dtype=_i64)
    seen = np.zeros(n + 1, dtype=_i64)
    order = np.empty(n, dtype=_i64)
    got = lib().orc_amd_kernel(_c64(n), _p(Cp), _p(Ci), _c64(nzmax), _c64(cnz), _p(heap), _c64(cap),
                               _p(seen), _p(order))
    if got != n:
        raise RuntimeError("ordering failed to converge")
    return order


def default_perm(K, kkt=None, cone=None) -> np.ndarray:
    """sparse.py:205-222 (`fill_reducing_order(..., "amd")`): the reference's AMD on the full KKT pattern."""
    cnz2 = 2 * int(K.col_pointers[-1])
    return amd_order(K.cols, K.col_pointers, K.row_indices,
                     heap_words=None if cnz2 < 50_000_000 else cnz2 // 2 + 4 * K.cols + 64)


@dataclass
class Symbolic:  # ldl.py:22-38
    fwd: np.ndarray
    etree: np.ndarray
    Lp: np.ndarray
    Li: np.ndarray
    permuted: object
    entry_map: np.ndarray

    @property
    def n(self):
        return self.etree.size


def symbolic_factor(K, fwd) -> Symbolic:  # ldl.py:48-69
    n = K.cols
    fwd = np.ascontiguousarray(fwd, dtype=_i64)
    perm, emap = symmetric_permute(K, fwd)
    parent = np.empty(n, dtype=_i64)
    lnz = np.empty(n, dtype=_i64)
    work = np.empty(n, dtype=_i64)
    if lib().orc_etree_and_counts(_c64(n), _p(perm.col_pointers), _p(perm.row_indices),
                                  _p(parent), _p(lnz), _p(work)):
        raise ValueError("pattern is not upper triangular")
    Lp = np.zeros(n + 1, dtype=_i64)
    np.cumsum(lnz, out=Lp[1:])
    Li = np.empty(int(Lp[n]), dtype=_i64)
    w1, w2, w3 = (np.empty(n, dtype=_i64) for _ in range(3))
    lib().orc_ldl_pattern(_c64(n), _p(perm.col_pointers), _p(perm.row_indices), _p(parent),
                          _p(Lp), _p(Li), _p(w1), _p(w2), _p(w3))
    return Symbolic(fwd, parent, Lp, Li, perm, emap)


def reg_signs(n, p, m) -> np.ndarray:  # kkt.py:48-52
    s = np.ones(n + p + m, dtype=_i64)
    s[n:] = -1
    return s


def numeric_factor(K_values, sym: Symbolic, static_reg, signs):  # ldl.py:72-122
    n = sym.n
    sg = np.ascontiguousarray(signs[sym.fwd], dtype=_i64)
    pv = np.empty(sym.entry_map.size)
    pv[sym.entry_map] = K_values
    sd = static_reg * sg.astype(_f64)
    D = np.empty(n)
    Lx = np.zeros(sym.Li.size)
    yv = np.empty(n)
    w = [np.empty(n, dtype=_i64) for _ in range(4)]
    bumps = lib().orc_ldl_factor(
        _c64(n), _p(sym.permuted.col_pointers), _p(sym.permuted.row_indices), _p(pv), _p(sym.etree),
        _p(sym.Lp), _p(sym.Li), _p(Lx), _p(D), _p(sd), ctypes.c_double(DYN_REG_EPS), _p(sg),
        _p(yv), _p(w[0]), _p(w[1]), _p(w[2]), _p(w[3]))
    if bumps < 0:
        raise NumericalError("non-finite pivot during LDL^T factorization")
    return SimpleNamespace(Lx=Lx, D=D, bumps=int(bumps))


def backsolve(fac, sym: Symbolic, rhs) -> np.ndarray:  # ldl.py:125-132
    x = np.ascontiguousarray(rhs[sym.fwd], dtype=_f64)
    lib().orc_ldl_solve_inplace(_c64(sym.n), _p(sym.Lp), _p(sym.Li), _p(fac.Lx), _p(fac.D), _p(x))
    out = np.empty_like(x)
    out[sym.fwd] = x
    return out


def solve_refine(fac, sym, K, rhs, refine_iters) -> np.ndarray:  # ldl.py:135-166
    rhs = _vec(rhs)
    x = backsolve(fac, sym, rhs)
    if not np.all(np.isfinite(x)):
        raise NumericalError("non-finite triangular solve result")
    if refine_iters <= 0:
        return x
    stop = REFINE_STOP_TOL * (1.0 + np.max(np.abs(rhs), initial=0.0))
    r = rhs - spmv_sym_upper(K, x)
    rn = np.max(np.abs(r), initial=0.0)
    for _ in range(refine_iters):
        if rn <= stop:
            break
        xn = x + backsolve(fac, sym, r)
        r2 = rhs - spmv_sym_upper(K, xn)
        rn2 = np.max(np.abs(r2), initial=0.0)
        if not np.isfinite(rn2):
            raise NumericalError("non-finite refinement residual")
        if rn2 >= rn:
            break
        x, r, rn = xn, r2, rn2
    return x


class Backend:  # linsys.py:54-108 (BuiltinBackend)
    def __init__(self, kkt: KKT, settings, perm=None, cone=None):
        self.kkt, self.settings = kkt, settings
        self.n_factor = self.n_solve = 0
        t = time.perf_counter()
        fwd = default_perm(kkt.matrix, kkt, cone) if perm is None else np.asarray(perm, dtype=_i64)
        self.sym = symbolic_factor(kkt.matrix, fwd)
        self.analysis_seconds = time.perf_counter() - t
        self.signs = reg_signs(kkt.n, kkt.p, kkt.m)
        self.fac = None
        self.t_factor = self.t_solve = 0.0

    def update(self, sc):
        write_scaling(self.kkt, sc)

    def factor(self):
        t = time.perf_counter()
        self.fac = numeric_factor(self.kkt.matrix.values, self.sym, self.settings.static_reg, self.signs)
        self.t_factor += time.perf_counter() - t
        self.n_factor += 1

    def solve(self, rhs):
        t = time.perf_counter()
        out = solve_refine(self.fac, self.sym, self.kkt.matrix, rhs, self.settings.refine_iters)
        self.t_solve += time.perf_counter() - t
        if not np.all(np.isfinite(out)):
            raise NumericalError("non-finite linear-system solution")
        self.n_solve += 1
        return out


# -------------------------------------------------------------------- ipm ----
@dataclass
class Iterate:  # ipm.py:28-37
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    s: np.ndarray
    mu: float


def _inf(v) -> float:
    return float(np.max(np.abs(v), initial=0.0))


def compute_residuals(data, it):  # ipm.py:70-103
    Px = spmv_sym_upper(data.P, it.x)
    Aty = spmv(data.A, it.y, True)
    Gtz = spmv(data.G, it.z, True)
    Ax = spmv(data.A, it.x)
    Gx = spmv(data.G, it.x)
    r = SimpleNamespace(
        r_dual=Px + data.c + Aty + Gtz, r_eq=Ax - data.b, r_cone=Gx + it.s - data.h,
        gap=float(np.dot(it.s, it.z)),
        objective_primal=0.5 * float(np.dot(it.x, Px)) + float(np.dot(data.c, it.x)),
        norm_Px=_inf(Px), norm_Aty=_inf(Aty), norm_Gtz=_inf(Gtz), norm_c=_inf(data.c),
        norm_Ax=_inf(Ax), norm_b=_inf(data.b), norm_Gx=_inf(Gx), norm_h=_inf(data.h))
    if not (np.all(np.isfinite(r.r_dual)) and np.all(np.isfinite(r.r_eq))
            and np.all(np.isfinite(r.r_cone)) and np.isfinite(r.gap)):
        raise NumericalError("non-finite residuals")
    return r


def check_termination(res, it, st) -> bool:  # ipm.py:106-119
    ea, er = st.eps_abs, st.eps_rel
    return bool(
        _inf(res.r_dual) <= ea + er * max(res.norm_Px, res.norm_Aty, res.norm_Gtz, res.norm_c)
        and _inf(res.r_eq) <= ea + er * max(res.norm_Ax, res.norm_b)
        and _inf(res.r_cone) <= ea + er * max(res.norm_Gx, _inf(it.s), res.norm_h)
        and res.gap <= ea + er * max(abs(res.objective_primal), 1.0))


def initialize_iterate(data, backend) -> Iterate:  # ipm.py:135-156
    n, p = data.n, data.p
    backend.update(identity_scaling(data.cone))
    backend.factor()
    sol = backend.solve(np.concatenate([-data.c, data.b, data.h]))
    x, y, zt = sol[:n], sol[n:n + p], sol[n + p:]
    s = bring_to_interior(-zt, data.cone)
    sol2 = backend.solve(np.concatenate([-data.c, np.zeros(data.p), np.zeros(data.m)]))
    z = bring_to_interior(sol2[n + p:], data.cone)
    it = Iterate(x.copy(), y.copy(), z, s, 0.0)
    it.mu = compute_mu(it.s, it.z, data.cone)
    if not np.isfinite(it.mu):
        raise NumericalError("non-finite initial iterate")
    return it


def ipm_step(data, backend, it, st, res=None, trace=None):  # ipm.py:159-235
    if res is None:
        res = compute_residuals(data, it)
    cone = data.cone
    n, p = data.n, data.p
    deg = cone_degree(cone)
    sc = compute_nt_scaling(it.s, it.z, cone)
    lam = sc.lam
    backend.update(sc)
    backend.factor()

    def direction(d_comp):
        d = jordan_divide(lam, d_comp, cone)
        wd = apply_scaling(sc, d)
        rhs = np.concatenate([-res.r_dual, -res.r_eq, -res.r_cone - wd])
        sol = backend.solve(rhs)
        dx, dy, dz = sol[:n].copy(), sol[n:n + p].copy(), sol[n + p:].copy()
        wdz = apply_scaling(sc, dz)
        ds = apply_scaling(sc, d - wdz)
        return dx, dy, dz, ds, wdz, rhs

    lam_sq = jordan_product(lam, lam, cone)
    dx_a, dy_a, dz_a, ds_a, wdz_a, rhs_a = direction(-lam_sq)
    step_s = max_step_to_boundary(it.s, ds_a, cone)
    step_z = max_step_to_boundary(it.z, dz_a, cone)
    alpha_aff = min(1.0, step_s, step_z)
    mu_aff = max(0.0, float(np.dot(it.s + alpha_aff * ds_a, it.z + alpha_aff * dz_a)) / deg)
    mu = compute_mu(it.s, it.z, cone)
    sigma = min(1.0, max(0.0, (mu_aff / mu) ** 3)) if mu > 0 else 0.0
    winv_ds = apply_scaling(sc, ds_a, inverse=True)
    corr = jordan_product(winv_ds, wdz_a, cone)
    d_comp = sigma * mu * cone_identity(cone) - lam_sq - corr
    dx, dy, dz, ds, _, rhs_c = direction(d_comp)
    step_s = max_step_to_boundary(it.s, ds, cone)
    step_z = max_step_to_boundary(it.z, dz, cone)
    alpha = min(1.0, st.step_fraction * min(step_s, step_z))
    if not np.isfinite(alpha) or alpha <= 0.0:
        raise NumericalError("non-positive or non-finite step length")
    nxt = Iterate(it.x + alpha * dx, it.y + alpha * dy, it.z + alpha * dz, it.s + alpha * ds, 0.0)
    nxt.mu = compute_mu(nxt.s, nxt.z, cone)
    if not all(np.all(np.isfinite(v)) for v in (nxt.x, nxt.y, nxt.z, nxt.s)):
        raise NumericalError("non-finite iterate")
    info = SimpleNamespace(alpha=alpha, alpha_affine=alpha_aff, sigma=sigma, mu_affine=mu_aff)
    if trace is not None:
        trace.append(dict(scaling=sc, lam_sq=lam_sq, rhs_a=rhs_a, rhs_c=rhs_c, ds_a=ds_a, dz_a=dz_a,
                          ds=ds, dz=dz, dx=dx, dy=dy, d_comp=d_comp, info=info))
    return nxt, info


@dataclass
class OracleSettings:  # problem.py:59-67
    eps_abs: float = 1e-7
    eps_rel: float = 1e-7
    max_iters: int = 100
    static_reg: float = 1e-8
    refine_iters: int = 3
    step_fraction: float = 0.99
    time_limit_seconds: float = 3600.0


@dataclass
class OracleResult:
    status: str
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    s: np.ndarray
    objective: float
    iterations: int
    setup_seconds: float
    solve_seconds: float
    factor_count: int
    solve_count: int
    timers: dict = field(default_factory=dict)


def solve(data, settings=None, perm=None, hook=None, trace=None) -> OracleResult:  # ipm.py:238-312
    st = settings or OracleSettings()
    t0 = time.perf_counter()
    d = SimpleNamespace(n=data.n, m=data.m, p=data.p, P=_csc(data.P), A=_csc(data.A), G=_csc(data.G),
                        c=_vec(data.c), b=_vec(data.b), h=_vec(data.h), cone=data.cone)
    kkt = assemble_kkt(d)
    backend = Backend(kkt, st, perm, d.cone)
    t1 = time.perf_counter()
    status, iters, stalls = "NumericalError", 0, 0
    it = Iterate(np.zeros(d.n), np.zeros(d.p), np.zeros(d.m), np.zeros(d.m), 0.0)
    t_hot = 0.0
    try:
        it = initialize_iterate(d, backend)
        if hook:
            hook(it)
        while True:
            th = time.perf_counter()
            res = compute_residuals(d, it)
            t_hot += time.perf_counter() - th
            if check_termination(res, it, st):
                status = "Solved"
                break
            if iters >= st.max_iters:
                status = "MaxIters"
                break
            if time.perf_counter() - t0 > st.time_limit_seconds:
                status = "TimeLimit"
                break
            th = time.perf_counter()
            f0, s0 = backend.t_factor, backend.t_solve
            it, info = ipm_step(d, backend, it, st, res, trace)
            t_hot += (time.perf_counter() - th) - (backend.t_factor - f0) - (backend.t_solve - s0)
            iters += 1
            if hook:
                hook(it)
            if info.alpha < TINY_STEP:
                stalls += 1
                if stalls >= MAX_CONSECUTIVE_STALLS:
                    break
            else:
                stalls = 0
    except NumericalError:
        status = "NumericalError"
    t2 = time.perf_counter()
    Px = spmv_sym_upper(d.P, it.x)
    obj = 0.5 * float(np.dot(it.x, Px)) + float(np.dot(d.c, it.x))
    return OracleResult(status, it.x, it.y, it.z, it.s, obj, iters, t1 - t0, t2 - t1,
                        backend.n_factor, backend.n_solve,
                        dict(factor=backend.t_factor, linsolve=backend.t_solve, hot_path=t_hot,
                             analysis=backend.analysis_seconds, L_nnz=int(backend.sym.Li.size)))


# ------------------------------------------------------------------- ruiz ----
def ruiz_scalings(data, iters):
    """NumPy restatement of the GPU path's Ruiz equilibration (csrc/ruiz_kernels.cu).

    PARITY UNPINNED: the reference has no equilibration; this
    follows upstream QOCO's scheme and only pins the CUDA kernels to a second,
    independent implementation.  Returns (D, E, F) with the scaled problem
    P^ = D P D, A^ = E A D, G^ = F G D, c^ = D c, b^ = E b, h^ = F h."""
    import scipy.sparse as sp

    def mat(M):
        return sp.csc_matrix((M.values, M.row_indices, M.col_pointers), shape=(M.rows, M.cols))

    n, p, m = data.n, data.p, data.m
    Pu = mat(data.P)
    P = (Pu + Pu.T - sp.diags(Pu.diagonal())).tocsr()
    A, G = mat(data.A).tocsr(), mat(data.G).tocsr()
    D, E, F = np.ones(n), np.ones(p), np.ones(m)
    starts, dims = soc_layout(data.cone)

    def rowmax(M):
        M = abs(M).tocsr()
        out = np.zeros(M.shape[0])
        if M.nnz:
            nz = np.diff(M.indptr) > 0
            out[nz] = np.maximum.reduceat(M.data, M.indptr[:-1][nz])
        return out

    for _ in range(iters):
        Ps = sp.diags(D) @ P @ sp.diags(D)
        As = sp.diags(E) @ A @ sp.diags(D) if p else A
        Gs = sp.diags(F) @ G @ sp.diags(D)
        nx = np.maximum(rowmax(Ps), rowmax(Gs.T.tocsr()))
        if p:
            nx = np.maximum(nx, rowmax(As.T.tocsr()))
        ny = rowmax(As) if p else np.zeros(0)
        nz_ = rowmax(Gs)
        for o, d in zip(starts.tolist(), dims.tolist()):
            nz_[o:o + d] = nz_[o:o + d].max()
        for sc, nr in ((D, nx), (E, ny), (F, nz_)):
            pos = nr > 0
            sc[pos] *= 1.0 / np.sqrt(nr[pos])
    return D, E, F
