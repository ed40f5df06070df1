"""KKT assembly at the API boundary (reference: pkg/src/qsocp/kkt.py:26-150).

``assemble_kkt`` returns the same ``KKTSystem`` fields as the reference -- the
upper-triangular CSC of [P A' G'; . 0 0; . . -W'W] with an explicit full
diagonal, the slot -> position map and the slot offsets -- and must match it
bit for bit.  The pattern is written directly by the host library (no triplet
sort; see csrc/host_setup.cpp) because the reference's Python slot loop costs
~4 us per slot.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .problem import ProblemData
from .sparse import SparseMatrixCSC


@dataclass
class KKTSystem:
    matrix: SparseMatrixCSC
    nt_entry_positions: np.ndarray
    nt_slot_offsets: np.ndarray
    soc_slot_starts: np.ndarray
    n: int
    p: int
    m: int

    @property
    def dim(self) -> int:
        return self.n + self.p + self.m


def reg_signs(n: int, p: int, m: int) -> np.ndarray:
    """+1 on the first n diagonal entries, -1 after (kkt.py:48-52)."""
    s = np.ones(n + p + m, dtype=np.int64)
    s[n:] = -1
    return s


def assemble_kkt(data: ProblemData) -> KKTSystem:
    lib = _lib.load()
    n, m, p = data.n, data.m, data.p
    l = data.cone.orthant_dim
    q = _lib.i64(data.cone.soc_dims)
    nsoc = q.size
    P, A, G = data.P, data.A, data.G
    Pp, Pi, Px = _lib.i64(P.col_pointers), _lib.i64(P.row_indices), _lib.f64(P.values)
    Ap, Ai, Ax = _lib.i64(A.col_pointers), _lib.i64(A.row_indices), _lib.f64(A.values)
    Gp, Gi, Gx = _lib.i64(G.col_pointers), _lib.i64(G.row_indices), _lib.f64(G.values)
    ptr = _lib.ptr
    nnz = lib.qs_kkt_nnz(n, m, p, l, nsoc, ptr(q), ptr(Pp), ptr(Pi), int(Ap[n]), int(Gp[n]))
    slots = lib.qs_kkt_slot_count(l, nsoc, ptr(q))
    N = n + p + m
    Kp, Ki, Kx = np.empty(N + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz, np.float64)
    pos = np.empty(slots, np.int64)
    nviews = (1 if l > 0 else 0) + nsoc
    off = np.zeros(nviews + 1, np.int64)
    soc_starts = np.empty(nsoc, np.int64)
    rc = lib.qs_kkt_assemble(n, m, p, l, nsoc, ptr(q), ptr(Pp), ptr(Pi), ptr(Px), ptr(Ap), ptr(Ai), ptr(Ax),
                             ptr(Gp), ptr(Gi), ptr(Gx), ptr(Kp), ptr(Ki), ptr(Kx), ptr(pos), ptr(off),
                             ptr(soc_starts))
    _lib.check(lib, None, rc, "assemble_kkt")
    return KKTSystem(SparseMatrixCSC(N, N, Kp, Ki, Kx), pos, off, soc_starts, n, p, m)
