"""Linear-system backend contract and the ``cuda`` backend.

Same plugin contract as the reference (pkg/src/qsocp/linsys.py:24-136): an ABC
with initialize / factor / solve / update / close, instrumentation counters
``n_factor`` / ``n_solve`` and a name -> class registry.  The reference's CPU
backends ("builtin", "parallel") are deliberately not re-implemented here:
this package is the GPU path only and has no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from abc import ABC, abstractmethod

import numpy as np

from . import _lib
from .cones import NTScalingSet
from .errors import NumericalError
from .problem import ConeSpec, ProblemData, Settings
from .sparse import SparseMatrixCSC, csc_from_triplets, empty_csc


class LinsysBackend(ABC):
    """The plugin contract a linear-system backend fulfils (reference: linsys.py:24-51).

    Lifecycle: ``initialize`` exactly once, then any number of ``update`` -> ``factor`` -> ``solve`` rounds, then
    ``close``.  ``n_factor`` / ``n_solve`` count completed factorisations and refined solves (the IPM driver relies on
    factors = iterations + 1 and solves = 2 iterations + 2).
    """

    name = "abstract"

    def __init__(self):
        self._initialized = False
        self.n_factor = 0  # completed numeric factorisations
        self.n_solve = 0   # completed refined solves

    @abstractmethod
    def initialize(self, kkt, settings: Settings, ordering: str = "amd") -> None:
        """Analyse the KKT pattern (ordering + symbolic factorisation).  A second call is a RuntimeError."""

    @abstractmethod
    def update(self, scaling: NTScalingSet) -> None:
        """Write the -W'W block of the given Nesterov-Todd scaling into the KKT values."""

    @abstractmethod
    def factor(self) -> None:
        """Refactorise the KKT matrix numerically with its current values."""

    @abstractmethod
    def solve(self, rhs: np.ndarray) -> np.ndarray:
        """K x = rhs by the current factor, with iterative refinement against the unregularised K."""

    def close(self) -> None:
        """Release whatever the backend holds; the default holds nothing."""


def _problem_from_kkt(kkt) -> ProblemData:
    """Recover (P, A, G, cone) from an assembled KKT system: P is the leading
    n x n block, A' and G' the (1,2) and (1,3) blocks (kkt.py:1-13)."""
    n, p, m = kkt.n, kkt.p, kkt.m
    K = kkt.matrix
    cols = np.repeat(np.arange(K.cols, dtype=np.int64), np.diff(K.col_pointers))
    rows, vals = K.row_indices, K.values
    top = rows < n
    sel = top & (cols < n)
    # drop the explicit zero diagonal the assembly added where P had none
    P = csc_from_triplets(n, n, (rows[sel], cols[sel], vals[sel]))
    sel = top & (cols >= n) & (cols < n + p)
    A = csc_from_triplets(p, n, (cols[sel] - n, rows[sel], vals[sel])) if p else empty_csc(0, n)
    sel = top & (cols >= n + p)
    G = csc_from_triplets(m, n, (cols[sel] - n - p, rows[sel], vals[sel]))
    off = np.asarray(kkt.nt_slot_offsets, dtype=np.int64)
    nsoc = len(kkt.soc_slot_starts)
    counts = np.diff(off)
    l = int(counts[0]) if len(counts) > nsoc else 0
    soc_counts = counts[len(counts) - nsoc:]
    q = tuple(int(round((np.sqrt(8.0 * c + 1.0) - 1.0) / 2.0)) for c in soc_counts)
    return ProblemData(n=n, m=m, p=p, P=P, c=np.zeros(n), A=A, b=np.zeros(p), G=G, h=np.zeros(m), cone=ConeSpec(l, q))


class CudaBackend(LinsysBackend):
    """KKT system resident on the GPU: -W'W scatter, sparse LDL' and refined
    solves all run through the C ABI (csrc/capi.cu)."""

    name = "cuda"

    def __init__(self):
        super().__init__()
        self.cone_executor = None  # the reference's host-thread executor has no meaning here
        self._dev = None
        self._factored = False

    def initialize(self, kkt, settings: Settings, ordering: str = "amd", data: ProblemData | None = None) -> None:
        if self._initialized:
            raise RuntimeError("backend already initialized")
        from .ipm import DeviceSolver

        self._initialized = True
        self._kkt = kkt
        self._dev = DeviceSolver(data if data is not None else _problem_from_kkt(kkt), settings, ordering=ordering)

    def factor(self) -> None:
        if not self._initialized:
            raise RuntimeError("backend not initialized")
        self._dev._check(self._dev.lib.qs_linsys_factor(self._dev.h), "factor")
        self._factored = True
        self.n_factor += 1

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        if not self._factored:
            raise RuntimeError("factor() must run before solve()")
        rhs = _lib.f64(rhs)
        out = np.empty_like(rhs)
        self._dev._check(self._dev.lib.qs_linsys_solve(self._dev.h, _lib.ptr(rhs), _lib.ptr(out)), "solve")
        if not np.all(np.isfinite(out)):
            raise NumericalError("non-finite linear-system solution")
        self.n_solve += 1
        return out

    def update(self, scaling: NTScalingSet) -> None:
        if not self._initialized:
            raise RuntimeError("backend not initialized")
        d = self._dev
        arrs = [_lib.f64(scaling.w_orthant), _lib.f64(scaling.soc_eta), _lib.f64(scaling.soc_wbar), _lib.f64(scaling.lam)]
        d._check(d.lib.qs_set_scaling(d.h, *[_lib.ptr(a) for a in arrs]))
        d._check(d.lib.qs_linsys_update(d.h), "update")

    def kkt_values(self) -> np.ndarray:
        """Current K.values on the device (for inspection / parity checks)."""
        return self._dev.kkt().matrix.values

    def close(self) -> None:
        if self._dev is not None:
            self._dev.close()
            self._dev = None


BACKENDS = {"cuda": CudaBackend}


def make_backend(name: str) -> LinsysBackend:
    try:
        cls = BACKENDS[name]
    except KeyError:
        raise ValueError(f"unknown backend {name!r}; expected one of {sorted(BACKENDS)}") from None
    return cls()
