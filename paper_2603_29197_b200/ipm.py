"""Interior-point driver for the ``cuda`` algebra.

Mirrors the reference driver step for step (pkg/src/qsocp/ipm.py:238-312):
validate -> assemble + analyse (setup_seconds) -> initialize_iterate -> loop
{compute_residuals, check_termination, limits, ipm_step, stall counter}.  The
iterate, the NT scaling, the KKT values and the factor never leave the GPU; the
host sees ~20 scalars per iteration (the termination norms and step lengths)
and the final iterate.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NumericalError
from .problem import ProblemData, Settings, SolveResult, SolveStatus, validate_problem

TINY_STEP = 1e-10  # ipm.py:24
MAX_CONSECUTIVE_STALLS = 3  # ipm.py:25

ORDERINGS = {"natural": 0, "amd": 1, "user": 2}
TIMER_NAMES = ("cone", "kkt_update", "residual", "factor", "solve", "refine_spmv", "analysis", "h2d")


@dataclass
class Iterate:  # ipm.py:28-37
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    s: np.ndarray
    mu: float


@dataclass
class StepInfo:  # ipm.py:58-63
    alpha: float
    alpha_affine: float
    sigma: float
    mu_affine: float


def check_termination(res, settings: Settings):
    """Solved when every mixed absolute/relative criterion holds, inclusive (ipm.py:106-119)."""
    ea, er = settings.eps_abs, settings.eps_rel
    dual_ok = res.norm_r_dual <= ea + er * max(res.norm_Px, res.norm_Aty, res.norm_Gtz, res.norm_c)
    eq_ok = res.norm_r_eq <= ea + er * max(res.norm_Ax, res.norm_b)
    cone_ok = res.norm_r_cone <= ea + er * max(res.norm_Gx, res.norm_s, res.norm_h)
    gap_ok = res.gap <= ea + er * max(abs(res.objective), 1.0)
    return SolveStatus.SOLVED if (dual_ok and eq_ok and cone_ok and gap_ok) else None


class DeviceSolver:
    """One problem resident on one GPU: the object behind Solver(algebra='cuda')."""

    def __init__(self, data: ProblemData, settings: Settings | None = None, ordering: str = "amd",
                 user_perm=None, kkt_literal: bool = False):
        self.settings = settings = settings or Settings()
        self.data = data
        self.lib = lib = _lib.require_device(settings.device)
        self.h = lib.qs_create(settings.device)
        if not self.h:
            raise _lib.CudaUnavailable((lib.qs_global_error() or b"").decode())
        st = _lib.QsSettings(settings.eps_abs, settings.eps_rel, settings.max_iters, settings.static_reg,
                             settings.refine_iters, settings.step_fraction, settings.time_limit_seconds,
                             settings.ruiz_iters, ORDERINGS["user" if user_perm is not None else ordering],
                             int(kkt_literal))
        q = _lib.i64(data.cone.soc_dims)
        P, A, G = data.P, data.A, data.G
        arrs = [_lib.i64(P.col_pointers), _lib.i64(P.row_indices), _lib.f64(P.values),
                _lib.i64(A.col_pointers), _lib.i64(A.row_indices), _lib.f64(A.values),
                _lib.i64(G.col_pointers), _lib.i64(G.row_indices), _lib.f64(G.values),
                _lib.f64(data.c), _lib.f64(data.b), _lib.f64(data.h)]
        perm = _lib.i64(user_perm) if user_perm is not None else None
        rc = lib.qs_setup(self.h, data.n, data.m, data.p, data.cone.orthant_dim, q.size, _lib.ptr(q),
                          *[_lib.ptr(a) for a in arrs], C.byref(st), _lib.ptr(perm))
        try:
            _lib.check(lib, self.h, rc, "setup")
        except Exception:
            self.close()
            raise

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.lib.qs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what=""):
        _lib.check(self.lib, self.h, rc, what)

    def update_values(self, P=None, A=None, G=None, c=None, b=None, h=None):
        """New numbers on the SAME sparsity pattern (qs_update_values): keeps the KKT pattern, ordering, symbolic
        analysis, index maps and launch graphs of this handle.  Matrices are SparseMatrixCSC with exactly the pattern
        given at setup (BadSparseStructure otherwise); vectors must keep their length.  The next run() is a fresh
        solve of the updated problem."""
        import dataclasses

        from .errors import BadSparseStructure, DimensionMismatch

        d = self.data
        new = {}
        vals = []
        for name, M in (("P", P), ("A", A), ("G", G)):
            if M is None:
                vals.append(None)
                continue
            old = getattr(d, name)
            if (M.rows, M.cols) != (old.rows, old.cols) or not np.array_equal(M.col_pointers, old.col_pointers) \
                    or not np.array_equal(M.row_indices, old.row_indices):
                raise BadSparseStructure(f"update_values: {name} must keep the sparsity pattern given at setup")
            vals.append(_lib.f64(M.values))
            new[name] = M
        for name, v in (("c", c), ("b", b), ("h", h)):
            if v is None:
                vals.append(None)
                continue
            v = _lib.f64(v)
            if v.shape != getattr(d, name).shape:
                raise DimensionMismatch(f"update_values: {name} must keep its length")
            if not np.all(np.isfinite(v)):
                pass  # non-finite data surfaces as NUMERICAL_ERROR from the solve, as in the reference (ipm.py:96-102)
            vals.append(v)
            new[name] = v
        self._check(self.lib.qs_update_values(self.h, *[_lib.ptr(v) for v in vals]), "update_values")
        self.data = dataclasses.replace(d, **new)

    def set_stream(self, cuda_stream: int):
        """Run on an existing CUDA stream (e.g. torch.cuda.current_stream().cuda_stream)."""
        self._check(self.lib.qs_set_stream(self.h, C.c_void_p(cuda_stream)))

    # -- IPM phases (each is one C-ABI call)
    def initialize_iterate(self) -> float:  # ipm.py:135-156
        mu = C.c_double()
        self._check(self.lib.qs_initialize_iterate(self.h, C.byref(mu)), "initialize_iterate")
        return mu.value

    def compute_residuals(self):  # ipm.py:70-103
        info = _lib.QsResidualInfo()
        self._check(self.lib.qs_residuals(self.h, C.byref(info)), "compute_residuals")
        return info

    def ipm_step(self):  # ipm.py:159-235
        info = _lib.QsStepInfo()
        self._check(self.lib.qs_step(self.h, C.byref(info)), "ipm_step")
        return info

    def iterate(self, mu=0.0) -> Iterate:
        d = self.data
        x, y, z, s = np.empty(d.n), np.empty(d.p), np.empty(d.m), np.empty(d.m)
        self._check(self.lib.qs_get_iterate(self.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), _lib.ptr(s)))
        return Iterate(x, y, z, s, mu)

    def set_iterate(self, x=None, y=None, z=None, s=None):
        a = [None if v is None else _lib.f64(v) for v in (x, y, z, s)]
        self._check(self.lib.qs_set_iterate(self.h, *[_lib.ptr(v) for v in a]))

    def ruiz_scalings(self):
        d = self.data
        D, E, F = np.empty(d.n), np.empty(d.p), np.empty(d.m)
        self._check(self.lib.qs_get_ruiz(self.h, _lib.ptr(D), _lib.ptr(E), _lib.ptr(F)))
        return D, E, F

    def scaling(self):
        from .cones import NTScalingSet

        c = self.data.cone
        w, eta, wbar, lam = np.empty(c.orthant_dim), np.empty(c.soc_count), np.empty(c.total_dim), np.empty(c.total_dim)
        self._check(self.lib.qs_get_scaling(self.h, *[_lib.ptr(v) for v in (w, eta, wbar, lam)]))
        return NTScalingSet(c, w, eta, wbar, lam)

    def kkt(self):
        """Host copy of the assembled KKT system with the CURRENT device values."""
        from .kkt import KKTSystem
        from .sparse import SparseMatrixCSC

        nnz, slots = C.c_int64(), C.c_int64()
        N = self.lib.qs_kkt_size(self.h, C.byref(nnz), C.byref(slots))
        Kp, Ki, Kx = np.empty(N + 1, np.int64), np.empty(nnz.value, np.int64), np.empty(nnz.value)
        pos = np.empty(slots.value, np.int64)
        self._check(self.lib.qs_get_kkt(self.h, _lib.ptr(Kp), _lib.ptr(Ki), _lib.ptr(Kx), _lib.ptr(pos)))
        from .cones import slot_layout

        off, starts = slot_layout(self.data.cone)
        return KKTSystem(SparseMatrixCSC(N, N, Kp, Ki, Kx), pos, off, starts, self.data.n, self.data.p, self.data.m)

    def counters(self):
        f, s, k = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib.qs_get_counters(self.h, C.byref(f), C.byref(s), C.byref(k))
        return f.value, s.value, k.value

    def transfer_bytes(self):
        """(host -> device, device -> host) bytes this handle has copied so far."""
        a, b = C.c_int64(), C.c_int64()
        self.lib.qs_get_transfer_bytes(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def timers(self) -> dict:
        t = np.zeros(8)
        self.lib.qs_get_timers(self.h, _lib.ptr(t))
        return dict(zip(TIMER_NAMES, t.tolist()))

    def factor_stats(self) -> dict:
        t = np.zeros(8)
        self._check(self.lib.qs_get_factor_stats(self.h, _lib.ptr(t)))
        keys = ("supernodes", "levels", "L_nnz", "factor_flops", "max_front_rows", "max_front_cols", "device_bytes",
                "direct_map")
        return dict(zip(keys, t.tolist()))

    def graph_stats(self) -> dict:
        """Linear-system calls replayed from a captured CUDA graph vs issued as direct launches."""
        a, b = C.c_int64(), C.c_int64()
        self.lib.qs_get_graph_stats(self.h, C.byref(a), C.byref(b))
        return {"graph_replays": a.value, "direct_launch_sequences": b.value}

    def time_kernel(self, kernel_id: int, reps: int = 20, cold: bool = False) -> float:
        """Mean milliseconds per launch of one hot-path kernel (CUDA events on the handle's stream).  cold=True
        flushes the L2 before every timed launch (the figure the kernel sees inside a solve)."""
        ms = C.c_double()
        fn = self.lib.qs_time_kernel_cold if cold else self.lib.qs_time_kernel
        self._check(fn(self.h, kernel_id, reps, C.byref(ms)))
        return ms.value

    # -- the loop
    def run(self, t0: float | None = None, iterate_hook=None):
        """ipm.py:259-297.  Returns (status, iterations, Iterate)."""
        st = self.settings
        t0 = time.perf_counter() if t0 is None else t0
        status, iterations, stalls = SolveStatus.NUMERICAL_ERROR, 0, 0
        mu = 0.0
        have_iterate = False
        try:
            mu = self.initialize_iterate()
            have_iterate = True
            if iterate_hook is not None:
                iterate_hook(self.iterate(mu))
            while True:
                res = self.compute_residuals()
                if check_termination(res, st) is SolveStatus.SOLVED:
                    status = SolveStatus.SOLVED
                    break
                if iterations >= st.max_iters:
                    status = SolveStatus.MAX_ITERS
                    break
                if time.perf_counter() - t0 > st.time_limit_seconds:
                    status = SolveStatus.TIME_LIMIT
                    break
                info = self.ipm_step()
                mu = info.mu
                iterations += 1
                if iterate_hook is not None:
                    iterate_hook(self.iterate(mu))
                if info.alpha < TINY_STEP:
                    stalls += 1
                    if stalls >= MAX_CONSECUTIVE_STALLS:
                        status = SolveStatus.NUMERICAL_ERROR
                        break
                else:
                    stalls = 0
        except NumericalError:
            status = SolveStatus.NUMERICAL_ERROR
        d = self.data
        it = self.iterate(mu) if have_iterate else Iterate(np.zeros(d.n), np.zeros(d.p), np.zeros(d.m), np.zeros(d.m), 0.0)
        return status, iterations, it


def _objective_pattern(P):
    """The pattern-only part of _objective (shared by every instance of a batch)."""
    cols = P.column_of_entry()
    rows = P.row_indices
    return rows, cols, np.where(rows == cols, 0.5, 1.0)


def _objective(data: ProblemData, x: np.ndarray, pattern=None) -> float:
    """0.5 x'Px + c'x from the upper-triangular P (ipm.py:296-297); O(nnz(P)) on the host, once."""
    P = data.P
    rows, cols, w = pattern if pattern is not None else _objective_pattern(P)
    return float(np.dot(w * P.values * x[rows], x[cols])) + float(np.dot(data.c, x))


def solve(data: ProblemData, settings: Settings | None = None, backend_name: str = "cuda", iterate_hook=None,
          ordering: str = "amd", user_perm=None) -> SolveResult:
    """Validate, assemble, and iterate until a termination status is reached
    (same contract as the reference's qsocp.solve, ipm.py:238-312)."""
    from .linsys import BACKENDS

    if backend_name not in BACKENDS:
        raise ValueError(f"unknown backend {backend_name!r}; expected one of {sorted(BACKENDS)}")
    settings = settings or Settings()
    t0 = time.perf_counter()
    validate_problem(data)
    dev = DeviceSolver(data, settings, ordering=ordering, user_perm=user_perm)
    try:
        return solve_on(dev, t0, iterate_hook)
    finally:
        dev.close()


def solve_on(dev: "DeviceSolver", t0: float, iterate_hook=None) -> SolveResult:
    """One solve on an existing handle (fresh from setup or after update_values); counters and byte counts in the
    result are those of THIS solve."""
    f0, s0, l0 = dev.counters()
    t1 = time.perf_counter()
    status, iterations, it = dev.run(t0, iterate_hook)
    solve_seconds = time.perf_counter() - t1
    n_factor, n_solve, launches = dev.counters()
    timers = dev.timers()
    timers["gpu_launches"] = launches - (l0 if f0 else 0)  # the first solve also owns the setup launches
    timers["h2d_bytes"], timers["d2h_bytes"] = dev.transfer_bytes()
    timers.update({f"factor_{k}": v for k, v in dev.factor_stats().items()})
    return SolveResult(status=status, x=it.x, y=it.y, z=it.z, s=it.s, objective=_objective(dev.data, it.x),
                       iterations=iterations, setup_seconds=t1 - t0, solve_seconds=solve_seconds,
                       factor_count=n_factor - f0, solve_count=n_solve - s0, timers=timers)
