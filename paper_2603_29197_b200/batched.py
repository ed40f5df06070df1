"""Batched small-problem mode: many instances with ONE sparsity pattern solved in lockstep on one GPU.

SURVEY section 8 f-4.  The reference's precedent for solving independent instances concurrently is the thread-pool
sweep of its bench runner (pkg/src/qsocp/bench/runner.py:107-117) and pkg/tests/test_api.py:101-118; on a GPU a
small instance (an MPC trajectory: 15 K KKT nonzeros) is bound by kernel latency, not by the machine, so here every
kernel launch of the ordinary solver carries ALL instances (gridDim.z = count) and one host synchronisation per
phase serves the whole batch (C ABI: qs_batch_*).  Each instance runs exactly the iteration of a stand-alone
solve -- same kernels, same reduction order -- so its result is bitwise the stand-alone result.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .errors import BadSparseStructure, NotInterior
from .ipm import ORDERINGS, _objective, _objective_pattern
from .problem import ProblemData, Settings, SolveResult, SolveStatus, validate_problem

_STATUS = {1: SolveStatus.SOLVED, 2: SolveStatus.MAX_ITERS, 3: SolveStatus.TIME_LIMIT, 4: SolveStatus.NUMERICAL_ERROR}
MAX_BATCH = 512  # instances per arena (32 MiB of device memory each)


def same_pattern(a: ProblemData, b: ProblemData) -> bool:
    return (a.n, a.m, a.p) == (b.n, b.m, b.p) and a.cone == b.cone and all(
        np.array_equal(getattr(a, k).col_pointers, getattr(b, k).col_pointers)
        and np.array_equal(getattr(a, k).row_indices, getattr(b, k).row_indices) for k in "PAG")


class BatchSolver:
    """`count` slots on one GPU for instances that share the pattern of `template`."""

    def __init__(self, template: ProblemData, count: int, settings: Settings | None = None, ordering: str = "amd"):
        self.settings = settings = settings or Settings()
        self.template = template = validate_problem(template)
        self.count = int(count)
        self.lib = lib = _lib.require_device(settings.device)
        t0 = time.perf_counter()
        self.h = lib.qs_batch_create(settings.device, self.count)
        if not self.h:
            raise _lib.CudaUnavailable((lib.qs_global_error() or b"").decode())
        st = _lib.QsSettings(settings.eps_abs, settings.eps_rel, settings.max_iters, settings.static_reg,
                             settings.refine_iters, settings.step_fraction, settings.time_limit_seconds,
                             0, ORDERINGS[ordering], 0)
        d = template
        q = _lib.i64(d.cone.soc_dims)
        arrs = [_lib.i64(d.P.col_pointers), _lib.i64(d.P.row_indices), _lib.f64(d.P.values),
                _lib.i64(d.A.col_pointers), _lib.i64(d.A.row_indices), _lib.f64(d.A.values),
                _lib.i64(d.G.col_pointers), _lib.i64(d.G.row_indices), _lib.f64(d.G.values),
                _lib.f64(d.c), _lib.f64(d.b), _lib.f64(d.h)]
        rc = lib.qs_batch_setup(self.h, d.n, d.m, d.p, d.cone.orthant_dim, q.size, _lib.ptr(q),
                                *[_lib.ptr(a) for a in arrs], C.byref(st))
        try:
            self._check(rc, "batch setup")
        except Exception:
            self.close()
            raise
        self.setup_seconds = time.perf_counter() - t0

    def _check(self, rc, what=""):
        if rc == _lib.QS_OK:
            return
        msg = (self.lib.qs_batch_last_error(self.h) or b"").decode()
        if rc == _lib.QS_E_MEMORY:
            raise MemoryError(f"{what}: {msg}")
        if rc == _lib.QS_E_INVALID:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: {msg}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.qs_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def stats(self) -> dict:
        out = np.zeros(4)
        self.lib.qs_batch_stats(self.h, _lib.ptr(out))
        return dict(zip(("gpu_launches", "host_syncs", "solve_seconds", "slot_bytes"), out.tolist()))

    def solve(self, problems, check_pattern: bool = True) -> list[SolveResult]:
        """Solve len(problems) <= count instances; slots beyond len(problems) repeat the last instance."""
        k = len(problems)
        if not 1 <= k <= self.count:
            raise ValueError(f"between 1 and {self.count} instances per call")
        t0 = time.perf_counter()
        d0 = self.template
        probs = list(problems)
        if check_pattern:
            for i, d in enumerate(probs):
                if not same_pattern(d0, d):
                    raise BadSparseStructure(f"instance {i} does not have the pattern the batch was set up with")
        probs += [probs[-1]] * (self.count - k)

        def stack(get):
            return np.ascontiguousarray(np.stack([_lib.f64(get(d)) for d in probs]))

        Px, Ax, Gx = stack(lambda d: d.P.values), stack(lambda d: d.A.values), stack(lambda d: d.G.values)
        c, b, h = stack(lambda d: d.c), stack(lambda d: d.b), stack(lambda d: d.h)
        self._check(self.lib.qs_batch_set_values(self.h, *[_lib.ptr(a) for a in (Px, Ax, Gx, c, b, h)]), "set_values")
        B, n, p, m = self.count, d0.n, d0.p, d0.m
        status, iters = np.zeros(B, np.int64), np.zeros(B, np.int64)
        x, y, z, s = np.empty((B, n)), np.empty((B, p)), np.empty((B, m)), np.empty((B, m))
        t1 = time.perf_counter()
        self._check(self.lib.qs_batch_solve(self.h, *[_lib.ptr(a) for a in (status, iters, x, y, z, s)]), "batch solve")
        t2 = time.perf_counter()
        bad = [i for i in range(k) if status[i] == 5]
        if bad:  # the reference lets NotInterior propagate (it is not a NumericalError, errors.py:32-37)
            raise NotInterior(f"instances {bad}: point is not strictly inside the cone")
        st = self.stats()
        pat = _objective_pattern(d0.P)  # one pattern for the whole batch
        out = []
        for i in range(k):
            timers = {"batch_size": B, "batch_seconds": t2 - t1, "gpu_launches": st["gpu_launches"],
                      "host_syncs": st["host_syncs"]}
            out.append(SolveResult(status=_STATUS[int(status[i])], x=x[i].copy(), y=y[i].copy(), z=z[i].copy(),
                                   s=s[i].copy(), objective=_objective(probs[i], x[i], pat), iterations=int(iters[i]),
                                   setup_seconds=(t1 - t0) / k, solve_seconds=(t2 - t1) / k,
                                   factor_count=int(iters[i]) + 1, solve_count=2 * int(iters[i]) + 2, timers=timers))
        return out


def solve_batched(problems, settings: Settings | None = None, max_batch: int = MAX_BATCH, side_by_side: int = 4) -> list[SolveResult]:
    """Solve same-pattern instances in lockstep batches on settings.device.

    Up to `side_by_side` batches (own arena, stream and host thread each) run concurrently once there is work for more
    than one full batch: the synchronisation gaps of one lockstep batch are filled by the launches of the others (C5
    on one B200, set-up excluded: 2590 instances/s as one batch of 512, 3390 as 2 x 512, 3460 as 4 x 256 over 1024
    instances).  A lane pays its own set-up (analysis, arena), so 512 instances stay ONE batch: with set-up inside
    the clock 4 x 128 took 0.40 s against 0.23 s.  Batches hold at most `max_batch` instances."""
    problems = list(problems)
    if not problems:
        return []
    count = len(problems)
    lanes = max(1, min(side_by_side, count // max_batch))  # a lane is worth its set-up cost from a full batch on
    size = min(max_batch, -(-count // lanes))
    chunks = [(k0, problems[k0:k0 + size]) for k0 in range(0, count, size)]
    out: list = [None] * count

    def run(lane):
        mine = chunks[lane::lanes]
        if not mine:
            return
        with BatchSolver(problems[0], size, settings) as bs:
            for k0, chunk in mine:
                out[k0:k0 + len(chunk)] = bs.solve(chunk)

    if lanes == 1:
        run(0)
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(lanes) as pool:
            list(pool.map(run, range(lanes)))  # list(): re-raise a lane's exception here
    return out
