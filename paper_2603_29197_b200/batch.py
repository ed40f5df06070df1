"""Batches of independent instances, sharded one instance per GPU.

A single solve stays on one GPU (the KKT factorisation does not shard); a
batch is partitioned statically -- instance i goes to rank i mod world -- with
NO data-path collective: each rank owns a private handle / stream / factor.
`torch.distributed` is used only to gather the per-instance result records on
rank 0 (NCCL on GPUs, gloo in the CPU tests).  The reference's analogue is the
thread-pool sweep of its bench runner (pkg/src/qsocp/bench/runner.py:107-117).
"""

from __future__ import annotations

import time
from dataclasses import dataclass


@dataclass
class InstanceRecord:
    index: int
    rank: int
    status: str
    iterations: int
    objective: float
    setup_seconds: float
    solve_seconds: float


def shard(count: int, rank: int, world: int) -> list[int]:
    """Instance indices owned by `rank` (round robin: i mod world == rank)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, count, world))


def _default_solve(data, settings):
    from .ipm import solve

    return solve(data, settings)


def rank_device(rank: int = 0, device_count: int | None = None) -> int:
    """The GPU of this rank: LOCAL_RANK under torchrun (one process per GPU), else rank mod the visible devices."""
    import os

    if "LOCAL_RANK" in os.environ:
        return int(os.environ["LOCAL_RANK"])
    if device_count is None:
        from . import _lib

        device_count = max(_lib.load().qs_device_count(), 1)
    return rank % device_count


def pattern_reuse_solver():
    """solve_fn for batches whose instances share one sparsity pattern (MPC trajectories, parametric sweeps): every
    worker thread keeps ONE device handle; the first instance pays setup + analysis, the following ones only upload
    their numbers (Solver.update -> qs_update_values)."""
    import threading

    import numpy as np

    from .api import Solver

    tls = threading.local()
    opened = []  # every worker's solver, so close() can release the device handles when the pool is done

    def same_pattern(a, b):
        return (a.n, a.m, a.p) == (b.n, b.m, b.p) and a.cone == b.cone and all(
            np.array_equal(getattr(a, k).col_pointers, getattr(b, k).col_pointers)
            and np.array_equal(getattr(a, k).row_indices, getattr(b, k).row_indices) for k in "PAG")

    def solve_fn(d, settings):
        s = getattr(tls, "solver", None)
        if s is not None and tls.settings is settings and same_pattern(s._data, d):
            s.update(P=d.P, c=d.c, A=d.A, b=d.b, G=d.G, h=d.h)
        else:
            kw = {} if settings is None else dict(vars(settings))
            s = Solver("cuda").setup(d.n, d.m, d.p, d.P, d.c, d.A, d.b, d.G, d.h, d.cone.orthant_dim,
                                     len(d.cone.soc_dims), d.cone.soc_dims, **kw)
            tls.solver, tls.settings = s, settings
            opened.append(s)
        return s.solve()

    def close():
        for s in opened:
            s.close()
        opened.clear()

    solve_fn.close = close
    return solve_fn


def solve_batch(make_instance, count: int, settings=None, rank: int = 0, world: int = 1, solve_fn=None, group=None,
                workers: int = 1, device: int | None = None):
    """Solve instances {i : i mod world == rank}; gather records on rank 0.

    The rank's GPU is `device` (default: rank_device(rank) = LOCAL_RANK under torchrun); it is written into the
    Settings every solve of this rank receives, so rank r never lands on device 0 by default.  A failing instance
    becomes a record with status "Error: ..." -- the gather always completes.

    make_instance(i) -> ProblemData.  solve_fn(data, settings) -> SolveResult
    (defaults to the CUDA path on settings.device).  workers > 1 keeps that many instances in flight on this rank's
    GPU, each on its own handle and CUDA stream (a handle is single-threaded, distinct handles are independent;
    ctypes releases the GIL inside the library): small instances are bound by kernel latency, not by the SMs, so
    their kernels overlap -- the reference's analogue is the thread pool of its bench runner
    (pkg/src/qsocp/bench/runner.py:107-117).  Returns
    (records sorted by index on rank 0 / this rank's records elsewhere, wall seconds of this rank).
    """
    import dataclasses

    from .problem import Settings

    solve_fn = solve_fn or _default_solve
    if device is None:
        device = rank_device(rank)
    settings = dataclasses.replace(settings or Settings(), device=device)

    def one(i):
        try:
            res = solve_fn(make_instance(i), settings)
        except Exception as exc:  # noqa: BLE001 -- one bad instance must not hang the other ranks in the gather
            return InstanceRecord(i, rank, f"Error: {type(exc).__name__}: {exc}", 0, float("nan"), 0.0, 0.0)
        return InstanceRecord(i, rank, getattr(res.status, "value", str(res.status)), int(res.iterations),
                              float(res.objective), float(res.setup_seconds), float(res.solve_seconds))

    t0 = time.perf_counter()
    todo = shard(count, rank, world)
    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers) as pool:
            mine = list(pool.map(one, todo))
    else:
        mine = [one(i) for i in todo]
    wall = time.perf_counter() - t0
    if hasattr(solve_fn, "close"):
        solve_fn.close()
    if world == 1:
        return mine, wall
    import torch.distributed as dist

    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0, group=group)
    if rank == 0:
        out = sorted((r for part in gathered for r in part), key=lambda r: r.index)
        if [r.index for r in out] != list(range(count)):
            raise RuntimeError("batch gather lost or duplicated instances")
        return out, wall
    return mine, wall


def solve_shard(problems, device: int, workers: int = 16, max_batch: int = 512):
    """This rank's share of a batch on GPU `device` -> (records, mode description).

    Same-pattern instances that fit a batch slot go through the lockstep batched mode (batched.py: every launch
    carries all instances); anything else keeps `workers` instances in flight, one handle + stream each, reusing the
    pattern where it repeats."""
    from .batched import same_pattern, solve_batched
    from .problem import Settings

    problems = list(problems)
    if len(problems) > 1 and all(same_pattern(problems[0], d) for d in problems[1:]):
        try:
            t0 = time.perf_counter()
            res = solve_batched(problems, Settings(device=device), max_batch)
            dt = time.perf_counter() - t0
            recs = [InstanceRecord(i, 0, r.status.value, int(r.iterations), float(r.objective), float(r.setup_seconds),
                                   float(r.solve_seconds)) for i, r in enumerate(res)]
            return recs, (f"lockstep batches of {res[0].timers['batch_size']} instances per launch (qs_batch_*), "
                          f"{dt / len(problems) * 1e3:.3f} ms per instance incl. set-up")
        except MemoryError:
            pass  # an instance does not fit a slot: per-instance handles below
    fn = pattern_reuse_solver()
    recs, _ = solve_batch(lambda i: problems[i], len(problems), Settings(device=device), solve_fn=fn, workers=workers,
                          device=device)
    return recs, f"{workers} instances in flight, one handle + stream each, pattern reuse (qs_update_values)"
