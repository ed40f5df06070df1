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


def pattern_reuse_solver():
    """solve_fn for batches whose instances share one sparsity pattern (MPC trajectories, parametric sweeps): every
    worker thread keeps ONE device handle; the first instance pays setup + analysis, the following ones only upload
    their numbers (Solver.update -> qs_update_values)."""
    import threading

    import numpy as np

    from .api import Solver

    tls = threading.local()

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
        return s.solve()

    return solve_fn


def solve_batch(make_instance, count: int, settings=None, rank: int = 0, world: int = 1, solve_fn=None, group=None,
                workers: int = 1):
    """Solve instances {i : i mod world == rank}; gather records on rank 0.

    make_instance(i) -> ProblemData.  solve_fn(data, settings) -> SolveResult
    (defaults to the CUDA path on settings.device).  workers > 1 keeps that many instances in flight on this rank's
    GPU, each on its own handle and CUDA stream (a handle is single-threaded, distinct handles are independent;
    ctypes releases the GIL inside the library): small instances are bound by kernel latency, not by the SMs, so
    their kernels overlap -- the reference's analogue is the thread pool of its bench runner
    (pkg/src/qsocp/bench/runner.py:107-117).  Returns
    (records sorted by index on rank 0 / this rank's records elsewhere, wall seconds of this rank).
    """
    solve_fn = solve_fn or _default_solve

    def one(i):
        res = solve_fn(make_instance(i), settings)
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
