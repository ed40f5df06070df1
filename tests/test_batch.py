"""Multi-rank batch sharding (one instance per GPU, no data-path collective):
partition logic and the rank-0 gather, exercised with gloo on CPU, world size 2.
The per-instance solver is the CPU oracle here (test infrastructure) -- on the
GPU box the same driver runs the CUDA path (tests/test_gpu_batch.py)."""

import os
import sys

import numpy as np

import pytest
import torch.multiprocessing as mp

from paper_2603_29197_b200.batch import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_is_a_partition():
    for count in (0, 1, 7, 512):
        for world in (1, 2, 4, 8):
            parts = [shard(count, r, world) for r in range(world)]
            assert sorted(i for p in parts for i in p) == list(range(count))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK=str(rank))  # as torchrun sets it
    import torch.distributed as dist

    from oracle import qsocp_oracle as orc
    from paper_2603_29197_b200 import configs
    from paper_2603_29197_b200.batch import solve_batch

    dist.init_process_group("gloo", rank=rank, world_size=world)
    devices = []

    def solve_fn(d, settings):
        devices.append(settings.device)  # what the CUDA path would hand to qs_create
        return orc.solve(d)

    recs, wall = solve_batch(lambda i: configs.make("C5_mpc", small=True, seed=i), 6, None, rank, world,
                             solve_fn=solve_fn)
    assert devices == [rank] * 3, devices  # every solve of rank r is placed on GPU r (settings=None included)
    if rank == 0:
        out.put([(r.index, r.rank, r.status, r.iterations, r.objective) for r in recs])
    dist.destroy_process_group()


def test_gloo_world2_batch_matches_serial(oracle):
    from paper_2603_29197_b200 import configs

    ctx = mp.get_context("spawn")
    out = ctx.SimpleQueue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = out.get()
    assert [g[0] for g in got] == list(range(6))
    assert [g[1] for g in got] == [0, 1, 0, 1, 0, 1]  # instance i ran on rank i mod 2
    for idx, _, status, iters, obj in got:
        ref = oracle.solve(configs.make("C5_mpc", small=True, seed=idx))
        assert status == ref.status == "Solved" and iters == ref.iterations and obj == ref.objective


def test_worker_pool_keeps_the_order_and_overlaps_instances():
    """workers > 1: several instances in flight on one rank (own handle / stream each on the GPU); records come
    back in instance order whatever the completion order."""
    import threading
    import time
    from types import SimpleNamespace

    from paper_2603_29197_b200.batch import solve_batch

    active, peak, lock = [0], [0], threading.Lock()

    def fake_solve(d, settings):
        with lock:
            active[0] += 1
            peak[0] = max(peak[0], active[0])
        time.sleep(0.02 * (5 - d % 5))  # later instances finish first
        with lock:
            active[0] -= 1
        return SimpleNamespace(status="Solved", iterations=d, objective=float(d), setup_seconds=0.0, solve_seconds=0.0)

    recs, _ = solve_batch(lambda i: i, 10, None, solve_fn=fake_solve, workers=4)
    assert [r.index for r in recs] == list(range(10))
    assert [r.iterations for r in recs] == list(range(10))
    assert peak[0] > 1


def test_rank_device_and_error_records(monkeypatch):
    from types import SimpleNamespace

    from paper_2603_29197_b200.batch import rank_device, solve_batch

    monkeypatch.delenv("LOCAL_RANK", raising=False)
    assert [rank_device(r, 4) for r in range(6)] == [0, 1, 2, 3, 0, 1]
    monkeypatch.setenv("LOCAL_RANK", "3")
    assert rank_device(0, 8) == 3
    seen = []

    def solve_fn(d, settings):
        seen.append(settings.device)
        if d == 2:
            raise RuntimeError("boom")
        return SimpleNamespace(status="Solved", iterations=1, objective=0.0, setup_seconds=0.0, solve_seconds=0.0)

    recs, _ = solve_batch(lambda i: i, 4, None, solve_fn=solve_fn, device=5)
    assert seen == [5, 5, 5, 5]
    assert [r.status for r in recs] == ["Solved", "Solved", "Error: RuntimeError: boom", "Solved"]


def test_same_pattern_is_about_structure_not_numbers():
    import dataclasses

    from paper_2603_29197_b200 import configs
    from paper_2603_29197_b200.batched import same_pattern

    a, b = configs.make("C5_mpc", small=True, seed=0), configs.make("C5_mpc", small=True, seed=1)
    assert same_pattern(a, b) and not np.array_equal(a.b, b.b)
    c = configs.make("C4_group_lasso", small=True, seed=0)
    assert not same_pattern(a, c)
    d = dataclasses.replace(a, cone=type(a.cone)(a.cone.orthant_dim + a.cone.soc_dims[-1], a.cone.soc_dims[:-1]))
    assert not same_pattern(a, d)  # same matrices, another cone layout
