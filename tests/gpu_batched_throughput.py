"""C5: 512 independent MPC trajectory SOCPs on ONE GPU through the lockstep batched mode (qs_batch_*), instances per
second as a function of the batch size; the multi-stream mode (one handle per instance in flight) beside it.
Not a pytest file.    python tests/gpu_batched_throughput.py [count]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.batch import pattern_reuse_solver, solve_batch
from paper_2603_29197_b200.batched import BatchSolver
from paper_2603_29197_b200.problem import Settings


def main(count=512):
    probs = [configs.make("C5_mpc", seed=i) for i in range(count)]
    out = {"lockstep": {}, "streams": {}}
    for size in (16, 64, 128, 256, 512):
        if size > count:
            break
        t0 = time.perf_counter()
        with BatchSolver(probs[0], size) as bs:
            t_setup = time.perf_counter() - t0
            bs.solve(probs[:size])  # warm-up: graph capture
            t = time.perf_counter()
            res = []
            for k0 in range(0, count, size):
                res += bs.solve(probs[k0:k0 + size], check_pattern=False)
            dt = time.perf_counter() - t
            st = bs.stats()
        assert all(r.status.value == "Solved" for r in res), [r.status for r in res if r.status.value != "Solved"][:3]
        out["lockstep"][size] = count / dt
        print(f"lockstep batch of {size:4d}: {count / dt:9.1f} instances/s  ({dt / count * 1e3:.3f} ms per instance, "
              f"setup {t_setup:.2f} s once, mean iterations {sum(r.iterations for r in res) / count:.2f}, "
              f"device seconds per batch {st['solve_seconds']:.4f}, slot {st['slot_bytes'] / 2**20:.2f} MiB)", flush=True)
    # several lockstep batches side by side (own arena + stream each, one host thread each): the synchronisation gaps
    # of one batch are filled by the launches of the others
    from concurrent.futures import ThreadPoolExecutor

    for nb, size in ((2, 256), (4, 128), (2, 512), (4, 256)):
        if nb * size > 2 * count:
            continue
        solvers = [BatchSolver(probs[0], size) for _ in range(nb)]
        chunks = [probs[k0:k0 + size] for k0 in range(0, count, size)]
        reps = max(1, (nb * size) // count)  # enough work for every solver
        chunks = chunks * reps

        def run(args):
            bs, mine = args
            return [r for c in mine for r in bs.solve(c, check_pattern=False)]

        with ThreadPoolExecutor(nb) as pool:
            list(pool.map(run, [(bs, [chunks[0]]) for bs in solvers]))  # warm-up
            t = time.perf_counter()
            res = list(pool.map(run, [(bs, chunks[i::nb]) for i, bs in enumerate(solvers)]))
            dt = time.perf_counter() - t
        total = sum(len(r) for r in res)
        assert all(r.status.value == "Solved" for rr in res for r in rr)
        for bs in solvers:
            bs.close()
        out.setdefault("concurrent_lockstep", {})[f"{nb}x{size}"] = total / dt
        print(f"{nb} lockstep batches of {size} side by side: {total / dt:9.1f} instances/s  ({total} instances in {dt:.3f} s)",
              flush=True)
    for workers in (8, 16, 32):
        fn = pattern_reuse_solver()
        n = min(count, 256)
        solve_batch(lambda i: probs[i], workers, Settings(), workers=workers, solve_fn=pattern_reuse_solver())
        t = time.perf_counter()
        recs, _ = solve_batch(lambda i: probs[i], n, Settings(), workers=workers, solve_fn=fn)
        dt = time.perf_counter() - t
        out["streams"][workers] = n / dt
        print(f"streams, {workers:3d} in flight: {n / dt:9.1f} instances/s", flush=True)
    print(json.dumps({"workload": "C5_mpc", "count": count, "instances_per_second": out}))


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
