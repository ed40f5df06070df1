"""C5: a batch of independent MPC trajectory SOCPs on ONE GPU, instances per second as a function of the number of
instances kept in flight (each on its own handle / stream).  Not a pytest file.
    python tests/gpu_batch_throughput.py [count]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.batch import pattern_reuse_solver, solve_batch
from paper_2603_29197_b200.problem import Settings


def main(count=128):
    probs = [configs.make("C5_mpc", seed=i) for i in range(count)]
    solve_batch(lambda i: probs[i], 8, Settings(), workers=4)  # warm-up (library load, first-use costs)
    out = {}
    for mode in ("fresh handle per instance", "one handle per worker, values updated (pattern reuse)"):
        res = {}
        for workers in (1, 2, 4, 8, 16):
            fn = pattern_reuse_solver() if mode.startswith("one") else None
            t = time.perf_counter()
            recs, _ = solve_batch(lambda i: probs[i], count, Settings(), workers=workers, solve_fn=fn)
            dt = time.perf_counter() - t
            assert all(r.status == "Solved" for r in recs), [r.status for r in recs if r.status != "Solved"][:3]
            res[workers] = count / dt
            print(f"{mode}: workers {workers:3d}: {count / dt:8.1f} instances/s   ({dt / count * 1e3:.2f} ms per "
                  f"instance, mean iterations {sum(r.iterations for r in recs) / count:.1f})", flush=True)
        out[mode] = res
    print(json.dumps({"workload": "C5_mpc", "count": count, "instances_per_second": out}))


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
