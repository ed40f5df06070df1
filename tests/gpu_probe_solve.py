"""Solve one named config on the GPU and print the timing breakdown (not a pytest file).
usage: python tests/gpu_probe_solve.py C4_group_lasso "dict(groups=1000)" """

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs


def main():
    name = sys.argv[1]
    kw = eval(sys.argv[2]) if len(sys.argv) > 2 else {}
    small = kw.pop("small", False)
    t = time.time()
    d = configs.make(name, small=small, **kw)
    print(f"generated {name} n={d.n} p={d.p} m={d.m} KKT nnz={configs.kkt_nnz(d)} in {time.time()-t:.2f}s", flush=True)
    res = qs.solve(d)
    tm = res.timers
    print(f"status={res.status.value} iters={res.iterations} obj={res.objective:.10g} setup={res.setup_seconds:.3f}s "
          f"solve={res.solve_seconds:.3f}s")
    print(json.dumps({k: (round(v, 6) if isinstance(v, float) else v) for k, v in tm.items()}))


if __name__ == "__main__":
    main()
