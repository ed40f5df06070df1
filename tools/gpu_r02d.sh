#!/bin/bash
# r02d: full GPU suite, microbench (new residual kernels), bench (lockstep C5 batch), torchrun 1-rank, C2 at 20k samples
set -u
O=gpurun_out/r02d; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 12 $O/pytest_gpu.log
python tests/gpu_microbench.py > $O/microbench.txt 2>&1; grep -i "resid\|scatter\|post_solve\|nt_scaling" $O/microbench.txt | head -20
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -n 3 $O/bench.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu --no-ladder > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err; echo "torchrun rc=$?"; tail -n 3 $O/bench_torchrun1.err
python - <<'PY' > $O/c2_20k.txt 2>&1
import time, sys
sys.path.insert(0, '.')
import paper_2603_29197_b200 as qs
from paper_2603_29197_b200 import configs
d = configs.make("C2_lasso", features=100_000, samples=20_000)
t = time.time(); r = qs.solve(d); print("C2 20k samples:", r.status, r.iterations, r.objective, "setup", r.setup_seconds, "solve", r.solve_seconds, "wall", time.time() - t)
print({k: v for k, v in r.timers.items() if not k.startswith("factor_")}); print({k: v for k, v in r.timers.items() if k.startswith("factor_")})
PY
tail -n 4 $O/c2_20k.txt
python -c "
import json; l=json.load(open('$O/bench.json')); print(json.dumps({k:l[k] for k in ('value','e2e','batch','hot_path')})[:3500])"
