"""One lockstep batch of C5 instances, for `ncu` launch lists of the batched mode (not a pytest file).
usage: python tests/gpu_batched_profile.py [batch size]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.batched import BatchSolver

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
probs = [configs.make("C5_mpc", seed=i) for i in range(B)]
with BatchSolver(probs[0], B) as bs:
    res = bs.solve(probs, check_pattern=False)
    print(B, "instances:", bs.stats(), sum(r.iterations for r in res) / B)
