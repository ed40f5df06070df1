"""One numeric factorisation + one triangular solve of the C4 KKT system, for `ncu` launch lists of the linear-system
kernels (not a pytest file).  usage: python tests/gpu_factor_profile.py [groups]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_29197_b200 import configs
from paper_2603_29197_b200.ipm import DeviceSolver
from paper_2603_29197_b200.problem import Settings

groups = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
d = configs.make("C4_group_lasso", groups=groups, qlo=20, qhi=250, samples=2000, nnz_per_col=3)
dev = DeviceSolver(d, Settings())
dev.initialize_iterate()
dev.compute_residuals()
dev.ipm_step()
print("factor ms", dev.time_kernel(12, 2), "solve ms", dev.time_kernel(13, 2))
dev.close()
