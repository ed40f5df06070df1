"""Solver settings, termination statuses and the result record of the ``cuda`` algebra.

The names, defaults and meanings are the reference's contract (pkg/src/qsocp/problem.py:52-95) -- a caller passes the
same keyword arguments and reads the same attributes -- plus the two GPU-only settings and the device-side timers.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np


class SolveStatus(enum.Enum):
    """How a solve ended (values are the reference's status strings)."""

    SOLVED = "Solved"                    # every termination criterion of ipm.py:106-119 holds
    MAX_ITERS = "MaxIters"               # iteration budget exhausted
    TIME_LIMIT = "TimeLimit"             # wall-clock budget exhausted (checked between iterations)
    NUMERICAL_ERROR = "NumericalError"   # non-finite data, pivot, step or iterate


@dataclass
class Settings:
    """Keyword settings of ``Solver.setup`` / ``solve``."""

    eps_abs: float = 1e-7                 # absolute part of every termination tolerance
    eps_rel: float = 1e-7                 # relative part
    max_iters: int = 100                  # interior-point iterations
    static_reg: float = 1e-8              # sign-matched diagonal shift of the factorised KKT copy
    refine_iters: int = 3                 # iterative-refinement rounds per linear solve, at most
    step_fraction: float = 0.99           # fraction of the step to the cone boundary
    time_limit_seconds: float = 3600.0    # wall-clock budget of one solve
    ruiz_iters: int = 0                   # GPU only: Ruiz equilibration passes (0 = iterate exactly like the reference)
    device: int = 0                       # GPU only: CUDA device ordinal

    def __post_init__(self):
        problems = []
        if not (self.eps_abs > 0 and self.eps_rel > 0):
            problems.append("tolerances must be positive")
        if not self.static_reg > 0:
            problems.append("static regularization must be positive")
        if not 0.0 < self.step_fraction < 1.0:
            problems.append("step_fraction must lie in (0, 1)")
        if self.max_iters < 1 or self.refine_iters < 0:
            problems.append("iteration counts out of range")
        if not self.time_limit_seconds > 0:
            problems.append("time limit must be positive")
        if self.ruiz_iters < 0:
            problems.append("ruiz_iters must be nonnegative")
        if problems:
            raise ValueError(problems[0])


@dataclass
class SolveResult:
    """What ``solve()`` returns: the final iterate on the host and the solve's bookkeeping."""

    status: SolveStatus
    x: np.ndarray                         # primal variables [n]
    y: np.ndarray                         # equality multipliers [p]
    z: np.ndarray                         # conic multipliers [m]
    s: np.ndarray                         # conic slacks [m]
    objective: float                      # 1/2 x'Px + c'x at the returned x
    iterations: int
    setup_seconds: float                  # validation + assembly + analysis + host-to-device
    solve_seconds: float                  # initial point + iterations + device-to-host
    factor_count: int = 0                 # numeric factorisations (iterations + 1)
    solve_count: int = 0                  # refined linear solves (2 iterations + 2)
    timers: dict | None = field(default=None)  # device-side phase seconds, launches, transfer bytes
