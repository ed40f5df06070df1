"""Shared helpers for the test-suite: golden fixture loading and seeded inputs."""

from __future__ import annotations

import os

import numpy as np

from paper_2603_29197_b200.problem import ConeSpec, ProblemData
from paper_2603_29197_b200.sparse import SparseMatrixCSC

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_problem_names():
    with open(os.path.join(GOLDEN, "problems.txt")) as f:
        return [ln.strip() for ln in f if ln.strip()]


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name if name.endswith(".npz") else f"problem_{name}.npz")))


def problem_from_golden(g) -> ProblemData:
    n, m, p, l = (int(v) for v in g["dims"])
    mats = {}
    for k in "PAG":
        r, c = (int(v) for v in g[f"{k}_shape"])
        mats[k] = SparseMatrixCSC(r, c, g[f"{k}_p"].astype(np.int64), g[f"{k}_i"].astype(np.int64),
                                  g[f"{k}_x"].astype(np.float64))
    return ProblemData(n=n, m=m, p=p, P=mats["P"], c=g["c"], A=mats["A"], b=g["b"], G=mats["G"], h=g["h"],
                       cone=ConeSpec(l, tuple(int(q) for q in g["soc_dims"])))


def random_interior_point(cone, rng):
    """Strictly interior point of the product cone (recipe of the reference's
    tests, pkg/tests/conftest.py:57-66), vectorised for large cone counts."""
    u = rng.standard_normal(cone.total_dim)
    l = cone.orthant_dim
    u[:l] = np.abs(u[:l]) + 0.1
    dims = np.asarray(cone.soc_dims, dtype=np.int64)
    if dims.size:
        starts = l + np.concatenate([[0], np.cumsum(dims)[:-1]])
        sq = u * u
        sq[starts] = 0.0
        sq[:l] = 0.0
        tail = np.add.reduceat(sq, starts) if dims.size else np.zeros(0)
        u[starts] = np.sqrt(tail) + np.abs(rng.standard_normal(dims.size)) + 0.1
    return u
