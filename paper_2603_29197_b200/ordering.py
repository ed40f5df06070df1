"""Fill-reducing ordering + supernodal symbolic analysis (host C++, csrc/host_setup.cpp).

The reference orders with its own numba AMD (pkg/src/qsocp/_amd.py), which is
out of the hot-path scope; here the ordering is the quotient-graph AMD of the
host library, which additionally takes the dense SOC blocks as cliques.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def analyze(N, col_pointers, row_indices, ordering="amd", user_perm=None, clique_starts=None, clique_sizes=None):
    """-> (perm[new] = old, stats dict)."""
    lib = _lib.load()
    Kp, Ki = _lib.i64(col_pointers), _lib.i64(row_indices)
    perm, stats = np.empty(N, np.int64), np.zeros(6)
    up = _lib.i64(user_perm) if user_perm is not None else None
    cs = _lib.i64(clique_starts) if clique_starts is not None else None
    cz = _lib.i64(clique_sizes) if clique_sizes is not None else None
    nc = 0 if cs is None else cs.size
    code = 2 if up is not None else {"natural": 0, "amd": 1}[ordering]
    rc = lib.qs_symbolic_stats(N, _lib.ptr(Kp), _lib.ptr(Ki), code, _lib.ptr(up), nc, _lib.ptr(cs), _lib.ptr(cz),
                               _lib.ptr(perm), _lib.ptr(stats))
    _lib.check(lib, None, rc, "symbolic analysis")
    keys = ("supernodes", "levels", "L_nnz", "factor_flops", "max_front_rows", "max_front_cols")
    return perm, dict(zip(keys, stats.tolist()))


def amd_order_upper(N, col_pointers, row_indices) -> np.ndarray:
    """AMD permutation (perm[new] = old) of the symmetric pattern given by its upper triangle."""
    return analyze(N, col_pointers, row_indices, "amd")[0]
