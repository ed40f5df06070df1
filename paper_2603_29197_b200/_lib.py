"""ctypes binding of libqsocp_cuda.so (C ABI declared in include/qsocp_cuda.h).

The library is the product path: if it is missing or no CUDA device is usable,
callers get ``CudaUnavailable`` -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

# Batches of small instances keep many streams busy at once; the driver maps streams onto 8 hardware queues by
# default, which caps the overlap at 8 instances (measured: 125 -> 373 instances/s at C5 with 32 queues).  Only
# effective when set before the process creates its CUDA context; an explicit setting of the user wins.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np

from .errors import CudaUnavailable, DimensionMismatch, NotInterior, NumericalError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QS_LIB_PATH") or os.path.join(HERE, "libqsocp_cuda.so")  # QS_LIB_PATH: A/B builds

QS_OK, QS_E_INVALID, QS_E_CUDA, QS_E_NOT_INTERIOR, QS_E_NUMERICAL, QS_E_MEMORY, QS_E_DIMENSION = range(7)

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class QsSettings(C.Structure):
    _fields_ = [("eps_abs", C.c_double), ("eps_rel", C.c_double), ("max_iters", C.c_int64),
                ("static_reg", C.c_double), ("refine_iters", C.c_int64), ("step_fraction", C.c_double),
                ("time_limit_seconds", C.c_double), ("ruiz_iters", C.c_int64), ("ordering", C.c_int64),
                ("kkt_literal", C.c_int64)]


class QsResidualInfo(C.Structure):
    _fields_ = [(k, C.c_double) for k in
                ("norm_r_dual", "norm_r_eq", "norm_r_cone", "gap", "objective", "norm_Px", "norm_Aty", "norm_Gtz",
                 "norm_c", "norm_Ax", "norm_b", "norm_Gx", "norm_h", "norm_s", "mu")] + [("flags", C.c_int64)]


class QsStepInfo(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("alpha", "alpha_affine", "sigma", "mu_affine", "mu", "step_s", "step_z")] \
        + [("flags", C.c_int64)]


# every exported symbol of include/qsocp_cuda.h: name -> (restype, argtypes)
SIGNATURES = {
    "qs_version": (C.c_int, []),
    "qs_device_count": (C.c_int, []),
    "qs_global_error": (C.c_char_p, []),
    "qs_create": (vp, [C.c_int]),
    "qs_destroy": (None, [vp]),
    "qs_last_error": (C.c_char_p, [vp]),
    "qs_set_stream": (C.c_int, [vp, vp]),
    "qs_sync": (C.c_int, [vp]),
    "qs_host_register": (C.c_int, [vp, C.c_int64]),
    "qs_host_unregister": (C.c_int, [vp]),
    "qs_kkt_nnz": (C.c_int64, [C.c_int64] * 5 + [vp, vp, vp, C.c_int64, C.c_int64]),
    "qs_kkt_slot_count": (C.c_int64, [C.c_int64, C.c_int64, vp]),
    "qs_kkt_assemble": (C.c_int, [C.c_int64] * 5 + [vp] * 16),
    "qs_symbolic_stats": (C.c_int, [C.c_int64, vp, vp, C.c_int64, vp, C.c_int64, vp, vp, vp, vp]),
    "qs_set_cones": (C.c_int, [vp, C.c_int64, C.c_int64, vp, C.c_int64]),
    "qs_nt_scaling": (C.c_int, [vp] * 8 + [C.POINTER(C.c_int)]),
    "qs_apply_w": (C.c_int, [vp] * 6 + [C.c_int]),
    "qs_jordan_product": (C.c_int, [vp] * 4),
    "qs_jordan_divide": (C.c_int, [vp] * 4),
    "qs_max_step": (C.c_int, [vp, vp, vp, f64p, f64p]),
    "qs_bring_to_interior": (C.c_int, [vp, vp, C.c_double, vp, f64p]),
    "qs_compute_mu": (C.c_int, [vp, vp, vp, f64p]),
    "qs_neg_wtw": (C.c_int, [vp, C.c_int] + [vp] * 7),
    "qs_get_graph_stats": (C.c_int, [vp, vp, vp]),
    "qs_batch_create": (vp, [C.c_int, C.c_int64]),
    "qs_batch_destroy": (None, [vp]),
    "qs_batch_last_error": (C.c_char_p, [vp]),
    "qs_batch_setup": (C.c_int, [vp] + [C.c_int64] * 5 + [vp] * 14),
    "qs_batch_set_values": (C.c_int, [vp] * 7),
    "qs_batch_solve": (C.c_int, [vp] * 7),
    "qs_batch_stats": (C.c_int, [vp, vp]),
    "qs_predictor_rhs": (C.c_int, [vp] * 11 + [C.POINTER(C.c_int)]),
    "qs_corrector_rhs": (C.c_int, [vp] * 9 + [C.c_double, C.c_double] + [vp] * 3),
    "qs_post_solve": (C.c_int, [vp] * 8 + [C.c_int, C.c_double, vp, vp, f64p]),
    "qs_update_iterate": (C.c_int, [vp, C.c_int64, C.c_int64] + [vp] * 6 + [C.c_double] + [vp] * 4 + [f64p]),
    "qs_spmv_csr": (C.c_int, [vp, C.c_int64, C.c_int64, vp, vp, vp, vp, vp, C.c_int]),
    "qs_spmv_sym_upper": (C.c_int, [vp, C.c_int64, vp, vp, vp, vp, vp]),
    "qs_setup": (C.c_int, [vp] + [C.c_int64] * 5 + [vp] * 13 + [C.POINTER(QsSettings), vp]),
    "qs_kkt_size": (C.c_int64, [vp, i64p, i64p]),
    "qs_get_kkt": (C.c_int, [vp, vp, vp, vp, vp]),
    "qs_linsys_update_identity": (C.c_int, [vp]),
    "qs_linsys_update": (C.c_int, [vp]),
    "qs_linsys_factor": (C.c_int, [vp]),
    "qs_linsys_solve": (C.c_int, [vp, vp, vp]),
    "qs_initialize_iterate": (C.c_int, [vp, f64p]),
    "qs_residuals": (C.c_int, [vp, C.POINTER(QsResidualInfo)]),
    "qs_step": (C.c_int, [vp, C.POINTER(QsStepInfo)]),
    "qs_get_iterate": (C.c_int, [vp] * 5),
    "qs_set_iterate": (C.c_int, [vp] * 5),
    "qs_get_ruiz": (C.c_int, [vp] * 4),
    "qs_get_scaling": (C.c_int, [vp] * 5),
    "qs_set_scaling": (C.c_int, [vp] * 5),
    "qs_get_counters": (C.c_int, [vp, i64p, i64p, i64p]),
    "qs_get_timers": (C.c_int, [vp, vp]),
    "qs_get_factor_stats": (C.c_int, [vp, vp]),
    "qs_update_values": (C.c_int, [vp] * 7),
    "qs_get_transfer_bytes": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "qs_time_kernel": (C.c_int, [vp, C.c_int, C.c_int, f64p]),
    "qs_time_kernel_cold": (C.c_int, [vp, C.c_int, C.c_int, f64p]),
}

_lib = None


def load():
    """Load the shared library (no GPU needed for this step)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaUnavailable(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the cuda algebra)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _lib = lib
    return _lib


def require_device(device: int = 0):
    lib = load()
    cnt = lib.qs_device_count()
    if device >= cnt:
        raise CudaUnavailable(f"CUDA device {device} requested but {cnt} visible; the cuda algebra has no CPU fallback")
    return lib


def ptr(a):
    """Host numpy array (or None) -> void*."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def check(lib, h, rc, what=""):
    if rc == QS_OK:
        return
    msg = (lib.qs_last_error(h) or b"").decode() if h else (lib.qs_global_error() or b"").decode()
    msg = f"{what}: {msg}" if what else msg
    if rc == QS_E_NOT_INTERIOR:
        raise NotInterior(msg)
    if rc == QS_E_NUMERICAL:
        raise NumericalError(msg)
    if rc == QS_E_DIMENSION:
        raise DimensionMismatch(msg)
    if rc == QS_E_MEMORY:
        raise MemoryError(msg)
    if rc == QS_E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)
