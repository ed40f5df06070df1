"""Cone algebra on the device, behind the reference's function names
(reference: pkg/src/qsocp/cones.py).

These wrappers exist for callers and tests that work op by op with host NumPy
arrays: every call copies its operands to the GPU, launches the CUDA kernel
through the C ABI and copies the result back.  The solver itself never goes
through here -- its state stays in HBM (ipm.py / csrc/capi.cu).
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NotInterior
from .problem import ConeSpec

STEP_UNBOUNDED = float(np.finfo(np.float64).max)  # _cone_kernels.py:13


class ScalingMode(enum.Enum):
    MULTIPLY = "multiply"
    MULTIPLY_INVERSE = "multiply_inverse"


@dataclass
class NTScalingSet:  # cones.py:120-143
    cone: ConeSpec
    w_orthant: np.ndarray
    soc_eta: np.ndarray
    soc_wbar: np.ndarray
    lam: np.ndarray


def cone_degree(cone: ConeSpec) -> int:  # cones.py:61-63
    return cone.orthant_dim + cone.soc_count


def soc_starts(cone: ConeSpec) -> np.ndarray:
    dims = np.asarray(cone.soc_dims, dtype=np.int64)
    if not dims.size:
        return np.zeros(0, np.int64)
    return cone.orthant_dim + np.concatenate([[0], np.cumsum(dims)[:-1]])


def cone_identity(cone: ConeSpec) -> np.ndarray:  # cones.py:66-71
    e = np.zeros(cone.total_dim)
    e[: cone.orthant_dim] = 1.0
    e[soc_starts(cone)] = 1.0
    return e


def identity_scaling(cone: ConeSpec) -> NTScalingSet:  # cones.py:146-156
    wbar = np.zeros(cone.total_dim)
    wbar[soc_starts(cone)] = 1.0
    return NTScalingSet(cone, np.ones(cone.orthant_dim), np.ones(cone.soc_count), wbar, cone_identity(cone))


def slot_layout(cone: ConeSpec):
    """(nt_slot_offsets, soc_slot_starts) of the reference's slot order (kkt.py:107-125)."""
    cnt = ([cone.orthant_dim] if cone.orthant_dim > 0 else []) + [q * (q + 1) // 2 for q in cone.soc_dims]
    off = np.zeros(len(cnt) + 1, np.int64)
    np.cumsum(np.asarray(cnt, np.int64), out=off[1:])
    starts = off[(1 if cone.orthant_dim > 0 else 0):-1].copy() if cone.soc_dims else np.zeros(0, np.int64)
    return off, starts


class DeviceCones:
    """A cone layout resident on one GPU plus the per-kernel entry points."""

    def __init__(self, cone: ConeSpec, device: int = 0, big_threshold: int = 0):
        import torch

        self._torch = torch
        self.lib = _lib.require_device(device)
        self.cone = cone
        self.device = torch.device("cuda", device)
        self.h = self.lib.qs_create(device)
        if not self.h:
            raise _lib.CudaUnavailable((self.lib.qs_global_error() or b"").decode())
        q = _lib.i64(cone.soc_dims)
        self._check(self.lib.qs_set_cones(self.h, cone.orthant_dim, q.size, _lib.ptr(q), big_threshold))

    def close(self):
        if self.h:
            self.lib.qs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what=""):
        _lib.check(self.lib, self.h, rc, what)

    # device buffers are torch tensors; the library only sees their addresses
    def dev(self, a):
        t = self._torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        self._torch.cuda.synchronize(self.device)
        return t

    def empty(self, n):
        return self._torch.empty(max(int(n), 1), dtype=self._torch.float64, device=self.device)

    def host(self, t, n):
        self.lib.qs_sync(self.h)
        return t[:n].cpu().numpy().copy()

    @staticmethod
    def p(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    # -- ops, named after the reference functions
    def compute_nt_scaling(self, s, z, with_lam_sq=False):
        cone = self.cone
        l, nsoc, m = cone.orthant_dim, cone.soc_count, cone.total_dim
        ds, dz = self.dev(s), self.dev(z)
        w, eta, lam, lsq = self.empty(l), self.empty(nsoc), self.empty(m), self.empty(m)
        wbar = self._torch.zeros(max(m, 1), dtype=self._torch.float64, device=self.device)
        flag = C.c_int(0)
        self._torch.cuda.synchronize(self.device)  # the zero fill above ran on torch's stream
        self._check(self.lib.qs_nt_scaling(self.h, self.p(ds), self.p(dz), self.p(w), self.p(eta), self.p(wbar),
                                           self.p(lam), self.p(lsq) if with_lam_sq else None, C.byref(flag)))
        if flag.value:
            raise NotInterior("point is not strictly inside the cone")
        sc = NTScalingSet(cone, self.host(w, l), self.host(eta, nsoc), self.host(wbar, m), self.host(lam, m))
        return (sc, self.host(lsq, m)) if with_lam_sq else sc

    def _scaling_dev(self, sc):
        return self.dev(sc.w_orthant), self.dev(sc.soc_eta), self.dev(sc.soc_wbar)

    def apply_scaling(self, sc, u, mode=ScalingMode.MULTIPLY):
        w, eta, wbar = self._scaling_dev(sc)
        du, out = self.dev(u), self.empty(self.cone.total_dim)
        self._check(self.lib.qs_apply_w(self.h, self.p(w), self.p(eta), self.p(wbar), self.p(du), self.p(out),
                                        int(mode is ScalingMode.MULTIPLY_INVERSE)))
        return self.host(out, self.cone.total_dim)

    def jordan_product(self, u, v):
        du, dv, out = self.dev(u), self.dev(v), self.empty(self.cone.total_dim)
        self._check(self.lib.qs_jordan_product(self.h, self.p(du), self.p(dv), self.p(out)))
        return self.host(out, self.cone.total_dim)

    def jordan_divide(self, lam, v):
        dl, dv, out = self.dev(lam), self.dev(v), self.empty(self.cone.total_dim)
        self._check(self.lib.qs_jordan_divide(self.h, self.p(dl), self.p(dv), self.p(out)))
        return self.host(out, self.cone.total_dim)

    def interior_violation(self, u) -> float:
        du = self.dev(u)
        step, viol = C.c_double(), C.c_double()
        self._check(self.lib.qs_max_step(self.h, self.p(du), None, C.byref(step), C.byref(viol)))
        return viol.value

    def max_step_to_boundary(self, u, du) -> float:
        a, b = self.dev(u), self.dev(du)
        step, viol = C.c_double(), C.c_double()
        self._check(self.lib.qs_max_step(self.h, self.p(a), self.p(b), C.byref(step), C.byref(viol)))
        if not viol.value < 0.0:  # check_interior, cones.py:297-299
            raise NotInterior("point is not strictly inside the cone")
        return step.value

    def bring_to_interior(self, u):
        du, out = self.dev(u), self.empty(self.cone.total_dim)
        alpha = C.c_double()
        self._check(self.lib.qs_bring_to_interior(self.h, self.p(du), 1.0, self.p(out), C.byref(alpha)))
        return self.host(out, self.cone.total_dim)

    def compute_mu(self, s, z) -> float:
        a, b = self.dev(s), self.dev(z)
        mu = C.c_double()
        self._check(self.lib.qs_compute_mu(self.h, self.p(a), self.p(b), C.byref(mu)))
        return mu.value

    # -- the fused kernels of one IPM step (ipm.py:180-234), vector in / vector out
    def predictor_rhs(self, s, z, r_cone):
        """-> (NTScalingSet, lam_sq, d = lam \\ (-lam o lam), rhs_z = -r_cone - W d)."""
        cone = self.cone
        l, nsoc, m = cone.orthant_dim, cone.soc_count, cone.total_dim
        a, b, r = self.dev(s), self.dev(z), self.dev(r_cone)
        w, eta, lam, lsq, d, rz = (self.empty(k) for k in (l, nsoc, m, m, m, m))
        wbar = self._torch.zeros(max(m, 1), dtype=self._torch.float64, device=self.device)
        flag = C.c_int(0)
        self._torch.cuda.synchronize(self.device)
        self._check(self.lib.qs_predictor_rhs(self.h, self.p(a), self.p(b), self.p(r), self.p(w), self.p(eta),
                                              self.p(wbar), self.p(lam), self.p(lsq), self.p(d), self.p(rz),
                                              C.byref(flag)))
        if flag.value:
            raise NotInterior("point is not strictly inside the cone")
        sc = NTScalingSet(cone, self.host(w, l), self.host(eta, nsoc), self.host(wbar, m), self.host(lam, m))
        return sc, self.host(lsq, m), self.host(d, m), self.host(rz, m)

    def corrector_rhs(self, sc, lam_sq, ds_a, wdz_a, r_cone, sigma, mu):
        """-> (d_comp, d = lam \\ d_comp, rhs_z = -r_cone - W d)."""
        m = self.cone.total_dim
        w, eta, wbar = self._scaling_dev(sc)
        lam, lsq, a, b, r = (self.dev(v) for v in (sc.lam, lam_sq, ds_a, wdz_a, r_cone))
        dc, d, rz = self.empty(m), self.empty(m), self.empty(m)
        self._check(self.lib.qs_corrector_rhs(self.h, self.p(w), self.p(eta), self.p(wbar), self.p(lam), self.p(lsq),
                                              self.p(a), self.p(b), self.p(r), float(sigma), float(mu), self.p(dc),
                                              self.p(d), self.p(rz)))
        return self.host(dc, m), self.host(d, m), self.host(rz, m)

    def post_solve(self, sc, d, dz, s, z, corrector=False, step_fraction=0.99):
        """-> (wdz = W dz, ds = W (d - W dz), dict of step_s, step_z, alpha_aff, alpha, mu, mu_aff, sigma, flags)."""
        m = self.cone.total_dim
        w, eta, wbar = self._scaling_dev(sc)
        dd, ddz, a, b = (self.dev(v) for v in (d, dz, s, z))
        wdz, ds = self.empty(m), self.empty(m)
        out = np.zeros(8)
        self._check(self.lib.qs_post_solve(self.h, self.p(w), self.p(eta), self.p(wbar), self.p(dd), self.p(ddz),
                                           self.p(a), self.p(b), int(corrector), float(step_fraction), self.p(wdz),
                                           self.p(ds), out.ctypes.data_as(C.POINTER(C.c_double))))
        keys = ("step_s", "step_z", "alpha_aff", "alpha", "mu", "mu_aff", "sigma", "flags")
        return self.host(wdz, m), self.host(ds, m), dict(zip(keys, out.tolist()))

    def update_iterate(self, x, y, z, s, sol, ds, alpha):
        """-> (x', y', z', s', mu', flags) with sol = (dx, dy, dz)."""
        n, p, m = len(x), len(y), self.cone.total_dim
        a = [self.dev(v) for v in (x, y, z, s, sol, ds)]
        o = [self.empty(k) for k in (n, p, m, m)]
        out = np.zeros(2)
        self._check(self.lib.qs_update_iterate(self.h, n, p, *[self.p(v) for v in a], float(alpha),
                                               *[self.p(v) for v in o], out.ctypes.data_as(C.POINTER(C.c_double))))
        return (*[self.host(t, k) for t, k in zip(o, (n, p, m, m))], out[0], int(out[1]))

    def neg_wtw_values(self, sc, out=None):
        """Slot values of -W'W in the reference's slot order (cones.py:319-336)."""
        off, _ = slot_layout(self.cone)
        w, eta, wbar = self._scaling_dev(sc)
        slots = self.empty(int(off[-1]))
        self._check(self.lib.qs_neg_wtw(self.h, 0, self.p(w), self.p(eta), self.p(wbar), None, None, None,
                                        self.p(slots)))
        res = self.host(slots, int(off[-1]))
        if out is not None:
            out[:] = res
        return res

    def write_scaling(self, kkt, sc, direct=False):
        """K.values[nt_entry_positions] = -W'W slots, on the device (kkt.py:146-150)."""
        torch = self._torch
        w, eta, wbar = self._scaling_dev(sc)
        vals = self.dev(kkt.matrix.values)
        n_p = kkt.n + kkt.p
        if direct:
            kp = torch.as_tensor(np.ascontiguousarray(kkt.matrix.col_pointers[n_p + 1:])).to(self.device)
            rc = self.lib.qs_neg_wtw(self.h, 2, self.p(w), self.p(eta), self.p(wbar), None, None,
                                     C.c_void_p(kp.data_ptr()), self.p(vals))
        else:
            pos = torch.as_tensor(np.ascontiguousarray(kkt.nt_entry_positions)).to(self.device)
            rc = self.lib.qs_neg_wtw(self.h, 1, self.p(w), self.p(eta), self.p(wbar), None,
                                     C.c_void_p(pos.data_ptr()), None, self.p(vals))
        self._check(rc)
        kkt.matrix.values[:] = self.host(vals, kkt.matrix.values.size)
