// Cone algebra kernels: Nesterov-Todd scaling, W / W^-1 application, Jordan
// product and division, max step to the boundary, interior violation, and the
// fused per-iteration kernels built from them.
//
// One launch covers the whole product cone.  The grid is cut into three block
// ranges: [orthant | small SOCs | big SOCs].
//   * orthant: grid-stride elementwise, 128-bit (double2) accesses;
//   * small SOCs: a power-of-two lane group (1..32 lanes, chosen from the mean
//     cone size at setup) per cone, segmented reductions by xor-shuffles; the
//     group keeps the whole cone in registers (R = 4 or 8 elements per lane,
//     every load issued before the first use), so a multi-pass op reads HBM
//     exactly once and its later passes touch no memory;
//   * big SOCs (dim > group * R): one CTA per cone, shuffles + a shared-memory
//     stage, registers up to dim 2048, chunked re-reads beyond that.
//
// Every op cites the reference lines whose arithmetic it reproduces
// (paths relative to /root/reference/pkg/src/qsocp/).
#include "cone_kernels.h"

namespace {

// ------------------------------------------------------------------ dispatch
struct NoAcc {};

// One lane group per small cone.  RESIDENT: the whole cone sits in registers (every small cone has dim <= 8 G); the
// number of register slots a cone really needs, ceil(dim / G), picks one of six instantiations of the op, so a cone
// of 40 entries executes two slots' worth of instructions, not eight (the cones of a CTA have similar sizes:
// small_ids is sorted by dimension, so the dispatch does not diverge).  The grid is persistent -- as many CTAs as
// are resident at once -- and the lane groups stride over the size-sorted cone list, largest cones first: every
// warp gets the same mix of sizes, the shortest cones fill the tail, and the per-warp reduction epilogue of the
// reducing ops is paid once per warp instead of once per cone.
template <int G, bool RESIDENT, class Op>
__global__ void __launch_bounds__(QS_THREADS, RESIDENT ? 2 : 3) cone_kernel(ConeLayout L, Op op, int nb_orth, int nb_small, int nb_big) {
  QS_BATCH(L, op);
  typename Op::Acc acc;
  op.init(acc);
  const int b = blockIdx.x;
  bool lanes01 = false;  // the step / violation candidates of this thread's cones sit in lanes 0 and 1 of each group
  if (b < nb_orth) {
    op.orthant(acc, L, b * blockDim.x + threadIdx.x, nb_orth * blockDim.x);
  } else if (b < nb_orth + nb_small) {
    // groups of one warp may diverge (their shuffles name only their own lanes)
    const int ngroups = nb_small * (QS_THREADS / G);
    lanes01 = G >= 2;
    // snake order over the size-sorted list (trip 0 forwards, trip 1 backwards, ...): every group's cones add up
    // to nearly the same number of entries
    const int g0 = ((b - nb_orth) * blockDim.x + threadIdx.x) / G;
    for (int base = 0, trip = 0; base < L.nsmall; base += ngroups, ++trip) {
      const int gid = base + ((trip & 1) ? ngroups - 1 - g0 : g0);
      if (gid >= L.nsmall) continue;
      const int k = L.small_ids ? L.small_ids[gid] : gid;
      const int o = L.soc_ptr[k];
      const int q = L.soc_ptr[k + 1] - o;
      if (RESIDENT) {
#ifndef QS_CONE_VARIANTS
#define QS_CONE_VARIANTS 4
#endif
        const int need = (q + G - 1) / G;
#if QS_CONE_VARIANTS == 6
        if (need <= 1) op.soc(acc, LaneGroup<G, 1, true>{}, k, o, q);
        else if (need == 2) op.soc(acc, LaneGroup<G, 2, true>{}, k, o, q);
        else if (need == 3) op.soc(acc, LaneGroup<G, 3, true>{}, k, o, q);
        else if (need == 4) op.soc(acc, LaneGroup<G, 4, true>{}, k, o, q);
        else if (need <= 6) op.soc(acc, LaneGroup<G, 6, true>{}, k, o, q);
        else op.soc(acc, LaneGroup<G, 8, true>{}, k, o, q);
#elif QS_CONE_VARIANTS == 4
        if (need <= 2) op.soc(acc, LaneGroup<G, 2, true>{}, k, o, q);
        else if (need <= 4) op.soc(acc, LaneGroup<G, 4, true>{}, k, o, q);
        else if (need <= 6) op.soc(acc, LaneGroup<G, 6, true>{}, k, o, q);
        else op.soc(acc, LaneGroup<G, 8, true>{}, k, o, q);
#elif QS_CONE_VARIANTS == 2
        if (need <= 4) op.soc(acc, LaneGroup<G, 4, true>{}, k, o, q);
        else op.soc(acc, LaneGroup<G, 8, true>{}, k, o, q);
#else
        op.soc(acc, LaneGroup<G, 8, true>{}, k, o, q);
#endif
      } else {
        op.soc(acc, LaneGroup<G, 4, false>{}, k, o, q);
      }
    }
  } else {
    __shared__ double scratch[128];
    CtaGroup g{scratch};
    for (int id = b - nb_orth - nb_small; id < L.nbig; id += nb_big) {
      const int k = L.big_ids[id];
      const int o = L.soc_ptr[k];
      op.soc(acc, g, k, o, L.soc_ptr[k + 1] - o);
    }
  }
  op.finish(acc, lanes01);
}

// CTAs of one kernel instantiation that fit the device at once (persistent grid size)
template <class K>
int resident_ctas(K kern) {
  static int cached = 0;  // one value per instantiation; every device of a node is the same part
  if (cached == 0) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, QS_THREADS, 0) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      per_sm = 2;
    }
    cached = per_sm * sms;
  }
  return cached;
}

template <class Op>
void launch(const ConeLayout& L, const Op& op, cudaStream_t st) {
  const int cap = QS_MAX_GRID / 4;
  int nb_orth = 0;
  if (L.l > 0) {
    nb_orth = (L.l / 2 + QS_THREADS - 1) / QS_THREADS;
    if (nb_orth < 1) nb_orth = 1;
    if (nb_orth > cap) nb_orth = cap;
  }
  const int G = L.group;
  const i64 nbs_all = L.nsmall > 0 ? ((i64)L.nsmall * G + QS_THREADS - 1) / QS_THREADS : 0;
  const int nb_big = L.nbig > cap ? cap : L.nbig;
  // Two decompositions per lane-group width G (every small cone has dim <= 8 G, see qs_set_cones):
  //   resident  the whole cone sits in registers, later passes touch no memory: the fused multi-vector ops;
  //   chunked   4 independent loads per vector per trip, later passes re-read L1/L2: fewer registers, more warps
  //             per SM; the 1-2 vector unit ops (measured: tests/gpu_cone_sweep.py).
  const bool resident = L.single >= 0 ? L.single != 0 : Op::kResident;
  auto go = [&](auto kern) {
    i64 nbs = nbs_all;
    const i64 res = (i64)resident_ctas(kern) * (L.waves > 0 ? L.waves : 1);
    if (nbs > res) nbs = res;
    if (nbs > 2 * cap) nbs = 2 * cap;
    const int grid = nb_orth + (int)nbs + nb_big;
    if (grid == 0) return;
    kern<<<qs_grid(grid), QS_THREADS, 0, st>>>(L, op, nb_orth, (int)nbs, nb_big);
  };
#define QS_CASE(GG)                                                                 \
  case GG:                                                                          \
    if (resident) go(cone_kernel<GG, true, Op>); else go(cone_kernel<GG, false, Op>); \
    break;
  switch (G) {
    QS_CASE(1)
    QS_CASE(2)
    QS_CASE(4)
    QS_CASE(8)
    QS_CASE(16)
    default:
    QS_CASE(32)
  }
#undef QS_CASE
}

#define QS_EMPTY_GUARD(L) ((L).l == 0 && (L).nsoc == 0)

// W u on one SOC (forward) or W^-1 u (inverse), _cone_kernels.py:56-74:
//   dot = wbar0 u0 + sgn * sum wbar_t u_t ; out0 = scale (2 wbar0 dot - u0)
//   out_t = scale (2 sgn wbar_t dot + u_t)
__device__ __forceinline__ double w_head(double scale, double wb0, double dot, double u0) {
  return scale * (2.0 * wb0 * dot - u0);
}
__device__ __forceinline__ double w_tail(double scale, double sgn, double wbt, double dot, double ut) {
  return scale * (2.0 * sgn * wbt * dot + ut);
}

// ----------------------------------------------------------------- NT scaling
// compute_nt_scaling (cones.py:159-184) + soc_nt_scaling (_cone_kernels.py:16-53), fused with
//   * lam o lam (ipm.py:191, _cone_kernels.py:77-89),
//   * the per-cone constants of the -W'W generator (4 sum wbar^2 and eta^2, _cone_kernels.py:172-175), and
//   * when r_cone is given, the predictor's third right-hand-side block (ipm.py:180-184,192 with
//     d_comp = -lam o lam):  d = lam \ (-lam o lam),  rhs_z = -r_cone - W d.
// s and z are read once; wbar, lam, lam o lam, d and rhs_z leave the registers once.
struct NtRhsOp {
  static constexpr bool kResident = true;
  const double* s;
  const double* z;
  double* w;
  double* eta;
  double* wbar;
  double* lam;
  double* lam_sq;  // may be null
  double* c4;      // may be null: [nsoc] 4 * sum wbar^2
  double* e2;      //              [nsoc] eta^2
  const double* r_cone;  // null: scaling only
  double* d;
  double* rhs_z;
  double* scalars;
  __device__ void shift(size_t off) {
    qs_shift(off, s);
    qs_shift(off, z);
    qs_shift(off, w);
    qs_shift(off, eta);
    qs_shift(off, wbar);
    qs_shift(off, lam);
    qs_shift(off, lam_sq);
    qs_shift(off, c4);
    qs_shift(off, e2);
    qs_shift(off, r_cone);
    qs_shift(off, d);
    qs_shift(off, rhs_z);
    qs_shift(off, scalars);
  }
  struct Acc {
    int bad;
  };
  __device__ void init(Acc& a) const { a.bad = 0; }
  __device__ void orthant(Acc& a, const ConeLayout& L, int tid, int nth) const {
    for (int i = tid; i < L.l; i += nth) {
      const double sv = s[i], zv = z[i];
      if (sv <= 0.0 || zv <= 0.0) a.bad = 1;
      const double wv = sqrt(sv / zv), lv = sqrt(sv * zv), lsq = lv * lv;
      w[i] = wv;
      lam[i] = lv;
      if (lam_sq) lam_sq[i] = lsq;
      if (r_cone) {
        const double di = (-1.0 * lsq) / lv;
        d[i] = di;
        rhs_z[i] = -r_cone[i] - di * wv;
      }
    }
  }
  template <class Grp>
  __device__ void soc(Acc& a, const Grp& g, int k, int o, int q) const {
    const double s0 = q ? s[o] : 1.0, z0 = q ? z[o] : 1.0;
    const double* sp = s + o;
    const double* zp = z + o;
    double sf[Grp::kR], zf[Grp::kR], rf[Grp::kR];
    double ss = 0.0, zz = 0.0, sz = 0.0;
    QS_CHUNKS(base) {
      qs_frag_load(g, sp, q, base, sf);
      qs_frag_load(g, zp, q, base, zf);
      if (Grp::kSingle && r_cone) qs_frag_load(g, r_cone + o, q, base, rf);  // lands during the passes below
#pragma unroll
      for (int r = 0; r < Grp::kR; ++r) {
        ss += sf[r] * sf[r];
        zz += zf[r] * zf[r];
        sz += sf[r] * zf[r];
      }
    }
    g.sum3(ss, zz, sz);
    const double sres = s0 * s0 - ss, zres = z0 * z0 - zz;
    // a cone that is not strictly interior raises the flag and writes nothing
    // (the reference aborts with NotInterior, cones.py:182-183)
    const bool ok = s0 > 0.0 && z0 > 0.0 && sres > 0.0 && zres > 0.0;
    if (!ok && q) a.bad = 1;
    if (!ok) q = 0;
    const double sa = ok ? sqrt(sres) : 1.0, za = ok ? sqrt(zres) : 1.0;
    const double gamma = sqrt((1.0 + (s0 * z0 + sz) / (sa * za)) / 2.0);
    const double nt0 = (s0 / sa + z0 / za) / (2.0 * gamma);
    const double den = sqrt(2.0 * (1.0 + nt0));
    const double wb0 = (nt0 + 1.0) / den;
    const double ek = sqrt(sa / za);
    // per-cone reciprocals: the tail of wbar is (s_t/sa - z_t/za) / (2 gamma) / den in the reference
    // (_cone_kernels.py:43-44); multiplying by 1/sa, 1/za, 1/(2 gamma den) moves each entry by <= 2 ulp
    // and takes four fp64 divisions per element off the critical path
    const double isa = 1.0 / sa, iza = 1.0 / za, ik = 1.0 / ((2.0 * gamma) * den);
    double wz = 0.0, ww = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, sp, q, base, sf);
        qs_frag_load(g, zp, q, base, zf);
      }
      QS_FRAG(r, t) {
        const double wbt = (sf[r] * isa - zf[r] * iza) * ik;
        if (QS_TAIL_OK(t, q)) wbar[o + t] = wbt;
        if (Grp::kSingle) sf[r] = wbt;  // s is no longer needed: the slot now holds wbar
        wz += wbt * zf[r];
        ww += wbt * wbt;
      }
    }
    g.sum2(wz, ww);
    wz = wz + wb0 * z0;
    const double lam0 = ek * (2.0 * wb0 * wz - z0);
    double ll = 0.0, cross = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, sf);  // written by this very thread in the previous pass
        qs_frag_load(g, zp, q, base, zf);
      }
      QS_FRAG(r, t) {
        const double lt = ek * (2.0 * sf[r] * wz + zf[r]);
        const double lsq = lam0 * lt + lam0 * lt;
        ll += lt * lt;
        cross += lt * (-1.0 * lsq);
        if (Grp::kSingle) zf[r] = lt;  // the slot now holds lam
        if (QS_TAIL_OK(t, q)) {
          lam[o + t] = lt;
          if (lam_sq) lam_sq[o + t] = lsq;
        }
      }
    }
    g.sum2(ll, cross);
    const double lsq0 = lam0 * lam0 + ll;
    if (g.lane() == 0 && q) {
      wbar[o] = wb0;
      eta[k] = ek;
      lam[o] = lam0;
      if (lam_sq) lam_sq[o] = lsq0;
      if (c4) {
        c4[k] = 4.0 * (wb0 * wb0 + ww);
        e2[k] = ek * ek;
      }
    }
    if (!r_cone) return;
    // ---- predictor right-hand side: d = lam \ v with v = -(lam o lam)   (_cone_kernels.py:92-106)
    const double v0 = -1.0 * lsq0;
    const double d0 = (lam0 * v0 - cross) / (lam0 * lam0 - ll);
    const double ia = 1.0 / lam0;
    double dot = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, sf);
        qs_frag_load(g, lam + o, q, base, zf);
      }
      QS_FRAG(r, t) {
        const double lt = zf[r];
        const double dt = (-1.0 * (lam0 * lt + lam0 * lt) - d0 * lt) * ia;
        if (QS_TAIL_OK(t, q)) d[o + t] = dt;
        dot += sf[r] * dt;
      }
    }
    dot = wb0 * d0 + g.sum(dot);
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, sf);
        qs_frag_load(g, lam + o, q, base, zf);
        qs_frag_load(g, r_cone + o, q, base, rf);
      }
      QS_FRAG(r, t) {
        const double lt = zf[r];
        const double dt = (-1.0 * (lam0 * lt + lam0 * lt) - d0 * lt) * ia;
        if (QS_TAIL_OK(t, q)) rhs_z[o + t] = -rf[r] - w_tail(ek, 1.0, sf[r], dot, dt);
      }
    }
    if (g.lane() == 0 && q) {
      d[o] = d0;
      rhs_z[o] = -r_cone[o] - w_head(ek, wb0, dot, d0);
    }
  }
  __device__ void finish(Acc& a, bool) const {
    if (a.bad) scalars[SC_FLAG_NOT_INTERIOR] = 1.0;
  }
};

// -------------------------------------------------------------- apply W / W^-1
// apply_scaling (cones.py:192-212) + soc_apply_w (_cone_kernels.py:56-74)
struct ApplyWOp {
  static constexpr bool kResident = false;
  const double* w;
  const double* eta;
  const double* wbar;
  const double* u;
  double* out;
  int inverse;
  __device__ void shift(size_t off) {
    qs_shift(off, w);
    qs_shift(off, eta);
    qs_shift(off, wbar);
    qs_shift(off, u);
    qs_shift(off, out);
  }
  typedef NoAcc Acc;
  __device__ void init(Acc&) const {}
  __device__ void orthant(Acc&, const ConeLayout& L, int tid, int nth) const {
    for (int i = tid; i < L.l; i += nth) out[i] = inverse ? u[i] / w[i] : u[i] * w[i];
  }
  template <class Grp>
  __device__ void soc(Acc&, const Grp& g, int k, int o, int q) const {
    const double sgn = inverse ? -1.0 : 1.0;
    const double wb0 = q ? wbar[o] : 0.0, u0 = q ? u[o] : 0.0;
    const double e = q ? eta[k] : 1.0;
    double wf[Grp::kR], uf[Grp::kR];
    double dot = 0.0;
    QS_CHUNKS(base) {
      qs_frag_load(g, wbar + o, q, base, wf);
      qs_frag_load(g, u + o, q, base, uf);
#pragma unroll
      for (int r = 0; r < Grp::kR; ++r) dot += sgn * wf[r] * uf[r];
    }
    dot = wb0 * u0 + g.sum(dot);
    const double scale = inverse ? 1.0 / e : e;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, u + o, q, base, uf);
      }
      QS_FRAG(r, t) {
        if (QS_TAIL_OK(t, q)) out[o + t] = w_tail(scale, sgn, wf[r], dot, uf[r]);
      }
    }
    if (g.lane() == 0 && q) out[o] = w_head(scale, wb0, dot, u0);
  }
  __device__ void finish(Acc&, bool) const {}
};

// ------------------------------------------------------------- Jordan product
// jordan_product (cones.py:215-228) + soc_jordan (_cone_kernels.py:77-89)
struct JordanProductOp {
  static constexpr bool kResident = false;
  const double* u;
  const double* v;
  double* out;
  __device__ void shift(size_t off) {
    qs_shift(off, u);
    qs_shift(off, v);
    qs_shift(off, out);
  }
  typedef NoAcc Acc;
  __device__ void init(Acc&) const {}
  __device__ void orthant(Acc&, const ConeLayout& L, int tid, int nth) const {
    for (int i = tid; i < L.l; i += nth) out[i] = u[i] * v[i];
  }
  template <class Grp>
  __device__ void soc(Acc&, const Grp& g, int k, int o, int q) const {
    const double u0 = q ? u[o] : 0.0, v0 = q ? v[o] : 0.0;
    double dot = 0.0;
    double uf[Grp::kR], vf[Grp::kR];
    QS_CHUNKS(base) {
      qs_frag_load(g, u + o, q, base, uf);
      qs_frag_load(g, v + o, q, base, vf);
      QS_FRAG(r, t) {
        dot += uf[r] * vf[r];
        if (QS_TAIL_OK(t, q)) out[o + t] = u0 * vf[r] + v0 * uf[r];
      }
    }
    dot = u0 * v0 + g.sum(dot);
    if (g.lane() == 0 && q) out[o] = dot;
  }
  __device__ void finish(Acc&, bool) const {}
};

// ------------------------------------------------------------ Jordan division
// jordan_divide (cones.py:231-244) + soc_jordan_div (_cone_kernels.py:92-106)
struct JordanDivideOp {
  static constexpr bool kResident = false;
  const double* lam;
  const double* v;
  double* out;
  __device__ void shift(size_t off) {
    qs_shift(off, lam);
    qs_shift(off, v);
    qs_shift(off, out);
  }
  typedef NoAcc Acc;
  __device__ void init(Acc&) const {}
  __device__ void orthant(Acc&, const ConeLayout& L, int tid, int nth) const {
    for (int i = tid; i < L.l; i += nth) out[i] = v[i] / lam[i];
  }
  template <class Grp>
  __device__ void soc(Acc&, const Grp& g, int k, int o, int q) const {
    const double a = q ? lam[o] : 1.0, v0 = q ? v[o] : 0.0;
    double ll = 0.0, cross = 0.0;
    double lf[Grp::kR], vf[Grp::kR];
    QS_CHUNKS(base) {
      qs_frag_load(g, lam + o, q, base, lf);
      qs_frag_load(g, v + o, q, base, vf);
#pragma unroll
      for (int r = 0; r < Grp::kR; ++r) {
        ll += lf[r] * lf[r];
        cross += lf[r] * vf[r];
      }
    }
    g.sum2(ll, cross);
    const double u0 = (a * v0 - cross) / (a * a - ll);
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, lam + o, q, base, lf);
        qs_frag_load(g, v + o, q, base, vf);
      }
      QS_FRAG(r, t) {
        if (QS_TAIL_OK(t, q)) out[o + t] = (vf[r] - u0 * lf[r]) / a;
      }
    }
    if (g.lane() == 0 && q) out[o] = u0;
  }
  __device__ void finish(Acc&, bool) const {}
};

// ------------------------------------------------ max step + interior check
// max_step_to_boundary (cones.py:247-272), check_interior/interior_violation
// (cones.py:275-299), soc_max_step (_cone_kernels.py:109-146), soc_violation
// (_cone_kernels.py:149-162).  Writes scalars[slot_step] and scalars[slot_viol].
struct MaxStepOp {
  static constexpr bool kResident = false;
  const double* u;
  const double* du;  // may be null: violation only
  double* scalars;
  int slot_step, slot_viol;
  GridRed gr;
  __device__ void shift(size_t off) {
    qs_shift(off, u);
    qs_shift(off, du);
    qs_shift(off, scalars);
    qs_shift(off, gr);
  }
  struct Acc {
    double step, viol;
  };
  __device__ void init(Acc& a) const {
    a.step = QS_UNBOUNDED;
    a.viol = -INFINITY;
  }
  __device__ void orthant(Acc& a, const ConeLayout& L, int tid, int nth) const {
    for (int i = tid; i < L.l; i += nth) {
      const double ui = u[i];
      a.viol = fmax(a.viol, -ui);
      if (du) {
        const double di = du[i];
        if (di < 0.0) a.step = fmin(a.step, -ui / di);
      }
    }
  }
  template <class Grp>
  __device__ void soc(Acc& acc, const Grp& g, int k, int o, int q) const {
    double uu = 0.0, dd = 0.0, ud = 0.0;
    double uf[Grp::kR], df[Grp::kR];
    QS_CHUNKS(base) {
      qs_frag_load(g, u + o, q, base, uf);
      if (du) qs_frag_load(g, du + o, q, base, df);
#pragma unroll
      for (int r = 0; r < Grp::kR; ++r) {
        uu += uf[r] * uf[r];
        if (du) {
          dd += df[r] * df[r];
          ud += uf[r] * df[r];
        }
      }
    }
    g.sum3(uu, dd, ud);
    if (q && g.lane() == 0) {
      const double u0 = u[o];
      acc.viol = fmax(acc.viol, sqrt(uu) - u0);
      if (du) {
        const double d0 = du[o];
        acc.step = fmin(acc.step, qs_soc_step(d0 * d0 - dd, 2.0 * (u0 * d0 - ud), u0 * u0 - uu));
      }
    }
  }
  __device__ void finish(Acc& a, bool) const {
    double v[2] = {a.step, a.viol};
    using Ops = RedOps<RED_MIN, RED_MAX>;
    double* sc = scalars;
    const int ss = slot_step, sv = slot_viol;
    qs_grid_reduce<Ops>(v, gr, [=](double (&t)[2]) {
      if (ss >= 0) sc[ss] = t[0];
      if (sv >= 0) sc[sv] = t[1];
    });
  }
};

// ------------------------------------------------------------ shift interior
// bring_to_interior (cones.py:302-311): out = u (+ (1 + alpha) e when the
// violation alpha = scalars[slot] is >= 0).  scale = -1 negates u first (the
// initial slack is -z~, ipm.py:146).
struct ShiftOp {
  static constexpr bool kResident = false;
  const double* u;
  double* out;
  const double* scalars;
  int slot;
  double scale;
  __device__ void shift(size_t off) {
    qs_shift(off, u);
    qs_shift(off, out);
    qs_shift(off, scalars);
  }
  typedef NoAcc Acc;
  __device__ void init(Acc&) const {}
  __device__ void orthant(Acc&, const ConeLayout& L, int tid, int nth) const {
    const double alpha = scalars[slot];
    const double add = (alpha < 0.0) ? 0.0 : 1.0 + alpha;
    for (int i = tid; i < L.l; i += nth) {
      const double v = scale * u[i];
      out[i] = (alpha < 0.0) ? v : v + add;
    }
  }
  template <class Grp>
  __device__ void soc(Acc&, const Grp& g, int k, int o, int q) const {
    const double alpha = scalars[slot];
    const double add = 1.0 + alpha;
    // tail: u + (1+alpha)*0.0 == u
    double uf[Grp::kR];
    QS_CHUNKS(base) {
      qs_frag_load(g, u + o, q, base, uf);
      QS_FRAG(r, t) {
        if (QS_TAIL_OK(t, q)) out[o + t] = scale * uf[r];
      }
    }
    if (g.lane() == 0 && q) {
      const double v = scale * u[o];
      out[o] = (alpha < 0.0) ? v : v + add;
    }
  }
  __device__ void finish(Acc&, bool) const {}
};

// ------------------------------------------- corrector right-hand side (a-10, a-11)
// d_comp = sigma mu e - lam o lam - (W^-1 ds_a) o (W dz_a)                       (ipm.py:209-211)
// d = lam \ d_comp ;  rhs_z = -r_cone - W d                                      (ipm.py:180-184)
// One pass over six vectors; d_comp itself is written only when asked for (parity tests).
struct CorrRhsOp {
  static constexpr bool kResident = true;
  const double* w;
  const double* eta;
  const double* wbar;
  const double* lam;
  const double* lam_sq;
  const double* ds_a;
  const double* wdz_a;
  const double* r_cone;
  double* dcomp;  // may be null
  double* d;
  double* rhs_z;
  const double* scalars;
  __device__ void shift(size_t off) {
    qs_shift(off, w);
    qs_shift(off, eta);
    qs_shift(off, wbar);
    qs_shift(off, lam);
    qs_shift(off, lam_sq);
    qs_shift(off, ds_a);
    qs_shift(off, wdz_a);
    qs_shift(off, r_cone);
    qs_shift(off, dcomp);
    qs_shift(off, d);
    qs_shift(off, rhs_z);
    qs_shift(off, scalars);
  }
  typedef NoAcc Acc;
  __device__ void init(Acc&) const {}
  __device__ void orthant(Acc&, const ConeLayout& L, int tid, int nth) const {
    const double sm = scalars[SC_SIGMA] * scalars[SC_MU];
    for (int i = tid; i < L.l; i += nth) {
      const double wi = w[i];
      const double winv = ds_a[i] / wi;
      const double dc = sm - lam_sq[i] - winv * wdz_a[i];
      if (dcomp) dcomp[i] = dc;
      const double di = (1.0 * dc) / lam[i];
      d[i] = di;
      rhs_z[i] = -r_cone[i] - di * wi;
    }
  }
  template <class Grp>
  __device__ void soc(Acc&, const Grp& g, int k, int o, int q) const {
    const double sm = scalars[SC_SIGMA] * scalars[SC_MU];
    const double wb0 = q ? wbar[o] : 0.0, u0 = q ? ds_a[o] : 0.0, y0 = q ? wdz_a[o] : 0.0;
    const double e = q ? eta[k] : 1.0;
    const double a = q ? lam[o] : 1.0;
    const double scale = 1.0 / e;
    double wf[Grp::kR], af[Grp::kR], yf[Grp::kR], cf[Grp::kR], lf[Grp::kR];
    // pass A: wbar . ds_a  ->  (W^-1 ds_a)_0
    double dot = 0.0;
    QS_CHUNKS(base) {
      qs_frag_load(g, wbar + o, q, base, wf);
      qs_frag_load(g, ds_a + o, q, base, af);
      if (Grp::kSingle) {  // operands of the next pass: issue their loads now, they land during the reduction
        qs_frag_load(g, wdz_a + o, q, base, yf);
        qs_frag_load(g, lam_sq + o, q, base, cf);
        qs_frag_load(g, lam + o, q, base, lf);
      }
#pragma unroll
      for (int r = 0; r < Grp::kR; ++r) dot += -1.0 * wf[r] * af[r];
    }
    dot = wb0 * u0 + g.sum(dot);
    const double x0 = w_head(scale, wb0, dot, u0);
    // pass B: d_comp tail, its head sum, and the two sums of the Jordan division
    double cr = 0.0, ll = 0.0, cross = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, ds_a + o, q, base, af);
        qs_frag_load(g, wdz_a + o, q, base, yf);
        qs_frag_load(g, lam_sq + o, q, base, cf);
        qs_frag_load(g, lam + o, q, base, lf);
      }
      QS_FRAG(r, t) {
        const double xt = w_tail(scale, -1.0, wf[r], dot, af[r]);
        const double yt = yf[r];
        const double dct = 0.0 - cf[r] - (x0 * yt + y0 * xt);
        const bool in = QS_TAIL_OK(t, q);
        if (in) {
          cr += xt * yt;
          ll += lf[r] * lf[r];
          cross += lf[r] * (1.0 * dct);
          if (dcomp || !Grp::kSingle) (dcomp ? dcomp : d)[o + t] = dct;  // chunked: parked in d until pass C
        }
        cf[r] = in ? dct : 0.0;
      }
    }
    double rf[Grp::kR];
    if (Grp::kSingle) qs_frag_load(g, r_cone + o, q, 0, rf);  // needed last; lands during the reductions
    g.sum3(cr, ll, cross);
    cr = x0 * y0 + cr;
    const double dc0 = q ? sm - lam_sq[o] - cr : 0.0;
    const double v0 = 1.0 * dc0;
    const double d0 = (a * v0 - cross) / (a * a - ll);
    const double ia = 1.0 / a;
    // pass C: d tail, wbar . d
    double dot2 = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, (dcomp ? dcomp : d) + o, q, base, cf);
        qs_frag_load(g, lam + o, q, base, lf);
      }
      QS_FRAG(r, t) {
        const double dt = (1.0 * cf[r] - d0 * lf[r]) * ia;
        if (QS_TAIL_OK(t, q)) d[o + t] = dt;
        cf[r] = dt;
        dot2 += wf[r] * dt;
      }
    }
    dot2 = wb0 * d0 + g.sum(dot2);
    // pass D: rhs_z
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, d + o, q, base, cf);
        qs_frag_load(g, r_cone + o, q, base, rf);
      }
      QS_FRAG(r, t) {
        if (QS_TAIL_OK(t, q)) rhs_z[o + t] = -rf[r] - w_tail(e, 1.0, wf[r], dot2, cf[r]);
      }
    }
    if (g.lane() == 0 && q) {
      if (dcomp) dcomp[o] = dc0;
      d[o] = d0;
      rhs_z[o] = -r_cone[o] - w_head(e, wb0, dot2, d0);
    }
  }
  __device__ void finish(Acc&, bool) const {}
};

// ----------------------------------------- after the solve: ds and both steps
// wdz = W dz ; ds = W (d - wdz)                                (ipm.py:187-188)
// step_s = max_step(s, ds), step_z = max_step(z, dz)           (ipm.py:195-196 / 214-215)
// final:  predictor  alpha_aff = min(1, step_s, step_z)        (ipm.py:197)
//                    mu_aff = max(0, (s + alpha_aff ds).(z + alpha_aff dz) / deg), mu = s.z / deg,
//                    sigma = clip((mu_aff / mu)^3, 0, 1)        (ipm.py:198-206)
//         corrector  alpha = min(1, step_fraction * min(..))   (ipm.py:216-218)
// The affine complementarity needs alpha_aff, a minimum over every cone, before its dot product can be formed;
// the kernel therefore accumulates the four dots s.z, s.dz, ds.z, ds.dz (its operands are in registers anyway)
// and the last block evaluates s.z + alpha (s.dz + ds.z) + alpha^2 ds.dz -- the same polynomial the reference
// sums term by term, rounded differently (relative difference of mu_aff ~1e-15 mu / mu_aff).
template <bool CORR>
struct PostSolveOp {
  static constexpr bool kResident = true;
  const double* w;
  const double* eta;
  const double* wbar;
  const double* d;
  const double* dz;
  const double* s;
  const double* z;
  double* wdz;  // may be null (corrector does not need it)
  double* ds;
  double* scalars;
  static constexpr int corrector = CORR;  // compile-time: the corrector instantiation carries no mu_aff sums
  double step_fraction;
  double deg;
  GridRed gr;
  __device__ void shift(size_t off) {
    qs_shift(off, w);
    qs_shift(off, eta);
    qs_shift(off, wbar);
    qs_shift(off, d);
    qs_shift(off, dz);
    qs_shift(off, s);
    qs_shift(off, z);
    qs_shift(off, wdz);
    qs_shift(off, ds);
    qs_shift(off, scalars);
    qs_shift(off, gr);
  }
  struct Acc {
    double step_s, step_z, viol_s, viol_z, sz, sdz, dsz, dsdz;
  };
  __device__ void init(Acc& a) const {
    a.step_s = a.step_z = QS_UNBOUNDED;
    a.viol_s = a.viol_z = -INFINITY;
    a.sz = a.sdz = a.dsz = a.dsdz = 0.0;
  }
  __device__ void orthant(Acc& a, const ConeLayout& L, int tid, int nth) const {
    for (int i = tid; i < L.l; i += nth) {
      const double wi = w[i], dzi = dz[i];
      const double y = dzi * wi;
      const double dsi = (d[i] - y) * wi;
      if (wdz) wdz[i] = y;
      ds[i] = dsi;
      const double si = s[i], zi = z[i];
      a.viol_s = fmax(a.viol_s, -si);
      a.viol_z = fmax(a.viol_z, -zi);
      if (dsi < 0.0) a.step_s = fmin(a.step_s, -si / dsi);
      if (dzi < 0.0) a.step_z = fmin(a.step_z, -zi / dzi);
      if (!corrector) {
        a.sz += si * zi;
        a.sdz += si * dzi;
        a.dsz += dsi * zi;
        a.dsdz += dsi * dzi;
      }
    }
  }
  template <class Grp>
  __device__ void soc(Acc& acc, const Grp& g, int k, int o, int q) const {
    const double wb0 = q ? wbar[o] : 0.0, e = q ? eta[k] : 1.0;
    const double dz0 = q ? dz[o] : 0.0, z0 = q ? z[o] : 1.0, s0 = q ? s[o] : 1.0, d0 = q ? d[o] : 0.0;
    // pass 1: w.dz and the (z, dz) quadratic
    double dot1 = 0.0, zz = 0.0, dd = 0.0, zd = 0.0;
    double wf[Grp::kR], gf[Grp::kR], df[Grp::kR], zf[Grp::kR], sf[Grp::kR];  // wbar, dz, d, z, s
    QS_CHUNKS(base) {
      qs_frag_load(g, wbar + o, q, base, wf);
      qs_frag_load(g, dz + o, q, base, gf);
      qs_frag_load(g, z + o, q, base, zf);
      if (Grp::kSingle) {
        qs_frag_load(g, d + o, q, base, df);
        qs_frag_load(g, s + o, q, base, sf);  // lands during the reductions and pass 2
      }
#pragma unroll
      for (int r = 0; r < Grp::kR; ++r) {
        dot1 += wf[r] * gf[r];
        zz += zf[r] * zf[r];
        dd += gf[r] * gf[r];
        zd += zf[r] * gf[r];
      }
    }
    g.sum4(dot1, zz, dd, zd);
    dot1 = wb0 * dz0 + dot1;
    const double y0 = w_head(e, wb0, dot1, dz0);
    // pass 2: w.(d - wdz)
    double dot2 = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, dz + o, q, base, gf);
        qs_frag_load(g, d + o, q, base, df);
      }
      QS_FRAG(r, t) {
        const double yt = w_tail(e, 1.0, wf[r], dot1, gf[r]);
        if (QS_TAIL_OK(t, q)) {
          if (wdz) wdz[o + t] = yt;
          dot2 += wf[r] * (df[r] - yt);
        }
      }
    }
    const double e0 = d0 - y0;
    dot2 = wb0 * e0 + g.sum(dot2);
    const double ds0 = w_head(e, wb0, dot2, e0);
    // pass 3: ds, the (s, ds) quadratic, and (predictor) the four dots of the affine complementarity
    double ss = 0.0, d2 = 0.0, sd = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, dz + o, q, base, gf);
        qs_frag_load(g, d + o, q, base, df);
        qs_frag_load(g, s + o, q, base, sf);
        if (!corrector) qs_frag_load(g, z + o, q, base, zf);
      }
      QS_FRAG(r, t) {
        const double yt = w_tail(e, 1.0, wf[r], dot1, gf[r]);
        const double dst = w_tail(e, 1.0, wf[r], dot2, df[r] - yt);
        if (QS_TAIL_OK(t, q)) {
          ds[o + t] = dst;
          const double st = sf[r];
          ss += st * st;
          d2 += dst * dst;
          sd += st * dst;
          if (!corrector) {
            acc.sz += st * zf[r];
            acc.sdz += st * gf[r];
            acc.dsz += dst * zf[r];
            acc.dsdz += dst * gf[r];
          }
        }
      }
    }
    g.sum3(ss, d2, sd);
    if (g.lane() == 0 && q) {
      if (wdz) wdz[o] = y0;
      ds[o] = ds0;
      if (!corrector) {
        acc.sz += s0 * z0;
        acc.sdz += s0 * dz0;
        acc.dsz += ds0 * z0;
        acc.dsdz += ds0 * dz0;
      }
    }
    // every thread holds all eight sums: lane 0 finishes the (s, ds) pair and lane 1 the (z, dz) pair side by
    // side (each is a sqrt + divisions chain); a one-lane group does both
    if (g.size() >= 2) {
      if (g.lane() < 2 && q) {
        const bool zs = g.lane() == 1;
        const double u0 = zs ? z0 : s0, du0 = zs ? dz0 : ds0, uu = zs ? zz : ss, d_d = zs ? dd : d2, ud = zs ? zd : sd;
        const double viol = sqrt(uu) - u0;
        const double step = qs_soc_step(du0 * du0 - d_d, 2.0 * (u0 * du0 - ud), u0 * u0 - uu);
        if (zs) {
          acc.viol_z = fmax(acc.viol_z, viol);
          acc.step_z = fmin(acc.step_z, step);
        } else {
          acc.viol_s = fmax(acc.viol_s, viol);
          acc.step_s = fmin(acc.step_s, step);
        }
      }
    } else if (q) {
      acc.viol_s = fmax(acc.viol_s, sqrt(ss) - s0);
      acc.viol_z = fmax(acc.viol_z, sqrt(zz) - z0);
      acc.step_s = fmin(acc.step_s, qs_soc_step(ds0 * ds0 - d2, 2.0 * (s0 * ds0 - sd), s0 * s0 - ss));
      acc.step_z = fmin(acc.step_z, qs_soc_step(dz0 * dz0 - dd, 2.0 * (z0 * dz0 - zd), z0 * z0 - zz));
    }
  }
  __device__ void finish(Acc& a, bool) const {
    double* sc = scalars;
    const int corr = corrector;
    const double sf = step_fraction, dg = deg;
    if (corr) {
      double v[4] = {a.step_s, a.step_z, a.viol_s, a.viol_z};
      using Ops = RedOps<RED_MIN, RED_MIN, RED_MAX, RED_MAX>;
      qs_grid_reduce<Ops>(v, gr, [=](double (&t)[4]) {
        sc[SC_STEP_S] = t[0];
        sc[SC_STEP_Z] = t[1];
        sc[SC_VIOL_S] = t[2];
        sc[SC_VIOL_Z] = t[3];
        if (!(t[2] < 0.0) || !(t[3] < 0.0)) sc[SC_FLAG_NOT_INTERIOR] = 1.0;
        const double al = fmin(1.0, sf * fmin(t[0], t[1]));
        sc[SC_ALPHA] = al;
        if (!qs_finite(al) || al <= 0.0) sc[SC_FLAG_BAD_STEP] = 1.0;
      });
    } else {
      double v[8] = {a.step_s, a.step_z, a.viol_s, a.viol_z, a.sz, a.sdz, a.dsz, a.dsdz};
      using Ops = RedOps<RED_MIN, RED_MIN, RED_MAX, RED_MAX, RED_SUM, RED_SUM, RED_SUM, RED_SUM>;
      qs_grid_reduce<Ops>(v, gr, [=](double (&t)[8]) {
        sc[SC_STEP_S] = t[0];
        sc[SC_STEP_Z] = t[1];
        sc[SC_VIOL_S] = t[2];
        sc[SC_VIOL_Z] = t[3];
        if (!(t[2] < 0.0) || !(t[3] < 0.0)) sc[SC_FLAG_NOT_INTERIOR] = 1.0;
        const double al = fmin(1.0, fmin(t[0], t[1]));
        sc[SC_ALPHA_AFF] = al;
        const double mu_aff = fmax(0.0, (t[4] + al * (t[5] + t[6]) + (al * al) * t[7]) / dg);
        const double mu = t[4] / dg;
        double sigma = 0.0;
        if (mu > 0.0) {
          const double r = mu_aff / mu;
          sigma = fmin(1.0, fmax(0.0, r * r * r));
        }
        sc[SC_MU_AFF] = mu_aff;
        sc[SC_MU] = mu;
        sc[SC_SIGMA] = sigma;
      });
    }
  }
};

// -------------------------------------------------- W^T W v = W (W v)  (a-13)
// Scaling block of the KKT operator, used by the refinement residual.
struct ApplyW2Op {
  static constexpr bool kResident = false;
  const double* w;
  const double* eta;
  const double* wbar;
  const double* u;
  double* out;
  __device__ void shift(size_t off) {
    qs_shift(off, w);
    qs_shift(off, eta);
    qs_shift(off, wbar);
    qs_shift(off, u);
    qs_shift(off, out);
  }
  typedef NoAcc Acc;
  __device__ void init(Acc&) const {}
  __device__ void orthant(Acc&, const ConeLayout& L, int tid, int nth) const {
    for (int i = tid; i < L.l; i += nth) out[i] = (w[i] * w[i]) * u[i];
  }
  template <class Grp>
  __device__ void soc(Acc&, const Grp& g, int k, int o, int q) const {
    const double wb0 = q ? wbar[o] : 0.0, u0 = q ? u[o] : 0.0, e = q ? eta[k] : 1.0;
    double dot1 = 0.0;
    double wf[Grp::kR], uf[Grp::kR];
    QS_CHUNKS(base) {
      qs_frag_load(g, wbar + o, q, base, wf);
      qs_frag_load(g, u + o, q, base, uf);
#pragma unroll
      for (int r = 0; r < Grp::kR; ++r) dot1 += wf[r] * uf[r];
    }
    dot1 = wb0 * u0 + g.sum(dot1);
    const double y0 = w_head(e, wb0, dot1, u0);
    double dot2 = 0.0;
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, u + o, q, base, uf);
      }
      QS_FRAG(r, t) {
        if (QS_TAIL_OK(t, q)) dot2 += wf[r] * w_tail(e, 1.0, wf[r], dot1, uf[r]);
      }
    }
    dot2 = wb0 * y0 + g.sum(dot2);
    QS_CHUNKS(base) {
      if (!Grp::kSingle) {
        qs_frag_load(g, wbar + o, q, base, wf);
        qs_frag_load(g, u + o, q, base, uf);
      }
      QS_FRAG(r, t) {
        if (QS_TAIL_OK(t, q)) out[o + t] = w_tail(e, 1.0, wf[r], dot2, w_tail(e, 1.0, wf[r], dot1, uf[r]));
      }
    }
    if (g.lane() == 0 && q) out[o] = w_head(e, wb0, dot2, y0);
  }
  __device__ void finish(Acc&, bool) const {}
};

// ------------------------------------------------------- plain vector kernels
// out = a + alpha * b over [0, len), four independent load pairs in flight per thread; returns whether every result
// is finite
__device__ __forceinline__ bool axpy_range(const double* __restrict__ a, const double* __restrict__ b, double alpha,
                                           double* __restrict__ out, int len, int tid, int nth) {
  bool fin = true;
  int i = tid;
  for (; i + 3 * nth < len; i += 4 * nth) {
    const double a0 = a[i], a1 = a[i + nth], a2 = a[i + 2 * nth], a3 = a[i + 3 * nth];
    const double b0 = b[i], b1 = b[i + nth], b2 = b[i + 2 * nth], b3 = b[i + 3 * nth];
    const double t0 = a0 + alpha * b0, t1 = a1 + alpha * b1, t2 = a2 + alpha * b2, t3 = a3 + alpha * b3;
    out[i] = t0;
    out[i + nth] = t1;
    out[i + 2 * nth] = t2;
    out[i + 3 * nth] = t3;
    fin = fin && qs_finite(t0) && qs_finite(t1) && qs_finite(t2) && qs_finite(t3);
  }
  for (; i < len; i += nth) {
    const double t = a[i] + alpha * b[i];
    out[i] = t;
    fin = fin && qs_finite(t);
  }
  return fin;
}

__global__ void __launch_bounds__(QS_THREADS) k_update_iterate(int n, int p, int m, const double* x, const double* y,
                                                               const double* z, const double* s, double* xo, double* yo,
                                                               double* zo, double* so, const double* sol,
                                                               const double* ds, double deg, double* scalars, GridRed gr) {
  // it' = it + alpha (dx, dy, dz, ds); mu' = s'.z' / deg; finite check (ipm.py:220-234).  The new iterate goes to
  // (xo, yo, zo, so): the reference builds `nxt` and raises before it replaces `it` (ipm.py:219-229), so a failed
  // step must leave the last good iterate intact -- the host swaps the buffers only when no flag is raised.
  QS_BATCH(x, y, z, s, xo, yo, zo, so, sol, ds, scalars, gr);
  const double a = scalars[SC_ALPHA];
  const bool bad_step = scalars[SC_FLAG_BAD_STEP] != 0.0;  // alpha <= 0 or non-finite: nothing to apply
  double v[2] = {0.0, 0.0};
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  if (!bad_step) {
    bool fin = axpy_range(x, sol, a, xo, n, tid, nth);
    fin = axpy_range(y, sol + n, a, yo, p, tid, nth) && fin;
    const double* dz = sol + n + p;
    int i = tid;
    for (; i + nth < m; i += 2 * nth) {  // two elements of four vectors in flight
      const double z0 = z[i], z1 = z[i + nth], g0 = dz[i], g1 = dz[i + nth];
      const double s0 = s[i], s1 = s[i + nth], h0 = ds[i], h1 = ds[i + nth];
      const double zt0 = z0 + a * g0, zt1 = z1 + a * g1, st0 = s0 + a * h0, st1 = s1 + a * h1;
      zo[i] = zt0;
      zo[i + nth] = zt1;
      so[i] = st0;
      so[i + nth] = st1;
      v[0] += st0 * zt0;
      v[0] += st1 * zt1;
      fin = fin && qs_finite(zt0) && qs_finite(zt1) && qs_finite(st0) && qs_finite(st1);
    }
    for (; i < m; i += nth) {
      const double zt = z[i] + a * dz[i];
      const double st = s[i] + a * ds[i];
      zo[i] = zt;
      so[i] = st;
      v[0] += st * zt;
      fin = fin && qs_finite(zt) && qs_finite(st);
    }
    if (!fin) v[1] = 1.0;
  }
  using Ops = RedOps<RED_SUM, RED_MAX>;
  qs_grid_reduce<Ops>(v, gr, [=](double (&t)[2]) {
    if (bad_step) return;  // SC_MU keeps the value of the iterate that stays
    if (t[1] != 0.0) {  // only the vectors are tested here (ipm.py:227-229); a non-finite s'.z' of finite
      scalars[SC_FLAG_NONFINITE] = 1.0;  // vectors surfaces in the next residual phase, as in the reference
      return;
    }
    scalars[SC_MU] = t[0] / deg;
  });
}

__global__ void __launch_bounds__(QS_THREADS) k_dot(int m, const double* a, const double* b, double scale, double* out,
                                                    GridRed gr) {
  QS_BATCH(a, b, out, gr);
  double v[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) v[0] += a[i] * b[i];
  using Ops = RedOps<RED_SUM>;
  qs_grid_reduce<Ops>(v, gr, [=](double (&t)[1]) { *out = t[0] * scale; });
}

int vec_grid(i64 n) {
  i64 g = (n + QS_THREADS - 1) / QS_THREADS;
  if (g < 1) g = 1;
  if (g > 148 * 8) g = 148 * 8;
  return (int)g;
}

}  // namespace

// ------------------------------------------------------------ host launchers
void qsk_nt_scaling(const ConeLayout& L, const double* s, const double* z, double* w, double* eta, double* wbar,
                    double* lam, double* lam_sq, double* c4, double* e2, const double* r_cone, double* d,
                    double* rhs_z, double* scalars, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, NtRhsOp{s, z, w, eta, wbar, lam, lam_sq, c4, e2, r_cone, d, rhs_z, scalars}, st);
}

void qsk_apply_w(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* u,
                 double* out, int inverse, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, ApplyWOp{w, eta, wbar, u, out, inverse}, st);
}

void qsk_apply_w2(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* u,
                  double* out, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, ApplyW2Op{w, eta, wbar, u, out}, st);
}

void qsk_jordan_product(const ConeLayout& L, const double* u, const double* v, double* out, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, JordanProductOp{u, v, out}, st);
}

void qsk_jordan_divide(const ConeLayout& L, const double* lam, const double* v, double* out, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, JordanDivideOp{lam, v, out}, st);
}

void qsk_max_step(const ConeLayout& L, const double* u, const double* du, double* scalars, int slot_step,
                  int slot_viol, GridRed gr, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, MaxStepOp{u, du, scalars, slot_step, slot_viol, gr}, st);
}

void qsk_shift(const ConeLayout& L, const double* u, double* out, const double* scalars, int slot, double scale,
               cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, ShiftOp{u, out, scalars, slot, scale}, st);
}

void qsk_corrector_rhs(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* lam,
                       const double* lam_sq, const double* ds_a, const double* wdz_a, const double* r_cone,
                       double* dcomp, double* d, double* rhs_z, const double* scalars, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  launch(L, CorrRhsOp{w, eta, wbar, lam, lam_sq, ds_a, wdz_a, r_cone, dcomp, d, rhs_z, scalars}, st);
}

void qsk_post_solve(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* d,
                    const double* dz, const double* s, const double* z, double* wdz, double* ds, double* scalars,
                    int corrector, double step_fraction, double deg, GridRed gr, cudaStream_t st) {
  if (QS_EMPTY_GUARD(L)) return;
  if (corrector) launch(L, PostSolveOp<true>{w, eta, wbar, d, dz, s, z, wdz, ds, scalars, step_fraction, deg, gr}, st);
  else launch(L, PostSolveOp<false>{w, eta, wbar, d, dz, s, z, wdz, ds, scalars, step_fraction, deg, gr}, st);
}

void qsk_update_iterate(int n, int p, int m, const double* x, const double* y, const double* z, const double* s,
                        double* xo, double* yo, double* zo, double* so, const double* sol, const double* ds, double deg,
                        double* scalars, GridRed gr, cudaStream_t st) {
  i64 big = n > m ? n : m;
  k_update_iterate<<<qs_grid(vec_grid(big)), QS_THREADS, 0, st>>>(n, p, m, x, y, z, s, xo, yo, zo, so, sol, ds, deg, scalars, gr);
}

void qsk_dot(int m, const double* a, const double* b, double scale, double* out, GridRed gr, cudaStream_t st) {
  k_dot<<<qs_grid(vec_grid(m)), QS_THREADS, 0, st>>>(m, a, b, scale, out, gr);
}
