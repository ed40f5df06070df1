// Shared device-side building blocks for the qsocp sm_100a kernels.
//
// Layout conventions (mirrors the reference's flat conic vectors,
// pkg/src/qsocp/cones.py:40-58): a conic vector has length m; the orthant
// block is [0, l); second-order cone k occupies [soc_ptr[k], soc_ptr[k+1]) with
// its head first.  All values fp64.  Indices are int32 on the device (m and
// nnz are checked < 2^31 at setup); int64 only where the reference contract
// exposes them (the slot -> position map).
#pragma once
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

typedef long long i64;

#define QS_THREADS 256
#define QS_MAX_GRID 8192  // every reducing kernel launches at most this many blocks
#define QS_RED_MAXK 16    // widest grid reduction (values per block)
#define QS_UNBOUNDED DBL_MAX  // _cone_kernels.py:13

// ------------------------------------------------------------------ scalars
// Device-resident scalar block of one solver instance.  Written by the last
// block of the reducing kernels, read by later kernels and (once per
// iteration) by the host through a pinned mirror.
enum QsScalar {
  SC_STEP_S = 0,
  SC_STEP_Z,
  SC_ALPHA_AFF,
  SC_ALPHA,
  SC_MU,
  SC_MU_AFF,
  SC_SIGMA,
  SC_VIOL_S,
  SC_VIOL_Z,
  SC_FLAG_NOT_INTERIOR,  // nonzero: NT scaling / max-step pre-check failed
  SC_FLAG_NONFINITE,     // nonzero: non-finite iterate / residual / step
  SC_FLAG_BAD_STEP,      // nonzero: alpha <= 0 or non-finite
  SC_GAP,
  SC_OBJ,
  SC_XPX,
  SC_CX,
  SC_NORM_PX,
  SC_NORM_ATY,
  SC_NORM_GTZ,
  SC_NORM_AX,
  SC_NORM_GX,
  SC_NORM_S,
  SC_NORM_RDUAL,
  SC_NORM_REQ,
  SC_NORM_RCONE,
  SC_REFINE_RNORM,   // ||rhs - K x||_inf of the last refinement residual
  SC_REFINE_NONFINITE,
  SC_SHIFT,          // bring_to_interior: violation alpha
  SC_TMP0,
  SC_TMP1,
  SC_TMP2,
  SC_TMP3,
  SC_PIVOT_BUMPS,
  SC_PIVOT_NONFINITE,
  SC_COUNT = 48
};

// ------------------------------------------------------------ instance batches
// Batched small-problem mode: B instances with ONE sparsity pattern live in B equal slots of one
// device arena, QS_BSTRIDE bytes apart; slot b is a byte-for-byte copy of slot 0's layout (pattern arrays included),
// so the address of anything belonging to instance b is the address in slot 0 plus b * QS_BSTRIDE.  A batched launch
// is the ordinary launch with gridDim.z = B: every kernel begins with QS_BATCH(...) over its pointer arguments
// (and structs of pointers), which moves them to the slot of blockIdx.z.  gridDim.z == 1 is the ordinary solver.
#define QS_BSTRIDE (size_t(1) << 25)  // 32 MiB per instance: "small" means the whole handle fits

// qs_moved(x, off): pointers move by `off` bytes (null stays null; T may be const), structs of pointers move their
// members (they provide  __device__ void shift(size_t off)), numbers stay.  By value and back by assignment, so
// __restrict__-qualified kernel parameters are fine.
template <class T>
__device__ __forceinline__ T* qs_moved(T* p, size_t off) {
  return p ? (T*)((char*)p + off) : p;
}
template <class T>
__device__ __forceinline__ typename std::enable_if<std::is_arithmetic<T>::value || std::is_enum<T>::value, T>::type
qs_moved(T v, size_t) {
  return v;
}
template <class T>
__device__ __forceinline__ typename std::enable_if<std::is_class<T>::value, T>::type qs_moved(T s, size_t off) {
  s.shift(off);
  return s;
}
// used inside the shift() members
template <class T>
__device__ __forceinline__ void qs_shift(size_t off, T& x) {
  x = qs_moved(x, off);
}
#define QS_FE_1(m, x) m(x)
#define QS_FE_2(m, x, ...) m(x) QS_FE_1(m, __VA_ARGS__)
#define QS_FE_3(m, x, ...) m(x) QS_FE_2(m, __VA_ARGS__)
#define QS_FE_4(m, x, ...) m(x) QS_FE_3(m, __VA_ARGS__)
#define QS_FE_5(m, x, ...) m(x) QS_FE_4(m, __VA_ARGS__)
#define QS_FE_6(m, x, ...) m(x) QS_FE_5(m, __VA_ARGS__)
#define QS_FE_7(m, x, ...) m(x) QS_FE_6(m, __VA_ARGS__)
#define QS_FE_8(m, x, ...) m(x) QS_FE_7(m, __VA_ARGS__)
#define QS_FE_9(m, x, ...) m(x) QS_FE_8(m, __VA_ARGS__)
#define QS_FE_10(m, x, ...) m(x) QS_FE_9(m, __VA_ARGS__)
#define QS_FE_11(m, x, ...) m(x) QS_FE_10(m, __VA_ARGS__)
#define QS_FE_12(m, x, ...) m(x) QS_FE_11(m, __VA_ARGS__)
#define QS_FE_13(m, x, ...) m(x) QS_FE_12(m, __VA_ARGS__)
#define QS_FE_14(m, x, ...) m(x) QS_FE_13(m, __VA_ARGS__)
#define QS_FE_15(m, x, ...) m(x) QS_FE_14(m, __VA_ARGS__)
#define QS_FE_16(m, x, ...) m(x) QS_FE_15(m, __VA_ARGS__)
#define QS_FE_17(m, x, ...) m(x) QS_FE_16(m, __VA_ARGS__)
#define QS_FE_18(m, x, ...) m(x) QS_FE_17(m, __VA_ARGS__)
#define QS_FE_19(m, x, ...) m(x) QS_FE_18(m, __VA_ARGS__)
#define QS_FE_20(m, x, ...) m(x) QS_FE_19(m, __VA_ARGS__)
#define QS_FE_21(m, x, ...) m(x) QS_FE_20(m, __VA_ARGS__)
#define QS_FE_22(m, x, ...) m(x) QS_FE_21(m, __VA_ARGS__)
#define QS_FE_23(m, x, ...) m(x) QS_FE_22(m, __VA_ARGS__)
#define QS_FE_24(m, x, ...) m(x) QS_FE_23(m, __VA_ARGS__)
#define QS_FE_PICK(_1, _2, _3, _4, _5, _6, _7, _8, _9, _10, _11, _12, _13, _14, _15, _16, _17, _18, _19, _20, _21, _22, _23, _24, NAME, ...) NAME
#define QS_FOR_EACH(m, ...) QS_FE_PICK(__VA_ARGS__, QS_FE_24, QS_FE_23, QS_FE_22, QS_FE_21, QS_FE_20, QS_FE_19, QS_FE_18, QS_FE_17, QS_FE_16, QS_FE_15, QS_FE_14, QS_FE_13, QS_FE_12, QS_FE_11, QS_FE_10, QS_FE_9, QS_FE_8, QS_FE_7, QS_FE_6, QS_FE_5, QS_FE_4, QS_FE_3, QS_FE_2, QS_FE_1)(m, __VA_ARGS__)
#define QS_MV_(x) x = qs_moved(x, qs_boff_);
#ifdef QS_NO_BATCH  // A/B builds: the cost of the prologue
#define QS_BATCH(...)
#else
#define QS_BATCH(...)                                               \
  if (gridDim.z > 1 && blockIdx.z > 0) {                            \
    const size_t qs_boff_ = (size_t)blockIdx.z * QS_BSTRIDE;        \
    QS_FOR_EACH(QS_MV_, __VA_ARGS__)                                \
  }
#endif

// Host side: the batch size of the launches issued by this thread (1 outside qs_batch_* calls).
extern thread_local int qs_tls_batch;
inline dim3 qs_grid(dim3 g) {
  g.z = (unsigned)qs_tls_batch;
  return g;
}
// memset / device-to-device copy of the same range in every slot
inline cudaError_t qs_memset_b(void* p, int value, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  if (qs_tls_batch <= 1) return cudaMemsetAsync(p, value, bytes, st);
  return cudaMemset2DAsync(p, QS_BSTRIDE, value, bytes, (size_t)qs_tls_batch, st);
}
inline cudaError_t qs_copy_b(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  if (qs_tls_batch <= 1) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st);
  return cudaMemcpy2DAsync(dst, QS_BSTRIDE, src, QS_BSTRIDE, bytes, (size_t)qs_tls_batch, cudaMemcpyDeviceToDevice, st);
}

// --------------------------------------------------------------- cone layout
struct ConeLayout {
  int m, l, nsoc;
  const int* soc_ptr;    // [nsoc+1]
  int group;             // lanes cooperating on one small cone (1,2,4,...,32)
  int single;            // -1: each op picks its own decomposition; 0 / 1 force chunked / register-resident
  int waves;             // persistent grid = waves x the CTAs resident at once (0 = 1; tuning knob QS_CONE_WAVES)
  int nsmall;            // cones handled by lane groups
  const int* small_ids;  // [nsmall] small cones sorted by dimension, largest first (nullptr: natural order)
  int nbig;              // cones handled by a whole CTA (dim > big threshold)
  const int* big_ids;    // [nbig]
  __device__ void shift(size_t off) {
    qs_shift(off, soc_ptr);
    qs_shift(off, small_ids);
    qs_shift(off, big_ids);
  }
};

// ------------------------------------------------------------ group policies
// A "group" is the set of threads that cooperates on one cone.  sum() is an
// all-reduce: every thread of the group gets the same bits back.
// kR = elements of the cone a thread keeps in registers per chunk; kSingle = the
// whole cone is one chunk (group * kR >= dim by construction of the layout), so
// multi-pass ops read HBM once and never touch memory again between passes.
template <int G, int R_ = 4, bool SINGLE_ = false>
struct LaneGroup {
  static constexpr int kSize = G;
  static constexpr int kR = R_;
  static constexpr bool kSingle = SINGLE_;
  __device__ __forceinline__ int lane() const { return threadIdx.x & (G - 1); }
  __device__ __forceinline__ int size() const { return G; }
  // shuffles name only this group's lanes, so groups of one warp may diverge
  __device__ __forceinline__ unsigned mask() const {
    return G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (threadIdx.x & 31 & ~(G - 1)));
  }
  __device__ __forceinline__ double sum(double v) const {
    const unsigned mk = mask();
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mk, v, o);
    return v;
  }
  // several independent reductions interleaved: same instruction count, the
  // shuffle latencies overlap instead of adding up
  __device__ __forceinline__ void sum2(double& a, double& b) const {
    const unsigned mk = mask();
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double ta = __shfl_xor_sync(mk, a, o), tb = __shfl_xor_sync(mk, b, o);
      a += ta;
      b += tb;
    }
  }
  __device__ __forceinline__ void sum3(double& a, double& b, double& c) const {
    const unsigned mk = mask();
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double ta = __shfl_xor_sync(mk, a, o), tb = __shfl_xor_sync(mk, b, o), tc = __shfl_xor_sync(mk, c, o);
      a += ta;
      b += tb;
      c += tc;
    }
  }
  __device__ __forceinline__ void sum4(double& a, double& b, double& c, double& d) const {
    const unsigned mk = mask();
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double ta = __shfl_xor_sync(mk, a, o), tb = __shfl_xor_sync(mk, b, o), tc = __shfl_xor_sync(mk, c, o),
                   td = __shfl_xor_sync(mk, d, o);
      a += ta;
      b += tb;
      c += tc;
      d += td;
    }
  }
};

struct CtaGroup {
  static constexpr int kR = 8;  // 256 threads x 8: cones up to 2048 stay in registers; longer ones are chunked
  static constexpr bool kSingle = false;
  double* scratch;  // [32 * 4] shared
  __device__ __forceinline__ int lane() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ void sum4(double& a, double& b, double& c, double& d) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ta = __shfl_xor_sync(0xffffffffu, a, o), tb = __shfl_xor_sync(0xffffffffu, b, o),
                   tc = __shfl_xor_sync(0xffffffffu, c, o), td = __shfl_xor_sync(0xffffffffu, d, o);
      a += ta;
      b += tb;
      c += tc;
      d += td;
    }
    __syncthreads();  // scratch may still be read from a previous reduction
    if ((threadIdx.x & 31) == 0) {
      double* sl = scratch + 4 * (threadIdx.x >> 5);
      sl[0] = a;
      sl[1] = b;
      sl[2] = c;
      sl[3] = d;
    }
    __syncthreads();
    a = b = c = d = 0.0;
    const int nw = (blockDim.x + 31) >> 5;
    for (int w = 0; w < nw; ++w) {
      a += scratch[4 * w];
      b += scratch[4 * w + 1];
      c += scratch[4 * w + 2];
      d += scratch[4 * w + 3];
    }
  }
  __device__ __forceinline__ double sum(double v) const {
    double b = 0.0, c = 0.0, d = 0.0;
    sum4(v, b, c, d);
    return v;
  }
  __device__ __forceinline__ void sum2(double& a, double& b) const {
    double c = 0.0, d = 0.0;
    sum4(a, b, c, d);
  }
  __device__ __forceinline__ void sum3(double& a, double& b, double& c) const {
    double d = 0.0;
    sum4(a, b, c, d);
  }
};

// ------------------------------------------------------------ cone fragments
// Slot r of a thread's fragment holds tail element t = base + lane + r * size of
// the cone (head t = 0 excluded: it is handled by scalar code), zero when t is
// outside [1, q).  All kR loads of a fragment are independent, so a thread has
// kR x (number of vectors) loads in flight before the first use.
#define QS_CHUNKS(base) for (int base = 0; base < (Grp::kSingle ? 1 : q); base += g.size() * Grp::kR)
#define QS_FRAG(r, t) _Pragma("unroll") for (int r = 0, t = base + g.lane(); r < Grp::kR; ++r, t += g.size())
#define QS_TAIL_OK(t, q) ((t) >= 1 && (t) < (q))

template <class Grp>
__device__ __forceinline__ void qs_frag_load(const Grp& g, const double* __restrict__ p, int q, int base,
                                             double (&f)[Grp::kR]) {
#pragma unroll
  for (int r = 0; r < Grp::kR; ++r) {
    const int t = base + g.lane() + r * g.size();
    f[r] = QS_TAIL_OK(t, q) ? p[t] : 0.0;
  }
}

// ------------------------------------------------------- grid-wide reduction
// Deterministic (fixed grid -> fixed order) reduction of K doubles across the
// whole grid with the "last block finishes" pattern: each block publishes its
// partials, takes a ticket, and the block drawing the last ticket combines all
// partials in block order and runs `fin(result)` on thread 0.
// RED_AMAX: max of NON-NEGATIVE doubles (|x| norms).  Their bit patterns order like unsigned integers and a
// NaN (sign cleared by fabs) is the largest pattern, so it propagates; a warp reduces one with two REDUX
// instructions instead of five shuffle rounds.
enum { RED_SUM = 0, RED_MIN = 1, RED_MAX = 2, RED_AMAX = 3 };

struct GridRed {
  double* partial;    // [>= gridDim.x * K]
  unsigned* counter;  // zero before the launch; left zero afterwards
  __device__ void shift(size_t off) {
    qs_shift(off, partial);
    qs_shift(off, counter);
  }
};

// The reduction operators of a launch are COMPILE-TIME constants (RedOps<RED_MIN, RED_MAX, ...>): after
// unrolling, every combine is a fixed two-or-three instruction sequence.  (With run-time operator codes the
// epilogue of the residual kernel was ~1000 instructions per thread -- more than its SpMV work.)
template <int OP>
__device__ __forceinline__ double qs_combine(double a, double b) {
  // NaN-propagating max/min so that non-finite data is never masked
  if (OP == RED_SUM) return a + b;
  if (OP == RED_AMAX)
    return ((unsigned long long)__double_as_longlong(b) > (unsigned long long)__double_as_longlong(a)) ? b : a;
  if (OP == RED_MIN) return (a != a) ? a : ((b < a || b != b) ? b : a);
  return (a != a) ? a : ((b > a || b != b) ? b : a);
}

template <int OP>
__device__ __forceinline__ double qs_identity() {
  return (OP == RED_SUM || OP == RED_AMAX) ? 0.0 : (OP == RED_MIN ? INFINITY : -INFINITY);
}

template <int... OPS>
struct RedOps {
  static constexpr int K = sizeof...(OPS);
};

// apply f.template operator()<k, OP_k>() for every k (C++17 fold over an index pack)
template <int... OPS, class F, int... IS>
__device__ __forceinline__ void qs_for_ops_impl(RedOps<OPS...>, F&& f, std::integer_sequence<int, IS...>) {
  (f(std::integral_constant<int, IS>{}, std::integral_constant<int, OPS>{}), ...);
}
template <int... OPS, class F>
__device__ __forceinline__ void qs_for_ops(RedOps<OPS...> o, F&& f) {
  qs_for_ops_impl(o, static_cast<F&&>(f), std::make_integer_sequence<int, sizeof...(OPS)>{});
}

template <class Ops>
__device__ __forceinline__ void qs_block_reduce(double (&v)[Ops::K], double* sm /*[32*K]*/) {
  constexpr int K = Ops::K;
  qs_for_ops(Ops{}, [&](auto kc, auto opc) {
    constexpr int k = decltype(kc)::value, OP = decltype(opc)::value;
    double x = v[k];
    if (OP == RED_AMAX) {
      const unsigned hi = (unsigned)__double2hiint(x), lo = (unsigned)__double2loint(x);
      const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
      const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
      x = __hiloint2double((int)mhi, (int)mlo);
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x = qs_combine<OP>(x, __shfl_xor_sync(0xffffffffu, x, o));
    }
    v[k] = x;
  });
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm[w * K + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    qs_for_ops(Ops{}, [&](auto kc, auto opc) {
      constexpr int k = decltype(kc)::value, OP = decltype(opc)::value;
      double x = sm[k];
      for (int j = 1; j < nw; ++j) x = qs_combine<OP>(x, sm[j * K + k]);
      v[k] = x;
    });
  }
}

// After the call, thread 0 of exactly one block (the last to arrive) has run
// fin(totals).  Every thread of every block must call this.
template <class Ops, class Fin>
__device__ __forceinline__ void qs_grid_reduce(double (&v)[Ops::K], GridRed gr, Fin fin) {
  constexpr int K = Ops::K;
  __shared__ double sm[32 * K];
  __shared__ int last;
  qs_block_reduce<Ops>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) gr.partial[(size_t)blockIdx.x * K + k] = v[k];
    __threadfence();
    const unsigned t = atomicInc(gr.counter, gridDim.x - 1);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc[K];
  qs_for_ops(Ops{}, [&](auto kc, auto opc) { acc[decltype(kc)::value] = qs_identity<decltype(opc)::value>(); });
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    qs_for_ops(Ops{}, [&](auto kc, auto opc) {
      constexpr int k = decltype(kc)::value;
      acc[k] = qs_combine<decltype(opc)::value>(acc[k], __ldcg(&gr.partial[(size_t)b * K + k]));
    });
  }
  qs_block_reduce<Ops>(acc, sm);
  if (threadIdx.x == 0) fin(acc);
}

// ------------------------------------------------------------------- helpers
__device__ __forceinline__ bool qs_finite(double v) { return fabs(v) <= DBL_MAX; }

// Exit step of one second-order cone from the quadratic's coefficients
// (a = du0^2 - |du1|^2, b = 2(u0 du0 - u1.du1), c = u0^2 - |u1|^2), branch for
// branch as the reference (_cone_kernels.py:124-143).
__device__ __forceinline__ double qs_soc_step(double a, double b, double c) {
  if (a == 0.0) return (b < 0.0) ? -c / b : QS_UNBOUNDED;
  const double disc = __dsub_rn(__dmul_rn(b, b), __dmul_rn(__dmul_rn(4.0, a), c));
  if (a > 0.0 && disc < 0.0) return QS_UNBOUNDED;
  const double sq = sqrt(disc);
  const double den = (b >= 0.0) ? (-b - sq) : (-b + sq);
  const double r1 = den / (2.0 * a);
  const double r2 = (den != 0.0) ? 2.0 * c / den : QS_UNBOUNDED;
  double step = QS_UNBOUNDED;
  if (0.0 < r1 && r1 < step) step = r1;
  if (0.0 < r2 && r2 < step) step = r2;
  return step;
}
