// Sparse products for the residuals and the refinement operator.
//
// The reference keeps P (upper), A and G in CSC and uses a column-scatter
// product for M x and a column gather-dot for M'x (sparse.py:119-150,
// _kernels.py:13-43).  A scatter needs atomics on a GPU, so setup builds, once,
// the row-major views the gathers need:
//     Pf  = P + P' - diag(P) in CSR      (n x n)
//     At  = CSC of A read as CSR of A'   (n x p)   -- zero-copy
//     Gt  = CSC of G read as CSR of G'   (n x m)   -- zero-copy
//     Ar  = CSR of A                     (p x n)
//     Gr  = CSR of G                     (m x n)
// Every product is then a gather-dot with `tpr` (1..32, power of two) lanes
// per row chosen from the mean row length; sums are deterministic.
//
// compute_residuals (ipm.py:70-103) is ONE launch over the row ranges
// [dual | eq | cone] with all norms reduced in the same pass.
#include "spmv_kernels.h"

#include <algorithm>

namespace {

__device__ __forceinline__ double row_dot(const Csr& M, int row, const double* __restrict__ x, int lane, int tpr,
                                          unsigned mask) {
  double acc = 0.0;
  if (row < M.rows) {
    const int e = M.ptr[row + 1];
    for (int p = M.ptr[row] + lane; p < e; p += tpr) acc += M.val[p] * x[M.idx[p]];
  }
  for (int o = tpr >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o);
  return acc;
}

// Four rows at once with the same lane group: four independent load chains
// (row pointer -> index/value -> x) are in flight per thread instead of one.
// Rows are short here (1..50 entries), so the products are latency-bound and
// memory-level parallelism is what buys bandwidth.
__device__ __forceinline__ void row_dot4(const Csr& M, const int (&row)[4], const double* __restrict__ x, int lane,
                                         int tpr, unsigned mask, double (&acc)[4]) {
  int b[4], e[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const bool ok = row[r] < M.rows;
    b[r] = ok ? M.ptr[row[r]] + lane : 0;
    e[r] = ok ? M.ptr[row[r] + 1] : 0;
    acc[r] = 0.0;
  }
  bool more = true;
  while (more) {
    more = false;
    int ix[4];
    double va[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const bool on = b[r] < e[r];
      ix[r] = on ? M.idx[b[r]] : 0;
      va[r] = on ? M.val[b[r]] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (b[r] < e[r]) {
        acc[r] += va[r] * x[ix[r]];
        b[r] += tpr;
        more |= b[r] < e[r];
      }
    }
  }
  for (int o = tpr >> 1; o > 0; o >>= 1) {
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[r] += __shfl_xor_sync(mask, acc[r], o);
  }
}

// One row of the fused dual-range matrix Dt = [Pf | A' | G']: three sums (P x, A'y, G'z), entries in the order Pf, A',
// G' and, inside a block, in the block's own order -- so each sum is bitwise the one row_dot_thread would produce.
__device__ __forceinline__ void row_dot_fused(const Csr& Dt, int row, const double* __restrict__ x,
                                              const double* __restrict__ y, const double* __restrict__ z, double& px,
                                              double& aty, double& gtz) {
  px = aty = gtz = 0.0;
  const int e = Dt.ptr[row + 1];
  for (int p = Dt.ptr[row]; p < e; ++p) {
    const int j = Dt.idx[p];
    const double v = Dt.val[p];
    const int tag = (unsigned)j >> QS_DT_TAG_SHIFT, col = j & QS_DT_COL_MASK;
    if (tag == 0) px += v * x[col];
    else if (tag == 1) aty += v * y[col];
    else gtz += v * z[col];
  }
}

// Short rows (a handful of entries): one thread per row, plain loop.  Few instructions and few registers, so
// many warps are resident and their load chains overlap; the generic lane-group machinery costs ~10x more
// instructions per entry on such rows.  Same summation order as a one-lane group.
__device__ __forceinline__ double row_dot_thread(const Csr& M, int row, const double* __restrict__ x) {
  double acc = 0.0;
  const int e = M.ptr[row + 1];
  for (int p = M.ptr[row]; p < e; ++p) acc += M.val[p] * x[M.idx[p]];
  return acc;
}

// Thread-per-row products with memory-level parallelism: NM matrices x NR rows per thread advance side by side, so
// the three dependent round trips of a row (row pointer -> index/value -> operand) are paid once per NM * NR rows
// instead of once per row -- with rows of 1-3 entries the kernel is bound by exactly that latency (ncu: 30 cycles of
// long-scoreboard stall per issue, 23 % DRAM utilisation with one row at a time).  Entry order within a row is
// unchanged, so the sums are bitwise those of row_dot_thread.  A matrix whose rows all hold exactly one entry
// (exact1: a signed permutation such as the G of an epigraph form or of bound constraints) needs no row pointers.
template <int NM, int NR>
__device__ __forceinline__ void thread_dots(const Csr* const (&M)[NM], const double* const (&x)[NM],
                                            const int (&row)[NR], int nrows, double (&acc)[NM][NR]) {
  int b[NM][NR], len[NM][NR], maxlen = 0;
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const bool ok = row[r] < nrows;
      if (M[m]->exact1) {
        b[m][r] = row[r];
        len[m][r] = ok ? 1 : 0;
      } else {
        b[m][r] = ok ? M[m]->ptr[row[r]] : 0;
        len[m][r] = ok ? M[m]->ptr[row[r] + 1] - b[m][r] : 0;
      }
      acc[m][r] = 0.0;
    }
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int r = 0; r < NR; ++r) maxlen = max(maxlen, len[m][r]);
  for (int k = 0; k < maxlen; ++k) {
    int ix[NM][NR];
    double va[NM][NR];
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const bool on = k < len[m][r];
        ix[m][r] = on ? M[m]->idx[b[m][r] + k] : 0;
        va[m][r] = on ? M[m]->val[b[m][r] + k] : 0.0;
      }
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (k < len[m][r]) acc[m][r] += va[m][r] * x[m][ix[m][r]];
  }
}

// The dual range needs three products per row (P x, A'y, G'z).  Run them side by side: NM matrices x NR rows =
// NM * NR independent load chains (row pointer -> index/value -> operand) per lane group, so a trip costs three
// dependent memory round trips instead of nine.
template <int NM, int NR>
__device__ __forceinline__ void row_dots(const Csr* const (&M)[NM], const double* const (&x)[NM], const int (&row)[NR],
                                         int lane, int tpr, unsigned mask, double (&acc)[NM][NR]) {
  int b[NM][NR], e[NM][NR];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const bool ok = row[r] < M[m]->rows;
      b[m][r] = ok ? M[m]->ptr[row[r]] + lane : 0;
      e[m][r] = ok ? M[m]->ptr[row[r] + 1] : 0;
      acc[m][r] = 0.0;
    }
  bool more = true;
  while (more) {
    more = false;
    int ix[NM][NR];
    double va[NM][NR];
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const bool on = b[m][r] < e[m][r];
        ix[m][r] = on ? M[m]->idx[b[m][r]] : 0;
        va[m][r] = on ? M[m]->val[b[m][r]] : 0.0;
      }
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (b[m][r] < e[m][r]) {
          acc[m][r] += va[m][r] * x[m][ix[m][r]];
          b[m][r] += tpr;
          more |= b[m][r] < e[m][r];
        }
      }
  }
  for (int o = tpr >> 1; o > 0; o >>= 1) {
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int r = 0; r < NR; ++r) acc[m][r] += __shfl_xor_sync(mask, acc[m][r], o);
  }
}

__device__ __forceinline__ unsigned lane_mask(int tpr) {
  return tpr == 32 ? 0xffffffffu : (((1u << tpr) - 1u) << (threadIdx.x & 31 & ~(tpr - 1)));
}

// Long rows (mean length >= 512, e.g. the 2000-entry rows of a design matrix): the whole CTA takes one row,
// 4 independent loads in flight per thread, fixed-order block reduction.  Every thread gets the sum.
#define QS_TPR_CTA 256
__device__ __forceinline__ double row_dot_cta(const Csr& M, int row, const double* __restrict__ x, double* sm /*[8]*/) {
  const int b = M.ptr[row], e = M.ptr[row + 1];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int p = b + threadIdx.x;
  for (; p + 3 * QS_THREADS < e; p += 4 * QS_THREADS) {
    const int i0 = M.idx[p], i1 = M.idx[p + QS_THREADS], i2 = M.idx[p + 2 * QS_THREADS], i3 = M.idx[p + 3 * QS_THREADS];
    const double v0 = M.val[p], v1 = M.val[p + QS_THREADS], v2 = M.val[p + 2 * QS_THREADS], v3 = M.val[p + 3 * QS_THREADS];
    a0 += v0 * x[i0];
    a1 += v1 * x[i1];
    a2 += v2 * x[i2];
    a3 += v3 * x[i3];
  }
  for (; p < e; p += QS_THREADS) a0 += M.val[p] * x[M.idx[p]];
  double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __syncthreads();  // sm may still be read from the previous row
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < QS_THREADS / 32; ++w) t += sm[w];
  return t;
}

struct RowRange {
  int which;  // 0 dual, 1 eq, 2 cone
  int row, stride, lane, tpr;
  unsigned mask;
};

// block ranges: the first nbe blocks stride over the eq rows (rows of A are the long ones when A is a design
// matrix: start them first), the next nbd over the dual rows, the rest over the cone rows; a group of tpr lanes
// owns a row (tpr == QS_TPR_CTA: the whole CTA)
__device__ __forceinline__ RowRange locate(int nbd, int nbe, int nbc, int tpr_d, int tpr_e, int tpr_c) {
  RowRange r;
  int b = blockIdx.x, nb;
  if (b < nbe) {
    r.which = 1;
    r.tpr = tpr_e;
    nb = nbe;
  } else if (b < nbe + nbd) {
    r.which = 0;
    r.tpr = tpr_d;
    b -= nbe;
    nb = nbd;
  } else {
    r.which = 2;
    r.tpr = tpr_c;
    b -= nbd + nbe;
    nb = nbc;
  }
  if (r.tpr == QS_TPR_CTA) {
    r.row = b;
    r.stride = nb;
    r.lane = threadIdx.x;
    r.mask = 0xffffffffu;
    return r;
  }
  r.row = (b * blockDim.x + threadIdx.x) / r.tpr;
  r.stride = nb * (QS_THREADS / r.tpr);
  r.lane = threadIdx.x & (r.tpr - 1);
  r.mask = lane_mask(r.tpr);
  return r;
}

__device__ __forceinline__ double absmax(double a, double v) {
  const double t = fabs(v);
  return (t > a || t != t) ? t : a;  // NaN sticks
}

// compute_residuals is three launches, one per row range (dual / eq / cone), each compiled for ONE row-product
// mode: a fused single kernel carried the registers of all nine (range, mode) paths (80 per thread, 3 CTAs per
// SM) and, with rows this short, the kernel is bound by how many load chains are in flight.
enum { MODE_THREAD = 0, MODE_GROUP = 1, MODE_CTA = 2, MODE_MLP = 3, MODE_FUSED = 4, MODE_SPLIT = 5 };  // MLP: thread per row, several rows in flight
enum { RANGE_DUAL = 0, RANGE_EQ = 1, RANGE_CONE = 2 };

__device__ __forceinline__ RowRange locate1(int tpr, int mode) {
  RowRange r;
  r.which = 0;
  r.tpr = tpr;
  if (mode == MODE_CTA) {
    r.row = blockIdx.x;
    r.stride = gridDim.x;
    r.lane = threadIdx.x;
    r.mask = 0xffffffffu;
    return r;
  }
  r.row = (blockIdx.x * blockDim.x + threadIdx.x) / tpr;
  r.stride = gridDim.x * (QS_THREADS / tpr);
  r.lane = threadIdx.x & (tpr - 1);
  r.mask = lane_mask(tpr);
  return r;
}

// partial[row * QS_ROW_SEGS + seg] = sum over segment `seg` of row `row` of M(row, :) x  -- a warp per segment
template <bool BATCH>
__global__ void __launch_bounds__(QS_THREADS) k_rowseg_partial(Csr M, const double* __restrict__ x, double* partial) {
  if (BATCH) {
    QS_BATCH(M, x, partial);
  }
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= M.rows * QS_ROW_SEGS) return;
  const int row = w / QS_ROW_SEGS, seg = w - row * QS_ROW_SEGS;
  const int b = M.ptr[row];
  const i64 len = M.ptr[row + 1] - b;
  const int s0 = b + (int)(len * seg / QS_ROW_SEGS), s1 = b + (int)(len * (seg + 1) / QS_ROW_SEGS);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int p = s0 + lane;
  for (; p + 96 < s1; p += 128) {
    const int i0 = M.idx[p], i1 = M.idx[p + 32], i2 = M.idx[p + 64], i3 = M.idx[p + 96];
    const double v0 = M.val[p], v1 = M.val[p + 32], v2 = M.val[p + 64], v3 = M.val[p + 96];
    a0 += v0 * x[i0];
    a1 += v1 * x[i1];
    a2 += v2 * x[i2];
    a3 += v3 * x[i3];
  }
  for (; p < s1; p += 32) a0 += M.val[p] * x[M.idx[p]];
  double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) partial[w] = acc;
}

// r_dual = P x + c + A'y + G'z (ipm.py:76), -r_dual -> rhs[0:n]; |Px|, |A'y|, |G'z|, |r_dual| (inf norms), x'Px, c'x
template <int MODE, bool BATCH>
__global__ void __launch_bounds__(QS_THREADS) k_resid_dual(ResidualArgs A) {
  if (BATCH) {  // moved pointers cost registers (the unmoved ones are read from the parameter bank): own instantiation
    QS_BATCH(A);
  }
  enum { PX, ATY, GTZ, RD, XPX, CX, NV };
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  const RowRange r = locate1((MODE == MODE_THREAD || MODE == MODE_MLP || MODE == MODE_FUSED) ? 1 : A.Pf.tpr, MODE);
  auto finish_row = [&](int row, double px, double aty, double gtz) {
    const double ci = A.c[row], xi = A.x[row];
    const double rd = px + ci + aty + gtz;
    A.rhs[row] = -rd;
    v[PX] = absmax(v[PX], px);
    v[ATY] = absmax(v[ATY], aty);
    v[GTZ] = absmax(v[GTZ], gtz);
    v[RD] = absmax(v[RD], rd);
    v[XPX] += xi * px;
    v[CX] += ci * xi;
  };
  if (MODE == MODE_THREAD) {
    for (int row = r.row; row < A.n; row += r.stride)
      finish_row(row, row_dot_thread(A.Pf, row, A.x), row_dot_thread(A.At, row, A.y), row_dot_thread(A.Gt, row, A.z));
  } else if (MODE == MODE_FUSED) {
    for (int row = r.row; row < A.n; row += r.stride) {
      double px, aty, gtz;
      row_dot_fused(A.Dt, row, A.x, A.y, A.z, px, aty, gtz);
      finish_row(row, px, aty, gtz);
    }
  } else if (MODE == MODE_MLP) {
    const Csr* const mats[3] = {&A.Pf, &A.At, &A.Gt};
    const double* const vecs[3] = {A.x, A.y, A.z};
    for (int row0 = r.row; row0 < A.n; row0 += 2 * r.stride) {
      const int rows[2] = {row0, row0 + r.stride};
      double d[3][2];
      thread_dots<3, 2>(mats, vecs, rows, A.n, d);
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (rows[q] < A.n) finish_row(rows[q], d[0][q], d[1][q], d[2][q]);
    }
  } else {
    const Csr* const mats[3] = {&A.Pf, &A.At, &A.Gt};
    const double* const vecs[3] = {A.x, A.y, A.z};
    for (int row0 = r.row; row0 < A.n; row0 += 2 * r.stride) {
      const int rows[2] = {row0, row0 + r.stride};
      double d[3][2];
      row_dots<3, 2>(mats, vecs, rows, r.lane, r.tpr, r.mask, d);
      if (r.lane == 0) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (rows[q] < A.n) finish_row(rows[q], d[0][q], d[1][q], d[2][q]);
      }
    }
  }
  using Ops = RedOps<RED_AMAX, RED_AMAX, RED_AMAX, RED_AMAX, RED_SUM, RED_SUM>;
  double* sc = A.scalars;
  const int p = A.p;
  qs_grid_reduce<Ops>(v, A.gr, [=](double (&t)[NV]) {
    sc[SC_NORM_PX] = t[PX];
    sc[SC_NORM_ATY] = t[ATY];
    sc[SC_NORM_GTZ] = t[GTZ];
    sc[SC_NORM_RDUAL] = t[RD];
    sc[SC_XPX] = t[XPX];
    sc[SC_CX] = t[CX];
    sc[SC_OBJ] = 0.5 * t[XPX] + t[CX];
    if (p == 0) sc[SC_NORM_AX] = sc[SC_NORM_REQ] = 0.0;  // no equality launch
    if (!qs_finite(t[RD])) sc[SC_FLAG_NONFINITE] = 1.0;   // ipm.py:96-102
  });
}

// r_eq = A x - b (ipm.py:77), -r_eq -> rhs[n:n+p]; |Ax|, |r_eq|
template <int MODE, bool BATCH>
__global__ void __launch_bounds__(QS_THREADS) k_resid_eq(ResidualArgs A) {
  if (BATCH) {  // moved pointers cost registers (the unmoved ones are read from the parameter bank): own instantiation
    QS_BATCH(A);
  }
  enum { AX, RE, NV };
  double v[NV] = {0.0, 0.0};
  const RowRange r = locate1((MODE == MODE_THREAD || MODE == MODE_MLP || MODE == MODE_SPLIT) ? 1 : A.Ar.tpr, MODE);
  auto finish_row = [&](int row, double ax) {
    const double re = ax - A.b[row];
    A.rhs[A.n + row] = -re;
    v[AX] = absmax(v[AX], ax);
    v[RE] = absmax(v[RE], re);
  };
  if (MODE == MODE_THREAD) {
    for (int row = r.row; row < A.p; row += r.stride) finish_row(row, row_dot_thread(A.Ar, row, A.x));
  } else if (MODE == MODE_SPLIT) {  // the products were formed by k_rowseg_partial: add the segments in order
    for (int row = r.row; row < A.p; row += r.stride) {
      double ax = 0.0;
#pragma unroll
      for (int sg = 0; sg < QS_ROW_SEGS; ++sg) ax += A.seg_partial[row * QS_ROW_SEGS + sg];
      finish_row(row, ax);
    }
  } else if (MODE == MODE_MLP) {
    const Csr* const mats[1] = {&A.Ar};
    const double* const vecs[1] = {A.x};
    for (int row0 = r.row; row0 < A.p; row0 += 4 * r.stride) {
      const int rows[4] = {row0, row0 + r.stride, row0 + 2 * r.stride, row0 + 3 * r.stride};
      double d[1][4];
      thread_dots<1, 4>(mats, vecs, rows, A.p, d);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (rows[q] < A.p) finish_row(rows[q], d[0][q]);
    }
  } else if (MODE == MODE_CTA) {
    __shared__ double rsm[QS_THREADS / 32];
    for (int row = r.row; row < A.p; row += r.stride) {
      const double ax = row_dot_cta(A.Ar, row, A.x, rsm);
      if (threadIdx.x == 0) finish_row(row, ax);
    }
  } else {
    for (int row0 = r.row; row0 < A.p; row0 += 4 * r.stride) {
      const int rows[4] = {row0, row0 + r.stride, row0 + 2 * r.stride, row0 + 3 * r.stride};
      double ax[4];
      row_dot4(A.Ar, rows, A.x, r.lane, r.tpr, r.mask, ax);
      if (r.lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (rows[q] < A.p) finish_row(rows[q], ax[q]);
      }
    }
  }
  using Ops = RedOps<RED_AMAX, RED_AMAX>;
  double* sc = A.scalars;
  qs_grid_reduce<Ops>(v, A.gr, [=](double (&t)[NV]) {
    sc[SC_NORM_AX] = t[AX];
    sc[SC_NORM_REQ] = t[RE];
    if (!qs_finite(t[RE])) sc[SC_FLAG_NONFINITE] = 1.0;
  });
}

// r_cone = G x + s - h (ipm.py:78); |Gx|, |s|, |r_cone|, gap = s'z (ipm.py:79)
template <int MODE, bool BATCH>
__global__ void __launch_bounds__(QS_THREADS) k_resid_cone(ResidualArgs A) {
  if (BATCH) {  // moved pointers cost registers (the unmoved ones are read from the parameter bank): own instantiation
    QS_BATCH(A);
  }
  enum { GX, SN, RC, GAP, NV };
  double v[NV] = {0.0, 0.0, 0.0, 0.0};
  const RowRange r = locate1((MODE == MODE_THREAD || MODE == MODE_MLP) ? 1 : A.Gr.tpr, MODE);
  auto finish_row = [&](int row, double gx) {
    const double si = A.s[row];
    const double rc = gx + si - A.h[row];
    A.r_cone[row] = rc;
    v[GX] = absmax(v[GX], gx);
    v[SN] = absmax(v[SN], si);
    v[RC] = absmax(v[RC], rc);
    v[GAP] += si * A.z[row];
  };
  if (MODE == MODE_THREAD) {
    for (int row = r.row; row < A.m; row += r.stride) finish_row(row, row_dot_thread(A.Gr, row, A.x));
  } else if (MODE == MODE_MLP) {
    const Csr* const mats[1] = {&A.Gr};
    const double* const vecs[1] = {A.x};
    for (int row0 = r.row; row0 < A.m; row0 += 4 * r.stride) {
      const int rows[4] = {row0, row0 + r.stride, row0 + 2 * r.stride, row0 + 3 * r.stride};
      // the row's own operands do not depend on the product: in flight together with the first loads of the chain
      double si[4], hi[4], zi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = rows[q] < A.m;
        si[q] = ok ? A.s[rows[q]] : 0.0;
        hi[q] = ok ? A.h[rows[q]] : 0.0;
        zi[q] = ok ? A.z[rows[q]] : 0.0;
      }
      double d[1][4];
      thread_dots<1, 4>(mats, vecs, rows, A.m, d);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (rows[q] < A.m) {
          const double gx = d[0][q], rc = gx + si[q] - hi[q];
          A.r_cone[rows[q]] = rc;
          v[GX] = absmax(v[GX], gx);
          v[SN] = absmax(v[SN], si[q]);
          v[RC] = absmax(v[RC], rc);
          v[GAP] += si[q] * zi[q];
        }
    }
  } else if (MODE == MODE_CTA) {
    __shared__ double rsm[QS_THREADS / 32];
    for (int row = r.row; row < A.m; row += r.stride) {
      const double gx = row_dot_cta(A.Gr, row, A.x, rsm);
      if (threadIdx.x == 0) finish_row(row, gx);
    }
  } else {
    for (int row0 = r.row; row0 < A.m; row0 += 4 * r.stride) {
      const int rows[4] = {row0, row0 + r.stride, row0 + 2 * r.stride, row0 + 3 * r.stride};
      double gx[4];
      row_dot4(A.Gr, rows, A.x, r.lane, r.tpr, r.mask, gx);
      if (r.lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (rows[q] < A.m) finish_row(rows[q], gx[q]);
      }
    }
  }
  using Ops = RedOps<RED_AMAX, RED_AMAX, RED_AMAX, RED_SUM>;
  double* sc = A.scalars;
  qs_grid_reduce<Ops>(v, A.gr, [=](double (&t)[NV]) {
    sc[SC_NORM_GX] = t[GX];
    sc[SC_NORM_S] = t[SN];
    sc[SC_NORM_RCONE] = t[RC];
    sc[SC_GAP] = t[GAP];
    if (!qs_finite(t[RC]) || !qs_finite(t[GAP])) sc[SC_FLAG_NONFINITE] = 1.0;
  });
}

// r = rhs - K v with K applied as an operator (blocks P, A, G and W'W):
//   r_x = rhs_x - (P v_x + A' v_y + G' v_z)
//   r_y = rhs_y - A v_x
//   r_z = rhs_z - (G v_x - (W'W v_z))         w2vz precomputed by qsk_apply_w2
// plus ||r||_inf -> scalars[slot].  Reference: ldl.py:152,159 (there the
// product runs over the stored entries of K; same operator, other rounding).
__global__ void __launch_bounds__(QS_THREADS)
    k_kkt_residual(KktResidualArgs A, int nbd, int nbe, int nbc, int eq_split) {
  QS_BATCH(A);
  double v[1] = {0.0};
  const RowRange r = locate(nbd, nbe, nbc, A.Pf.tpr, eq_split ? 1 : A.Ar.tpr, A.Gr.tpr);
  const double* vx = A.v;
  const double* vy = A.v + A.n;
  const double* vz = A.v + A.n + A.p;
  if (r.which == 0 && r.tpr == 1 && A.Dt.ptr) {
    for (int row = r.row; row < A.n; row += r.stride) {
      double px, aty, gtz;
      row_dot_fused(A.Dt, row, vx, vy, vz, px, aty, gtz);
      const double t = A.rhs[row] - (px + aty + gtz);
      A.r[row] = t;
      v[0] = absmax(v[0], t);
    }
  } else if (r.which == 0 && r.tpr == 1) {
    const Csr* const mats[3] = {&A.Pf, &A.At, &A.Gt};
    const double* const vecs[3] = {vx, vy, vz};
    for (int row0 = r.row; row0 < A.n; row0 += 2 * r.stride) {
      const int rows[2] = {row0, row0 + r.stride};
      double d[3][2];
      thread_dots<3, 2>(mats, vecs, rows, A.n, d);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (rows[q] >= A.n) continue;
        const double t = A.rhs[rows[q]] - (d[0][q] + d[1][q] + d[2][q]);
        A.r[rows[q]] = t;
        v[0] = absmax(v[0], t);
      }
    }
  } else if (r.which == 0) {
    const Csr* const mats[3] = {&A.Pf, &A.At, &A.Gt};
    const double* const vecs[3] = {vx, vy, vz};
    for (int row0 = r.row; row0 < A.n; row0 += 2 * r.stride) {
      const int rows[2] = {row0, row0 + r.stride};
      double d[3][2];
      row_dots<3, 2>(mats, vecs, rows, r.lane, r.tpr, r.mask, d);
      if (r.lane == 0) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (rows[q] >= A.n) continue;
          const double t = A.rhs[rows[q]] - (d[0][q] + d[1][q] + d[2][q]);
          A.r[rows[q]] = t;
          v[0] = absmax(v[0], t);
        }
      }
    }
  } else if (r.which == 1 && eq_split) {  // products formed by k_rowseg_partial: add the segments in order
    for (int row = r.row; row < A.p; row += r.stride) {
      double ax = 0.0;
#pragma unroll
      for (int sg = 0; sg < QS_ROW_SEGS; ++sg) ax += A.seg_partial[row * QS_ROW_SEGS + sg];
      const double t = A.rhs[A.n + row] - ax;
      A.r[A.n + row] = t;
      v[0] = absmax(v[0], t);
    }
  } else if (r.which == 1 && r.tpr == QS_TPR_CTA) {
    __shared__ double rsm[QS_THREADS / 32];
    for (int row = r.row; row < A.p; row += r.stride) {
      const double ax = row_dot_cta(A.Ar, row, vx, rsm);
      if (threadIdx.x == 0) {
        const double t = A.rhs[A.n + row] - ax;
        A.r[A.n + row] = t;
        v[0] = absmax(v[0], t);
      }
    }
  } else if (r.which == 1 && r.tpr == 1) {
    for (int row = r.row; row < A.p; row += r.stride) {
      const double t = A.rhs[A.n + row] - row_dot_thread(A.Ar, row, vx);
      A.r[A.n + row] = t;
      v[0] = absmax(v[0], t);
    }
  } else if (r.which == 1) {
    for (int row0 = r.row; row0 < A.p; row0 += 4 * r.stride) {
      const int rows[4] = {row0, row0 + r.stride, row0 + 2 * r.stride, row0 + 3 * r.stride};
      double ax[4];
      row_dot4(A.Ar, rows, vx, r.lane, r.tpr, r.mask, ax);
      if (r.lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (rows[q] >= A.p) continue;
          const double t = A.rhs[A.n + rows[q]] - ax[q];
          A.r[A.n + rows[q]] = t;
          v[0] = absmax(v[0], t);
        }
      }
    }
  } else if (r.tpr == QS_TPR_CTA) {
    __shared__ double rsm2[QS_THREADS / 32];
    for (int row = r.row; row < A.m; row += r.stride) {
      const double gx = row_dot_cta(A.Gr, row, vx, rsm2);
      if (threadIdx.x == 0) {
        const int i = A.n + A.p + row;
        const double t = A.rhs[i] - (gx - A.w2vz[row]);
        A.r[i] = t;
        v[0] = absmax(v[0], t);
      }
    }
  } else if (r.tpr == 1) {
    const Csr* const mats[1] = {&A.Gr};
    const double* const vecs[1] = {vx};
    for (int row0 = r.row; row0 < A.m; row0 += 4 * r.stride) {
      const int rows[4] = {row0, row0 + r.stride, row0 + 2 * r.stride, row0 + 3 * r.stride};
      double rh[4], w2[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = rows[q] < A.m;
        rh[q] = ok ? A.rhs[A.n + A.p + rows[q]] : 0.0;
        w2[q] = ok ? A.w2vz[rows[q]] : 0.0;
      }
      double d[1][4];
      thread_dots<1, 4>(mats, vecs, rows, A.m, d);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (rows[q] >= A.m) continue;
        const double t = rh[q] - (d[0][q] - w2[q]);
        A.r[A.n + A.p + rows[q]] = t;
        v[0] = absmax(v[0], t);
      }
    }
  } else {
    for (int row0 = r.row; row0 < A.m; row0 += 4 * r.stride) {
      const int rows[4] = {row0, row0 + r.stride, row0 + 2 * r.stride, row0 + 3 * r.stride};
      double gx[4];
      row_dot4(A.Gr, rows, vx, r.lane, r.tpr, r.mask, gx);
      if (r.lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (rows[q] >= A.m) continue;
          const int i = A.n + A.p + rows[q];
          const double t = A.rhs[i] - (gx[q] - A.w2vz[rows[q]]);
          A.r[i] = t;
          v[0] = absmax(v[0], t);
        }
      }
    }
  }
  using Ops = RedOps<RED_AMAX>;
  double* out = A.scalars + A.slot;
  qs_grid_reduce<Ops>(v, A.gr, [=](double (&t)[1]) { *out = t[0]; });
}

// plain y (+)= M x, gather form
__global__ void __launch_bounds__(QS_THREADS) k_spmv_csr(Csr M, const double* x, double* y, int accumulate) {
  QS_BATCH(M, x, y);
  if (M.tpr == QS_TPR_CTA) {
    __shared__ double rsm[QS_THREADS / 32];
    for (int row = blockIdx.x; row < M.rows; row += gridDim.x) {
      const double d = row_dot_cta(M, row, x, rsm);
      if (threadIdx.x == 0) y[row] = accumulate ? y[row] + d : d;
    }
    return;
  }
  const int tpr = M.tpr;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / tpr;
  const double d = row_dot(M, row, x, threadIdx.x & (tpr - 1), tpr, lane_mask(tpr));
  if ((threadIdx.x & (tpr - 1)) == 0 && row < M.rows) y[row] = accumulate ? y[row] + d : d;
}

// out += sym(M) x for M stored as its upper triangle in CSC -- the reference's
// literal KKT product (_kernels.py:33-43), kept as the checked alternative to
// the operator form.  Scatter side uses fp64 atomics (order not fixed).
__global__ void __launch_bounds__(QS_THREADS)
    k_spmv_sym_upper_csc(int ncols, const i64* cp, const int* ri, const double* vx, const double* x, double* out) {
  QS_BATCH(cp, ri, vx, x, out);
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= ncols) return;
  const double xj = x[col];
  double acc = 0.0;
  for (i64 p = cp[col] + lane; p < cp[col + 1]; p += 32) {
    const int i = ri[p];
    const double v = vx[p];
    atomicAdd(&out[i], v * xj);
    if (i != col) acc += v * x[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) atomicAdd(&out[col], acc);
}

__global__ void __launch_bounds__(QS_THREADS) k_axpby(i64 n, double a, const double* x, double b, const double* y,
                                                      double* out) {
  QS_BATCH(x, y, out);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = a * x[i] + (y ? b * y[i] : 0.0);
}

__global__ void __launch_bounds__(QS_THREADS) k_gather(i64 n, const double* __restrict__ src,
                                                       const int* __restrict__ map, double* __restrict__ dst) {
  QS_BATCH(src, map, dst);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) dst[i] = src[map[i]];
}

__global__ void __launch_bounds__(QS_THREADS) k_absmax(i64 n, const double* x, double* out, double* nonfinite,
                                                       GridRed gr) {
  QS_BATCH(x, out, nonfinite, gr);
  double v[1] = {0.0};
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    v[0] = absmax(v[0], x[i]);
  using Ops = RedOps<RED_AMAX>;
  qs_grid_reduce<Ops>(v, gr, [=](double (&t)[1]) {
    *out = t[0];
    if (nonfinite && !qs_finite(t[0])) *nonfinite = 1.0;
  });
}

int blocks_for(int rows, int tpr) {
  if (rows <= 0) return 0;
  if (tpr == QS_TPR_CTA) return rows > QS_MAX_GRID ? QS_MAX_GRID : rows;
  const int rpb = QS_THREADS / tpr;
  return (rows + rpb - 1) / rpb;
}

int blocks_capped(int rows, int tpr, int rows_per_trip = 4) {
  // a lane group takes 4 rows per trip; at most 8 blocks per SM and range, so that on large problems every
  // group makes several trips and the 12-value block reduction at the end is amortised
  if (tpr == QS_TPR_CTA) return blocks_for(rows, tpr);
  if (tpr == 1) rows_per_trip = 1;  // thread-per-row path
  const int b = blocks_for((rows + rows_per_trip - 1) / rows_per_trip, tpr), cap = 148 * 8;
  return b > cap ? cap : b;
}

int vgrid(i64 n) {
  i64 g = (n + QS_THREADS - 1) / QS_THREADS;
  if (g < 1) g = 1;
  if (g > 148 * 8) g = 148 * 8;
  return (int)g;
}


__global__ void __launch_bounds__(QS_THREADS) k_gather3(i64 n, const double* __restrict__ s0, const double* __restrict__ s1,
                                                        const double* __restrict__ s2, const int* __restrict__ map,
                                                        double* __restrict__ dst) {
  QS_BATCH(s0, s1, s2, map, dst);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const int j = map[i];
    const int tag = (unsigned)j >> QS_DT_TAG_SHIFT, k = j & QS_DT_COL_MASK;
    dst[i] = tag == 0 ? s0[k] : (tag == 1 ? s1[k] : s2[k]);
  }
}

// Dt = [Pf | At | Gt] row by row with tagged indices (spmv_kernels.h), built on the device from the three row views
// that are already there: a thread per row (the host version of this loop cost 0.08 s at C4, more than the fused
// matrix saves in a whole solve).
__global__ void __launch_bounds__(QS_THREADS) k_build_dt(int n, Csr Pf, Csr At, Csr Gt, int* dp, int* di, double* dv,
                                                         int* dmap) {
  QS_BATCH(Pf, At, Gt, dp, di, dv, dmap);
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row > n) return;
  int at = Pf.ptr[row] + At.ptr[row] + Gt.ptr[row];
  dp[row] = at;
  if (row == n) return;
  for (int k = Pf.ptr[row]; k < Pf.ptr[row + 1]; ++k, ++at) {
    di[at] = Pf.idx[k];
    dmap[at] = k;
    dv[at] = Pf.val[k];
  }
  for (int k = At.ptr[row]; k < At.ptr[row + 1]; ++k, ++at) {
    di[at] = At.idx[k] | (1 << QS_DT_TAG_SHIFT);
    dmap[at] = k | (1 << QS_DT_TAG_SHIFT);
    dv[at] = At.val[k];
  }
  for (int k = Gt.ptr[row]; k < Gt.ptr[row + 1]; ++k, ++at) {
    di[at] = (int)((unsigned)Gt.idx[k] | (2u << QS_DT_TAG_SHIFT));
    dmap[at] = (int)((unsigned)k | (2u << QS_DT_TAG_SHIFT));
    dv[at] = Gt.val[k];
  }
}

// dst[i] = src[i] where *flag != 0 (the flag is a scalar of the instance: accept / reject decided on the host)
__global__ void __launch_bounds__(QS_THREADS) k_copy_if(i64 n, const double* flag, const double* src, double* dst) {
  QS_BATCH(flag, src, dst);
  if (*flag == 0.0) return;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) dst[i] = src[i];
}

// slot z of the batch arena receives the bytes of slot 0 (8-byte words); z = blockIdx.z + 1
__global__ void __launch_bounds__(QS_THREADS) k_broadcast(i64 nwords, unsigned long long* p) {
  unsigned long long* dst = (unsigned long long*)((char*)p + (size_t)(blockIdx.z + 1) * QS_BSTRIDE);
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < nwords; i += (i64)gridDim.x * blockDim.x) dst[i] = p[i];
}

}  // namespace

int qsk_pick_tpr(i64 nnz, i64 rows) {
  if (rows <= 0) return 1;
  const double mean = (double)nnz / (double)rows;
  if (mean >= 512.0) return QS_TPR_CTA;  // long rows: a CTA per row
  if (mean <= 6.0) return 1;             // short rows: a thread per row
  int t = 1;
  while (t < 32 && t * 2 <= mean) t <<= 1;  // largest power of two <= mean row length
  return t;
}

int qsk_residuals(const ResidualArgs& A, cudaStream_t st) {
  // thread-per-row ranges.  MLP variant (QS_RESID_MLP=0 selects the one-row-at-a-time kernels everywhere, =2 the MLP
  // kernels everywhere): `per` rows per thread and trip, about one trip per thread, at most the CTAs resident at
  // once.  Measured at C4 (ncu, profiles/r02e_resid_*): cone range 31.7 -> 23.9 us with four rows in flight; the
  // dual range (three matrices per row) is SLOWER with two rows in flight (62 registers, 4 CTAs per SM: 44.5 ->
  // 52.7 us), so it keeps one row per thread and trip.
  static const int mlp_env = getenv("QS_RESID_MLP") ? atoi(getenv("QS_RESID_MLP")) : 1;
  static const bool mlp = mlp_env != 0;
  static const bool mlp_dual = mlp_env == 2;
  static const bool split_rows = !(getenv("QS_RESID_SPLIT") && atoi(getenv("QS_RESID_SPLIT")) == 0);
  auto tgrid = [](int rows, int per) {
    if (!mlp) return std::max(1, std::min(148 * 16, (rows + 2 * QS_THREADS - 1) / (2 * QS_THREADS)));
    return std::max(1, std::min(148 * 8, (rows + per * QS_THREADS - 1) / (per * QS_THREADS)));
  };
  const bool bt = qs_tls_batch > 1;
#define QS_RESID(kern, MODE, grid)                                                       \
  do {                                                                                   \
    if (bt) kern<MODE, true><<<qs_grid(grid), QS_THREADS, 0, st>>>(A);                   \
    else kern<MODE, false><<<qs_grid(grid), QS_THREADS, 0, st>>>(A);                     \
  } while (0)
#define QS_RESID_T(kern, rows, per)                                                      \
  do {                                                                                   \
    if (mlp) QS_RESID(kern, MODE_MLP, tgrid(rows, per));                                 \
    else QS_RESID(kern, MODE_THREAD, tgrid(rows, per));                                  \
  } while (0)
  int launches = 0;
  if (A.p > 0) {  // rows of A are the long ones when A is a design matrix: start them first
    const int t = A.Ar.tpr;
    if (t == 1) QS_RESID_T(k_resid_eq, A.p, 4);
    else if (t == QS_TPR_CTA && A.seg_partial && split_rows) {
      const int nw = A.p * QS_ROW_SEGS, nb = (nw * 32 + QS_THREADS - 1) / QS_THREADS;
      if (bt) k_rowseg_partial<true><<<qs_grid(nb), QS_THREADS, 0, st>>>(A.Ar, A.x, A.seg_partial);
      else k_rowseg_partial<false><<<qs_grid(nb), QS_THREADS, 0, st>>>(A.Ar, A.x, A.seg_partial);
      QS_RESID(k_resid_eq, MODE_SPLIT, (A.p + QS_THREADS - 1) / QS_THREADS);
      ++launches;
    } else if (t == QS_TPR_CTA) QS_RESID(k_resid_eq, MODE_CTA, blocks_for(A.p, t));
    else QS_RESID(k_resid_eq, MODE_GROUP, blocks_capped(A.p, t));
    ++launches;
  }
  static const bool fused_dual = !(getenv("QS_RESID_FUSED") && atoi(getenv("QS_RESID_FUSED")) == 0);
  if (A.Pf.tpr == 1 && A.Dt.ptr && fused_dual) {
    QS_RESID(k_resid_dual, MODE_FUSED, std::max(1, std::min(148 * 16, (A.n + 2 * QS_THREADS - 1) / (2 * QS_THREADS))));
  } else if (A.Pf.tpr == 1) {
    if (mlp_dual) QS_RESID(k_resid_dual, MODE_MLP, tgrid(A.n, 2));
    else QS_RESID(k_resid_dual, MODE_THREAD, std::max(1, std::min(148 * 16, (A.n + 2 * QS_THREADS - 1) / (2 * QS_THREADS))));
  }
  else QS_RESID(k_resid_dual, MODE_GROUP, blocks_capped(A.n, A.Pf.tpr, 2));
  {
    const int t = A.Gr.tpr;
    if (t == 1) QS_RESID_T(k_resid_cone, A.m, 4);
    else if (t == QS_TPR_CTA) QS_RESID(k_resid_cone, MODE_CTA, blocks_for(A.m, t));
    else QS_RESID(k_resid_cone, MODE_GROUP, blocks_capped(A.m, t));
  }
#undef QS_RESID_T
#undef QS_RESID
  return launches + 2;
}

void qsk_kkt_residual(const KktResidualArgs& A, cudaStream_t st) {
  static const bool split_rows = !(getenv("QS_RESID_SPLIT") && atoi(getenv("QS_RESID_SPLIT")) == 0);
  const int eq_split = A.p > 0 && A.Ar.tpr == QS_TPR_CTA && A.seg_partial && split_rows;
  if (eq_split) {
    const int nw = A.p * QS_ROW_SEGS, nb = (nw * 32 + QS_THREADS - 1) / QS_THREADS;
    if (qs_tls_batch > 1) k_rowseg_partial<true><<<qs_grid(nb), QS_THREADS, 0, st>>>(A.Ar, A.v, A.seg_partial);
    else k_rowseg_partial<false><<<qs_grid(nb), QS_THREADS, 0, st>>>(A.Ar, A.v, A.seg_partial);
  }
  const int nbd = blocks_capped(A.n, A.Pf.tpr, 2), nbc = blocks_capped(A.m, A.Gr.tpr);
  const int nbe = eq_split ? (A.p + QS_THREADS - 1) / QS_THREADS : blocks_capped(A.p, A.Ar.tpr);
  k_kkt_residual<<<qs_grid(nbd + nbe + nbc), QS_THREADS, 0, st>>>(A, nbd, nbe, nbc, eq_split);
}

void qsk_spmv_csr(const Csr& M, const double* x, double* y, int accumulate, cudaStream_t st) {
  if (M.rows <= 0) return;
  k_spmv_csr<<<qs_grid(blocks_for(M.rows, M.tpr)), QS_THREADS, 0, st>>>(M, x, y, accumulate);
}

void qsk_spmv_sym_upper_csc(int ncols, const i64* cp, const int* ri, const double* vx, const double* x, double* out,
                            cudaStream_t st) {
  if (ncols <= 0) return;
  const i64 blocks = ((i64)ncols * 32 + QS_THREADS - 1) / QS_THREADS;
  k_spmv_sym_upper_csc<<<qs_grid((unsigned)blocks), QS_THREADS, 0, st>>>(ncols, cp, ri, vx, x, out);
}

void qsk_gather(i64 n, const double* src, const int* map, double* dst, cudaStream_t st) {
  if (n <= 0) return;
  k_gather<<<qs_grid(vgrid(n)), QS_THREADS, 0, st>>>(n, src, map, dst);
}

void qsk_axpby(i64 n, double a, const double* x, double b, const double* y, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_axpby<<<qs_grid(vgrid(n)), QS_THREADS, 0, st>>>(n, a, x, b, y, out);
}

void qsk_absmax(i64 n, const double* x, double* out, double* nonfinite, GridRed gr, cudaStream_t st) {
  k_absmax<<<qs_grid(vgrid(n)), QS_THREADS, 0, st>>>(n, x, out, nonfinite, gr);
}

void qsk_copy_if(i64 n, const double* flag, const double* src, double* dst, cudaStream_t st) {
  if (n > 0) k_copy_if<<<qs_grid(vgrid(n)), QS_THREADS, 0, st>>>(n, flag, src, dst);
}

void qsk_broadcast(i64 nwords, void* p, int slots, cudaStream_t st) {
  if (nwords > 0 && slots > 1)
    k_broadcast<<<dim3((unsigned)vgrid(nwords), 1, (unsigned)(slots - 1)), QS_THREADS, 0, st>>>(nwords, (unsigned long long*)p);
}

void qsk_gather3(i64 n, const double* src0, const double* src1, const double* src2, const int* map, double* dst,
                 cudaStream_t st) {
  if (n > 0) k_gather3<<<qs_grid(vgrid(n)), QS_THREADS, 0, st>>>(n, src0, src1, src2, map, dst);
}

void qsk_build_dt(int n, const Csr& Pf, const Csr& At, const Csr& Gt, int* dp, int* di, double* dv, int* dmap,
                  cudaStream_t st) {
  k_build_dt<<<qs_grid((n + 1 + QS_THREADS - 1) / QS_THREADS), QS_THREADS, 0, st>>>(n, Pf, At, Gt, dp, di, dv, dmap);
}
