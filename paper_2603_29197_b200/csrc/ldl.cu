// GPU supernodal multifrontal LDL' (see ldl.h).
#include "ldl.h"

#include "devmem.h"

#include <cooperative_groups.h>

#include <chrono>
#include <cstdio>
#include <thread>

namespace cg = cooperative_groups;

namespace {

#define LDL_THREADS 256

struct Front {
  int c0, ns, nr, nu;
  const int* rows;
  double* Lp;
  double* Up;
};

// Update matrices are symmetric: only the lower triangle is stored, packed by columns (column j holds rows j..nu-1),
// nu (nu + 1) / 2 doubles per front -- half the memory and half the zero-fill of a full nu x nu square (C4: 13 -> 6.5 GB;
// SURVEY's denser C4, 170 GB of squares, fits only in this form).  Element (i, j), i >= j, is Up[qs_ucol(j, nu) + i].
__device__ __forceinline__ i64 qs_ucol(i64 j, i64 nu) { return j * nu - j * (j + 1) / 2; }

__device__ __forceinline__ Front front_of(const DevSym& S, int s, double* L, double* U) {
  Front f;
  f.c0 = S.col0[s];
  f.ns = S.col0[s + 1] - f.c0;
  f.nr = (int)(S.rowptr[s + 1] - S.rowptr[s]);
  f.nu = f.nr - f.ns;
  f.rows = S.rowidx + S.rowptr[s];
  f.Lp = L + S.Loff[s];
  f.Up = U ? U + S.Uoff[s] : nullptr;
  return f;
}

// K entry -> panel offset (run once at analysis)
__global__ void __launch_bounds__(LDL_THREADS) k_build_amap(int N, const i64* Kp, const int* Ki, DevSym S, i64* amap) {
  QS_BATCH(Kp, Ki, S, amap);
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= N) return;
  const int b = S.iperm[col];
  for (i64 p = Kp[col] + lane; p < Kp[col + 1]; p += 32) {
    const int a = S.iperm[Ki[p]];
    const int c = a < b ? a : b, r = a < b ? b : a;
    const int s = S.sup_of[c];
    const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
    const i64 rp = S.rowptr[s];
    const int nr = (int)(S.rowptr[s + 1] - rp);
    int lr;
    if (r < c0 + ns) {
      lr = r - c0;
    } else {
      const int* rows = S.rowidx + rp;
      int lo = ns, hi = nr;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rows[mid] < r)
          lo = mid + 1;
        else
          hi = mid;
      }
      lr = lo;  // present by construction of the symbolic structure
    }
    amap[p] = S.Loff[s] + lr + (i64)(c - c0) * nr;
  }
}

__global__ void __launch_bounds__(LDL_THREADS) k_scatter_values(i64 nnz, const double* __restrict__ Kx,
                                                                const i64* __restrict__ amap, double* __restrict__ L) {
  QS_BATCH(Kx, amap, L);
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < nnz; p += (i64)gridDim.x * blockDim.x)
    L[amap[p]] = Kx[p];
}

// The G' entries above the block in the SOC columns of K: a warp per column.  (Everything before the first SOC column
// -- P, A', the orthant part -- holds no block and goes through k_scatter_values entry by entry: a K column there can be
// one dense equality row, 10^5 entries in a budget constraint, which no per-column scheme should own.)
__global__ void __launch_bounds__(LDL_THREADS) k_scatter_other(int N, ConeBlocks C, const double* __restrict__ Kx,
                                                               const i64* __restrict__ amap, double* __restrict__ L) {
  QS_BATCH(C, Kx, amap, L);
  const int lane = threadIdx.x & 31;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 col = C.n_p + C.l + (((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5); col < N; col += nwarps) {
    const int cc = (int)col - C.n_p;  // conic index, >= l
    const int k = C.cone_of_col[cc - C.l];
    const i64 b = C.Kp[col];
    const i64 e = C.Kp[col + 1] - ((cc - C.soc_ptr[k]) + 1);  // the last j + 1 entries of the column are the block's
    for (i64 p = b + lane; p < e; p += 32) L[amap[p]] = Kx[p];
  }
}

// one 32 x 32 tile (ti <= tj) of a cone's packed upper triangle: read along the K columns, write along the panel
// columns (whatever the map says: the transposition only makes the common case coalesced)
__global__ void __launch_bounds__(256) k_scatter_blocks(ConeBlocks C, const double* __restrict__ Kx,
                                                        const i64* __restrict__ amap, double* __restrict__ L) {
  QS_BATCH(C, Kx, amap, L);
  __shared__ double v[32][33];
  __shared__ i64 a[32][33];
  const int t = blockIdx.x;
  const int k = C.tile_cone[t];
  const int ti = C.tile_ij[2 * t], tj = C.tile_ij[2 * t + 1];
  const int o = C.soc_ptr[k], q = C.soc_ptr[k + 1] - o;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int jj = ty; jj < 32; jj += 8) {
    const int j = 32 * tj + jj, i = 32 * ti + tx;
    i64 off = -1;
    double val = 0.0;
    if (j < q && i <= j) {
      const i64 kpos = C.kp_conic[o + j] - (j + 1) + i;
      val = Kx[kpos];
      off = amap[kpos];
    }
    v[jj][tx] = val;
    a[jj][tx] = off;
  }
  __syncthreads();
  for (int ii = ty; ii < 32; ii += 8) {
    const i64 off = a[tx][ii];  // entry (i = 32 ti + ii, j = 32 tj + tx): consecutive lanes, consecutive panel rows
    if (off >= 0) L[off] = v[tx][ii];
  }
}

__global__ void __launch_bounds__(LDL_THREADS) k_add_reg(int N, DevSym S, const double* reg, double* L) {
  QS_BATCH(S, reg, L);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    const int s = S.sup_of[j];
    const int lc = j - S.col0[s];
    const i64 nr = S.rowptr[s + 1] - S.rowptr[s];
    L[S.Loff[s] + lc + lc * nr] += reg[j];
  }
}

// Extend-add (assembly of the children's update matrices into a front), one
// launch per level.  A CTA owns a slab of 8 consecutive front columns of one
// front; warp w owns column c_lo + w outright and walks the children in their
// fixed order, so every front entry is summed by one warp in a fixed order:
// deterministic, no atomics.  The search "does child c have a column that maps
// to mine?" runs 32 children at a time (one per lane, binary search in the
// sorted relative-index list); hits are then processed one by one with the
// whole warp striding over the child's rows.
__global__ void __launch_bounds__(LDL_THREADS)
    k_extend_add(DevSym S, const SlabItem* items, double* L, double* U) {
  QS_BATCH(S, items, L, U);
  const SlabItem it = items[blockIdx.x];
  const int s = it.front;
  const Front f = front_of(S, s, L, U);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pc = it.c_lo + warp;
  if (pc >= f.nr) return;
  const i64 nr = f.nr, nu = f.nu;
  double* dstcol = (pc < f.ns) ? f.Lp + pc * nr : f.Up + qs_ucol(pc - f.ns, nu) - f.ns;  // indexed by parent row
  const int ch0 = S.childptr[s], ch1 = S.childptr[s + 1];
  for (int base = ch0; base < ch1; base += 32) {
    int hit = -1;
    const int ci = base + lane;
    if (ci < ch1) {
      const int c = S.child[ci];
      const int nsc = S.col0[c + 1] - S.col0[c];
      const int nuc = (int)(S.rowptr[c + 1] - S.rowptr[c]) - nsc;
      const int* rel = S.rel + S.relptr[c];
      int lo = 0, hi = nuc;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rel[mid] < pc)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < nuc && rel[lo] == pc) hit = lo;
    }
    unsigned ballot = __ballot_sync(0xffffffffu, hit >= 0);
    while (ballot) {
      const int src = __ffs(ballot) - 1;
      ballot &= ballot - 1;
      const int cc = __shfl_sync(0xffffffffu, hit, src);
      const int c = S.child[base + src];
      const int nsc = S.col0[c + 1] - S.col0[c];
      const int nuc = (int)(S.rowptr[c + 1] - S.rowptr[c]) - nsc;
      const double* Ucol = U + S.Uoff[c] + qs_ucol(cc, nuc);
      const int* rel = S.rel + S.relptr[c];
      for (int r = cc + lane; r < nuc; r += 32) dstcol[rel[r]] += Ucol[r];
    }
  }
}

// List-driven extend-add (see AsmLists): a warp owns (column slot, row band) of a front outright and walks the
// slot's child entries in their fixed order -- deterministic, no atomics, no searching.
// TPR lanes own one work item.  TPR = 32 (root: ~50 rows per child and band): the per-child metadata (six
// dependent loads: child id -> offsets, sizes, band bounds) is fetched for 32 list entries at a time, one entry per
// lane, so the chains run in parallel and the entries are then processed from registers via shuffles.  TPR = 4
// (children with a handful of update rows, e.g. the 1.35 M one-column leaves of C4): eight items per warp.
template <int TPR>
__global__ void __launch_bounds__(LDL_THREADS)
    k_extend_add_list(DevSym S, AsmLists A, const EaItem* items, i64 slot0, i64 nitems, double* L, double* U) {
  QS_BATCH(S, A, items, L, U);
  const i64 w = (blockIdx.x * (i64)blockDim.x + threadIdx.x) / TPR;
  const int lane = threadIdx.x & (TPR - 1);
  if (TPR == 32 ? w >= nitems : false) return;
  const bool on = w < nitems;
  // items == nullptr: the level has no banded front, item w is simply column slot slot0 + w (whole column)
  const EaItem it = on ? (items ? items[w] : EaItem{(int)(slot0 + w), -1}) : EaItem{(int)slot0, -1};
  const int s = A.slot_front[it.slot], pc = A.slot_row[it.slot];
  const Front f = front_of(S, s, L, U);
  const i64 nr = f.nr, nu = f.nu;
  double* dstcol = (pc < f.ns) ? f.Lp + pc * nr : f.Up + qs_ucol(pc - f.ns, nu) - f.ns;  // indexed by parent row
  const i64 e0 = on ? A.gptr[it.slot] : 0, e1 = on ? A.gptr[it.slot + 1] : 0;
  if (TPR == 32) {
    for (i64 eb = e0; eb < e1; eb += 32) {
      // lane i: metadata of entry eb + i
      const i64 e = eb + lane;
      i64 uoff = 0, roff = 0;
      int r_lo = 0, r_hi = 0;
      if (e < e1) {
        const int c = A.gchild[e];
        const int cc = A.gsrc[e] - (int)S.Boff[c];
        const int nuc = (int)(S.rowptr[c + 1] - S.rowptr[c]) - (S.col0[c + 1] - S.col0[c]);
        r_lo = cc;
        r_hi = nuc;
        if (it.band >= 0) {
          const int* bs = A.bandstart + A.bandptr[c];
          r_lo = max(cc, bs[it.band]);
          r_hi = bs[it.band + 1];
        }
        uoff = S.Uoff[c] + qs_ucol(cc, nuc);
        roff = S.relptr[c];
      }
      const int cnt = (int)min((i64)32, e1 - eb);
      // Fixed child order; the FIRST 32-row chunk of entry q + 1 (its relative row and its value) is loaded before
      // entry q is added: the adds of successive children may hit the same parent row and stay ordered, their loads
      // need not wait for them (a band holds ~50 rows of a child, so the first chunk is usually the whole entry).
      i64 uo = __shfl_sync(0xffffffffu, uoff, 0), ro = __shfl_sync(0xffffffffu, roff, 0);
      int lo = __shfl_sync(0xffffffffu, r_lo, 0), hi = __shfl_sync(0xffffffffu, r_hi, 0);
      int rel0 = 0;
      double u0 = 0.0;
      bool ok0 = lo + lane < hi;
      if (ok0) {
        rel0 = S.rel[ro + lo + lane];
        u0 = U[uo + lo + lane];
      }
      for (int q = 0; q < cnt; ++q) {
        const i64 uo_c = uo, ro_c = ro;
        const int lo_c = lo, hi_c = hi, rel_c = rel0;
        const double u_c = u0;
        const bool ok_c = ok0;
        if (q + 1 < cnt) {  // warp-uniform
          uo = __shfl_sync(0xffffffffu, uoff, q + 1);
          ro = __shfl_sync(0xffffffffu, roff, q + 1);
          lo = __shfl_sync(0xffffffffu, r_lo, q + 1);
          hi = __shfl_sync(0xffffffffu, r_hi, q + 1);
          ok0 = lo + lane < hi;
          if (ok0) {
            rel0 = S.rel[ro + lo + lane];
            u0 = U[uo + lo + lane];
          }
        }
        if (ok_c) dstcol[rel_c] += u_c;
        const double* Ucol = U + uo_c;
        const int* rel = S.rel + ro_c;
        for (int r = lo_c + 32 + lane; r < hi_c; r += 32) dstcol[rel[r]] += Ucol[r];
      }
    }
  } else {
    for (i64 e = e0; e < e1; ++e) {
      const int c = A.gchild[e];
      const int cc = A.gsrc[e] - (int)S.Boff[c];
      const int nuc = (int)(S.rowptr[c + 1] - S.rowptr[c]) - (S.col0[c + 1] - S.col0[c]);
      int r_lo = cc, r_hi = nuc;
      if (it.band >= 0) {
        const int* bs = A.bandstart + A.bandptr[c];
        r_lo = max(cc, bs[it.band]);
        r_hi = bs[it.band + 1];
      }
      const double* Ucol = U + S.Uoff[c] + qs_ucol(cc, nuc);
      const int* rel = S.rel + S.relptr[c];
      for (int r = r_lo + lane; r < r_hi; r += TPR) dstcol[rel[r]] += Ucol[r];
    }
  }
}

// List-driven forward-solve gather: `tpr` lanes per slot sum the slot's child contributions in a fixed order.
__global__ void __launch_bounds__(LDL_THREADS)
    k_gather_fwd_list(AsmLists A, i64 slot0, i64 nslots, int tpr, double* xw, double* B) {
  QS_BATCH(A, xw, B);
  const i64 g = (blockIdx.x * (i64)blockDim.x + threadIdx.x) / tpr;
  const int lane = threadIdx.x & (tpr - 1);
  const unsigned mask = tpr == 32 ? 0xffffffffu : (((1u << tpr) - 1u) << (threadIdx.x & 31 & ~(tpr - 1)));
  double acc = 0.0;
  const bool on = g < nslots;
  if (on) {
    const i64 e1 = A.gptr[slot0 + g + 1];
    for (i64 e = A.gptr[slot0 + g] + lane; e < e1; e += tpr) acc += B[A.gsrc[e]];
  }
  for (int o = tpr >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o);
  if (on && lane == 0) {
    const i64 d = A.gdst[slot0 + g];
    if (d >= 0) xw[d] += acc;
    else B[-d - 1] = acc;
  }
}

// Leaf fronts with one pivot column and at most 33 rows (the private x columns of a cone block: millions of them):
// G lanes per front, G = smallest power of two >= the widest leaf's update rows (4 at C4: three sample rows and
// the cone row, so a warp handles eight leaves).
template <int G>
__device__ __forceinline__ unsigned leaf_mask() {
  return G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (threadIdx.x & 31 & ~(G - 1)));
}

template <int G>
__global__ void __launch_bounds__(LDL_THREADS)
    k_leaf_factor(DevSym S, const int* list, int count, double* L, double* U, double* Dg, const double* reg,
                  double dyn_eps, double* scalars) {
  QS_BATCH(S, list, L, U, Dg, reg, scalars);
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / G, lane = threadIdx.x & (G - 1);
  if (w >= count) return;
  const unsigned mask = leaf_mask<G>();
  const int s = list[w];
  const int c0 = S.col0[s];
  const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]), nu = nr - 1;
  double* Lp = L + S.Loff[s];
  double* Up = U + S.Uoff[s];
  double d = Lp[0];
  if (!qs_finite(d)) {
    if (lane == 0) scalars[SC_PIVOT_NONFINITE] = 1.0;
  } else if (fabs(d) < dyn_eps) {
    d = (reg[c0] >= 0.0) ? dyn_eps : -dyn_eps;
    if (lane == 0) atomicAdd(&scalars[SC_PIVOT_BUMPS], 1.0);
  }
  if (lane == 0) Dg[c0] = d;
  // lane r holds a_r = L[1+r]
  const double a = (lane < nu) ? Lp[1 + lane] : 0.0;
  const double l = a / d;
  if (lane < nu) Lp[1 + lane] = l;
  for (int j = 0; j < nu; ++j) {
    const double lj = __shfl_sync(mask, l, j, G);
    if (lane >= j && lane < nu) Up[qs_ucol(j, nu) + lane] -= a * lj;
  }
}

template <int G>
__global__ void __launch_bounds__(LDL_THREADS)
    k_leaf_fwd(DevSym S, const int* list, int count, const double* L, const double* xw, double* B) {
  QS_BATCH(S, list, L, xw, B);
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / G, lane = threadIdx.x & (G - 1);
  if (w >= count) return;
  const int s = list[w];
  const int nu = (int)(S.rowptr[s + 1] - S.rowptr[s]) - 1;
  const double x1 = xw[S.col0[s]];
  if (lane < nu) B[S.Boff[s] + lane] = -(L[S.Loff[s] + 1 + lane] * x1);
}

template <int G>
__global__ void __launch_bounds__(LDL_THREADS)
    k_leaf_bwd(DevSym S, const int* list, int count, const double* L, double* xw) {
  QS_BATCH(S, list, L, xw);
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / G, lane = threadIdx.x & (G - 1);
  if (w >= count) return;
  const unsigned mask = leaf_mask<G>();
  const int s = list[w];
  const i64 rp = S.rowptr[s];
  const int nu = (int)(S.rowptr[s + 1] - rp) - 1;
  double acc = (lane < nu) ? L[S.Loff[s] + 1 + lane] * xw[S.rowidx[rp + 1 + lane]] : 0.0;
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o);
  if (lane == 0) xw[S.col0[s]] -= acc;
}

#define QS_LEAF_DISPATCH(kern, grid, ...)                                                 \
  switch (leaf_group) {                                                                   \
    case 4: kern<4><<<qs_grid(grid(4)), LDL_THREADS, 0, st>>>(__VA_ARGS__); break;                 \
    case 8: kern<8><<<qs_grid(grid(8)), LDL_THREADS, 0, st>>>(__VA_ARGS__); break;                 \
    case 16: kern<16><<<qs_grid(grid(16)), LDL_THREADS, 0, st>>>(__VA_ARGS__); break;              \
    default: kern<32><<<qs_grid(grid(32)), LDL_THREADS, 0, st>>>(__VA_ARGS__); break;              \
  }

// One CTA per front of the level (children already assembled by k_extend_add):
// factor the pivot panel, form this front's own update matrix.
// Small fronts (at most QS_SMALL_NR rows and QS_SMALL_NS pivots: the panel is <= 36 KB) are factored IN SHARED MEMORY:
// one coalesced load of the panel, every pivot step at shared-memory latency, one coalesced store; the update matrix
// is then formed from the shared copy.  (In global memory every one of the ~2 ns barrier-separated steps paid an L2
// round trip; a chain of 100 small fronts is bound by exactly that latency.)
#define QS_SMALL_NR 96
#define QS_SMALL_NS 48

__device__ void front_factor_body(const DevSym& S, int s, double* L, double* U, double* Dg, const double* reg,
                                  double dyn_eps, double* scalars) {
  __shared__ double Ls[QS_SMALL_NR * QS_SMALL_NS];
  __shared__ double dsm[QS_SMALL_NS];
  const Front f = front_of(S, s, L, U);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int nr = f.nr, ns = f.ns, nu = f.nu;
  __syncthreads();  // the shared arrays may still be read by the previous front of a chain
  for (int e = tid; e < nr * ns; e += blockDim.x) Ls[e] = f.Lp[e];
  // ---- right-looking LDL' on the pivot panel (nr x ns)
  for (int k = 0; k < ns; ++k) {
    __syncthreads();
    double d = Ls[k + k * nr];
    if (!qs_finite(d)) {
      if (tid == 0) scalars[SC_PIVOT_NONFINITE] = 1.0;
    } else if (fabs(d) < dyn_eps) {  // dynamic floor, sign from the expected inertia (_kernels.py:160-165)
      d = (reg[f.c0 + k] >= 0.0) ? dyn_eps : -dyn_eps;
      if (tid == 0) atomicAdd(&scalars[SC_PIVOT_BUMPS], 1.0);
    }
    if (tid == 0) {
      Dg[f.c0 + k] = d;
      dsm[k] = d;
    }
    for (int j = k + 1 + warp; j < ns; j += nwarps) {
      const double ljk = Ls[j + k * nr] / d;
      for (int i = j + lane; i < nr; i += 32) Ls[i + j * nr] -= Ls[i + k * nr] * ljk;
    }
    __syncthreads();
    for (int i = k + 1 + tid; i < nr; i += blockDim.x) Ls[i + k * nr] /= d;
  }
  __syncthreads();
  for (int e = tid; e < nr * ns; e += blockDim.x) f.Lp[e] = Ls[e];
  // ---- update matrix: U -= L21 D L21'
  if (nu > 0) {
    const double* L21 = Ls + ns;
    for (int j = warp; j < nu; j += nwarps) {
      for (int i0 = j; i0 < nu; i0 += 32) {
        const int i = i0 + lane;
        double acc = 0.0;
        for (int k = 0; k < ns; ++k) {
          const double t = L21[j + k * nr] * dsm[k];
          if (i < nu) acc += L21[i + k * nr] * t;
        }
        if (i < nu) f.Up[qs_ucol(j, nu) + i] -= acc;
      }
    }
  }
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_front_factor(DevSym S, const int* list, double* L, double* U, double* Dg, const double* reg, double dyn_eps,
                   double* scalars) {
  QS_BATCH(S, list, L, U, Dg, reg, scalars);
  front_factor_body(S, list[blockIdx.x], L, U, Dg, reg, dyn_eps, scalars);
}

// ============================ blocked path for large fronts ==================
// Fronts too large for one CTA are factored by panels of NB = 32 pivot columns,
// every front of the level advancing in lockstep (blockIdx.y = front):
//   k_blk_diag    factor the NB x NB diagonal block (one CTA per front)
//   k_blk_panel   rows below it: L21 = A21 L11^-T D^-1 (thread per row)
//   k_blk_update  rank-NB update of the remaining pivot columns (64x64 tiles)
// and, once the panel is done, k_blk_update in SCHUR mode forms the front's
// update matrix U -= L21 D L21' with the full pivot depth.
#define NB 32
#define TS 64  // update tile edge

// One WARP per front: lane i keeps row i of the 32 x 32 block in registers; step k broadcasts the pivot and the
// multipliers by shuffles, so the whole block costs ~500 shuffles and ~500 FMAs and touches memory twice (load,
// store).  (The first version used a CTA with a shared-memory copy and three barriers per pivot: 40 us for one
// block, 1 ms for the 10^4 fronts of a level; this one is ~20x faster.)
__global__ void __launch_bounds__(LDL_THREADS)
    k_blk_diag(DevSym S, const int* list, int count, int kb, double* L, double* Dg, const double* reg, double dyn_eps,
               double* scalars) {
  QS_BATCH(S, list, L, Dg, reg, scalars);
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= count) return;
  const int s = list[w];
  const Front f = front_of(S, s, L, nullptr);
  if (kb >= f.ns) return;
  const int nb = min(NB, f.ns - kb);
  const i64 nr = f.nr;
  double a[NB];  // a[j] = A(kb + lane, kb + j), j <= lane
#pragma unroll
  for (int j = 0; j < NB; ++j) a[j] = (j <= lane && lane < nb) ? f.Lp[(kb + lane) + (i64)(kb + j) * nr] : 0.0;
  double dmine = 1.0;  // pivot of column `lane`
  int bumps = 0, bad = 0;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    double d = __shfl_sync(0xffffffffu, a[k], k);  // A(k, k) after the previous updates
    if (k < nb) {
      if (!qs_finite(d)) {
        bad = 1;
      } else if (fabs(d) < dyn_eps) {  // dynamic floor, sign from the expected inertia (_kernels.py:160-165)
        d = (reg[f.c0 + kb + k] >= 0.0) ? dyn_eps : -dyn_eps;
        bumps += (lane == 0);
      }
    } else {
      d = 1.0;
    }
    if (lane == k) dmine = d;
    const double lik = a[k] / d;  // multiplier of this lane's row (rows > k)
#pragma unroll
    for (int j = k + 1; j < NB; ++j) {
      const double ljk = __shfl_sync(0xffffffffu, lik, j);  // L(j, k)
      // A(i, j) -= L(i, k) d L(j, k) for i >= j (lanes below j hold no a[j])
      if (lane >= j) a[j] -= a[k] * ljk;
    }
    if (lane > k) a[k] = lik;
  }
#pragma unroll
  for (int j = 0; j < NB; ++j)
    if (j < lane && lane < nb) f.Lp[(kb + lane) + (i64)(kb + j) * nr] = a[j];
  if (lane < nb) {
    Dg[f.c0 + kb + lane] = dmine;
    f.Lp[(kb + lane) + (i64)(kb + lane) * nr] = dmine;
  }
  if (bad) scalars[SC_PIVOT_NONFINITE] = 1.0;
  if (bumps) atomicAdd(&scalars[SC_PIVOT_BUMPS], (double)bumps);
}

template <int T, int MINB>
__global__ void __launch_bounds__(T, MINB)
    k_blk_panel(DevSym S, const int* list, int kb, double* L, const double* Dg) {
  QS_BATCH(S, list, L, Dg);
  const int s = list[blockIdx.y];
  const Front f = front_of(S, s, L, nullptr);
  if (kb >= f.ns) return;
  const int nb = min(NB, f.ns - kb);
  const int row0 = kb + nb + blockIdx.x * blockDim.x;
  if (row0 >= f.nr) return;
  const i64 nr = f.nr;
  __shared__ double l11[NB][NB + 1];
  __shared__ double dinv[NB];
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    l11[i][j] = (i > j) ? f.Lp[(kb + i) + (i64)(kb + j) * nr] : 0.0;
  }
  for (int k = tid; k < nb; k += blockDim.x) dinv[k] = 1.0 / Dg[f.c0 + kb + k];
  __syncthreads();
  const int row = row0 + tid;
  if (row >= f.nr) return;
  double y[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) y[k] = (k < nb) ? f.Lp[row + (i64)(kb + k) * nr] : 0.0;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    if (k < nb) {
      double acc = y[k];
#pragma unroll
      for (int mm = 0; mm < NB; ++mm)
        if (mm < k) acc -= y[mm] * l11[k][mm];
      y[k] = acc;
    }
  }
#pragma unroll
  for (int k = 0; k < NB; ++k)
    if (k < nb) f.Lp[row + (i64)(kb + k) * nr] = y[k] * dinv[k];
}

// C(i, j) -= sum_k A(i, k) d_k A(j, k) over 64 x 64 tiles of the lower triangle.
//   PANEL mode, left-looking : C = panel columns [kb, kb+nb), rows [col, nr);  k in [0, kb)
//   PANEL mode, right-looking: C = panel columns [kb+nb, ns), rows [col, nr);  k in [kb, kb+nb)
//   SCHUR mode: C = U (nu x nu);                              k in [0, ns)
// Inner product on the fp64 tensor pipe: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; 37 TFLOP/s measured on B200,
// tests/probes/dmma_probe.cu -- the same peak as DFMA, at an eighth of the issue slots and a quarter of the
// shared-memory operand traffic).  8 warps as 2 x 4; a warp owns 32 x 16 of the tile = 4 x 2 DMMA blocks.
// k-blocks of 32 are staged in shared memory [k][row] with a row stride of 68 doubles (= 4 mod 16: within each
// half-warp the four k rows of a fragment fall on disjoint banks, so a fragment load is the minimal two wavefronts);
// the next k-block is fetched into registers while the current one is multiplied.
#define TSP (TS + 4)

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool SCHUR>
__global__ void __launch_bounds__(LDL_THREADS, 3)
    k_blk_update(DevSym S, const int* list, const TileItem* tiles, int kb, int left, double* L, double* U,
                 const double* Dg) {
  QS_BATCH(S, list, tiles, L, U, Dg);
  // SCHUR mode runs over an exact tile list built at analysis (no empty CTAs); PANEL mode keeps the lockstep grid
  TileItem item{0, 0, 0};
  if (SCHUR) item = tiles[blockIdx.x];
  const int s = SCHUR ? item.front : list[blockIdx.y];
  const Front f = front_of(S, s, L, U);
  int k_lo, k_hi, c_lo, c_hi;
  if (SCHUR) {
    k_lo = 0;
    k_hi = f.ns;
    c_lo = f.ns;
    c_hi = f.nr;
  } else {
    // left-looking panel step: block column [kb, kb+NB) (rows kb .. nr) receives the updates of ALL previous
    // pivot columns at once -- one pass with inner depth kb instead of kb/32 rank-32 passes over the panel
    if (kb >= f.ns) return;
    if (left == 3) {
      // wide left-looking step: TWO block columns [kb, kb + 2 NB) receive the updates of all previous pivots --
      // the 64 x 64 tile is full (a 32-column step keeps half of the CTA's warps out of the multiply)
      if (kb == 0) return;
      k_lo = 0;
      k_hi = kb;
      c_lo = kb;
      c_hi = min(f.ns, kb + 2 * NB);
    } else if (left == 2) {
      // second half of a wide step: pivots [kb, kb + NB) update the block column [kb + NB, kb + 2 NB) only
      k_lo = kb;
      k_hi = min(f.ns, kb + NB);
      c_lo = k_hi;
      c_hi = min(f.ns, kb + 2 * NB);
    } else if (left) {
      if (kb == 0) return;
      k_lo = 0;
      k_hi = kb;
      c_lo = kb;
      c_hi = min(f.ns, kb + NB);
    } else {
      // right-looking step: pivots [kb, kb+NB) update every remaining pivot column -- many tiles of depth 32,
      // which is what a level with ONE big front (the root) needs to fill the machine
      k_lo = kb;
      k_hi = min(f.ns, kb + NB);
      c_lo = k_hi;
      c_hi = f.ns;
    }
  }
  if (c_lo >= c_hi || k_lo >= k_hi) return;
  const int ntj = (c_hi - c_lo + TS - 1) / TS;
  const int nti = (f.nr - c_lo + TS - 1) / TS;
  if (!SCHUR && (int)blockIdx.x >= nti * ntj) return;
  const int tj = SCHUR ? item.tj : blockIdx.x / nti, ti = SCHUR ? item.ti : blockIdx.x % nti;
  const int i0 = c_lo + ti * TS, j0 = c_lo + tj * TS;  // front-local row / column of the tile origin
  if (i0 + TS <= j0) return;                         // entirely above the diagonal
  const i64 nr = f.nr;
  __shared__ double As[NB][TSP];
  __shared__ double Bs[NB][TSP];
  __shared__ double dsm[NB];  // pivots of the current k-block
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = 32 * (warp & 1), wj = 16 * (warp >> 1);
  const int g = lane >> 2, t = lane & 3;
  // a warp whose 32 x 16 block lies outside the front or strictly above the diagonal only helps with the staging
  // (edge tiles of a 390-row update matrix hold 6 useful rows: most of their warps have nothing to multiply)
  const bool live = (i0 + wi < f.nr) && (j0 + wj < c_hi) && (i0 + wi + 31 >= j0 + wj);
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b2 = 0; b2 < 2; ++b2) acc[a][b2][0] = acc[a][b2][1] = 0.0;
  // staging map: element e = tid + 256 u  ->  row r = e % 64 (consecutive threads, consecutive rows), k = e / 64
  const int sr = tid & 63, sk = tid >> 6;  // k = sk + 4 u
  // fetch() only ISSUES loads (raw values into registers, no arithmetic on them), so that they stay in flight
  // across the multiply of the current k-block; the pivot scaling d_k is applied when a B fragment is read
  double ra[8], rb[8], rd = 0.0;
  auto fetch = [&](int k0) {
    const int kn = min(NB, k_hi - k0);
    const int gi = i0 + sr, gj = j0 + sr;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = sk + 4 * u;
      const bool ka = k < kn && gi < f.nr, kb2 = k < kn && gj < c_hi;
      ra[u] = ka ? f.Lp[gi + (i64)(k0 + k) * nr] : 0.0;
      rb[u] = kb2 ? f.Lp[gj + (i64)(k0 + k) * nr] : 0.0;
    }
    if (tid < NB) rd = tid < kn ? Dg[f.c0 + k0 + tid] : 0.0;
  };
  auto stage = [&]() {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      As[sk + 4 * u][sr] = ra[u];
      Bs[sk + 4 * u][sr] = rb[u];
    }
    if (tid < NB) dsm[tid] = rd;
  };
  fetch(k_lo);
  stage();
  __syncthreads();
  for (int k0 = k_lo; k0 < k_hi; k0 += NB) {
    const bool more = k0 + NB < k_hi;
    if (more) fetch(k0 + NB);  // in flight during the multiply below
    if (live)
#pragma unroll
    for (int kk = 0; kk < NB; kk += 4) {
      double av[4], bv[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk + t][wi + 8 * a + g];
#pragma unroll
      for (int b2 = 0; b2 < 2; ++b2) bv[b2] = Bs[kk + t][wj + 8 * b2 + g] * dsm[kk + t];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) dmma_8x8x4(acc[a][b2], av[a], bv[b2]);
    }
    __syncthreads();
    if (more) {
      stage();
      __syncthreads();
    }
  }
  // accumulator (a, b2, h) is C(i0 + wi + 8a + g, j0 + wj + 8 b2 + 2t + h)
  if (!live) return;
#pragma unroll
  for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gj = j0 + wj + 8 * b2 + 2 * t + h;
      if (gj >= c_hi) continue;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int gi = i0 + wi + 8 * a + g;
        if (gi >= f.nr || gi < gj) continue;
        if (SCHUR)
          f.Up[qs_ucol(gj - f.ns, f.nu) + (gi - f.ns)] -= acc[a][b2][h];
        else
          f.Lp[gi + (i64)gj * nr] -= acc[a][b2][h];
      }
    }
}

// ---- fused panel factorisation: ONE CTA per front walks all block steps of its panel -----------------------------
// The lockstep path above launches update / diag / panel once per 32-column step for ALL fronts of a level and
// re-reads every panel from DRAM at each step (left-looking: columns [0, kb) again and again).  A level with thousands
// of independent mid-size fronts (the 10^4 cone fronts of C4: ~135 pivots x ~500 rows, 0.5 MB each) does not need the
// lockstep: a CTA can factor its front from the first to the last step on its own -- the panel stays in the L2 while
// the CTA works on it, barriers replace launches, and the grid (fronts sorted by size, largest first) balances
// itself.  MEASURED SLOWER than the lockstep path at C4 (see factor_launches): opt-in, QS_LDL_FUSED=1.  Same arithmetic in the same order as the lockstep kernels (the tile / diagonal / row routines are the
// same code), so the factor is bitwise the same.  Used for levels with more than QS_FUSED_MIN fronts; a level with a
// few big fronts (the root) keeps the lockstep / right-looking path, which is what fills the machine there.
__device__ __forceinline__ void fused_update_tile(const Front& f, const double* Dg, int k_hi, int c_lo, int c_hi, int ti,
                                                  double (*As)[TSP], double (*Bs)[TSP], double* dsm) {
  // left-looking: block column [c_lo, c_hi) rows [c_lo + ti * TS, ...) -= L[:, 0:k_hi] D L[c_lo:c_hi, 0:k_hi]'
  const int i0 = c_lo + ti * TS, j0 = c_lo;
  const i64 nr = f.nr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = 32 * (warp & 1), wj = 16 * (warp >> 1);
  const int g = lane >> 2, t = lane & 3;
  const bool live = (i0 + wi < f.nr) && (j0 + wj < c_hi) && (i0 + wi + 31 >= j0 + wj);
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b2 = 0; b2 < 2; ++b2) acc[a][b2][0] = acc[a][b2][1] = 0.0;
  const int sr = tid & 63, sk = tid >> 6;
  double ra[8], rb[8], rd = 0.0;
  auto fetch = [&](int k0) {
    const int kn = min(NB, k_hi - k0);
    const int gi = i0 + sr, gj = j0 + sr;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = sk + 4 * u;
      const bool ka = k < kn && gi < f.nr, kb2 = k < kn && gj < c_hi;
      ra[u] = ka ? f.Lp[gi + (i64)(k0 + k) * nr] : 0.0;
      rb[u] = kb2 ? f.Lp[gj + (i64)(k0 + k) * nr] : 0.0;
    }
    if (tid < NB) rd = tid < kn ? Dg[f.c0 + k0 + tid] : 0.0;
  };
  auto stage = [&]() {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      As[sk + 4 * u][sr] = ra[u];
      Bs[sk + 4 * u][sr] = rb[u];
    }
    if (tid < NB) dsm[tid] = rd;
  };
  fetch(0);
  __syncthreads();  // the previous tile's multiply has finished reading the staging buffers
  stage();
  __syncthreads();
  for (int k0 = 0; k0 < k_hi; k0 += NB) {
    const bool more = k0 + NB < k_hi;
    if (more) fetch(k0 + NB);
    if (live)
#pragma unroll
      for (int kk = 0; kk < NB; kk += 4) {
        double av[4], bv[2];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk + t][wi + 8 * a + g];
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) bv[b2] = Bs[kk + t][wj + 8 * b2 + g] * dsm[kk + t];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b2 = 0; b2 < 2; ++b2) dmma_8x8x4(acc[a][b2], av[a], bv[b2]);
      }
    __syncthreads();
    if (more) {
      stage();
      __syncthreads();
    }
  }
  if (!live) return;
#pragma unroll
  for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gj = j0 + wj + 8 * b2 + 2 * t + h;
      if (gj >= c_hi) continue;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int gi = i0 + wi + 8 * a + g;
        if (gi >= f.nr || gi < gj) continue;
        f.Lp[gi + (i64)gj * nr] -= acc[a][b2][h];
      }
    }
}

// 32 x 32 diagonal block by ONE warp (the body of k_blk_diag)
__device__ __forceinline__ void fused_diag_warp(const Front& f, int kb, double* Dg, const double* reg, double dyn_eps,
                                                double* scalars) {
  const int lane = threadIdx.x & 31;
  const int nb = min(NB, f.ns - kb);
  const i64 nr = f.nr;
  double a[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) a[j] = (j <= lane && lane < nb) ? f.Lp[(kb + lane) + (i64)(kb + j) * nr] : 0.0;
  double dmine = 1.0;
  int bumps = 0, bad = 0;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    double d = __shfl_sync(0xffffffffu, a[k], k);
    if (k < nb) {
      if (!qs_finite(d)) {
        bad = 1;
      } else if (fabs(d) < dyn_eps) {
        d = (reg[f.c0 + kb + k] >= 0.0) ? dyn_eps : -dyn_eps;
        bumps += (lane == 0);
      }
    } else {
      d = 1.0;
    }
    if (lane == k) dmine = d;
    const double lik = a[k] / d;
#pragma unroll
    for (int j = k + 1; j < NB; ++j) {
      const double ljk = __shfl_sync(0xffffffffu, lik, j);
      if (lane >= j) a[j] -= a[k] * ljk;
    }
    if (lane > k) a[k] = lik;
  }
#pragma unroll
  for (int j = 0; j < NB; ++j)
    if (j < lane && lane < nb) f.Lp[(kb + lane) + (i64)(kb + j) * nr] = a[j];
  if (lane < nb) {
    Dg[f.c0 + kb + lane] = dmine;
    f.Lp[(kb + lane) + (i64)(kb + lane) * nr] = dmine;
  }
  if (bad) scalars[SC_PIVOT_NONFINITE] = 1.0;
  if (bumps) atomicAdd(&scalars[SC_PIVOT_BUMPS], (double)bumps);
}

template <int MINB>
__global__ void __launch_bounds__(LDL_THREADS, MINB)
    k_front_blocked(DevSym S, const int* list, double* L, double* Dg, const double* reg, double dyn_eps,
                    double* scalars) {
  QS_BATCH(S, list, L, Dg, reg, scalars);
  const int s = list[blockIdx.x];
  const Front f = front_of(S, s, L, nullptr);
  __shared__ double As[NB][TSP];
  __shared__ double Bs[NB][TSP];
  __shared__ double dsm[NB];
  __shared__ double l11[NB][NB + 1];
  __shared__ double dinv[NB];
  const int tid = threadIdx.x;
  const i64 nr = f.nr;
  for (int kb = 0; kb < f.ns; kb += NB) {
    const int nb = min(NB, f.ns - kb);
    if (kb > 0) {
      const int nti = (f.nr - kb + TS - 1) / TS;
      for (int ti = 0; ti < nti; ++ti) fused_update_tile(f, Dg, kb, kb, kb + nb, ti, As, Bs, dsm);
      __syncthreads();  // the updated block column is visible to the whole CTA
    }
    if (tid < 32) fused_diag_warp(f, kb, Dg, reg, dyn_eps, scalars);
    __syncthreads();
    // rows below the diagonal block: L21 = A21 L11^-T D^-1, a thread per row (the body of k_blk_panel)
    for (int e = tid; e < nb * nb; e += blockDim.x) {
      const int i = e % nb, j = e / nb;
      l11[i][j] = (i > j) ? f.Lp[(kb + i) + (i64)(kb + j) * nr] : 0.0;
    }
    for (int k = tid; k < nb; k += blockDim.x) dinv[k] = 1.0 / Dg[f.c0 + kb + k];
    __syncthreads();
    for (int row = kb + nb + tid; row < f.nr; row += blockDim.x) {
      double y[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) y[k] = (k < nb) ? f.Lp[row + (i64)(kb + k) * nr] : 0.0;
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        if (k < nb) {
          double acc = y[k];
#pragma unroll
          for (int mm = 0; mm < NB; ++mm)
            if (mm < k) acc -= y[mm] * l11[k][mm];
          y[k] = acc;
        }
      }
#pragma unroll
      for (int k = 0; k < NB; ++k)
        if (k < nb) f.Lp[row + (i64)(kb + k) * nr] = y[k] * dinv[k];
    }
    __syncthreads();  // the finished block column is visible before the next step reads it
  }
}

__global__ void __launch_bounds__(LDL_THREADS) k_zero_cb(DevSym S, const int* list, double* B) {
  QS_BATCH(S, list, B);
  const int s = list[blockIdx.x];
  if (S.childptr[s + 1] != S.childptr[s]) return;
  const int nu = (int)(S.rowptr[s + 1] - S.rowptr[s]) - (S.col0[s + 1] - S.col0[s]);
  for (int r = threadIdx.x; r < nu; r += blockDim.x) B[S.Boff[s] + r] = 0.0;
}

// ---- forward-solve gather: contributions of the children into a front, same
// ownership scheme as k_extend_add (warp w of a slab owns front row c_lo + w).
__global__ void __launch_bounds__(LDL_THREADS)
    k_gather_fwd(DevSym S, const SlabItem* items, double* xw, double* B) {
  QS_BATCH(S, items, xw, B);
  const SlabItem it = items[blockIdx.x];
  const int s = it.front;
  const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
  const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pr = it.c_lo + warp;
  if (pr >= nr) return;
  double acc = 0.0;
  const int ch0 = S.childptr[s], ch1 = S.childptr[s + 1];
  for (int base = ch0; base < ch1; base += 32) {
    double v = 0.0;
    const int ci = base + lane;
    if (ci < ch1) {
      const int c = S.child[ci];
      const int nsc = S.col0[c + 1] - S.col0[c];
      const int nuc = (int)(S.rowptr[c + 1] - S.rowptr[c]) - nsc;
      const int* rel = S.rel + S.relptr[c];
      int lo = 0, hi = nuc;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rel[mid] < pr)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < nuc && rel[lo] == pr) v = B[S.Boff[c] + lo];
    }
    // fixed-order sum over the 32 children of this batch
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc += v;
  }
  if (lane == 0) {
    if (pr < ns)
      xw[c0 + pr] += acc;
    else
      B[S.Boff[s] + pr - ns] = acc;
  }
}

// ---- blocked triangular solves for the large fronts (lockstep over the level)
__global__ void __launch_bounds__(32) k_fwd_diag(DevSym S, const int* list, int kb, const double* L, double* xw) {
  QS_BATCH(S, list, L, xw);
  const int s = list[blockIdx.x];
  const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
  if (kb >= ns) return;
  const int nb = min(NB, ns - kb);
  const i64 nr = S.rowptr[s + 1] - S.rowptr[s];
  const double* Lp = L + S.Loff[s];
  const int lane = threadIdx.x;
  double x = (lane < nb) ? xw[c0 + kb + lane] : 0.0;
  for (int k = 0; k < nb - 1; ++k) {
    const double xk = __shfl_sync(0xffffffffu, x, k);
    if (lane > k && lane < nb) x -= Lp[(kb + lane) + (i64)(kb + k) * nr] * xk;
  }
  if (lane < nb) xw[c0 + kb + lane] = x;
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_fwd_update(DevSym S, const int* list, int kb, const double* L, double* xw, double* B) {
  QS_BATCH(S, list, L, xw, B);
  const int s = list[blockIdx.y];
  const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
  if (kb >= ns) return;
  const int nb = min(NB, ns - kb);
  const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]);
  const int row0 = kb + nb + blockIdx.x * blockDim.x;
  if (row0 >= nr) return;
  __shared__ double xs[NB];
  if (threadIdx.x < NB) xs[threadIdx.x] = (threadIdx.x < nb) ? xw[c0 + kb + threadIdx.x] : 0.0;
  __syncthreads();
  const int r = row0 + threadIdx.x;
  if (r >= nr) return;
  const double* Lp = L + S.Loff[s] + r + (i64)kb * nr;
  double acc = 0.0;
#pragma unroll 8
  for (int k = 0; k < nb; ++k) acc += Lp[(i64)k * nr] * xs[k];
  if (r < ns)
    xw[c0 + r] -= acc;
  else
    B[S.Boff[s] + r - ns] -= acc;
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_bwd_partial(DevSym S, const int* list, const i64* poff, int kb, const double* L, const double* xw,
                  double* partial) {
  QS_BATCH(S, list, poff, L, xw, partial);
  const int s = list[blockIdx.y];
  const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
  if (kb >= ns) return;
  const int nb = min(NB, ns - kb);
  const i64 rp = S.rowptr[s];
  const int nr = (int)(S.rowptr[s + 1] - rp);
  const int row0 = kb + nb + blockIdx.x * blockDim.x;
  if (row0 >= nr) return;
  const int r = row0 + threadIdx.x;
  __shared__ double red[LDL_THREADS / 32][NB];
  double xr = 0.0;
  const double* Lp = L + S.Loff[s] + (i64)kb * nr;
  if (r < nr) xr = (r < ns) ? xw[c0 + r] : xw[S.rowidx[rp + r]];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < nb; ++k) {
    double v = (r < nr) ? Lp[r + (i64)k * nr] * xr : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    double t = 0.0;
    for (int w = 0; w < LDL_THREADS / 32; ++w) t += red[w][threadIdx.x];
    partial[poff[blockIdx.y] + (i64)blockIdx.x * NB + threadIdx.x] = t;
  }
}

__global__ void __launch_bounds__(32)
    k_bwd_diag(DevSym S, const int* list, const i64* poff, int kb, const double* L, double* xw,
               const double* partial) {
  QS_BATCH(S, list, poff, L, xw, partial);
  const int s = list[blockIdx.x];
  const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
  if (kb >= ns) return;
  const int nb = min(NB, ns - kb);
  const i64 nr = S.rowptr[s + 1] - S.rowptr[s];
  const double* Lp = L + S.Loff[s];
  const int lane = threadIdx.x;
  const int rows_below = (int)nr - kb - nb;
  const int ntiles = rows_below > 0 ? (rows_below + LDL_THREADS - 1) / LDL_THREADS : 0;
  double x = (lane < nb) ? xw[c0 + kb + lane] : 0.0;
  if (lane < nb)
    for (int t = 0; t < ntiles; ++t) x -= partial[poff[blockIdx.x] + (i64)t * NB + lane];
  for (int k = nb - 1; k > 0; --k) {
    const double xk = __shfl_sync(0xffffffffu, x, k);
    if (lane < k) x -= Lp[(kb + k) + (i64)(kb + lane) * nr] * xk;
  }
  if (lane < nb) xw[c0 + kb + lane] = x;
}

// ---- triangular solves of a level with only a few large fronts (the root of a conic KKT system: one dense
// 2000 x 2000 front): ONE launch per direction instead of two launches per 32-column step.  A thread-block
// cluster of QS_CL CTAs owns a front; cluster barriers order the steps, so the 63 steps of a 2000-column front
// cost 63 hardware barriers instead of 126 kernel launches, and eight SMs stream the panel together.
// The cluster size is a launch attribute (cudaLaunchAttributeClusterDimension), 8 CTAs per front.
#define QS_CL_MAX 8

__global__ void __launch_bounds__(LDL_THREADS)
    k_cluster_fwd(DevSym S, const int* list, const double* L, double* xw, double* B) {
  QS_BATCH(S, list, L, xw, B);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int QS_CL = (int)cluster.num_blocks();
  const int s = list[blockIdx.x / QS_CL];
  const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
  const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]);
  const double* Lp = L + S.Loff[s];
  double* cb = B + S.Boff[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gt = rank * LDL_THREADS + tid, gstride = QS_CL * LDL_THREADS;
  __shared__ double xs[NB];
  if (S.childptr[s + 1] == S.childptr[s]) {  // no children: nothing was gathered, start from zero
    for (int r = gt; r < nr - ns; r += gstride) cb[r] = 0.0;
    __threadfence();
    cluster.sync();
  }
  double solved = 0.0;
  int solved_at = -1;
  for (int kb = 0; kb < ns; kb += NB) {
    const int nb = min(NB, ns - kb);
    if (warp == 0) {
      // the previous block's solution becomes visible only now: every CTA has finished reading the unsolved values
      if (rank == 0 && solved_at >= 0 && lane < NB) xw[c0 + solved_at + lane] = solved;
      // every CTA solves the 32 x 32 unit-lower block itself (8 KB of L, no communication)
      double x = (lane < nb) ? xw[c0 + kb + lane] : 0.0;
      double lrow[NB];  // row kb + lane of the block, fetched up front: the serial loop below touches no memory
#pragma unroll
      for (int k = 0; k < NB; ++k) lrow[k] = (k < lane && lane < nb) ? Lp[(kb + lane) + (i64)(kb + k) * nr] : 0.0;
#pragma unroll
      for (int k = 0; k < NB - 1; ++k) {
        const double xk = __shfl_sync(0xffffffffu, x, k);
        x -= lrow[k] * xk;  // zero unless k < lane < nb
      }
      xs[lane] = (lane < nb) ? x : 0.0;
      solved = x;
      solved_at = (nb == NB) ? kb : -2 - kb;  // a short last block is written under its own guard below
    }
    __syncthreads();
    for (int r = kb + nb + gt; r < nr; r += gstride) {
      const double* Lr = Lp + r + (i64)kb * nr;
      double acc = 0.0;
#pragma unroll 8
      for (int k = 0; k < nb; ++k) acc += Lr[(i64)k * nr] * xs[k];
      if (r < ns)
        xw[c0 + r] -= acc;
      else
        cb[r - ns] -= acc;
    }
    __threadfence();
    cluster.sync();
  }
  if (rank == 0 && warp == 0) {  // the last block
    const int last_kb = ((ns - 1) / NB) * NB, nb = ns - last_kb;
    if (lane < nb) xw[c0 + last_kb + lane] = solved;
  }
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_cluster_bwd(DevSym S, const int* list, const double* L, double* xw) {
  QS_BATCH(S, list, L, xw);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int QS_CL = (int)cluster.num_blocks();
  const int s = list[blockIdx.x / QS_CL];
  const int c0 = S.col0[s], ns = S.col0[s + 1] - c0;
  const i64 rp = S.rowptr[s];
  const int nr = (int)(S.rowptr[s + 1] - rp);
  const double* Lp = L + S.Loff[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double part[LDL_THREADS / 32];  // this CTA's partial sums (one per warp), read by rank 0 through DSMEM
  const int last_kb = ((ns - 1) / NB) * NB;
  // Column-oriented products: the 8 x QS_CL = 64 warps of the cluster take the 32 columns of the block, two warps
  // per column (even / odd 32-row groups); a lane strides down its column (contiguous in memory), so a step costs
  // one 5-round shuffle reduction per warp instead of 32 of them.
  const int gw = rank * (LDL_THREADS / 32) + warp;  // 0 .. 63
  const int kcol = gw & (NB - 1), half = gw >> 5;
  for (int kb = last_kb; kb >= 0; kb -= NB) {
    const int nb = min(NB, ns - kb);
    double acc = 0.0;
    if (kcol < nb) {
      const double* Lc = Lp + (i64)(kb + kcol) * nr;
      for (int r = kb + nb + lane + 32 * half; r < nr; r += 64) {
        const double xr = (r < ns) ? xw[c0 + r] : xw[S.rowidx[rp + r]];
        acc += Lc[r] * xr;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[warp] = acc;
    cluster.sync();  // all partials published
    if (rank == 0 && warp == 0) {
      double x = (lane < nb) ? xw[c0 + kb + lane] : 0.0;
      // column `lane` was summed by global warps `lane` (even row groups) and `lane + 32` (odd ones): fixed order
      if (lane < nb) {
        const double* r0p = cluster.map_shared_rank(part, lane >> 3);
        const double* r1p = cluster.map_shared_rank(part, (lane >> 3) + 4);
        x -= r0p[lane & 7] + r1p[lane & 7];
      }
      double lcol[NB];  // column kb + lane of the block below its diagonal, fetched up front
#pragma unroll
      for (int k = 0; k < NB; ++k) lcol[k] = (k > lane && k < nb) ? Lp[(kb + k) + (i64)(kb + lane) * nr] : 0.0;
#pragma unroll
      for (int k = NB - 1; k > 0; --k) {
        const double xk = __shfl_sync(0xffffffffu, x, k);
        x -= lcol[k] * xk;  // zero unless lane < k < nb
      }
      if (lane < nb) xw[c0 + kb + lane] = x;
      __threadfence();
    }
    cluster.sync();  // the block's solution is visible to every CTA; `part` may be overwritten
  }
}

// ---- triangular solves, one CTA per front of the level
__device__ void solve_fwd_body(const DevSym& S, int s, const double* L, double* xw, double* B) {
  __shared__ double L11[QS_SMALL_NS * QS_SMALL_NS];
  __shared__ double xs[QS_SMALL_NS];
  const Front f = front_of(S, s, const_cast<double*>(L), nullptr);
  const int tid = threadIdx.x;
  const int nr = f.nr, ns = f.ns;
  double* cb = B + S.Boff[s];
  const bool childless = S.childptr[s + 1] == S.childptr[s];  // nothing was gathered: start from zero
  double* x1 = xw + f.c0;
  __syncthreads();  // shared arrays may still be read by the previous front of a chain
  for (int e = tid; e < ns * ns; e += blockDim.x) L11[e] = f.Lp[(e % ns) + (i64)(e / ns) * nr];
  if (tid < ns) xs[tid] = x1[tid];
  __syncthreads();
  if (ns <= 32) {
    // one warp, entry i in lane i, pivots broadcast by shuffles: no CTA barrier per pivot (a chain of ~50 narrow
    // levels per sweep pays every barrier in latency).  Same update order per entry as the loop below: bitwise equal.
    if (tid < 32) {
      double x = tid < ns ? xs[tid] : 0.0;
      for (int k = 0; k < ns - 1; ++k) {
        const double xk = __shfl_sync(0xffffffffu, x, k);
        if (tid > k && tid < ns) x -= L11[tid + k * ns] * xk;
      }
      if (tid < ns) xs[tid] = x;
    }
    __syncthreads();
  } else {
    for (int k = 0; k < ns - 1; ++k) {  // unit lower triangular solve at shared-memory latency
      const double xk = xs[k];
      for (int i = k + 1 + tid; i < ns; i += blockDim.x) xs[i] -= L11[i + k * ns] * xk;
      __syncthreads();
    }
  }
  if (tid < ns) x1[tid] = xs[tid];
  for (int r = tid; r < f.nu; r += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < ns; ++k) acc += f.Lp[ns + r + (i64)k * nr] * xs[k];
    cb[r] = (childless ? 0.0 : cb[r]) - acc;
  }
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_solve_fwd(DevSym S, const int* list, const double* L, double* xw, double* B) {
  QS_BATCH(S, list, L, xw, B);
  solve_fwd_body(S, list[blockIdx.x], L, xw, B);
}

__global__ void __launch_bounds__(LDL_THREADS) k_solve_diag(int N, const double* Dg, double* xw) {
  QS_BATCH(Dg, xw);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) xw[j] /= Dg[j];
}

__device__ void solve_bwd_body(const DevSym& S, int s, const double* L, double* xw) {
  __shared__ double L11[QS_SMALL_NS * QS_SMALL_NS];
  __shared__ double xs[QS_SMALL_NS];
  const Front f = front_of(S, s, const_cast<double*>(L), nullptr);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int nr = f.nr, ns = f.ns;
  double* x1 = xw + f.c0;
  __syncthreads();  // shared arrays may still be read by the previous front of a chain
  for (int e = tid; e < ns * ns; e += blockDim.x) L11[e] = f.Lp[(e % ns) + (i64)(e / ns) * nr];
  // x1 -= L21' x2
  for (int k = warp; k < ns; k += nwarps) {
    double acc = 0.0;
    for (int r = lane; r < f.nu; r += 32) acc += f.Lp[ns + r + (i64)k * nr] * xw[f.rows[ns + r]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) xs[k] = x1[k] - acc;
  }
  __syncthreads();
  // x1 <- L11^{-T} x1
  if (ns <= 32) {  // one warp, no CTA barrier per pivot (see solve_fwd_body); bitwise the loop below
    if (tid < 32) {
      double x = tid < ns ? xs[tid] : 0.0;
      for (int k = ns - 1; k > 0; --k) {
        const double xk = __shfl_sync(0xffffffffu, x, k);
        if (tid < k) x -= L11[k + tid * ns] * xk;
      }
      if (tid < ns) xs[tid] = x;
    }
    __syncthreads();
  } else {
    for (int k = ns - 1; k > 0; --k) {
      const double xk = xs[k];
      for (int i = tid; i < k; i += blockDim.x) xs[i] -= L11[k + i * ns] * xk;
      __syncthreads();
    }
  }
  if (tid < ns) x1[tid] = xs[tid];
}

__global__ void __launch_bounds__(LDL_THREADS) k_solve_bwd(DevSym S, const int* list, const double* L, double* xw) {
  QS_BATCH(S, list, L, xw);
  solve_bwd_body(S, list[blockIdx.x], L, xw);
}

// ---- narrow-level chains (the upper part of the elimination tree of a banded / staged problem such as an MPC
// trajectory is a long chain of small fronts, one or two per level): ONE CTA walks a run of consecutive narrow levels,
// barriers between the steps, instead of 3-5 launches per level -- a small problem is bound by the number of
// dependent launches, not by bytes or flops.
struct ChainArgs {
  int lv0, lv1;             // levels [lv0, lv1)
  const int* smallptr;      // [nlevels+1] offsets into small_list
  const int* small_list;
  const i64* eaptr;         // [nlevels+1] extend-add item ranges
  const EaItem* eaitems;
  const i64* lvslot;        // [nlevels+1] slot ranges
  __device__ void shift(size_t off) {
    qs_shift(off, smallptr);
    qs_shift(off, small_list);
    qs_shift(off, eaptr);
    qs_shift(off, eaitems);
    qs_shift(off, lvslot);
  }
};

__global__ void __launch_bounds__(LDL_THREADS)
    k_chain_factor(DevSym S, AsmLists A, ChainArgs C, double* L, double* U, double* Dg, const double* reg, double dyn_eps,
                   double* scalars) {
  QS_BATCH(S, A, C, L, U, Dg, reg, scalars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int lv = C.lv0; lv < C.lv1; ++lv) {
    // extend-add of the level: a warp per (column slot) item, children in list order
    for (i64 w = C.eaptr[lv] + warp; w < C.eaptr[lv + 1]; w += nwarps) {
      const EaItem it = C.eaitems[w];
      const int s = A.slot_front[it.slot], pc = A.slot_row[it.slot];
      const Front f = front_of(S, s, L, U);
      const i64 nr = f.nr, nu = f.nu;
      double* dstcol = (pc < f.ns) ? f.Lp + pc * nr : f.Up + qs_ucol(pc - f.ns, nu) - f.ns;
      for (i64 e = A.gptr[it.slot]; e < A.gptr[it.slot + 1]; ++e) {
        const int c = A.gchild[e];
        const int cc = A.gsrc[e] - (int)S.Boff[c];
        const int nuc = (int)(S.rowptr[c + 1] - S.rowptr[c]) - (S.col0[c + 1] - S.col0[c]);
        const double* Ucol = U + S.Uoff[c] + qs_ucol(cc, nuc);
        const int* rel = S.rel + S.relptr[c];
        for (int r = cc + lane; r < nuc; r += 32) dstcol[rel[r]] += Ucol[r];
      }
    }
    __syncthreads();
    for (int k = C.smallptr[lv]; k < C.smallptr[lv + 1]; ++k) {
      front_factor_body(S, C.small_list[k], L, U, Dg, reg, dyn_eps, scalars);
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_chain_fwd(DevSym S, AsmLists A, ChainArgs C, const double* L, double* xw, double* B) {
  QS_BATCH(S, A, C, L, xw, B);
  for (int lv = C.lv0; lv < C.lv1; ++lv) {
    for (i64 g = C.lvslot[lv] + threadIdx.x; g < C.lvslot[lv + 1]; g += blockDim.x) {  // thread per slot
      double acc = 0.0;
      for (i64 e = A.gptr[g]; e < A.gptr[g + 1]; ++e) acc += B[A.gsrc[e]];
      const i64 d = A.gdst[g];
      if (d >= 0) xw[d] += acc;
      else B[-d - 1] = acc;
    }
    __syncthreads();
    for (int k = C.smallptr[lv]; k < C.smallptr[lv + 1]; ++k) {
      solve_fwd_body(S, C.small_list[k], L, xw, B);
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(LDL_THREADS) k_chain_bwd(DevSym S, ChainArgs C, const double* L, double* xw) {
  QS_BATCH(S, C, L, xw);
  for (int lv = C.lv1 - 1; lv >= C.lv0; --lv)
    for (int k = C.smallptr[lv]; k < C.smallptr[lv + 1]; ++k) {
      solve_bwd_body(S, C.small_list[k], L, xw);
      __syncthreads();
    }
}

__global__ void __launch_bounds__(LDL_THREADS) k_permute_in(int N, const int* perm, const double* rhs, double* xw) {
  QS_BATCH(perm, rhs, xw);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) xw[j] = rhs[perm[j]];
}
__global__ void __launch_bounds__(LDL_THREADS) k_permute_out(int N, const int* perm, const double* xw, double* sol) {
  QS_BATCH(perm, xw, sol);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) sol[perm[j]] = xw[j];
}

// Host-side parallel loop over [0, n): fn(lo, hi) on up to 8 threads (the analysis runs once per problem; its loops
// over 10^6 supernodes / 10^7 list entries are memory-bound and independent per parent).
template <class Fn>
void parallel_ranges(i64 n, Fn fn) {
  const int nt = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (n < 200000 || nt == 1) {
    fn((i64)0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(fn, n * t / nt, n * (t + 1) / nt);
  for (auto& th : pool) th.join();
}

template <class... Args>
void launch_clustered(void (*kern)(Args...), int nfronts, int cl, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nfronts * cl), 1, (unsigned)qs_tls_batch);
  cfg.blockDim = dim3(LDL_THREADS, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

// Threads of the single-CTA chain kernels (runs of narrow levels: a handful of small fronts per level).  Their
// bodies are written for any block size; with fronts of ~30 rows most of 256 threads only wait at the barriers.
int chain_threads() {
  static const int t = [] {
    int v = getenv("QS_CHAIN_THREADS") ? atoi(getenv("QS_CHAIN_THREADS")) : LDL_THREADS;
    v = (v / 32) * 32;
    return v < 32 ? 32 : (v > LDL_THREADS ? LDL_THREADS : v);
  }();
  return t;
}

int grid_for(i64 n) {
  i64 g = (n + LDL_THREADS - 1) / LDL_THREADS;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

thread_local size_t g_upload_bytes = 0;  // bytes copied by upload() since analyze() reset it (analysis is single-threaded per call)

template <class T>
T* upload(const std::vector<T>& v, std::vector<void*>* owned, size_t* bytes, cudaStream_t st) {
  g_upload_bytes += v.size() * sizeof(T);
  T* d = nullptr;
  const size_t sz = std::max<size_t>(v.size(), 1) * sizeof(T);
  if (qs_dev_malloc((void**)&d, sz) != cudaSuccess) return nullptr;
  if (!v.empty()) cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st);
  owned->push_back(d);
  *bytes += sz;
  return d;
}

}  // namespace

std::string LinSys::analyze(i64 N_, const i64* Kp, const i64* Ki, i64 knnz_full, const i64* d_Kp, const int* d_Ki, int order,
                            const i64* user_perm, i64 ncliques, const i64* clique_start, const i64* clique_size,
                            i64 n_pos, double static_reg, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  const size_t upload_mark = g_upload_bytes;
  N = N_;
  knnz = knnz_full;
  std::string err = hs_symbolic_cliques(N, Kp, Ki, order, user_perm, ncliques, clique_start, clique_size, &S);
  if (!err.empty()) return err;
  const bool verbose = getenv("QS_VERBOSE") != nullptr;
  auto t_mark = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (verbose) {
      cudaStreamSynchronize(st);
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[qs ldl setup] %-28s %8.3f s\n", what, std::chrono::duration<double>(now - t_mark).count());
      t_mark = now;
    }
  };
  lap("(symbolic total)");
  D.nsup = S.nsup;
#define UP(field, vec)                                   \
  D.field = upload(vec, &owned, &device_bytes, st);      \
  if (!D.field) return "cudaMalloc failed for LDL symbolic data";
  UP(col0, S.col0)
  UP(rowptr, S.rowptr)
  UP(rowidx, S.rowidx)
  UP(childptr, S.childptr)
  UP(child, S.child)
  UP(relptr, S.relptr)
  UP(rel, S.rel)
  UP(Loff, S.Loff)
  UP(Uoff, S.Uoff)
  UP(Boff, S.Boff)
  UP(sup_of, S.sup_of)
  UP(iperm, S.iperm)
  UP(perm, S.perm)
#undef UP
  d_levelsup = upload(S.levelsup, &owned, &device_bytes, st);
  // work lists: simple leaves (warp per front), general fronts per level (CTA per front),
  // extend-add slabs per level (8 front columns per CTA; only fronts that have children)
  std::vector<int> leaf, gen, small, blk;
  int leaf_max_nu = 0;
  std::vector<SlabItem> slabs;
  smallptr.assign(S.nlevels + 1, 0);
  blkptr.assign(S.nlevels + 1, 0);
  blk_max_ns.assign(S.nlevels, 0);
  blk_max_nr.assign(S.nlevels, 0);
  blk_max_nu.assign(S.nlevels, 0);
  genptr.assign(S.nlevels + 1, 0);
  slabptr.assign(S.nlevels + 1, 0);
  for (int lv = 0; lv < S.nlevels; ++lv) {
    for (int k = S.levelptr[lv]; k < S.levelptr[lv + 1]; ++k) {
      const int s = S.levelsup[k];
      const int ns = S.col0[s + 1] - S.col0[s];
      const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]);
      const bool has_children = S.childptr[s + 1] > S.childptr[s];
      if (!has_children && ns == 1 && nr <= 33) {
        leaf.push_back(s);
        leaf_max_nu = std::max(leaf_max_nu, nr - 1);
        continue;
      }
      gen.push_back(s);
      if (nr > QS_SMALL_NR || ns > QS_SMALL_NS) {
        blk.push_back(s);
        blk_max_ns[lv] = std::max(blk_max_ns[lv], ns);
        blk_max_nr[lv] = std::max(blk_max_nr[lv], nr);
        blk_max_nu[lv] = std::max(blk_max_nu[lv], nr - ns);
      } else {
        small.push_back(s);
      }
      if (has_children)
        for (int c = 0; c < nr; c += 8) slabs.push_back(SlabItem{s, c});
    }
    genptr[lv + 1] = (int)gen.size();
    smallptr[lv + 1] = (int)small.size();
    blkptr[lv + 1] = (int)blk.size();
    slabptr[lv + 1] = (int)slabs.size();
    // widest panels first: the fronts of a chunk (below) then need the same number of block steps
    std::stable_sort(blk.begin() + blkptr[lv], blk.end(), [&](int a, int b) {
      const int na = S.col0[a + 1] - S.col0[a], nb = S.col0[b + 1] - S.col0[b];
      if (na != nb) return na > nb;
      return (S.rowptr[a + 1] - S.rowptr[a]) > (S.rowptr[b + 1] - S.rowptr[b]);
    });
  }
  n_leaf = (int)leaf.size();
  leaf_group = 4;
  while (leaf_group < 32 && leaf_group < leaf_max_nu) leaf_group <<= 1;
  d_leaf = upload(leaf, &owned, &device_bytes, st);
  d_gen = upload(gen, &owned, &device_bytes, st);
  d_small = upload(small, &owned, &device_bytes, st);
  d_blk = upload(blk, &owned, &device_bytes, st);
  // per blocked front: offset of its row-tile partial sums (backward solve); the workspace is reused per level
  std::vector<i64> poff(blk.size() + 1, 0);
  i64 pmax = 0;
  for (int lv = 0; lv < S.nlevels; ++lv) {
    i64 at = 0;
    for (int k = blkptr[lv]; k < blkptr[lv + 1]; ++k) {
      const int fs = blk[k];
      const i64 nrf = S.rowptr[fs + 1] - S.rowptr[fs];
      poff[k] = at;
      at += ((nrf + LDL_THREADS - 1) / LDL_THREADS) * NB;
    }
    pmax = std::max(pmax, at);
  }
  d_poff = upload(poff, &owned, &device_bytes, st);
  {
    std::vector<TileItem> tiles;
    tileptr.assign(S.nlevels + 1, 0);
    blk_chunks.clear();
    chunkptr.assign(S.nlevels + 1, 0);
    // chunk budget: panel bytes per chunk (QS_LDL_CHUNK_MB; default 0 = one chunk per level).  Measured at C4 (10^4
    // cone fronts, 4.9 GB of panels): 16 / 32 / 48 / 96 / 200 MB chunks -> 138 / 90 / 76 / 62 / 55 ms per
    // factorisation against 50.8 ms unchunked -- the lockstep launches need the whole level to fill the machine;
    // L2 residency of the panels buys less than the extra launch tails cost.
    const i64 chunk_bytes = (i64)(getenv("QS_LDL_CHUNK_MB") ? atoi(getenv("QS_LDL_CHUNK_MB")) : 0) << 20;
    for (int lv = 0; lv < S.nlevels; ++lv) {
      BlkChunk c{blkptr[lv], 0, 0, 0, (i64)tiles.size(), 0};
      i64 bytes = 0;
      auto close = [&]() {
        if (c.count == 0) return;
        c.t1 = (i64)tiles.size();
        blk_chunks.push_back(c);
        c = BlkChunk{c.b0 + c.count, 0, 0, 0, (i64)tiles.size(), 0};
        bytes = 0;
      };
      for (int k = blkptr[lv]; k < blkptr[lv + 1]; ++k) {
        const int fs = blk[k];
        const int nsf = S.col0[fs + 1] - S.col0[fs], nrf = (int)(S.rowptr[fs + 1] - S.rowptr[fs]);
        const int nu = nrf - nsf;
        const int nt = (nu + TS - 1) / TS;
        for (int tj = 0; tj < nt; ++tj)
          for (int ti = tj; ti < nt; ++ti) tiles.push_back(TileItem{fs, (short)ti, (short)tj});
        c.count++;
        c.max_ns = std::max(c.max_ns, nsf);
        c.max_nr = std::max(c.max_nr, nrf);
        bytes += (i64)nsf * nrf * 8;
        if (c.count >= 65535 || (chunk_bytes > 0 && bytes >= chunk_bytes)) close();
      }
      close();
      tileptr[lv + 1] = (i64)tiles.size();
      chunkptr[lv + 1] = (int)blk_chunks.size();
    }
    d_tiles = upload(tiles, &owned, &device_bytes, st);
    if (!d_tiles) return "cudaMalloc failed for the Schur tile list";
    cudaStreamSynchronize(st);
  }
  if (qs_dev_malloc((void**)&partial, std::max<i64>(pmax, 1) * 8) != cudaSuccess) return "cudaMalloc failed (solve partials)";
  owned.push_back(partial);
  device_bytes += pmax * 8;
  d_slabs = upload(slabs, &owned, &device_bytes, st);
  if (!d_leaf || !d_gen || !d_small || !d_blk || !d_slabs) return "cudaMalloc failed for LDL work lists";
  lap("symbolic upload + work lists");
  // ---- assembly lists (AsmLists): slots of the fronts that have children, level by level
  use_cluster = getenv("QS_LDL_LOCKSTEP") == nullptr;
  use_graphs = getenv("QS_NO_GRAPH") == nullptr;
  use_lists = getenv("QS_LDL_SEARCH") == nullptr && S.Boff[S.nsup] < ((i64)1 << 31);
  if (use_lists) {
    std::vector<i64> slot_base(S.nsup, -1);
    lvslot.assign(S.nlevels + 1, 0);
    i64 nslots = 0;
    for (int lv = 0; lv < S.nlevels; ++lv) {
      for (int k = S.levelptr[lv]; k < S.levelptr[lv + 1]; ++k) {
        const int s = S.levelsup[k];
        if (S.childptr[s + 1] == S.childptr[s]) continue;
        slot_base[s] = nslots;
        nslots += S.rowptr[s + 1] - S.rowptr[s];
      }
      lvslot[lv + 1] = nslots;
    }
    lap("  lists: slot bases");
    std::vector<int> slot_front(nslots), slot_row(nslots);
    std::vector<i64> gptr(nslots + 1, 0), gdst(nslots);
    // every loop below is partitioned by PARENT supernode: a thread touches only the slots of its own parents
    parallel_ranges(S.nsup, [&](i64 lo, i64 hi) {
      for (i64 s = lo; s < hi; ++s) {
        if (slot_base[s] < 0) continue;
        const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]), ns = S.col0[s + 1] - S.col0[s];
        for (int r = 0; r < nr; ++r) {
          const i64 k = slot_base[s] + r;
          slot_front[k] = (int)s;
          slot_row[k] = r;
          gdst[k] = (r < ns) ? (i64)(S.col0[s] + r) : -(S.Boff[s] + (r - ns)) - 1;
        }
        for (int ci = S.childptr[s]; ci < S.childptr[s + 1]; ++ci) {
          const int c = S.child[ci];
          for (i64 t = S.relptr[c]; t < S.relptr[c + 1]; ++t) gptr[slot_base[s] + S.rel[t] + 1]++;
        }
      }
    });
    lap("  lists: slots + counts");
    for (i64 k = 0; k < nslots; ++k) gptr[k + 1] += gptr[k];
    std::vector<int> gsrc(gptr[nslots]), gchild(gptr[nslots]);
    {
      std::vector<i64> next(gptr.begin(), gptr.end() - 1);
      parallel_ranges(S.nsup, [&](i64 lo, i64 hi) {
        for (i64 s = lo; s < hi; ++s)  // children in their fixed (ascending) order
          for (int ci = S.childptr[s]; ci < S.childptr[s + 1]; ++ci) {
            const int c = S.child[ci];
            const i64 nuc = S.relptr[c + 1] - S.relptr[c];
            for (i64 t = 0; t < nuc; ++t) {
              const i64 e = next[slot_base[s] + S.rel[S.relptr[c] + t]]++;
              gsrc[e] = (int)(S.Boff[c] + t);
              gchild[e] = c;
            }
          }
      });
    }
    lap("  lists: fill");
    // row bands for fronts with many children
    std::vector<i64> bandptr(S.nsup + 1, 0);
    std::vector<char> banded(S.nsup, 0);
    for (int s = 0; s < S.nsup; ++s) {
      const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]);
      // bands pay off when many children each bring many rows (the root: 10^4 children x ~400 rows); a cone
      // front with 135 one-column leaves of 4 rows gains nothing from them
      i64 child_rows = 0;
      const int nch = S.childptr[s + 1] - S.childptr[s];
      for (int ci = S.childptr[s]; ci < S.childptr[s + 1]; ++ci)
        child_rows += S.relptr[S.child[ci] + 1] - S.relptr[S.child[ci]];
      banded[s] = (nch >= 64 && nr > QS_EA_BAND && child_rows > 32 * (i64)nch);
    }
    for (int c = 0; c < S.nsup; ++c) {
      const int par = S.parent[c];
      i64 cntb = 0;
      if (par >= 0 && banded[par]) {
        const int nrp = (int)(S.rowptr[par + 1] - S.rowptr[par]);
        cntb = (nrp + QS_EA_BAND - 1) / QS_EA_BAND + 1;
      }
      bandptr[c + 1] = bandptr[c] + cntb;
    }
    std::vector<int> bandstart(std::max<i64>(bandptr[S.nsup], 1));
    for (int c = 0; c < S.nsup; ++c) {
      const i64 nb1 = bandptr[c + 1] - bandptr[c];
      if (!nb1) continue;
      const int* rel = S.rel.data() + S.relptr[c];
      const int nuc = (int)(S.relptr[c + 1] - S.relptr[c]);
      int r = 0;
      for (i64 b = 0; b < nb1; ++b) {
        while (r < nuc && rel[r] < b * QS_EA_BAND) ++r;
        bandstart[bandptr[c] + b] = r;
      }
    }
    lap("  lists: bands");
    // extend-add items per level
    std::vector<EaItem> items;
    eaptr.assign(S.nlevels + 1, 0);
    ea_wide.clear();
    lv_tpr.assign(S.nlevels, 1);
    ea_direct.assign(S.nlevels, 0);
    items.reserve(1 << 16);
    for (int lv = 0; lv < S.nlevels; ++lv) {
      // a wide level without banded fronts needs no item list: item w is column slot lvslot[lv] + w (an explicit
      // list would be 8 bytes x 7 M slots at C4, built and uploaded for nothing)
      bool any_banded = false;
      for (int k = S.levelptr[lv]; k < S.levelptr[lv + 1] && !any_banded; ++k) any_banded = banded[S.levelsup[k]];
      ea_direct[lv] = !any_banded && lvslot[lv + 1] - lvslot[lv] > 4096;
      for (i64 k = lvslot[lv]; k < lvslot[lv + 1] && !ea_direct[lv]; ++k) {
        if (gptr[k + 1] == gptr[k]) continue;  // nothing lands on this column
        const int s = slot_front[k];
        if (!banded[s]) {
          items.push_back(EaItem{(int)k, -1});
        } else {
          const int nr = (int)(S.rowptr[s + 1] - S.rowptr[s]);
          const int nbands = (nr + QS_EA_BAND - 1) / QS_EA_BAND;
          for (int b = slot_row[k] / QS_EA_BAND; b < nbands; ++b) items.push_back(EaItem{(int)k, b});
        }
      }
      eaptr[lv + 1] = (i64)items.size();
      {  // mean number of update rows of the children assembled at this level decides the lanes per item
        i64 rows = 0, kids = 0;
        for (int k = S.levelptr[lv]; k < S.levelptr[lv + 1]; ++k) {
          const int s2 = S.levelsup[k];
          for (int ci = S.childptr[s2]; ci < S.childptr[s2 + 1]; ++ci) {
            rows += S.relptr[S.child[ci] + 1] - S.relptr[S.child[ci]];
            ++kids;
          }
        }
        ea_wide.push_back(kids == 0 || rows > 16 * kids);
      }
      const i64 ns_lv = lvslot[lv + 1] - lvslot[lv];
      const double mean = ns_lv ? (double)(gptr[lvslot[lv + 1]] - gptr[lvslot[lv]]) / (double)ns_lv : 1.0;
      int t = 1;
      while (t < 32 && t * 2 <= mean) t <<= 1;
      lv_tpr[lv] = t;
    }
    lap("  lists: items + lanes");
    if (nslots >= ((i64)1 << 31)) {
      use_lists = false;
    } else {
      A.gptr = upload(gptr, &owned, &device_bytes, st);
      A.gsrc = upload(gsrc, &owned, &device_bytes, st);
      A.gchild = upload(gchild, &owned, &device_bytes, st);
      A.gdst = upload(gdst, &owned, &device_bytes, st);
      A.slot_front = upload(slot_front, &owned, &device_bytes, st);
      A.slot_row = upload(slot_row, &owned, &device_bytes, st);
      A.bandptr = upload(bandptr, &owned, &device_bytes, st);
      A.bandstart = upload(bandstart, &owned, &device_bytes, st);
      d_eaitems = upload(items, &owned, &device_bytes, st);
      if (!A.gptr || !A.gsrc || !A.gchild || !A.gdst || !A.slot_front || !A.slot_row || !A.bandptr || !A.bandstart ||
          !d_eaitems)
        return "cudaMalloc failed for the LDL assembly lists";
      cudaStreamSynchronize(st);  // the host vectors above die at the end of this block
    }
  }
  lap("  lists: uploads");
  // ---- narrow-level chains: maximal runs of >= 3 consecutive levels that hold only a few small fronts each
  chain_end.assign(S.nlevels, 0);
  chain_start_of_end.assign(S.nlevels, -1);
  for (int lv = 0; lv < S.nlevels; ++lv) chain_end[lv] = lv + 1;
  if (use_lists && getenv("QS_LDL_NO_CHAIN") == nullptr) {
    auto narrow = [&](int lv) {
      const int nsm = smallptr[lv + 1] - smallptr[lv];
      return lv > 0 && blkptr[lv + 1] == blkptr[lv] && nsm >= 1 && nsm <= 8 && lvslot[lv + 1] - lvslot[lv] <= 4096;
    };
    for (int lv = 0; lv < S.nlevels;) {
      int e = lv;
      while (e < S.nlevels && narrow(e)) ++e;
      if (e - lv >= 3) {
        chain_end[lv] = e;
        lv = e;
      } else {
        lv = std::max(e, lv + 1);
      }
    }
    chain_start_of_end.assign(S.nlevels, -1);
    for (int lv = 0; lv < S.nlevels; ++lv)
      if (chain_end[lv] > lv + 1) chain_start_of_end[chain_end[lv] - 1] = lv;
    d_smallptr = upload(smallptr, &owned, &device_bytes, st);
    d_eaptr = upload(eaptr, &owned, &device_bytes, st);
    d_lvslot = upload(lvslot, &owned, &device_bytes, st);
    if (!d_smallptr || !d_eaptr || !d_lvslot) return "cudaMalloc failed for the chain tables";
    cudaStreamSynchronize(st);
  }
  lap("assembly lists");
  std::vector<double> regh(N);
  for (i64 k = 0; k < N; ++k) regh[k] = (S.perm[k] < n_pos) ? static_reg : -static_reg;  // kkt.py:48-52
  reg = upload(regh, &owned, &device_bytes, st);
  auto alloc = [&](void** p, size_t bytes) {
    if (qs_dev_malloc(p, std::max<size_t>(bytes, 8)) != cudaSuccess) return false;
    owned.push_back(*p);
    device_bytes += bytes;
    return true;
  };
  const i64 lsz = S.Loff[S.nsup], usz = S.Uoff[S.nsup], bsz = S.Boff[S.nsup];
  if (!alloc((void**)&L, lsz * 8) || !alloc((void**)&U, usz * 8) || !alloc((void**)&Dg, N * 8) ||
      !alloc((void**)&B, bsz * 8) || !alloc((void**)&xw, N * 8) || !alloc((void**)&amap, knnz * 8) || !d_levelsup ||
      !reg) {
    cudaGetLastError();
    return "out of device memory for the LDL' factor (panels " + std::to_string(lsz * 8 >> 20) + " MiB, updates " +
           std::to_string(usz * 8 >> 20) + " MiB)";
  }
  k_build_amap<<<qs_grid((unsigned)((N * 32 + LDL_THREADS - 1) / LDL_THREADS)), LDL_THREADS, 0, st>>>((int)N, d_Kp, d_Ki, D,
                                                                                              amap);
  cudaStreamSynchronize(st);  // host vectors above must outlive the async copies
  if (cudaGetLastError() != cudaSuccess) return "LDL' analysis kernels failed";
  lap("factor storage + amap");
  h2d_bytes = g_upload_bytes - upload_mark;
  analysis_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return std::string();
}

namespace {
// Replay the launches of `body` from a graph captured on first use for the argument pair (a, b).
template <class Body>
void run_graphed(std::vector<LinSys::GraphEntry>& cache, bool enabled, const void* a, const void* b, cudaStream_t st,
                 long long* counts /*[2]: graph replays, direct launch sequences*/, Body body) {
  if (!enabled) {
    counts[1]++;
    body();
    return;
  }
  for (const LinSys::GraphEntry& e : cache)
    if (e.a == a && e.b == b) {
      counts[0]++;
      cudaGraphLaunch(e.exec, st);
      return;
    }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone || cache.size() >= 16 ||
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    counts[1]++;
    body();  // already inside someone else's capture, too many variants, or capture unavailable
    return;
  }
  body();
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  if (cudaStreamEndCapture(st, &g) == cudaSuccess && g && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) {
    cache.push_back(LinSys::GraphEntry{a, b, exec});
    counts[0]++;
    cudaGraphLaunch(exec, st);
  } else {
    cudaGetLastError();
    counts[1]++;
    body();
  }
  if (g) cudaGraphDestroy(g);
}
}  // namespace

std::string LinSys::set_cone_blocks(int n_p, int l, int nsoc, const i64* q_host, const int* d_soc_ptr,
                                    const i64* d_kp_conic, const int* d_cone_of_col, const i64* d_Kp, i64 flat_nnz,
                                    cudaStream_t st) {
  have_cb = false;
  if (nsoc <= 0) return "";
  std::vector<int> tc;
  std::vector<short> tij;
  for (int k = 0; k < nsoc; ++k) {
    const int T = (int)((q_host[k] + 31) / 32);
    if (T > 32767) return "";  // a cone of more than 10^6 entries: keep the entry-by-entry scatter
    for (int tj = 0; tj < T; ++tj)
      for (int ti = 0; ti <= tj; ++ti) {
        tc.push_back(k);
        tij.push_back((short)ti);
        tij.push_back((short)tj);
      }
  }
  if (tc.size() >= ((size_t)1 << 31)) return "";
  cb = ConeBlocks{n_p, l, nsoc, d_soc_ptr, d_kp_conic, d_cone_of_col, d_Kp, flat_nnz, (int)tc.size(), nullptr, nullptr};
  cb.tile_cone = upload(tc, &owned, &device_bytes, st);
  cb.tile_ij = upload(tij, &owned, &device_bytes, st);
  cudaStreamSynchronize(st);
  if (!cb.tile_cone || !cb.tile_ij) return "cudaMalloc failed for the SOC block tile list";
  have_cb = true;
  return "";
}

void LinSys::factor(const double* d_Kx, double* scalars, cudaStream_t st) {
  run_graphed(factor_graphs, use_graphs, d_Kx, scalars, st, graph_counts, [&]() { factor_launches(d_Kx, scalars, st); });
}

void LinSys::solve(const double* d_rhs, double* d_sol, cudaStream_t st) {
  run_graphed(solve_graphs, use_graphs, d_rhs, d_sol, st, graph_counts, [&]() { solve_launches(d_rhs, d_sol, st); });
}

void LinSys::factor_launches(const double* d_Kx, double* scalars, cudaStream_t st) {
  qs_memset_b(L, 0, S.Loff[S.nsup] * 8, st);
  if (S.Uoff[S.nsup] > 0) qs_memset_b(U, 0, S.Uoff[S.nsup] * 8, st);
  static const bool tiled_scatter = !(getenv("QS_LDL_TILED_SCATTER") && atoi(getenv("QS_LDL_TILED_SCATTER")) == 0);
  if (have_cb && tiled_scatter) {
    if (cb.flat_nnz > 0) k_scatter_values<<<qs_grid(grid_for(cb.flat_nnz)), LDL_THREADS, 0, st>>>(cb.flat_nnz, d_Kx, amap, L);
    k_scatter_other<<<qs_grid(grid_for((N - cb.n_p - cb.l) * 32)), LDL_THREADS, 0, st>>>((int)N, cb, d_Kx, amap, L);
    k_scatter_blocks<<<qs_grid(cb.ntiles), 256, 0, st>>>(cb, d_Kx, amap, L);
  } else {
    k_scatter_values<<<qs_grid(grid_for(knnz)), LDL_THREADS, 0, st>>>(knnz, d_Kx, amap, L);
  }
  k_add_reg<<<qs_grid(grid_for(N)), LDL_THREADS, 0, st>>>((int)N, D, reg, L);
  auto leaf_grid = [&](int g) { return (unsigned)(((i64)n_leaf * g + LDL_THREADS - 1) / LDL_THREADS); };
  if (n_leaf > 0) QS_LEAF_DISPATCH(k_leaf_factor, leaf_grid, D, d_leaf, n_leaf, L, U, Dg, reg, dyn_eps, scalars)
  for (int lv = 0; lv < S.nlevels; ++lv) {
    if (chain_end[lv] > lv + 1) {  // a run of narrow levels: one single-CTA launch
      const ChainArgs C{lv, chain_end[lv], d_smallptr, d_small, d_eaptr, d_eaitems, d_lvslot};
      k_chain_factor<<<qs_grid(1), chain_threads(), 0, st>>>(D, A, C, L, U, Dg, reg, dyn_eps, scalars);
      lv = chain_end[lv] - 1;
      continue;
    }
    const int nslab = slabptr[lv + 1] - slabptr[lv];
    if (use_lists) {
      const i64 ni = eaptr[lv + 1] - eaptr[lv];
      const bool direct = ea_direct[lv];
      const i64 nit = direct ? lvslot[lv + 1] - lvslot[lv] : ni;
      const EaItem* itp = direct ? nullptr : d_eaitems + eaptr[lv];
      if (nit > 0) {
        if (ea_wide[lv])
          k_extend_add_list<32><<<qs_grid((unsigned)((nit * 32 + LDL_THREADS - 1) / LDL_THREADS)), LDL_THREADS, 0, st>>>(
              D, A, itp, lvslot[lv], nit, L, U);
        else
          k_extend_add_list<4><<<qs_grid((unsigned)((nit * 4 + LDL_THREADS - 1) / LDL_THREADS)), LDL_THREADS, 0, st>>>(
              D, A, itp, lvslot[lv], nit, L, U);
      }
    } else if (nslab > 0) {
      k_extend_add<<<qs_grid(nslab), LDL_THREADS, 0, st>>>(D, d_slabs + slabptr[lv], L, U);
    }
    const int cnt = smallptr[lv + 1] - smallptr[lv];
    if (cnt > 0)
      k_front_factor<<<qs_grid(cnt), LDL_THREADS, 0, st>>>(D, d_small + smallptr[lv], L, U, Dg, reg, dyn_eps, scalars);
    // blocked fronts of this level, chunk by chunk (see BlkChunk)
    for (int ci = chunkptr[lv]; ci < chunkptr[lv + 1]; ++ci) {
      const BlkChunk& ch = blk_chunks[ci];
      const int nb_fronts = ch.count;
      const int* lst = d_blk + ch.b0;
      const int mx_ns = ch.max_ns, mx_nr = ch.max_nr;
      // many fronts: left-looking (each panel block is written once, inner depth kb); a few big fronts:
      // right-looking (rank-32 updates over (ns/64) x (nr/64) tiles keep all SMs busy)
      const bool left = (blkptr[lv + 1] - blkptr[lv]) > 16;
      // many independent fronts: one CTA per front can walk all its block steps (k_front_blocked, QS_LDL_FUSED=1;
      // QS_FUSED_MIN sets the front count from which it is used).  Correct (bitwise the lockstep factor, the solve
      // tests pass with it) but SLOWER at C4: 58.2 ms per factorisation with two CTAs per SM (128 registers, 888
      // bytes of spills), 73.7 ms with one, against 50.4 ms for the lockstep launches -- 16 warps per SM with a barrier
      // after every k-block expose the fetch latency that 10^5-CTA lockstep grids hide.  Kept as an opt-in experiment.
      static const bool fused_on = getenv("QS_LDL_FUSED") && atoi(getenv("QS_LDL_FUSED")) != 0;
      static const int fused_min = getenv("QS_FUSED_MIN") ? atoi(getenv("QS_FUSED_MIN")) : 592;
      const bool fused = fused_on && (blkptr[lv + 1] - blkptr[lv]) >= fused_min;
      static const int fused_minb = getenv("QS_FUSED_MINB") ? atoi(getenv("QS_FUSED_MINB")) : 2;
      if (fused && fused_minb == 1)
        k_front_blocked<1><<<qs_grid(nb_fronts), LDL_THREADS, 0, st>>>(D, lst, L, Dg, reg, dyn_eps, scalars);
      else if (fused)
        k_front_blocked<2><<<qs_grid(nb_fronts), LDL_THREADS, 0, st>>>(D, lst, L, Dg, reg, dyn_eps, scalars);
      // left-looking levels advance two block columns per update launch (QS_LDL_WIDE=0: one)
      static const bool wide = !(getenv("QS_LDL_WIDE") && atoi(getenv("QS_LDL_WIDE")) == 0);
      for (int kb = 0; kb < mx_ns && !fused; kb += NB) {
        if (left && wide) {
          const int nti = (mx_nr - kb + TS - 1) / TS;
          dim3 gu(nti, nb_fronts);
          if ((kb / NB) % 2 == 0) {
            if (kb > 0) k_blk_update<false><<<qs_grid(gu), LDL_THREADS, 0, st>>>(D, lst, nullptr, kb, 3, L, U, Dg);
          } else {  // the odd block column: only the pivots of the block column before it are missing
            k_blk_update<false><<<qs_grid(gu), LDL_THREADS, 0, st>>>(D, lst, nullptr, kb - NB, 2, L, U, Dg);
          }
        } else if (left && kb > 0) {  // bring block column kb up to date with the pivots [0, kb)
          const int nti = (mx_nr - kb + TS - 1) / TS;
          dim3 gu(nti, nb_fronts);
          k_blk_update<false><<<qs_grid(gu), LDL_THREADS, 0, st>>>(D, lst, nullptr, kb, 1, L, U, Dg);
        }
        k_blk_diag<<<qs_grid((nb_fronts * 32 + LDL_THREADS - 1) / LDL_THREADS), LDL_THREADS, 0, st>>>(D, lst, nb_fronts, kb, L, Dg,
                                                                                              reg, dyn_eps, scalars);
        const int rows_below = mx_nr - kb - 1;
        if (rows_below > 0) {
          // thread-per-row trsm: 144 registers = ONE 256-thread CTA per SM (ncu r02g: 11 % of the warp slots active);
          // capped at 128 registers (32 bytes of spills) two CTAs fit: 53.4 -> 51.0 ms per C4 factorisation.
          // QS_PANEL_CFG: 0 = uncapped, 1 = 256 x 2 (default), 2 = 128 x 4, 3 = 128 x 3, 4 = 64 x 8 (all measured)
          static const int cfg = getenv("QS_PANEL_CFG") ? atoi(getenv("QS_PANEL_CFG")) : 1;
          const int T = (cfg == 2 || cfg == 3) ? 128 : (cfg == 4 ? 64 : LDL_THREADS);
          dim3 gp((rows_below + T - 1) / T, nb_fronts);
          switch (cfg) {
            case 0: k_blk_panel<256, 1><<<qs_grid(gp), T, 0, st>>>(D, lst, kb, L, Dg); break;
            case 2: k_blk_panel<128, 4><<<qs_grid(gp), T, 0, st>>>(D, lst, kb, L, Dg); break;
            case 3: k_blk_panel<128, 3><<<qs_grid(gp), T, 0, st>>>(D, lst, kb, L, Dg); break;
            case 4: k_blk_panel<64, 8><<<qs_grid(gp), T, 0, st>>>(D, lst, kb, L, Dg); break;
            default: k_blk_panel<256, 2><<<qs_grid(gp), T, 0, st>>>(D, lst, kb, L, Dg); break;
          }
        }
        const int cols_left = mx_ns - kb - 1;
        if (!left && cols_left > 0) {
          const int ntj = (cols_left + TS - 1) / TS, nti = (mx_nr - kb - 1 + TS - 1) / TS;
          dim3 gu(ntj * nti, nb_fronts);
          k_blk_update<false><<<qs_grid(gu), LDL_THREADS, 0, st>>>(D, lst, nullptr, kb, 0, L, U, Dg);
        }
      }
      // Schur complements of the chunk's fronts (exact tile list), while their panels are still in the L2
      const i64 ntile = ch.t1 - ch.t0;
      for (i64 t0 = 0; t0 < ntile; t0 += (i64)1 << 30) {
        const unsigned cnt2 = (unsigned)std::min<i64>((i64)1 << 30, ntile - t0);
        k_blk_update<true><<<qs_grid(cnt2), LDL_THREADS, 0, st>>>(D, nullptr, d_tiles + ch.t0 + t0, 0, 0, L, U, Dg);
      }
    }
  }
}



void LinSys::solve_launches(const double* d_rhs, double* d_sol, cudaStream_t st) {
  k_permute_in<<<qs_grid(grid_for(N)), LDL_THREADS, 0, st>>>((int)N, D.perm, d_rhs, xw);
  auto leaf_grid = [&](int g) { return (unsigned)(((i64)n_leaf * g + LDL_THREADS - 1) / LDL_THREADS); };
  if (n_leaf > 0) QS_LEAF_DISPATCH(k_leaf_fwd, leaf_grid, D, d_leaf, n_leaf, L, xw, B)
  for (int lv = 0; lv < S.nlevels; ++lv) {
    if (chain_end[lv] > lv + 1) {
      const ChainArgs C{lv, chain_end[lv], d_smallptr, d_small, d_eaptr, d_eaitems, d_lvslot};
      k_chain_fwd<<<qs_grid(1), chain_threads(), 0, st>>>(D, A, C, L, xw, B);
      lv = chain_end[lv] - 1;
      continue;
    }
    const int nslab = slabptr[lv + 1] - slabptr[lv];
    if (use_lists) {
      const i64 nsl = lvslot[lv + 1] - lvslot[lv];
      if (nsl > 0)
        k_gather_fwd_list<<<qs_grid((unsigned)((nsl * lv_tpr[lv] + LDL_THREADS - 1) / LDL_THREADS)), LDL_THREADS, 0, st>>>(
            A, lvslot[lv], nsl, lv_tpr[lv], xw, B);
    } else if (nslab > 0) {
      k_gather_fwd<<<qs_grid(nslab), LDL_THREADS, 0, st>>>(D, d_slabs + slabptr[lv], xw, B);
    }
    const int cnt = smallptr[lv + 1] - smallptr[lv];
    if (cnt > 0) k_solve_fwd<<<qs_grid(cnt), LDL_THREADS, 0, st>>>(D, d_small + smallptr[lv], L, xw, B);
    const int nblk_lv = blkptr[lv + 1] - blkptr[lv];
    // few large fronts (the root): one clustered launch; thousands of fronts: the lockstep path below, which keeps
    // every SM streaming panels (a CTA per front walking its own blocks is latency-bound: 9.2 vs 5.1 ms at C4)
    const bool clustered = use_cluster && nblk_lv > 0 && nblk_lv <= 16;
    if (clustered)
      launch_clustered(k_cluster_fwd, nblk_lv, QS_CL_MAX, st, D, (const int*)(d_blk + blkptr[lv]),
                       (const double*)L, xw, B);
    for (int b0 = blkptr[lv]; b0 < blkptr[lv + 1] && !clustered; b0 += 65535) {
      const int nbf = std::min(65535, blkptr[lv + 1] - b0);
      const int* lst = d_blk + b0;
      // childless blocked fronts start their contribution vector from zero (the others were set by the gather)
      k_zero_cb<<<qs_grid(nbf), LDL_THREADS, 0, st>>>(D, lst, B);
      for (int kb = 0; kb < blk_max_ns[lv]; kb += NB) {
        k_fwd_diag<<<qs_grid(nbf), 32, 0, st>>>(D, lst, kb, L, xw);
        const int rows_below = blk_max_nr[lv] - kb - 1;
        if (rows_below > 0) {
          dim3 g((rows_below + LDL_THREADS - 1) / LDL_THREADS, nbf);
          k_fwd_update<<<qs_grid(g), LDL_THREADS, 0, st>>>(D, lst, kb, L, xw, B);
        }
      }
    }
  }
  k_solve_diag<<<qs_grid(grid_for(N)), LDL_THREADS, 0, st>>>((int)N, Dg, xw);
  // chain_start[e - 1] = first level of the chain that ends at level e - 1 (or -1)
  for (int lv = S.nlevels - 1; lv >= 0; --lv) {
    if (chain_start_of_end[lv] >= 0) {
      const int b = chain_start_of_end[lv];
      const ChainArgs C{b, lv + 1, d_smallptr, d_small, d_eaptr, d_eaitems, d_lvslot};
      k_chain_bwd<<<qs_grid(1), chain_threads(), 0, st>>>(D, C, L, xw);
      lv = b;
      continue;
    }
    const int nblk_lv = blkptr[lv + 1] - blkptr[lv];
    const bool clustered = use_cluster && nblk_lv > 0 && nblk_lv <= 16;
    if (clustered)
      launch_clustered(k_cluster_bwd, nblk_lv, QS_CL_MAX, st, D, (const int*)(d_blk + blkptr[lv]),
                       (const double*)L, xw);
    for (int b0 = blkptr[lv]; b0 < blkptr[lv + 1] && !clustered; b0 += 65535) {
      const int nbf = std::min(65535, blkptr[lv + 1] - b0);
      const int* lst = d_blk + b0;
      const i64* po = d_poff + b0;
      const int last_kb = ((blk_max_ns[lv] - 1) / NB) * NB;
      for (int kb = last_kb; kb >= 0; kb -= NB) {
        const int rows_below = blk_max_nr[lv] - kb - 1;
        if (rows_below > 0) {
          dim3 g((rows_below + LDL_THREADS - 1) / LDL_THREADS, nbf);
          k_bwd_partial<<<qs_grid(g), LDL_THREADS, 0, st>>>(D, lst, po, kb, L, xw, partial);
        }
        k_bwd_diag<<<qs_grid(nbf), 32, 0, st>>>(D, lst, po, kb, L, xw, partial);
      }
    }
    const int cnt = smallptr[lv + 1] - smallptr[lv];
    if (cnt > 0) k_solve_bwd<<<qs_grid(cnt), LDL_THREADS, 0, st>>>(D, d_small + smallptr[lv], L, xw);
  }
  if (n_leaf > 0) QS_LEAF_DISPATCH(k_leaf_bwd, leaf_grid, D, d_leaf, n_leaf, L, xw)
  k_permute_out<<<qs_grid(grid_for(N)), LDL_THREADS, 0, st>>>((int)N, D.perm, xw, d_sol);
}

int LinSys::launches_per_factor() const {
  int k = 2 + (n_leaf > 0);  // own kernels only (the two memsets are not counted)
  for (int lv = 0; lv < S.nlevels; ++lv) {
    if (chain_end[lv] > lv + 1) {
      k += 1;
      lv = chain_end[lv] - 1;
      continue;
    }
    k += (slabptr[lv + 1] > slabptr[lv]) + (smallptr[lv + 1] > smallptr[lv]);
    for (int ci = chunkptr[lv]; ci < chunkptr[lv + 1]; ++ci)  // update + diag + panel per block step, Schur
      k += 3 * ((blk_chunks[ci].max_ns + NB - 1) / NB) + 1;
  }
  return k;
}

int LinSys::launches_per_solve() const {
  int k = 3 + 2 * (n_leaf > 0);
  for (int lv = 0; lv < S.nlevels; ++lv) {
    if (chain_end[lv] > lv + 1) {
      k += 2;
      lv = chain_end[lv] - 1;
      continue;
    }
    k += (slabptr[lv + 1] > slabptr[lv]) + 2 * (smallptr[lv + 1] > smallptr[lv]);
    const int nblk_lv = blkptr[lv + 1] - blkptr[lv];
    if (use_cluster && nblk_lv > 0 && nblk_lv <= 16) {
      k += 2;
    } else if (blkptr[lv + 1] > blkptr[lv]) {
      const int chunks = (blkptr[lv + 1] - blkptr[lv] + 65534) / 65535;
      k += chunks * (1 + 4 * ((blk_max_ns[lv] + NB - 1) / NB));
    }
  }
  return k;
}

void LinSys::release() {
  for (GraphEntry& e : factor_graphs) cudaGraphExecDestroy(e.exec);
  for (GraphEntry& e : solve_graphs) cudaGraphExecDestroy(e.exec);
  factor_graphs.clear();
  solve_graphs.clear();
  for (void* p : owned) qs_dev_free(p);
  owned.clear();
  L = U = Dg = B = xw = reg = nullptr;
  amap = nullptr;
}
