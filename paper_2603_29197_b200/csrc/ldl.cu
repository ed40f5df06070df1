// GPU supernodal multifrontal LDL' (see ldl.h).
#include "ldl.h"

#include <chrono>

namespace {

#define LDL_THREADS 256

struct Front {
  int c0, ns, nr, nu;
  const int* rows;
  double* Lp;
  double* Up;
};

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
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < nnz; p += (i64)gridDim.x * blockDim.x)
    L[amap[p]] = Kx[p];
}

__global__ void __launch_bounds__(LDL_THREADS) k_add_reg(int N, DevSym S, const double* reg, double* L) {
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
  const SlabItem it = items[blockIdx.x];
  const int s = it.front;
  const Front f = front_of(S, s, L, U);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pc = it.c_lo + warp;
  if (pc >= f.nr) return;
  const i64 nr = f.nr, nu = f.nu;
  double* dstcol = (pc < f.ns) ? f.Lp + pc * nr : f.Up + (i64)(pc - f.ns) * nu - f.ns;  // indexed by parent row
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
      const double* Ucol = U + S.Uoff[c] + (i64)cc * nuc;
      const int* rel = S.rel + S.relptr[c];
      for (int r = cc + lane; r < nuc; r += 32) dstcol[rel[r]] += Ucol[r];
    }
  }
}

// Leaf fronts with one pivot column and at most 33 rows (the private x columns
// of a cone block: millions of them): one warp per front.
__global__ void __launch_bounds__(LDL_THREADS)
    k_leaf_factor(DevSym S, const int* list, int count, double* L, double* U, double* Dg, const double* reg,
                  double dyn_eps, double* scalars) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= count) return;
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
    const double lj = __shfl_sync(0xffffffffu, l, j);
    if (lane >= j && lane < nu) Up[lane + (i64)j * nu] -= a * lj;
  }
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_leaf_fwd(DevSym S, const int* list, int count, const double* L, const double* xw, double* B) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= count) return;
  const int s = list[w];
  const int nu = (int)(S.rowptr[s + 1] - S.rowptr[s]) - 1;
  const double x1 = xw[S.col0[s]];
  if (lane < nu) B[S.Boff[s] + lane] = -(L[S.Loff[s] + 1 + lane] * x1);
}

__global__ void __launch_bounds__(LDL_THREADS)
    k_leaf_bwd(DevSym S, const int* list, int count, const double* L, double* xw) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= count) return;
  const int s = list[w];
  const i64 rp = S.rowptr[s];
  const int nu = (int)(S.rowptr[s + 1] - rp) - 1;
  double acc = (lane < nu) ? L[S.Loff[s] + 1 + lane] * xw[S.rowidx[rp + 1 + lane]] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) xw[S.col0[s]] -= acc;
}

// One CTA per front of the level (children already assembled by k_extend_add):
// factor the pivot panel, form this front's own update matrix.
__global__ void __launch_bounds__(LDL_THREADS)
    k_front_factor(DevSym S, const int* list, double* L, double* U, double* Dg, const double* reg, double dyn_eps,
                   double* scalars) {
  const int s = list[blockIdx.x];
  const Front f = front_of(S, s, L, U);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const i64 nr = f.nr, nu = f.nu;
  // ---- right-looking LDL' on the pivot panel (nr x ns)
  for (int k = 0; k < f.ns; ++k) {
    __syncthreads();
    double d = f.Lp[k + k * nr];
    if (!qs_finite(d)) {
      if (tid == 0) scalars[SC_PIVOT_NONFINITE] = 1.0;
    } else if (fabs(d) < dyn_eps) {  // dynamic floor, sign from the expected inertia (_kernels.py:160-165)
      d = (reg[f.c0 + k] >= 0.0) ? dyn_eps : -dyn_eps;
      if (tid == 0) atomicAdd(&scalars[SC_PIVOT_BUMPS], 1.0);
    }
    if (tid == 0) Dg[f.c0 + k] = d;
    for (int j = k + 1 + warp; j < f.ns; j += nwarps) {
      const double ljk = f.Lp[j + k * nr] / d;
      for (int i = j + lane; i < f.nr; i += 32) f.Lp[i + j * nr] -= f.Lp[i + k * nr] * ljk;
    }
    __syncthreads();
    for (int i = k + 1 + tid; i < f.nr; i += blockDim.x) f.Lp[i + k * nr] /= d;
  }
  __syncthreads();
  // ---- update matrix: U -= L21 D L21'
  if (f.nu > 0) {
    const double* L21 = f.Lp + f.ns;
    for (int j = warp; j < f.nu; j += nwarps) {
      for (int i0 = j; i0 < f.nu; i0 += 32) {
        const int i = i0 + lane;
        double acc = 0.0;
        for (int k = 0; k < f.ns; ++k) {
          const double t = L21[j + k * nr] * Dg[f.c0 + k];
          if (i < f.nu) acc += L21[i + k * nr] * t;
        }
        if (i < f.nu) f.Up[i + j * nu] -= acc;
      }
    }
  }
}

// ---- triangular solves, one CTA per front of the level
__global__ void __launch_bounds__(LDL_THREADS)
    k_solve_fwd(DevSym S, const int* list, const double* L, double* xw, double* B) {
  const int s = list[blockIdx.x];
  const Front f = front_of(S, s, const_cast<double*>(L), nullptr);
  const int tid = threadIdx.x;
  const i64 nr = f.nr;
  double* cb = B + S.Boff[s];
  for (int r = tid; r < f.nu; r += blockDim.x) cb[r] = 0.0;
  __syncthreads();
  for (int ci = S.childptr[s]; ci < S.childptr[s + 1]; ++ci) {
    const int c = S.child[ci];
    const int nsc = S.col0[c + 1] - S.col0[c];
    const int nuc = (int)(S.rowptr[c + 1] - S.rowptr[c]) - nsc;
    const double* cbc = B + S.Boff[c];
    const int* rel = S.rel + S.relptr[c];
    for (int r = tid; r < nuc; r += blockDim.x) {
      const int pr = rel[r];
      if (pr < f.ns)
        xw[f.c0 + pr] += cbc[r];
      else
        cb[pr - f.ns] += cbc[r];
    }
    __syncthreads();
  }
  double* x1 = xw + f.c0;
  for (int k = 0; k < f.ns - 1; ++k) {
    const double xk = x1[k];
    for (int i = k + 1 + tid; i < f.ns; i += blockDim.x) x1[i] -= f.Lp[i + k * nr] * xk;
    __syncthreads();
  }
  __syncthreads();
  for (int r = tid; r < f.nu; r += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < f.ns; ++k) acc += f.Lp[f.ns + r + k * nr] * x1[k];
    cb[r] -= acc;
  }
}

__global__ void __launch_bounds__(LDL_THREADS) k_solve_diag(int N, const double* Dg, double* xw) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) xw[j] /= Dg[j];
}

__global__ void __launch_bounds__(LDL_THREADS) k_solve_bwd(DevSym S, const int* list, const double* L, double* xw) {
  const int s = list[blockIdx.x];
  const Front f = front_of(S, s, const_cast<double*>(L), nullptr);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const i64 nr = f.nr;
  double* x1 = xw + f.c0;
  // x1 -= L21' x2
  for (int k = warp; k < f.ns; k += nwarps) {
    double acc = 0.0;
    for (int r = lane; r < f.nu; r += 32) acc += f.Lp[f.ns + r + k * nr] * xw[f.rows[f.ns + r]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) x1[k] -= acc;
  }
  __syncthreads();
  // x1 <- L11^{-T} x1
  for (int k = f.ns - 1; k > 0; --k) {
    const double xk = x1[k];
    for (int i = tid; i < k; i += blockDim.x) x1[i] -= f.Lp[k + i * nr] * xk;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(LDL_THREADS) k_permute_in(int N, const int* perm, const double* rhs, double* xw) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) xw[j] = rhs[perm[j]];
}
__global__ void __launch_bounds__(LDL_THREADS) k_permute_out(int N, const int* perm, const double* xw, double* sol) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) sol[perm[j]] = xw[j];
}

int grid_for(i64 n) {
  i64 g = (n + LDL_THREADS - 1) / LDL_THREADS;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

template <class T>
T* upload(const std::vector<T>& v, std::vector<void*>* owned, size_t* bytes, cudaStream_t st) {
  T* d = nullptr;
  const size_t sz = std::max<size_t>(v.size(), 1) * sizeof(T);
  if (cudaMalloc(&d, sz) != cudaSuccess) return nullptr;
  if (!v.empty()) cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st);
  owned->push_back(d);
  *bytes += sz;
  return d;
}

}  // namespace

std::string LinSys::analyze(i64 N_, const i64* Kp, const i64* Ki, const i64* d_Kp, const int* d_Ki, int order,
                            const i64* user_perm, i64 ncliques, const i64* clique_start, const i64* clique_size,
                            i64 n_pos, double static_reg, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  N = N_;
  knnz = Kp[N];
  std::string err = hs_symbolic_cliques(N, Kp, Ki, order, user_perm, ncliques, clique_start, clique_size, &S);
  if (!err.empty()) return err;
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
  std::vector<int> leaf, gen;
  std::vector<SlabItem> slabs;
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
        continue;
      }
      gen.push_back(s);
      if (has_children)
        for (int c = 0; c < nr; c += 8) slabs.push_back(SlabItem{s, c});
    }
    genptr[lv + 1] = (int)gen.size();
    slabptr[lv + 1] = (int)slabs.size();
  }
  n_leaf = (int)leaf.size();
  d_leaf = upload(leaf, &owned, &device_bytes, st);
  d_gen = upload(gen, &owned, &device_bytes, st);
  d_slabs = upload(slabs, &owned, &device_bytes, st);
  if (!d_leaf || !d_gen || !d_slabs) return "cudaMalloc failed for LDL work lists";
  std::vector<double> regh(N);
  for (i64 k = 0; k < N; ++k) regh[k] = (S.perm[k] < n_pos) ? static_reg : -static_reg;  // kkt.py:48-52
  reg = upload(regh, &owned, &device_bytes, st);
  auto alloc = [&](void** p, size_t bytes) {
    if (cudaMalloc(p, std::max<size_t>(bytes, 8)) != cudaSuccess) return false;
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
  k_build_amap<<<(unsigned)((N * 32 + LDL_THREADS - 1) / LDL_THREADS), LDL_THREADS, 0, st>>>((int)N, d_Kp, d_Ki, D,
                                                                                              amap);
  cudaStreamSynchronize(st);  // host vectors above must outlive the async copies
  if (cudaGetLastError() != cudaSuccess) return "LDL' analysis kernels failed";
  analysis_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return std::string();
}

void LinSys::factor(const double* d_Kx, double* scalars, cudaStream_t st) {
  cudaMemsetAsync(L, 0, S.Loff[S.nsup] * 8, st);
  if (S.Uoff[S.nsup] > 0) cudaMemsetAsync(U, 0, S.Uoff[S.nsup] * 8, st);
  k_scatter_values<<<grid_for(knnz), LDL_THREADS, 0, st>>>(knnz, d_Kx, amap, L);
  k_add_reg<<<grid_for(N), LDL_THREADS, 0, st>>>((int)N, D, reg, L);
  if (n_leaf > 0)
    k_leaf_factor<<<(unsigned)(((i64)n_leaf * 32 + LDL_THREADS - 1) / LDL_THREADS), LDL_THREADS, 0, st>>>(
        D, d_leaf, n_leaf, L, U, Dg, reg, dyn_eps, scalars);
  for (int lv = 0; lv < S.nlevels; ++lv) {
    const int nslab = slabptr[lv + 1] - slabptr[lv];
    if (nslab > 0) k_extend_add<<<nslab, LDL_THREADS, 0, st>>>(D, d_slabs + slabptr[lv], L, U);
    const int cnt = genptr[lv + 1] - genptr[lv];
    if (cnt > 0)
      k_front_factor<<<cnt, LDL_THREADS, 0, st>>>(D, d_gen + genptr[lv], L, U, Dg, reg, dyn_eps, scalars);
  }
}

void LinSys::solve(const double* d_rhs, double* d_sol, cudaStream_t st) {
  k_permute_in<<<grid_for(N), LDL_THREADS, 0, st>>>((int)N, D.perm, d_rhs, xw);
  const unsigned leaf_grid = (unsigned)(((i64)n_leaf * 32 + LDL_THREADS - 1) / LDL_THREADS);
  if (n_leaf > 0) k_leaf_fwd<<<leaf_grid, LDL_THREADS, 0, st>>>(D, d_leaf, n_leaf, L, xw, B);
  for (int lv = 0; lv < S.nlevels; ++lv) {
    const int cnt = genptr[lv + 1] - genptr[lv];
    if (cnt > 0) k_solve_fwd<<<cnt, LDL_THREADS, 0, st>>>(D, d_gen + genptr[lv], L, xw, B);
  }
  k_solve_diag<<<grid_for(N), LDL_THREADS, 0, st>>>((int)N, Dg, xw);
  for (int lv = S.nlevels - 1; lv >= 0; --lv) {
    const int cnt = genptr[lv + 1] - genptr[lv];
    if (cnt > 0) k_solve_bwd<<<cnt, LDL_THREADS, 0, st>>>(D, d_gen + genptr[lv], L, xw);
  }
  if (n_leaf > 0) k_leaf_bwd<<<leaf_grid, LDL_THREADS, 0, st>>>(D, d_leaf, n_leaf, L, xw);
  k_permute_out<<<grid_for(N), LDL_THREADS, 0, st>>>((int)N, D.perm, xw, d_sol);
}

int LinSys::launches_per_factor() const {
  int k = 4 + (n_leaf > 0);
  for (int lv = 0; lv < S.nlevels; ++lv) k += (slabptr[lv + 1] > slabptr[lv]) + (genptr[lv + 1] > genptr[lv]);
  return k;
}

int LinSys::launches_per_solve() const {
  int k = 3 + 2 * (n_leaf > 0);
  for (int lv = 0; lv < S.nlevels; ++lv) k += 2 * (genptr[lv + 1] > genptr[lv]);
  return k;
}

void LinSys::release() {
  for (void* p : owned) cudaFree(p);
  owned.clear();
  L = U = Dg = B = xw = reg = nullptr;
  amap = nullptr;
}
