// Ruiz equilibration of the KKT data  M = [P A' G'; A 0 0; G 0 0].
//
// NOT in the reference (it never equilibrates); north_star lists it, so it is
// built as an optional setup-time pass (Settings.ruiz_iters, default 0 = the
// reference's iteration).  Scheme (as in upstream QOCO): repeat
//     delta_i = 1 / sqrt(|| row i of the currently scaled M ||_inf)
//     D <- D delta_x,  E <- E delta_y,  F <- F delta_z
// with F held constant inside each second-order cone (s in K <=> F s in K needs a
// scalar per cone; the cone takes the largest of its rows' norms), then
//     P <- D P D, A <- E A D, G <- F G D, c <- D c, b <- E b, h <- F h.
// The solve runs on the scaled problem; qs_get_iterate returns
//     x = D x^, s = s^ / F, y = E y^, z = F z^.
// Row norms are gather-max passes over the same five CSR views the residual
// kernel uses; all scalings are applied on the fly until the final pass.
#include "ruiz_kernels.h"

namespace {

__device__ __forceinline__ double row_absmax(const Csr& M, int row, double rs, const double* cs) {
  double t = 0.0;
  for (int p = M.ptr[row]; p < M.ptr[row + 1]; ++p) t = fmax(t, fabs(M.val[p]) * rs * cs[M.idx[p]]);
  return t;
}

__global__ void __launch_bounds__(QS_THREADS)
    k_ruiz_norms(RuizArgs A, double* dx, double* dy, double* dz) {
  QS_BATCH(A, dx, dy, dz);
  const int N = A.n + A.p + A.m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (i < A.n) {
      const double d = A.D[i];
      double t = row_absmax(A.Pf, i, d, A.D);
      t = fmax(t, row_absmax(A.At, i, d, A.E));
      t = fmax(t, row_absmax(A.Gt, i, d, A.F));
      dx[i] = t;
    } else if (i < A.n + A.p) {
      const int r = i - A.n;
      dy[r] = row_absmax(A.Ar, r, A.E[r], A.D);
    } else {
      const int r = i - A.n - A.p;
      dz[r] = row_absmax(A.Gr, r, A.F[r], A.D);
    }
  }
}

// one scalar per second-order cone: the largest row norm of the cone
__global__ void __launch_bounds__(QS_THREADS) k_ruiz_cone_max(int nsoc, const int* soc_ptr, double* dz) {
  QS_BATCH(soc_ptr, dz);
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (k >= nsoc) return;
  const int o = soc_ptr[k], e = soc_ptr[k + 1];
  double t = 0.0;
  for (int i = o + lane; i < e; i += 32) t = fmax(t, dz[i]);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, s));
  for (int i = o + lane; i < e; i += 32) dz[i] = t;
}

__global__ void __launch_bounds__(QS_THREADS) k_ruiz_update(int n, const double* norm, double* scale) {
  QS_BATCH(norm, scale);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double t = norm[i];
    if (t > 0.0) scale[i] *= 1.0 / sqrt(t);
  }
}

__global__ void __launch_bounds__(QS_THREADS) k_scale_csr(Csr M, double* val, const double* rs, const double* cs) {
  QS_BATCH(M, val, rs, cs);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int row = warp; row < M.rows; row += (gridDim.x * blockDim.x) >> 5) {
    const double r = rs[row];
    for (int p = M.ptr[row] + lane; p < M.ptr[row + 1]; p += 32) val[p] *= r * cs[M.idx[p]];
  }
}

// entries of K with row < n (the P, A', G' blocks); the scaling block is untouched
__global__ void __launch_bounds__(QS_THREADS)
    k_scale_kkt(int n, int p, int m, const i64* Kp, const int* Ki, double* Kx, const double* D, const double* E,
                const double* F) {
  QS_BATCH(Kp, Ki, Kx, D, E, F);
  const int N = n + p + m;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int col = warp; col < N; col += (gridDim.x * blockDim.x) >> 5) {
    const double cs = col < n ? D[col] : (col < n + p ? E[col - n] : F[col - n - p]);
    for (i64 q = Kp[col] + lane; q < Kp[col + 1]; q += 32) {
      const int row = Ki[q];
      if (row < n) Kx[q] *= cs * D[row];
    }
  }
}

__global__ void __launch_bounds__(QS_THREADS) k_vec_scale(int n, double* v, const double* s, int divide) {
  QS_BATCH(v, s);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[i] = divide ? v[i] / s[i] : v[i] * s[i];
}

int vg(i64 n) {
  i64 g = (n + QS_THREADS - 1) / QS_THREADS;
  if (g < 1) g = 1;
  return (int)(g > 148 * 16 ? 148 * 16 : g);
}

}  // namespace

void qsk_ruiz(const RuizArgs& A, int iters, double* work_x, double* work_y, double* work_z, cudaStream_t st) {
  const i64 N = (i64)A.n + A.p + A.m;
  for (int it = 0; it < iters; ++it) {
    k_ruiz_norms<<<qs_grid(vg(N)), QS_THREADS, 0, st>>>(A, work_x, work_y, work_z);
    if (A.nsoc > 0)
      k_ruiz_cone_max<<<qs_grid((A.nsoc * 32 + QS_THREADS - 1) / QS_THREADS), QS_THREADS, 0, st>>>(A.nsoc, A.soc_ptr, work_z);
    k_ruiz_update<<<qs_grid(vg(A.n)), QS_THREADS, 0, st>>>(A.n, work_x, A.D);
    if (A.p > 0) k_ruiz_update<<<qs_grid(vg(A.p)), QS_THREADS, 0, st>>>(A.p, work_y, A.E);
    k_ruiz_update<<<qs_grid(vg(A.m)), QS_THREADS, 0, st>>>(A.m, work_z, A.F);
  }
}

void qsk_ruiz_apply(const RuizArgs& A, const i64* Kp, const int* Ki, double* Kx, double* c, double* b, double* h,
                    cudaStream_t st) {
  auto sc = [&](const Csr& M, const double* rs, const double* cs) {
    if (M.rows > 0) k_scale_csr<<<qs_grid(vg((i64)M.rows * 32)), QS_THREADS, 0, st>>>(M, const_cast<double*>(M.val), rs, cs);
  };
  sc(A.Pf, A.D, A.D);
  sc(A.At, A.D, A.E);
  sc(A.Gt, A.D, A.F);
  sc(A.Ar, A.E, A.D);
  sc(A.Gr, A.F, A.D);
  k_scale_kkt<<<qs_grid(vg(((i64)A.n + A.p + A.m) * 32)), QS_THREADS, 0, st>>>(A.n, A.p, A.m, Kp, Ki, Kx, A.D, A.E, A.F);
  qsk_vec_scale(A.n, c, A.D, 0, st);
  qsk_vec_scale(A.p, b, A.E, 0, st);
  qsk_vec_scale(A.m, h, A.F, 0, st);
}

void qsk_vec_scale(int n, double* v, const double* s, int divide, cudaStream_t st) {
  if (n > 0) k_vec_scale<<<qs_grid(vg(n)), QS_THREADS, 0, st>>>(n, v, s, divide);
}
