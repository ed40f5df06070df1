// Sparse gather products, fused residuals and small vector kernels (spmv_kernels.cu).
#pragma once
#include "common.cuh"

struct Csr {
  int rows, cols;
  const int* ptr;  // [rows+1]
  const int* idx;
  const double* val;
  int tpr;  // lanes per row (power of two, 1..32)
  int exact1;  // every row holds exactly one entry (ptr[r] == r): the thread-per-row products skip the row pointers
  __device__ void shift(size_t off) {
    qs_shift(off, ptr);
    qs_shift(off, idx);
    qs_shift(off, val);
  }
};

// compute_residuals (ipm.py:70-103): writes rhs[0:n] = -r_dual, rhs[n:n+p] = -r_eq,
// r_cone, and every scalar check_termination (ipm.py:106-119) needs.
// Dual range in ONE pass: Dt = [Pf | A' | G'] row by row (n rows), each index tagged in its top two bits with the block
// it came from (0: P, operand x; 1: A', operand y; 2: G', operand z).  One row pointer pair and one entry stream per
// row instead of three: the dependent chain row pointer -> entry -> operand is paid once.  Built at setup when the
// dual range runs thread-per-row (short rows); ptr == nullptr otherwise.
// Long rows (mean >= 512 entries: the sample rows of a design matrix) are cut into QS_ROW_SEGS segments, a warp per
// segment with eight loads in flight per lane and no barrier; a second, tiny pass adds the partials of a row in
// fixed order.  (A CTA per row spent a third of its stall cycles at its two barriers: ncu r02e.)
#define QS_ROW_SEGS 8
#define QS_DT_TAG_SHIFT 30
#define QS_DT_COL_MASK 0x3fffffff

struct ResidualArgs {
  int n, p, m;
  Csr Pf, At, Gt, Ar, Gr;  // Pf.tpr is used for the whole dual range
  Csr Dt;
  double* seg_partial;  // [p * QS_ROW_SEGS] scratch of the split long-row product of the equality range, or null
  const double *x, *y, *z, *s, *c, *b, *h;
  double* rhs;
  double* r_cone;
  double* scalars;
  GridRed gr;
  __device__ void shift(size_t off) {
    Pf.shift(off), At.shift(off), Gt.shift(off), Ar.shift(off), Gr.shift(off), Dt.shift(off), gr.shift(off);
    qs_shift(off, x), qs_shift(off, y), qs_shift(off, z), qs_shift(off, s), qs_shift(off, c), qs_shift(off, b);
    qs_shift(off, h), qs_shift(off, rhs), qs_shift(off, r_cone), qs_shift(off, scalars), qs_shift(off, seg_partial);
  }
};

struct KktResidualArgs {
  int n, p, m;
  Csr Pf, At, Gt, Ar, Gr;
  Csr Dt;
  double* seg_partial;  // as in ResidualArgs, or null
  const double* v;     // [n+p+m] candidate solution
  const double* rhs;   // [n+p+m]
  const double* w2vz;  // [m]  W'W v_z
  double* r;           // [n+p+m] out
  double* scalars;
  int slot;            // scalars[slot] = ||r||_inf
  GridRed gr;
  __device__ void shift(size_t off) {
    Pf.shift(off), At.shift(off), Gt.shift(off), Ar.shift(off), Gr.shift(off), Dt.shift(off), gr.shift(off);
    qs_shift(off, v), qs_shift(off, rhs), qs_shift(off, w2vz), qs_shift(off, r), qs_shift(off, scalars);
    qs_shift(off, seg_partial);
  }
};

int qsk_pick_tpr(i64 nnz, i64 rows);
int qsk_residuals(const ResidualArgs& A, cudaStream_t st);  // returns the number of kernels launched (2 or 3)
void qsk_kkt_residual(const KktResidualArgs& A, cudaStream_t st);
void qsk_spmv_csr(const Csr& M, const double* x, double* y, int accumulate, cudaStream_t st);
void qsk_spmv_sym_upper_csc(int ncols, const i64* cp, const int* ri, const double* vx, const double* x, double* out,
                            cudaStream_t st);
void qsk_gather(i64 n, const double* src, const int* map, double* dst, cudaStream_t st);  // dst[i] = src[map[i]]
// dst[i] = src_t[map[i] & QS_DT_COL_MASK] with t = map[i] >> QS_DT_TAG_SHIFT (values of the fused dual-range matrix)
void qsk_gather3(i64 n, const double* src0, const double* src1, const double* src2, const int* map, double* dst,
                 cudaStream_t st);
void qsk_axpby(i64 n, double a, const double* x, double b, const double* y, double* out, cudaStream_t st);
void qsk_absmax(i64 n, const double* x, double* out, double* nonfinite, GridRed gr, cudaStream_t st);
// batched mode (common.cuh): per-instance conditional copy; replication of slot 0's words into the other slots
void qsk_copy_if(i64 n, const double* flag, const double* src, double* dst, cudaStream_t st);
void qsk_broadcast(i64 nwords, void* p, int slots, cudaStream_t st);
// Dt = [Pf | At | Gt] with tagged indices, plus the value map for qsk_gather3 (all arrays preallocated)
void qsk_build_dt(int n, const Csr& Pf, const Csr& At, const Csr& Gt, int* dp, int* di, double* dv, int* dmap,
                  cudaStream_t st);
