// Ruiz equilibration kernels (ruiz_kernels.cu).
#pragma once
#include "spmv_kernels.h"

struct RuizArgs {
  int n, p, m, nsoc;
  const int* soc_ptr;
  Csr Pf, At, Gt, Ar, Gr;
  double *D, *E, *F;  // [n], [p], [m]; start at 1
  __device__ void shift(size_t off) {
    qs_shift(off, soc_ptr);
    qs_shift(off, Pf);
    qs_shift(off, At);
    qs_shift(off, Gt);
    qs_shift(off, Ar);
    qs_shift(off, Gr);
    qs_shift(off, D);
    qs_shift(off, E);
    qs_shift(off, F);
  }
};

void qsk_ruiz(const RuizArgs& A, int iters, double* work_x, double* work_y, double* work_z, cudaStream_t st);
void qsk_ruiz_apply(const RuizArgs& A, const i64* Kp, const int* Ki, double* Kx, double* c, double* b, double* h,
                    cudaStream_t st);
void qsk_vec_scale(int n, double* v, const double* s, int divide, cudaStream_t st);
