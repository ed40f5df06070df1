// Host-callable launchers of the cone-algebra kernels (cone_kernels.cu).
// Every pointer is a device pointer; launches are asynchronous on `st`.
#pragma once
#include "common.cuh"

// NT scaling + lam o lam (+ c4/e2: the per-cone constants of the -W'W generator; + when r_cone is given the
// predictor's d = lam \ (-lam o lam) and rhs_z = -r_cone - W d).  lam_sq, c4/e2, r_cone/d/rhs_z may be null.
void qsk_nt_scaling(const ConeLayout& L, const double* s, const double* z, double* w, double* eta, double* wbar,
                    double* lam, double* lam_sq, double* c4, double* e2, const double* r_cone, double* d,
                    double* rhs_z, double* scalars, cudaStream_t st);
void qsk_apply_w(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* u,
                 double* out, int inverse, cudaStream_t st);
void qsk_apply_w2(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* u,
                  double* out, cudaStream_t st);
void qsk_jordan_product(const ConeLayout& L, const double* u, const double* v, double* out, cudaStream_t st);
void qsk_jordan_divide(const ConeLayout& L, const double* lam, const double* v, double* out, cudaStream_t st);
void qsk_max_step(const ConeLayout& L, const double* u, const double* du, double* scalars, int slot_step,
                  int slot_viol, GridRed gr, cudaStream_t st);
void qsk_shift(const ConeLayout& L, const double* u, double* out, const double* scalars, int slot, double scale,
               cudaStream_t st);
// corrector: d_comp = sigma mu e - lam o lam - (W^-1 ds_a) o (W dz_a) (scalars[SC_SIGMA], scalars[SC_MU]),
// d = lam \ d_comp, rhs_z = -r_cone - W d.  dcomp may be null (not materialised).
void qsk_corrector_rhs(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* lam,
                       const double* lam_sq, const double* ds_a, const double* wdz_a, const double* r_cone,
                       double* dcomp, double* d, double* rhs_z, const double* scalars, cudaStream_t st);
// wdz = W dz, ds = W (d - wdz), both max steps + interior checks; predictor (corrector = 0) also alpha_aff, mu_aff,
// mu and sigma; corrector: alpha.  Results in scalars[].
void qsk_post_solve(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* d,
                    const double* dz, const double* s, const double* z, double* wdz, double* ds, double* scalars,
                    int corrector, double step_fraction, double deg, GridRed gr, cudaStream_t st);
void qsk_update_iterate(int n, int p, int m, const double* x, const double* y, const double* z, const double* s,
                        double* xo, double* yo, double* zo, double* so, const double* sol, const double* ds, double deg,
                        double* scalars, GridRed gr, cudaStream_t st);
void qsk_dot(int m, const double* a, const double* b, double scale, double* out, GridRed gr, cudaStream_t st);
