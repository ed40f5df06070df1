// Host-callable launchers of the cone-algebra kernels (cone_kernels.cu).
// Every pointer is a device pointer; launches are asynchronous on `st`.
#pragma once
#include "common.cuh"

void qsk_nt_scaling(const ConeLayout& L, const double* s, const double* z, double* w, double* eta, double* wbar,
                    double* lam, double* lam_sq, double* scalars, cudaStream_t st);
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
void qsk_dcomp(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* ds_a,
               const double* wdz_a, const double* lam_sq, double* dcomp, const double* scalars, cudaStream_t st);
void qsk_rhs_cone(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* lam,
                  const double* dc, double sign, const double* r_cone, double* d, double* rhs_z, cudaStream_t st);
void qsk_post_solve(const ConeLayout& L, const double* w, const double* eta, const double* wbar, const double* d,
                    const double* dz, const double* s, const double* z, double* wdz, double* ds, double* scalars,
                    int corrector, double step_fraction, GridRed gr, cudaStream_t st);
void qsk_mu_aff(int m, const double* s, const double* z, const double* ds, const double* dz, double deg,
                double* scalars, GridRed gr, cudaStream_t st);
void qsk_update_iterate(int n, int p, int m, const double* x, const double* y, const double* z, const double* s,
                        double* xo, double* yo, double* zo, double* so, const double* sol, const double* ds, double deg,
                        double* scalars, GridRed gr, cudaStream_t st);
void qsk_dot(int m, const double* a, const double* b, double scale, double* out, GridRed gr, cudaStream_t st);
