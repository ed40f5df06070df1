/*
 * qsocp_cuda.h -- C ABI of libqsocp_cuda.so, the B200 (sm_100a) implementation
 * of the per-iteration hot path of the qsocp interior-point solver.
 *
 * The reference (pure Python + numba, /root/reference/pkg/src/qsocp) has no
 * FFI of its own; each entry point below names the reference function whose
 * role it takes (file:line relative to pkg/src/qsocp/).  A binding a
 * maintainer would add to the reference is shown in INTEGRATION.md.
 *
 * Conventions
 *   - plain C types only: int64_t / double / int pointers and sizes;
 *   - every function returns 0 on success or a QS_E_* code; the text of the
 *     last error of a handle is qs_last_error(h);
 *   - "host" pointers are caller-owned host memory, copied during the call;
 *     "dev" pointers are device memory on the handle's device (e.g. a torch
 *     tensor's data_ptr());
 *   - a handle owns one CUDA stream and all device state of one solver
 *     instance; a handle is single-threaded, distinct handles are independent;
 *   - all vectors are fp64, all host-visible indices int64, exactly as in the
 *     reference (sparse.py:18-19).
 */
#ifndef QSOCP_CUDA_H
#define QSOCP_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qs_handle qs_handle;

enum {
  QS_OK = 0,
  QS_E_INVALID = 1,      /* bad argument / call order            (ValueError, RuntimeError)  */
  QS_E_CUDA = 2,         /* CUDA runtime error                                                */
  QS_E_NOT_INTERIOR = 3, /* cones.py:169-170,182-183,297-299     (errors.NotInterior)         */
  QS_E_NUMERICAL = 4,    /* non-finite residual / iterate / pivot (errors.NumericalError)     */
  QS_E_MEMORY = 5,       /* out of device memory                                              */
  QS_E_DIMENSION = 6     /* sizes disagree                        (errors.DimensionMismatch)  */
};

/* problem.py:59-67 */
typedef struct qs_settings {
  double eps_abs, eps_rel;
  int64_t max_iters;
  double static_reg;
  int64_t refine_iters;
  double step_fraction;
  double time_limit_seconds;
  int64_t ruiz_iters;     /* 0 = off (reference behaviour) */
  int64_t ordering;       /* 0 natural, 1 AMD, 2 user permutation */
  int64_t kkt_literal;    /* 1: refine against the stored K entries (ldl.py:152) instead of the operator form */
} qs_settings;

/* scalars returned by qs_residuals: everything check_termination (ipm.py:106-119) reads */
typedef struct qs_residual_info {
  double norm_r_dual, norm_r_eq, norm_r_cone, gap, objective;
  double norm_Px, norm_Aty, norm_Gtz, norm_c, norm_Ax, norm_b, norm_Gx, norm_h, norm_s;
  double mu;
  int64_t flags; /* bit0 not interior, bit1 non-finite, bit2 bad step, bit3 pivot non-finite */
} qs_residual_info;

/* StepInfo (ipm.py:58-63) + what the driver needs after a step */
typedef struct qs_step_info {
  double alpha, alpha_affine, sigma, mu_affine, mu;
  double step_s, step_z;
  int64_t flags;
} qs_step_info;

/* ---- library / device ---------------------------------------------------- */
int qs_version(void);
int qs_device_count(void);
const char* qs_global_error(void);

/* ---- handle -------------------------------------------------------------- */
qs_handle* qs_create(int device);
void qs_destroy(qs_handle* h);
const char* qs_last_error(qs_handle* h);
/* run the handle's work on an existing stream (e.g. torch's current stream) */
int qs_set_stream(qs_handle* h, void* cuda_stream);
int qs_sync(qs_handle* h);
/* page-lock / release caller-owned host memory (a mapped problem file, fileio.py of this package; the reference
 * reads its text format into fresh arrays, fileio.py:120-122) so that qs_setup's copies are not staged */
int qs_host_register(const void* ptr, int64_t bytes);
int qs_host_unregister(const void* ptr);

/* ---- host-side structure (no GPU needed) ---------------------------------
 * assemble_kkt (kkt.py:55-135): pattern, values with the scaling block at -I,
 * slot -> position map, per-view slot offsets, per-SOC slot starts.          */
int64_t qs_kkt_nnz(int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q, const int64_t* Pp,
                   const int64_t* Pi, int64_t nnzA, int64_t nnzG);
int64_t qs_kkt_slot_count(int64_t l, int64_t nsoc, const int64_t* q);
int qs_kkt_assemble(int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q, const int64_t* Pp,
                    const int64_t* Pi, const double* Px, const int64_t* Ap, const int64_t* Ai, const double* Ax,
                    const int64_t* Gp, const int64_t* Gi, const double* Gx, int64_t* Kp, int64_t* Ki, double* Kx,
                    int64_t* nt_entry_positions, int64_t* nt_slot_offsets, int64_t* soc_slot_starts);
/* fill-reducing order + supernodal analysis of an upper-CSC pattern (host);
 * out_perm[new] = old; stats = {nsup, nlevels, lnz, flops, max_front_rows, max_front_cols} */
int qs_symbolic_stats(int64_t N, const int64_t* Kp, const int64_t* Ki, int64_t ordering, const int64_t* user_perm,
                      int64_t ncliques, const int64_t* clique_start, const int64_t* clique_size, int64_t* out_perm,
                      double* stats6);

/* ---- cone layout (cones.py:40-58) ----------------------------------------
 * big_threshold: SOCs larger than this use the block-per-cone path (<=0: default). */
int qs_set_cones(qs_handle* h, int64_t l, int64_t nsoc, const int64_t* q_host, int64_t big_threshold);

/* The fused per-iteration kernels of qs_step on caller-owned DEVICE vectors (vector-level parity against the
 * reference's ipm_step intermediates, pkg/src/qsocp/ipm.py:180-234).  Need qs_set_cones.
 * qs_predictor_rhs: compute_nt_scaling + lam o lam (cones.py:159-184, ipm.py:191), d = lam \ (-lam o lam) and the
 *   third RHS block rhs_z = -r_cone - W d (ipm.py:180-184).
 * qs_corrector_rhs: d_comp = sigma mu e - lam o lam - (W^-1 ds_a) o (W dz_a) (ipm.py:209-211), d, rhs_z as above.
 * qs_post_solve: wdz = W dz, ds = W (d - W dz) (ipm.py:187-188), max_step_to_boundary for (s, ds), (z, dz) with
 *   check_interior (cones.py:247-299); corrector = 0 also alpha_aff, mu_aff, mu, sigma (ipm.py:195-206), corrector = 1
 *   alpha (ipm.py:214-218).  out8 = {step_s, step_z, alpha_aff, alpha, mu, mu_aff, sigma, flags}.
 * qs_update_iterate: the new iterate, finite check, new mu (ipm.py:219-234); sol = (dx, dy, dz).  out2 = {mu, flags}. */
int qs_predictor_rhs(qs_handle* h, const double* s, const double* z, const double* r_cone, double* w, double* eta,
                     double* wbar, double* lam, double* lam_sq, double* d, double* rhs_z, int* not_interior_host);
int qs_corrector_rhs(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* lam,
                     const double* lam_sq, const double* ds_a, const double* wdz_a, const double* r_cone, double sigma,
                     double mu, double* dcomp, double* d, double* rhs_z);
int qs_post_solve(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* d,
                  const double* dz, const double* s, const double* z, int corrector, double step_fraction, double* wdz,
                  double* ds, double* out8_host);
int qs_update_iterate(qs_handle* h, int64_t n, int64_t p, const double* x, const double* y, const double* z,
                      const double* s, const double* sol, const double* ds, double alpha, double* xo, double* yo,
                      double* zo, double* so, double* out2_host);

/* ---- per-kernel entry points (dev pointers; unit parity tests, ncu) ------ */
/* compute_nt_scaling cones.py:159-184; lam_sq may be NULL.  flag_host != NULL forces a sync. */
int qs_nt_scaling(qs_handle* h, const double* s, const double* z, double* w, double* eta, double* wbar, double* lam,
                  double* lam_sq, int* not_interior_host);
/* apply_scaling cones.py:192-212 */
int qs_apply_w(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* u, double* out,
               int inverse);
/* jordan_product cones.py:215-228 / jordan_divide cones.py:231-244 */
int qs_jordan_product(qs_handle* h, const double* u, const double* v, double* out);
int qs_jordan_divide(qs_handle* h, const double* lam, const double* v, double* out);
/* max_step_to_boundary cones.py:247-272 (du may be NULL: violation only, cones.py:275-290) */
int qs_max_step(qs_handle* h, const double* u, const double* du, double* step_host, double* violation_host);
/* bring_to_interior cones.py:302-311: out = scale*u shifted by (1+alpha)e when alpha >= 0 */
int qs_bring_to_interior(qs_handle* h, const double* u, double scale, double* out, double* alpha_host);
/* compute_mu cones.py:314-316 */
int qs_compute_mu(qs_handle* h, const double* s, const double* z, double* mu_host);
/* neg_wtw_values cones.py:319-336 (mode 0: dense slots) and write_scaling
 * kkt.py:146-150 (mode 1: through positions[S]; mode 2: closed-form positions,
 * needs kp_conic[m] = K.col_pointers[n+p+1 ...]).                            */
int qs_neg_wtw(qs_handle* h, int mode, const double* w, const double* eta, const double* wbar,
               const int64_t* soc_slot_starts_dev, const int64_t* positions_dev, const int64_t* kp_conic_dev,
               double* out);
/* spmv sparse.py:119-140 on a CSR view (gather): y = M x (+ y when accumulate) */
int qs_spmv_csr(qs_handle* h, int64_t rows, int64_t cols, const int32_t* ptr, const int32_t* idx, const double* val,
                const double* x, double* y, int accumulate);
/* spmv_sym_upper sparse.py:143-150: out += sym(M) x, M = upper CSC */
int qs_spmv_sym_upper(qs_handle* h, int64_t ncols, const int64_t* colptr, const int32_t* rowidx, const double* val,
                      const double* x, double* out);

/* ---- solver instance -------------------------------------------------------
 * qs_setup takes the problem exactly as the reference's ProblemData holds it
 * (problem.py:31-49: CSC int64/fp64, P upper triangle) plus the cone sizes;
 * it assembles the KKT system, builds the row views, copies everything to the
 * device and analyses the factorisation (ipm.py:251-256).  user_perm may be
 * NULL.                                                                       */
int qs_setup(qs_handle* h, int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q,
             const int64_t* Pp, const int64_t* Pi, const double* Px, const int64_t* Ap, const int64_t* Ai,
             const double* Ax, const int64_t* Gp, const int64_t* Gi, const double* Gx, const double* c,
             const double* b, const double* hvec, const qs_settings* settings, const int64_t* user_perm);
/* KKT system of the instance (host copies out; any pointer may be NULL) */
int64_t qs_kkt_size(qs_handle* h, int64_t* nnz, int64_t* slots);
int qs_get_kkt(qs_handle* h, int64_t* Kp, int64_t* Ki, double* Kx, int64_t* positions);
/* LinsysBackend contract (linsys.py:24-51) on the device-resident system */
int qs_linsys_update_identity(qs_handle* h);                 /* update(identity_scaling), ipm.py:142 */
int qs_linsys_update(qs_handle* h);                          /* update(current NT scaling), ipm.py:177 */
int qs_linsys_factor(qs_handle* h);                          /* factor(), ipm.py:178 */
int qs_linsys_solve(qs_handle* h, const double* rhs_host, double* sol_host); /* solve(rhs) with refinement, ldl.py:135-166 */
/* IPM phases (ipm.py:135-156, 70-103, 159-235) */
int qs_initialize_iterate(qs_handle* h, double* mu_host);
int qs_residuals(qs_handle* h, qs_residual_info* out);
int qs_step(qs_handle* h, qs_step_info* out);
int qs_get_iterate(qs_handle* h, double* x, double* y, double* z, double* s);
/* Ruiz scalings D[n], E[p], F[m] (only when settings.ruiz_iters > 0; not a reference feature) */
int qs_get_ruiz(qs_handle* h, double* D, double* E, double* F);
int qs_set_iterate(qs_handle* h, const double* x, const double* y, const double* z, const double* s);
int qs_get_scaling(qs_handle* h, double* w, double* eta, double* wbar, double* lam);
/* load an NTScalingSet (cones.py:120-143) computed elsewhere; used by LinsysBackend.update(scaling) */
int qs_set_scaling(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* lam);
/* counters (linsys.py:30-31) and device timers in seconds:
 * timers = {cone, kkt_update, residual, factor, solve, refine_spmv, analysis, h2d}; launches of own kernels so far */
int qs_get_counters(qs_handle* h, int64_t* n_factor, int64_t* n_solve, int64_t* n_launches);
/* Pattern reuse (no reference counterpart -- SPEC.md lists parametric updates as a non-goal): new
 * VALUES for P (upper CSC order), A, G (CSC order) and/or c, b, h with the sparsity pattern given to qs_setup.  Null =
 * unchanged.  Ordering, symbolic analysis, index maps and launch graphs are kept; the next solve starts from
 * qs_initialize_iterate. */
int qs_update_values(qs_handle* h, const double* Px, const double* Ax, const double* Gx, const double* c,
                     const double* b, const double* hvec);
int qs_get_timers(qs_handle* h, double* timers8);
/* bytes copied host -> device (problem data, KKT column pointers, analysis structures) and device -> host (scalar
 * blocks per phase, the final iterate) by this handle so far */
int qs_get_transfer_bytes(qs_handle* h, int64_t* h2d, int64_t* d2h);
/* factor / solve calls of the linear system replayed from a captured CUDA graph vs issued as direct launches
 * (capture is impossible on the legacy NULL stream and inside a foreign capture) */
int qs_get_graph_stats(qs_handle* h, int64_t* replays, int64_t* direct);
int qs_get_factor_stats(qs_handle* h, double* stats8);
/* time `reps` launches of one hot-path kernel on the current state (CUDA events on the handle's stream);
 * kernel ids in INTEGRATION.md.  Returns mean milliseconds per launch. */
int qs_time_kernel(qs_handle* h, int kernel_id, int reps, double* ms_host);
/* same, but the L2 is flushed (256 MiB rewritten) before every timed launch and each launch is bracketed by its own
 * pair of events: the cold-cache figure a kernel sees inside a solve */
int qs_time_kernel_cold(qs_handle* h, int kernel_id, int reps, double* ms_host);

/* ---- Batched small-problem mode (the reference's precedent is its thread-pool sweep over
 * independent instances, pkg/src/qsocp/bench/runner.py:107-117, pkg/tests/test_api.py:101-118).  `count` instances
 * with ONE sparsity pattern and cone layout are solved in lockstep on one GPU: every kernel launch carries all
 * instances (gridDim.z = count), the ordering / symbolic analysis / index maps / launch graphs exist once, and one
 * host synchronisation per phase serves the whole batch.  Each instance follows exactly the iteration of qs_step /
 * qs_residuals (same kernels), so its iterates are those of a stand-alone solve.  An instance (all device memory
 * of one handle) must fit a 32 MiB slot.  A qs_batch is single-threaded like a handle.
 *   qs_batch_setup       same arguments as qs_setup: the pattern and the numbers of instance 0
 *   qs_batch_set_values  numbers of ALL instances, each array [count][len] row-major, or NULL (= as at setup)
 *   qs_batch_solve       status[count] (1 Solved, 2 MaxIters, 3 TimeLimit, 4 NumericalError, 5 NotInterior),
 *                        iterations[count], x [count][n], y [count][p], z [count][m], s [count][m]
 *   qs_batch_stats       out4 = {kernel launches, host synchronisations, seconds of the last solve, bytes per slot} */
typedef struct qs_batch qs_batch;
qs_batch* qs_batch_create(int device, int64_t count);
void qs_batch_destroy(qs_batch* bt);
const char* qs_batch_last_error(qs_batch* bt);
int qs_batch_setup(qs_batch* bt, int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q,
                   const int64_t* Pp, const int64_t* Pi, const double* Px, const int64_t* Ap, const int64_t* Ai,
                   const double* Ax, const int64_t* Gp, const int64_t* Gi, const double* Gx, const double* c,
                   const double* b, const double* h, const qs_settings* settings);
int qs_batch_set_values(qs_batch* bt, const double* Px, const double* Ax, const double* Gx, const double* c,
                        const double* b, const double* h);
int qs_batch_solve(qs_batch* bt, int64_t* status, int64_t* iterations, double* x, double* y, double* z, double* s);
int qs_batch_stats(qs_batch* bt, double* out4);

#ifdef __cplusplus
}
#endif
#endif /* QSOCP_CUDA_H */
