// -W'W generation + scatter into the KKT value array (kkt_kernels.cu).
#pragma once
#include "common.cuh"
#include "spmv_kernels.h"

#define QS_WTW_TILE 8192       // target block entries per CTA
#define QS_WTW_MAXCOLS 512     // at most this many columns per tile (metadata lives in shared memory)
#define QS_WTW_WCAP 16384      // wbar window staged in shared memory when it fits (doubles)
#define QS_WTW_STAGE 4096      // staged variant: output doubles per CTA (32 KiB of shared memory; 4 CTAs per SM)
#define QS_WTW_SCOLS 192       // staged variant: columns per CTA at most (their constants sit in shared memory too)
#define QS_WTW_SWIN 1024       // staged variant: wbar window staged in shared memory when it fits (doubles)

// Built once at setup (host side in capi.cu); all pointers are device pointers.
struct WtwPlan {
  int l, nsoc, m;
  const int* soc_ptr;      // [nsoc+1]
  const int* cone_of_col;  // [m-l]  cone index of conic column l + c
  int ntiles;
  const int* tile_ptr;     // [ntiles+1] global conic column ranges of ~QS_WTW_TILE entries
  int max_tile_cols;       // widest tile (columns)
  int max_tile_window;     // longest wbar window [first cone start, tile end) over the tiles
  const i64* slot_start;   // [nsoc]  the reference's soc_slot_starts (kkt.py:113-125)
  const i64* kp_conic;     // [m]  kp_conic[c] = K.col_pointers[n+p+c+1]  (DIRECT mode), may be null
  const int* g_ptr;        // [m+1] CSR row pointers of G, or null: DIRECT mode then also re-stores the G' entries
  const double* g_val;     //       of every conic K column so that the columns are written without holes
  // staged (bulk-store) variant: tiles whose contiguous output run fits QS_WTW_STAGE doubles
  const int* stile_ptr;         // [n_stiles_slots+1] tiling by packed-slot count (dense slot output), or null
  int n_stiles_slots;
  const int* stile_ptr_direct;  // [n_stiles_direct+1] tiling by whole-K-column length (needs kstart), or null
  int n_stiles_direct;
  const i64* kstart;            // K.col_pointers + n + p: kstart[c] .. kstart[c+1] is conic column c, or null
  double* c4;              // [nsoc] scratch: 4 * sum wbar^2
  double* e2;              // [nsoc] scratch: eta^2
};

// mode: 0 dense slots, 1 explicit int64 positions map, 2 closed-form positions
// have_consts: P.c4 / P.e2 already hold the constants of this scaling (written by qsk_nt_scaling)
void qsk_neg_wtw(const WtwPlan& P, int mode, const double* w, const double* eta, const double* wbar,
                 const i64* positions, double* out, cudaStream_t st, bool have_consts = false);
void qsk_check_direct_map(const WtwPlan& P, const i64* positions, int* flag, cudaStream_t st);

// KKT assembly on the device: row indices (int32), initial values and the slot -> position map of every column,
// given the column pointers Kp (device) and the row views Pu = CSC of P's upper triangle, Ar / Gr = CSR of A / G.
void qsk_kkt_fill(const WtwPlan& P, int n, int p, const Csr& Pu, const Csr& Ar, const Csr& Gr, const i64* Kp, int* Ki,
                  double* Kx, i64* pos, cudaStream_t st);
