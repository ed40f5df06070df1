// KKT scaling-block update: generate the -W'W slot values and write them into
// the KKT value array (reference: write_scaling kkt.py:146-150, neg_wtw_values
// cones.py:319-336, soc_neg_wtw _cone_kernels.py:165-186).
//
// The reference materialises `slots` and scatters through an int64 index map.
// Here the values are generated and stored in one pass; nothing of size S is
// ever read except (in MAP mode) the map itself:
//   SLOTS  out[slot]                      -- dense slot array (parity checks)
//   MAP    out[positions[slot]]           -- the reference's explicit map
//   DIRECT out[colend(col) - (j+1) + i]   -- closed form of the same map: in a
//          conic column the block rows sort after every G' row, so the block
//          entries are the last j+1 entries of column n+p+o+j.  Validated
//          against the explicit map at setup (qsk_check_direct_map).
//
// Work decomposition: global conic columns [l, m) are cut at setup into tiles
// of ~TILE entries (tile_ptr); one CTA per tile, one warp per column, lanes
// over the rows i <= j, so every warp store is a contiguous run of doubles.
// w_bar re-reads hit L1/L2 (each element is used by q/2 columns on average).
#include "kkt_kernels.h"

namespace {

enum { MODE_SLOTS = 0, MODE_MAP = 1, MODE_DIRECT = 2 };

// per-cone c = sum wbar^2 (all entries, head included) and eta^2
__global__ void __launch_bounds__(QS_THREADS) k_wtw_prepass(int nsoc, const int* soc_ptr, const double* wbar,
                                                            const double* eta, double* c4, double* e2) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nsoc) return;
  const int o = soc_ptr[warp], q = soc_ptr[warp + 1] - o;
  double acc = 0.0;
  for (int t = lane; t < q; t += 32) {
    const double v = wbar[o + t];
    acc += v * v;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) {
    c4[warp] = 4.0 * acc;
    e2[warp] = eta[warp] * eta[warp];
  }
}

// Per-column constants staged once per tile.  With A = -eta^2 (4c+4) w_j every
// tail-tail entry is A*w_i; row 0 uses A0 = -eta^2 4c w_j, the (0,0) entry
// -eta^2((4c-4) w_0^2 + 1), the diagonal adds -eta^2.  Algebraically identical
// to _cone_kernels.py:176-185 (the +-2 w_i w_j terms cancel or double); it
// differs from the reference's expression by rounding only (<= a few ulp).
struct ColMeta {
  double A, A0, ne2;
  i64 base;  // destination of row 0 of this column
  int j;     // local column index inside its cone
  int woff;  // offset of the cone's wbar inside the staged window
};

template <int MODE>
__global__ void __launch_bounds__(QS_THREADS)
    k_neg_wtw(int l, int nb_orth, int max_cols, int wcap, const double* __restrict__ w,
              const double* __restrict__ wbar, const int* __restrict__ soc_ptr, const int* __restrict__ cone_of_col,
              const int* __restrict__ tile_ptr, const double* __restrict__ c4, const double* __restrict__ e2,
              const i64* __restrict__ slot_start, const i64* __restrict__ positions,
              const i64* __restrict__ kp_conic, double* __restrict__ out) {
  if ((int)blockIdx.x < nb_orth) {
    // orthant diagonal: slot i holds -(w_i^2)                    (cones.py:324-326)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < l; i += nb_orth * blockDim.x) {
      const double v = -(w[i] * w[i]);
      if (MODE == MODE_SLOTS) out[i] = v;
      if (MODE == MODE_MAP) out[positions[i]] = v;
      if (MODE == MODE_DIRECT) out[kp_conic[i] - 1] = v;
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ColMeta* meta = reinterpret_cast<ColMeta*>(smem_raw);
  double* wst = reinterpret_cast<double*>(smem_raw + (size_t)max_cols * sizeof(ColMeta));
  const int tile = blockIdx.x - nb_orth;
  const int col0 = tile_ptr[tile], col1 = tile_ptr[tile + 1];
  const int ncols = col1 - col0;
  // window of wbar covering every cone touched by the tile: [wlo, col1)
  const int wlo = soc_ptr[cone_of_col[col0 - l]];
  const int wlen = col1 - wlo;
  const bool staged = wlen <= wcap;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    const int col = col0 + c;
    const int k = cone_of_col[col - l];
    const int o = soc_ptr[k];
    const int j = col - o;
    const double cc = c4[k], ne2 = -e2[k], wj = wbar[col];
    ColMeta m;
    m.ne2 = ne2;
    m.j = j;
    m.woff = o - wlo;
    if (j == 0) {
      m.A = 0.0;
      m.A0 = ne2 * ((cc - 4.0) * wj);  // times w_0 below, then the diagonal term
    } else {
      m.A = ne2 * ((cc + 4.0) * wj);
      m.A0 = ne2 * (cc * wj);
    }
    m.base = (MODE == MODE_DIRECT) ? kp_conic[col] - (j + 1) : slot_start[k] + (i64)j * (j + 1) / 2;
    meta[c] = m;
  }
  if (staged)
    for (int t = threadIdx.x; t < wlen; t += blockDim.x) wst[t] = wbar[wlo + t];
  __syncthreads();
  // streaming phase: a warp owns a contiguous chunk of the tile's columns; the
  // interior of a column (0 < i < j) is a pure multiply-store stream, the two
  // special entries (row 0, diagonal) are written by one lane each.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int per = (ncols + nwarp - 1) / nwarp;
  const int cbeg = warp * per, cend = min(ncols, cbeg + per);
  for (int c = cbeg; c < cend; ++c) {
    const double A = meta[c].A;
    const int j = meta[c].j;
    const i64 base = meta[c].base;
    const double* wc = (staged ? wst : wbar + wlo) + meta[c].woff;
    if (MODE == MODE_MAP) {
      const i64* pmap = positions + base;
#pragma unroll 2
      for (int i = 1 + lane; i < j; i += 32) out[pmap[i]] = A * wc[i];
      if (lane == 0) {
        const double v0 = meta[c].A0 * wc[0];
        out[pmap[0]] = (j == 0) ? v0 + meta[c].ne2 : v0;
      } else if (lane == 1 && j > 0) {
        out[pmap[j]] = A * wc[j] + meta[c].ne2;
      }
    } else {
      double* dst = out + base;
#pragma unroll 2
      for (int i = 1 + lane; i < j; i += 32) dst[i] = A * wc[i];
      if (lane == 0) {
        const double v0 = meta[c].A0 * wc[0];
        dst[0] = (j == 0) ? v0 + meta[c].ne2 : v0;
      } else if (lane == 1 && j > 0) {
        dst[j] = A * wc[j] + meta[c].ne2;
      }
    }
  }
}

// positions[slot] == closed form for every slot?  flag[0] set to 1 otherwise.
__global__ void __launch_bounds__(QS_THREADS)
    k_check_direct(int l, int nb_orth, const int* soc_ptr, const int* cone_of_col, const int* tile_ptr,
                   const i64* slot_start, const i64* positions, const i64* kp_conic, int* flag) {
  int bad = 0;
  if ((int)blockIdx.x < nb_orth) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < l; i += nb_orth * blockDim.x)
      if (positions[i] != kp_conic[i] - 1) bad = 1;
  } else {
    const int tile = blockIdx.x - nb_orth;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    for (int col = tile_ptr[tile] + warp; col < tile_ptr[tile + 1]; col += nwarp) {
      const int k = cone_of_col[col - l];
      const int j = col - soc_ptr[k];
      const i64 sb = slot_start[k] + (i64)j * (j + 1) / 2, pb = kp_conic[col] - (j + 1);
      for (int i = lane; i <= j; i += 32)
        if (positions[sb + i] != pb + i) bad = 1;
    }
  }
  if (bad) *flag = 1;
}

int orth_blocks(int l) {
  if (l <= 0) return 0;
  int nb = (l + QS_THREADS - 1) / QS_THREADS;
  return nb > 148 * 4 ? 148 * 4 : nb;
}

}  // namespace

void qsk_neg_wtw(const WtwPlan& P, int mode, const double* w, const double* eta, const double* wbar,
                 const i64* positions, double* out, cudaStream_t st) {
  if (P.nsoc > 0)
    k_wtw_prepass<<<(P.nsoc * 32 + QS_THREADS - 1) / QS_THREADS, QS_THREADS, 0, st>>>(P.nsoc, P.soc_ptr, wbar, eta,
                                                                                        P.c4, P.e2);
  const int nb_orth = orth_blocks(P.l);
  const int grid = nb_orth + P.ntiles;
  if (grid == 0) return;
  const int wcap = P.max_tile_window < QS_WTW_WCAP ? P.max_tile_window : QS_WTW_WCAP;
  const size_t smem = (size_t)P.max_tile_cols * sizeof(ColMeta) + (size_t)wcap * sizeof(double);
  static bool attr_set[3] = {false, false, false};
  auto launch = [&](auto kern, int idx, const i64* pos, const i64* kpc) {
    if (smem > 48 * 1024 && !attr_set[idx]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr_set[idx] = true;
    }
    kern<<<grid, QS_THREADS, smem, st>>>(P.l, nb_orth, P.max_tile_cols, wcap, w, wbar, P.soc_ptr, P.cone_of_col,
                                         P.tile_ptr, P.c4, P.e2, P.slot_start, pos, kpc, out);
  };
  if (mode == MODE_SLOTS)
    launch(k_neg_wtw<MODE_SLOTS>, 0, nullptr, nullptr);
  else if (mode == MODE_MAP)
    launch(k_neg_wtw<MODE_MAP>, 1, positions, nullptr);
  else
    launch(k_neg_wtw<MODE_DIRECT>, 2, nullptr, P.kp_conic);
}

void qsk_check_direct_map(const WtwPlan& P, const i64* positions, int* flag, cudaStream_t st) {
  const int nb_orth = orth_blocks(P.l);
  const int grid = nb_orth + P.ntiles;
  if (grid == 0) return;
  k_check_direct<<<grid, QS_THREADS, 0, st>>>(P.l, nb_orth, P.soc_ptr, P.cone_of_col, P.tile_ptr, P.slot_start,
                                              positions, P.kp_conic, flag);
}
