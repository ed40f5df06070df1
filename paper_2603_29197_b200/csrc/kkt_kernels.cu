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
  QS_BATCH(soc_ptr, wbar, eta, c4, e2);
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

// Per-column constants, staged once per tile as structure-of-arrays in shared
// memory.  With A = -eta^2 (4c+4) w_j every tail-tail entry of column j is
// A * w_i; row 0 uses A0 = -eta^2 4c w_j, the (0,0) entry is
// -eta^2((4c-4) w_0^2 + 1), the diagonal adds -eta^2.  Algebraically identical
// to _cone_kernels.py:176-185 (the +-2 w_i w_j terms cancel or double); it
// differs from the reference's expression by rounding only (<= a few ulp).
//
// Streaming phase: HALF a warp per column (two adjacent columns per warp, whose
// lengths differ by one, so the two halves stay in step): the average column of
// the C4 layout has 68 entries, and 16-lane groups waste fewer lanes and halve
// the per-column instruction overhead per warp instruction.  Each 16-lane store
// is a contiguous 128-byte run.
template <int MODE, bool STAGED, bool BATCH>
__global__ void __launch_bounds__(QS_THREADS)
    k_neg_wtw(int l, int nb_orth, int max_cols, int wcap, const double* __restrict__ w,
              const double* __restrict__ wbar, const int* __restrict__ soc_ptr, const int* __restrict__ cone_of_col,
              const int* __restrict__ tile_ptr, const double* __restrict__ c4, const double* __restrict__ e2,
              const i64* __restrict__ slot_start, const i64* __restrict__ positions,
              const i64* __restrict__ kp_conic, const int* __restrict__ g_ptr, const double* __restrict__ g_val,
              double* __restrict__ out) {
  // moved pointers live in registers for the whole kernel (unmoved ones are read from the parameter bank at every
  // use): +8 registers = one CTA per SM less, 186 -> 209 us.  The single-instance launch uses BATCH = false.
  if (BATCH) {
    QS_BATCH(w, wbar, soc_ptr, cone_of_col, tile_ptr, c4, e2, slot_start, positions, kp_conic, g_ptr, g_val, out);
  }
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
  double* mA = reinterpret_cast<double*>(smem_raw);
  double* mA0 = mA + max_cols;
  double* mne2 = mA0 + max_cols;
  i64* mbase = reinterpret_cast<i64*>(mne2 + max_cols);
  int* mj = reinterpret_cast<int*>(mbase + max_cols);
  int* mwoff = mj + max_cols;
  int* mg0 = mwoff + max_cols;   // first entry of the column's row of G (DIRECT mode with whole columns)
  int* mng = mg0 + max_cols;     // its length
  double* mgv = reinterpret_cast<double*>(mng + max_cols);  // its first value (most rows of G hold one entry)
  double* wst = mgv + max_cols;  // 4 * max_cols ints: 8-byte aligned
  const int tile = blockIdx.x - nb_orth;
  const int col0 = tile_ptr[tile], col1 = tile_ptr[tile + 1];
  const int ncols = col1 - col0;
  // window of wbar covering every cone touched by the tile: [wlo, col1)
  const int wlo = soc_ptr[cone_of_col[col0 - l]];
  const int wlen = col1 - wlo;
  for (int c = threadIdx.x; c < ncols; c += QS_THREADS) {
    const int col = col0 + c;
    const int k = cone_of_col[col - l];
    const int o = soc_ptr[k];
    const int j = col - o;
    const double cc = c4[k], ne2 = -e2[k], wj = wbar[col];
    mne2[c] = ne2;
    mj[c] = j;
    mwoff[c] = o - wlo;
    mA[c] = (j == 0) ? 0.0 : ne2 * ((cc + 4.0) * wj);
    mA0[c] = (j == 0) ? ne2 * ((cc - 4.0) * wj) : ne2 * (cc * wj);
    mbase[c] = (MODE == MODE_DIRECT) ? kp_conic[col] - (j + 1) : slot_start[k] + (i64)j * (j + 1) / 2;
    if (MODE == MODE_DIRECT && g_ptr) {  // every load chain of the column runs here, in parallel over the columns:
      const int g0 = g_ptr[col], ng = g_ptr[col + 1] - g0;  // the streaming loop below waits on no global load
      mg0[c] = g0;
      mng[c] = ng;
      mgv[c] = ng > 0 ? g_val[g0] : 0.0;
    }
  }
  if (STAGED)
    for (int t = threadIdx.x; t < wlen; t += QS_THREADS) wst[t] = wbar[wlo + t];
  __syncthreads();
  constexpr int NW = QS_THREADS / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 4, sl = lane & 15;
  // Column pairs are dealt round-robin to the warps (the two halves of a warp take the two columns of a pair, whose
  // lengths differ by one, so they stay in step).  Column lengths grow along a cone, so contiguous chunks per warp
  // left the warps of the first chunks idle early: 197 -> 194 us.
  for (int c = 2 * warp + sub; c < ncols; c += 2 * NW) {
    const int j = mj[c];
    const double A = mA[c];
    const i64 base = mbase[c];
    const double* wc = STAGED ? wst + mwoff[c] : wbar + wlo + mwoff[c];
    if (MODE == MODE_MAP) {
      const i64* pmap = positions + base;
      for (int i = sl; i <= j; i += 16) out[pmap[i]] = A * wc[i];
      if (sl == 0) out[pmap[0]] = (j == 0) ? mA0[c] * wc[0] + mne2[c] : mA0[c] * wc[0];
      if (j > 0 && sl == (j & 15)) out[pmap[j]] = A * wc[j] + mne2[c];
    } else {
      double* dst = out + base;
      if (MODE == MODE_DIRECT && g_ptr) {
        // Re-store the G' entries that precede the block in this K column (values from the compact CSR
        // of G).  The column is then written in full, adjacent columns tile K.values without holes, and
        // no 32-byte sector is left partially written: measured, that is the difference between ~3.2 and
        // ~6 TB/s of store bandwidth (tests/probes/store_probe.cu).
        const int g0 = mg0[c], ng = mng[c];
        if (sl == 0 && ng > 0) dst[-ng] = mgv[c];
        for (int t = 1 + sl; t < ng; t += 16) dst[t - ng] = g_val[g0 + t];
      }
      // 64-bit stores, 16 lanes = one contiguous 128-byte run.  (A 128-bit variant -- aligned pairs, odd head
      // peeled -- halves the store instructions but measured 217 vs 213 us: the stall is back-pressure from the
      // memory system, not store issue.)
      for (int i = sl; i <= j; i += 16) dst[i] = A * wc[i];
      // the two special entries are rewritten by the lane that just wrote them
      if (sl == 0) dst[0] = (j == 0) ? mA0[c] * wc[0] + mne2[c] : mA0[c] * wc[0];
      if (j > 0 && sl == (j & 15)) dst[j] = A * wc[j] + mne2[c];
    }
  }
}


// ------------------------------------------------------------ staged variant
// Whole conic K columns are adjacent in K.values (a conic column is its G'
// entries followed by its block entries, and the next column starts where it
// ends), and so are the packed slots of adjacent SOC columns.  A tile of
// columns therefore owns ONE contiguous run of the output.  The CTA builds that
// run in shared memory (half-warp per column, as in the streaming kernel) and
// hands it to the TMA engine as 16-byte-aligned bulk stores
// (cp.async.bulk.global.shared::cta): HBM sees full, aligned lines only, the
// SM's LSU issues no global stores, and the next CTA of the SM computes while
// this one's stores drain.  An odd first/last element goes out as a scalar.
//   SLOTS : run = slot range of the tile's columns
//   DIRECT: run = [kstart[col0], kstart[col1]) with kstart = K.col_pointers + n + p
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE, bool BULK>
__global__ void __launch_bounds__(QS_THREADS)
    k_neg_wtw_staged(int l, int nb_orth, const double* __restrict__ w, const double* __restrict__ wbar,
                     const int* __restrict__ soc_ptr, const int* __restrict__ cone_of_col,
                     const int* __restrict__ tile_ptr, const double* __restrict__ c4, const double* __restrict__ e2,
                     const i64* __restrict__ slot_start, const i64* __restrict__ kstart,
                     const int* __restrict__ g_ptr, const double* __restrict__ g_val, double* __restrict__ out) {
  QS_BATCH(w, wbar, soc_ptr, cone_of_col, tile_ptr, c4, e2, slot_start, kstart, g_ptr, g_val, out);
  if ((int)blockIdx.x < nb_orth) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < l; i += nb_orth * blockDim.x) {
      const double v = -(w[i] * w[i]);
      if (MODE == MODE_SLOTS) out[i] = v;
      if (MODE == MODE_DIRECT) out[kstart[i + 1] - 1] = v;
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* buf = reinterpret_cast<double*>(smem_raw);          // [QS_WTW_STAGE + 4] the output run
  double* mA = buf + QS_WTW_STAGE + 4;                         // per-column constants, structure of arrays
  double* mA0 = mA + QS_WTW_SCOLS;
  double* mne2 = mA0 + QS_WTW_SCOLS;
  int* mj = reinterpret_cast<int*>(mne2 + QS_WTW_SCOLS);       // row count - 1 of the block part
  int* mdst = mj + QS_WTW_SCOLS;                               // offset of the column's first entry in buf
  int* mng = mdst + QS_WTW_SCOLS;                              // G' entries in front of the block part
  int* mo = mng + QS_WTW_SCOLS;                                // first wbar index of the column's cone
  int* mg0 = mo + QS_WTW_SCOLS;                                // first entry of G's CSR row
  double* wst = reinterpret_cast<double*>(mg0 + QS_WTW_SCOLS); // [QS_WTW_SWIN] wbar window of the tile's cones
  __shared__ i64 run[2];
  __shared__ int win[2];
  const int tile = blockIdx.x - nb_orth;
  const int col0 = tile_ptr[tile], col1 = tile_ptr[tile + 1];
  const int ncols = col1 - col0;
  if (threadIdx.x == 0) {
    if (MODE == MODE_DIRECT) {
      run[0] = kstart[col0];
      run[1] = kstart[col1];
    } else {
      const int ka = cone_of_col[col0 - l], kb = cone_of_col[col1 - 1 - l];
      const i64 ja = col0 - soc_ptr[ka], jb = col1 - 1 - soc_ptr[kb];
      run[0] = slot_start[ka] + ja * (ja + 1) / 2;
      run[1] = slot_start[kb] + (jb + 1) * (jb + 2) / 2;
    }
    win[0] = soc_ptr[cone_of_col[col0 - l]];  // column c of cone k reads wbar[soc_ptr[k] .. c]: window [win0, col1)
  }
  __syncthreads();
  const i64 r0 = run[0], r1 = run[1];
  const int wlo = win[0], wlen = col1 - wlo;
  const bool wstaged = wlen <= QS_WTW_SWIN;
  if (wstaged)
    for (int t = threadIdx.x; t < wlen; t += QS_THREADS) wst[t] = wbar[wlo + t];
  const int shift = (int)(r0 & 1);  // global even indices land on even (16-byte aligned) shared indices
  // phase 0: one thread per column gathers the column constants (all columns' load chains run in parallel)
  for (int c = threadIdx.x; c < ncols; c += QS_THREADS) {
    const int col = col0 + c;
    const int k = cone_of_col[col - l];
    const int o = soc_ptr[k];
    const int j = col - o;
    const double cc = c4[k], ne2 = -e2[k], wj = wbar[col];
    mne2[c] = ne2;
    mj[c] = j;
    mo[c] = o;
    mA[c] = (j == 0) ? 0.0 : ne2 * ((cc + 4.0) * wj);
    mA0[c] = (j == 0) ? ne2 * ((cc - 4.0) * wj) : ne2 * (cc * wj);
    if (MODE == MODE_DIRECT) {
      const i64 cs = kstart[col];
      mdst[c] = shift + (int)(cs - r0);
      mng[c] = (int)(kstart[col + 1] - cs) - (j + 1);
      mg0[c] = g_ptr[col];
    } else {
      mdst[c] = shift + (int)(slot_start[k] + (i64)j * (j + 1) / 2 - r0);
      mng[c] = 0;
    }
  }
  __syncthreads();
  // phase 1: half a warp per column fills the run in shared memory
  const int hw = threadIdx.x >> 4, sl = threadIdx.x & 15;
  for (int c = hw; c < ncols; c += QS_THREADS / 16) {
    const int j = mj[c];
    const double A = mA[c], ne2 = mne2[c];
    double* dst = buf + mdst[c];
    if (MODE == MODE_DIRECT) {
      const int ng = mng[c], g0 = mg0[c];
      for (int t = sl; t < ng; t += 16) dst[t] = g_val[g0 + t];
      dst += ng;
    }
    const double* wc = wstaged ? wst + (mo[c] - wlo) : wbar + mo[c];
#pragma unroll 4
    for (int i = sl; i <= j; i += 16) {
      double v = A * wc[i];
      if (i == 0) v = (j == 0) ? mA0[c] * wc[0] + ne2 : mA0[c] * wc[0];
      else if (i == j) v = v + ne2;
      dst[i] = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> visible to the bulk engine
  __syncthreads();
  // phase 2: the run leaves as 16-byte aligned bulk stores
  const int total = (int)(r1 - r0);
  const int nbulk = (total - shift) & ~1;  // doubles moved by bulk stores
  if (!BULK) {  // comparison variant: the same run leaves as aligned 128-bit stores issued by every thread
    const double2* src = reinterpret_cast<const double2*>(buf + 2 * shift);
    double2* dst = reinterpret_cast<double2*>(out + r0 + shift);
    for (int i = threadIdx.x; i < nbulk / 2; i += QS_THREADS) dst[i] = src[i];
    if (threadIdx.x == 0) {
      if (shift) out[r0] = buf[1];
      if ((total - shift) & 1) out[r1 - 1] = buf[shift + total - 1];
    }
    return;
  }
  if (threadIdx.x == 0) {
    const i64 g0 = r0 + shift;
    if (nbulk > 0)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + g0),
                   "r"(smem_addr(buf + 2 * shift)), "r"(nbulk * 8)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (shift) out[r0] = buf[1];
    if ((total - shift) & 1) out[r1 - 1] = buf[shift + total - 1];
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // shared memory must outlive the reads
  }
}

// positions[slot] == closed form for every slot?  flag[0] set to 1 otherwise.
__global__ void __launch_bounds__(QS_THREADS)
    k_check_direct(int l, int nb_orth, const int* soc_ptr, const int* cone_of_col, const int* tile_ptr,
                   const i64* slot_start, const i64* positions, const i64* kp_conic, int* flag) {
  QS_BATCH(soc_ptr, cone_of_col, tile_ptr, slot_start, positions, kp_conic, flag);
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

// KKT assembly on the device (reference: assemble_kkt, kkt.py:55-135): one warp per K column writes the row
// indices, the initial values and the slot -> position map of that column.  Column layout (upper triangle, rows
// ascending): x column j = P(:, j) plus an explicit diagonal; equality column = row of A then its zero diagonal;
// conic column = row of G, then the -I block entries (orthant: the diagonal; SOC column j: rows o .. o+j).
__global__ void __launch_bounds__(QS_THREADS)
    k_kkt_fill(int n, int p, int m, int l, Csr Pu, Csr Ar, Csr Gr, const int* __restrict__ soc_ptr,
               const int* __restrict__ cone_of_col, const i64* __restrict__ slot_start, const i64* __restrict__ Kp,
               int* __restrict__ Ki, double* __restrict__ Kx, i64* __restrict__ pos) {
  QS_BATCH(Pu, Ar, Gr, soc_ptr, cone_of_col, slot_start, Kp, Ki, Kx, pos);
  const i64 col = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (col >= (i64)n + p + m) return;
  i64 at = Kp[col];
  if (col < n) {
    const int b = Pu.ptr[col], e = Pu.ptr[col + 1];
    for (int k = b + lane; k < e; k += 32) {
      const int i = Pu.idx[k];
      Ki[at + (k - b)] = i;
      Kx[at + (k - b)] = (i == col) ? Pu.val[k] + 0.0 : Pu.val[k];  // the explicit 0.0 diagonal is summed onto P_jj
    }
    if (lane == 0 && !(e > b && Pu.idx[e - 1] == col)) {
      Ki[at + (e - b)] = (int)col;
      Kx[at + (e - b)] = 0.0;
    }
    return;
  }
  if (col < n + p) {
    const int r = (int)(col - n);
    const int b = Ar.ptr[r], e = Ar.ptr[r + 1];
    for (int k = b + lane; k < e; k += 32) {
      Ki[at + (k - b)] = Ar.idx[k];
      Kx[at + (k - b)] = Ar.val[k];
    }
    if (lane == 0) {
      Ki[at + (e - b)] = (int)col;
      Kx[at + (e - b)] = 0.0;
    }
    return;
  }
  const int c = (int)(col - n - p);
  const int b = Gr.ptr[c], e = Gr.ptr[c + 1];
  for (int k = b + lane; k < e; k += 32) {
    Ki[at + (k - b)] = Gr.idx[k];
    Kx[at + (k - b)] = Gr.val[k];
  }
  at += e - b;
  if (c < l) {
    if (lane == 0) {
      Ki[at] = (int)col;
      Kx[at] = -1.0;
      pos[c] = at;
    }
    return;
  }
  const int k = cone_of_col[c - l];
  const int o = soc_ptr[k], j = c - o;
  const i64 sb = slot_start[k] + (i64)j * (j + 1) / 2;
  for (int i = lane; i <= j; i += 32) {
    Ki[at + i] = n + p + o + i;
    Kx[at + i] = (i == j) ? -1.0 : 0.0;
    pos[sb + i] = at + i;
  }
}

int orth_blocks(int l) {
  if (l <= 0) return 0;
  int nb = (l + QS_THREADS - 1) / QS_THREADS;
  return nb > 148 * 4 ? 148 * 4 : nb;
}

}  // namespace

void qsk_neg_wtw(const WtwPlan& P, int mode, const double* w, const double* eta, const double* wbar,
                 const i64* positions, double* out, cudaStream_t st, bool have_consts) {
  if (P.nsoc > 0 && !have_consts)  // the NT-scaling kernel of the solver leaves c4 / e2 behind
    k_wtw_prepass<<<qs_grid((P.nsoc * 32 + QS_THREADS - 1) / QS_THREADS), QS_THREADS, 0, st>>>(P.nsoc, P.soc_ptr, wbar, eta,
                                                                                        P.c4, P.e2);
  const int nb_orth = orth_blocks(P.l);
  const int grid = nb_orth + P.ntiles;
  if (grid == 0) return;
  // Staged bulk-store path (opt-in, QS_WTW_STAGED=1): contiguous output run per tile (dense slots, or whole K
  // columns), 16-byte aligned base.  Measured on B200 at C4 it is SLOWER than the streaming kernel below (360 us
  // vs 212 us: three dependent phases per tile with CTA-wide barriers and only 4 CTAs per SM leave the SM waiting
  // on latency), so the streaming kernel stays the default; see DESIGN.md section 3.
  if ((mode == MODE_SLOTS || (mode == MODE_DIRECT && P.g_ptr && P.kstart)) && P.stile_ptr &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0 && getenv("QS_WTW_STAGED")) {
    const bool direct = mode == MODE_DIRECT;
    const int nt = direct ? P.n_stiles_direct : P.n_stiles_slots;
    const int* tp = direct ? P.stile_ptr_direct : P.stile_ptr;
    const size_t sm = (size_t)(QS_WTW_STAGE + 4 + QS_WTW_SWIN) * sizeof(double) +
                      (size_t)QS_WTW_SCOLS * (3 * sizeof(double) + 5 * sizeof(int));
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<qs_grid(nb_orth + nt), QS_THREADS, sm, st>>>(P.l, nb_orth, w, wbar, P.soc_ptr, P.cone_of_col, tp, P.c4, P.e2,
                                                 P.slot_start, P.kstart, P.g_ptr, P.g_val, out);
    };
    if (nb_orth + nt == 0) return;
    const bool bulk = !getenv("QS_WTW_PLAIN");
    if (direct) {
      if (bulk) go(k_neg_wtw_staged<MODE_DIRECT, true>);
      else go(k_neg_wtw_staged<MODE_DIRECT, false>);
    } else {
      if (bulk) go(k_neg_wtw_staged<MODE_SLOTS, true>);
      else go(k_neg_wtw_staged<MODE_SLOTS, false>);
    }
    return;
  }
  const bool staged = P.max_tile_window <= QS_WTW_WCAP;
  const int wcap = staged ? P.max_tile_window : 0;
  const int mc = P.max_tile_cols;
  const size_t smem = (size_t)mc * (5 * sizeof(double) + 4 * sizeof(int)) + 16 + (size_t)wcap * sizeof(double);
  auto launch = [&](auto kern, const i64* pos, const i64* kpc) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<qs_grid(grid), QS_THREADS, smem, st>>>(P.l, nb_orth, mc, wcap, w, wbar, P.soc_ptr, P.cone_of_col, P.tile_ptr,
                                         P.c4, P.e2, P.slot_start, pos, kpc, P.g_ptr, P.g_val, out);
  };
#define LAUNCH_WTW(M, S, pos, kpc)                                   \
  do {                                                                \
    if (qs_tls_batch > 1) launch(k_neg_wtw<M, S, true>, pos, kpc);    \
    else launch(k_neg_wtw<M, S, false>, pos, kpc);                    \
  } while (0)
  if (mode == MODE_SLOTS) {
    if (staged) LAUNCH_WTW(MODE_SLOTS, true, nullptr, nullptr);
    else LAUNCH_WTW(MODE_SLOTS, false, nullptr, nullptr);
  } else if (mode == MODE_MAP) {
    if (staged) LAUNCH_WTW(MODE_MAP, true, positions, nullptr);
    else LAUNCH_WTW(MODE_MAP, false, positions, nullptr);
  } else {
    if (staged) LAUNCH_WTW(MODE_DIRECT, true, nullptr, P.kp_conic);
    else LAUNCH_WTW(MODE_DIRECT, false, nullptr, P.kp_conic);
  }
}

void qsk_kkt_fill(const WtwPlan& P, int n, int p, const Csr& Pu, const Csr& Ar, const Csr& Gr, const i64* Kp, int* Ki,
                  double* Kx, i64* pos, cudaStream_t st) {
  const i64 N = (i64)n + p + P.m;
  const i64 blocks = (N * 32 + QS_THREADS - 1) / QS_THREADS;
  k_kkt_fill<<<qs_grid((unsigned)blocks), QS_THREADS, 0, st>>>(n, p, P.m, P.l, Pu, Ar, Gr, P.soc_ptr, P.cone_of_col,
                                                      P.slot_start, Kp, Ki, Kx, pos);
}

void qsk_check_direct_map(const WtwPlan& P, const i64* positions, int* flag, cudaStream_t st) {
  const int nb_orth = orth_blocks(P.l);
  const int grid = nb_orth + P.ntiles;
  if (grid == 0) return;
  k_check_direct<<<qs_grid(grid), QS_THREADS, 0, st>>>(P.l, nb_orth, P.soc_ptr, P.cone_of_col, P.tile_ptr, P.slot_start,
                                              positions, P.kp_conic, flag);
}
