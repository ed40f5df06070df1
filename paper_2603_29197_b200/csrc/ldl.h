// GPU supernodal multifrontal LDL' of the quasidefinite KKT matrix.
//
// Stands where the paper's cuDSS calls stand (analysis once, numeric
// refactorisation per iteration, triangular solves): cuDSS is not present in
// this image, so the factorisation is implemented here.  Semantics follow the
// reference's LDL (ldl.py:72-122, _kernels.py:102-184): no pivoting, a
// sign-matched static diagonal shift (+reg on the first n pivots, -reg on the
// rest) added to the matrix being factorised only, and a dynamic floor
// |d| < 1e-14 -> +-1e-14 on the pivots.
//
// Structure: host symbolic analysis (host_setup.cpp) -> supernodes with dense
// column-major fronts; numeric phase runs level by level over the supernodal
// tree (leaves first), one launch per level per phase.  180 GB of HBM lets
// every front keep its own panel AND update matrix, so there is no stack
// management and the assembly is a pure gather from the children.
#pragma once
#include <string>

#include "common.cuh"
#include "host_setup.h"

struct DevSym {
  int nsup;
  const int* col0;
  const i64* rowptr;
  const int* rowidx;
  const int* childptr;
  const int* child;
  const i64* relptr;
  const int* rel;
  const i64* Loff;
  const i64* Uoff;
  const i64* Boff;
  const int* sup_of;
  const int* iperm;
  const int* perm;
  __device__ void shift(size_t off) {
    qs_shift(off, col0);
    qs_shift(off, rowptr);
    qs_shift(off, rowidx);
    qs_shift(off, childptr);
    qs_shift(off, child);
    qs_shift(off, relptr);
    qs_shift(off, rel);
    qs_shift(off, Loff);
    qs_shift(off, Uoff);
    qs_shift(off, Boff);
    qs_shift(off, sup_of);
    qs_shift(off, iperm);
    qs_shift(off, perm);
  }
};

// extend-add work item: front `front`, columns [c_lo, c_lo + 8)
struct SlabItem {
  int front, c_lo;
};

// Assembly lists built at analysis.  A "slot" is one (front, local row) pair of a front that has children; the
// slots of a level are contiguous.  Slot lists hold, in child order, every child entry that lands on that row:
//   gptr[slot] .. gptr[slot+1]   range in gsrc / gchild
//   gsrc[e]    offset of the entry in the solve contribution storage B (= Boff[child] + position in the child)
//   gchild[e]  the child supernode
//   gdst[slot] where the forward-solve sum goes: >= 0 -> xw[gdst] += sum,  < 0 -> B[-gdst-1] = sum
// By symmetry the same list serves the numeric extend-add: entry e of column slot (s, pc) is child column
// cc = gsrc[e] - Boff[child], whose rows cc.. are added into column pc of the front.
// Fronts with many children are cut into row bands of QS_EA_BAND rows so that several warps share one column:
// bandptr[child] .. : for each band b of the PARENT, the first child update row whose parent row is >= b * BAND.
#define QS_EA_BAND 256
struct AsmLists {
  const i64* gptr;
  const int* gsrc;
  const int* gchild;
  const i64* gdst;
  const int* slot_front;  // [nslots]
  const int* slot_row;    // [nslots] local row / column of the slot inside its front
  const i64* bandptr;     // [nsup+1] offsets into bandstart (only children of banded fronts have entries)
  const int* bandstart;
  __device__ void shift(size_t off) {
    qs_shift(off, gptr);
    qs_shift(off, gsrc);
    qs_shift(off, gchild);
    qs_shift(off, gdst);
    qs_shift(off, slot_front);
    qs_shift(off, slot_row);
    qs_shift(off, bandptr);
    qs_shift(off, bandstart);
  }
};
// Schur-complement work item: 64 x 64 tile (ti, tj), ti >= tj, of the update matrix of front `front`
struct TileItem {
  int front;
  short ti, tj;
};
// extend-add work item of the list-driven kernel: column slot + row band (band = -1: whole column)
struct EaItem {
  int slot, band;
};

// Dense SOC blocks of K (upper triangles packed by columns) land TRANSPOSED in the panels of L: entry (i, j), i <= j,
// of a cone goes to row j, column i of its front.  Scattering K entry by entry writes 8 bytes per 4 KB stride (each
// store its own 32-byte sector).  With the block structure at hand the scatter runs tile by tile through shared
// memory: read 32 x 32 along the K columns, write along the panel columns.
struct ConeBlocks {
  int n_p, l, nsoc;         // first conic K column, orthant size, cones
  const int* soc_ptr;       // [nsoc+1] conic index of each cone's first row (starts at l)
  const i64* kp_conic;      // [m] kp_conic[c] = K.col_pointers[n_p + c + 1]
  const int* cone_of_col;   // [m - l]
  const i64* Kp;            // K column pointers
  i64 flat_nnz;             // K entries before the first SOC column: no block among them (scattered entry by entry)
  int ntiles;
  const int* tile_cone;     // [ntiles]
  const short* tile_ij;     // [2 ntiles] (ti, tj), ti <= tj, of the cone's upper triangle
  __device__ void shift(size_t off) {
    qs_shift(off, soc_ptr), qs_shift(off, kp_conic), qs_shift(off, cone_of_col), qs_shift(off, Kp);
    qs_shift(off, tile_cone), qs_shift(off, tile_ij);
  }
};

struct LinSys {
  Symbolic S;
  ConeBlocks cb{};
  bool have_cb = false;
  // after analyze(): the cone layout of the KKT matrix whose closed-form block positions were validated (capi.cu)
  std::string set_cone_blocks(int n_p, int l, int nsoc, const i64* q_host, const int* d_soc_ptr, const i64* d_kp_conic,
                              const int* d_cone_of_col, const i64* d_Kp, i64 flat_nnz, cudaStream_t st);
  DevSym D{};
  i64 N = 0, knnz = 0;
  // device storage
  double* L = nullptr;     // panels
  double* U = nullptr;     // update matrices
  double* Dg = nullptr;    // pivots (new numbering)
  double* B = nullptr;     // solve contribution vectors
  double* xw = nullptr;    // permuted work vector
  double* reg = nullptr;   // sign-matched static shift per new column
  i64* amap = nullptr;     // K entry -> panel storage offset
  int* d_levelsup = nullptr;
  // work lists built at analysis (see ldl.cu)
  int n_leaf = 0;
  int leaf_group = 32;  // lanes per leaf front (4, 8, 16 or 32)
  int* d_leaf = nullptr;
  int* d_gen = nullptr;
  SlabItem* d_slabs = nullptr;
  int* d_small = nullptr;  // general fronts factored by one CTA
  int* d_blk = nullptr;    // general fronts factored by the blocked multi-CTA path
  i64* d_poff = nullptr;   // per blocked front: offset into `partial`
  double* partial = nullptr;  // backward-solve row-tile partial sums
  std::vector<int> genptr, slabptr, smallptr, blkptr, blk_max_ns, blk_max_nr, blk_max_nu;
  // The blocked fronts of a level, sorted by pivot count, are factored chunk by chunk (one chunk per level unless
  // QS_LDL_CHUNK_MB asks for L2-sized chunks -- measured slower, see ldl.cu); a chunk's launch grids use its own
  // maxima and its Schur tiles follow its panel steps.
  struct BlkChunk {
    int b0, count, max_ns, max_nr;
    i64 t0, t1;  // range in d_tiles
  };
  std::vector<BlkChunk> blk_chunks;
  std::vector<int> chunkptr;  // [nlevels+1] ranges in blk_chunks
  AsmLists A{};
  EaItem* d_eaitems = nullptr;
  TileItem* d_tiles = nullptr;      // Schur tiles of the blocked fronts, level by level
  std::vector<i64> tileptr;         // [nlevels+1]
  std::vector<i64> lvslot, eaptr;   // per level: slot range, extend-add item range
  std::vector<int> lv_tpr;          // per level: lanes per slot in the forward-solve gather
  std::vector<char> ea_wide;        // per level: 32 lanes per extend-add item (else 4)
  std::vector<char> ea_direct;      // per level: no item list, item w = column slot lvslot[lv] + w
  bool use_lists = true;
  bool use_cluster = true;  // cluster-of-CTAs triangular solves for levels with at most 16 large fronts
  std::vector<void*> owned;
  double dyn_eps = 1e-14;
  double analysis_seconds = 0.0;
  size_t device_bytes = 0;
  size_t h2d_bytes = 0;  // host -> device bytes copied by analyze()

  // Kp/Ki: host pattern (upper CSC) -- the full matrix or its compact form without the off-diagonal entries of
  // the clique blocks; knnz_full / d_Kp / d_Ki: the full matrix on the device.
  std::string analyze(i64 N, const i64* Kp, const i64* Ki, i64 knnz_full, const i64* d_Kp, const int* d_Ki, int order,
                      const i64* user_perm, i64 ncliques, const i64* clique_start, const i64* clique_size, i64 n_pos,
                      double static_reg, cudaStream_t st);
  // The launch sequences of factor() and solve() depend only on the analysis, so each is captured once into a CUDA
  // graph (per distinct argument tuple) and replayed: a small problem (MPC instance, 10^3 launches of a few
  // microseconds each) is otherwise bound by launch overhead.  QS_NO_GRAPH=1 launches directly.
  void factor(const double* d_Kx, double* scalars, cudaStream_t st);
  void solve(const double* d_rhs, double* d_sol, cudaStream_t st);  // (L D L')^{-1} rhs, no refinement
  void factor_launches(const double* d_Kx, double* scalars, cudaStream_t st);
  void solve_launches(const double* d_rhs, double* d_sol, cudaStream_t st);
  struct GraphEntry {
    const void* a;
    const void* b;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> factor_graphs, solve_graphs;
  bool use_graphs = true;
  long long graph_counts[2] = {0, 0};  // factor / solve calls replayed from a graph, issued as direct launches
  // narrow-level chains: chain_end[lv] > lv + 1 when levels [lv, chain_end[lv]) are fused into one single-CTA launch
  std::vector<int> chain_end, chain_start_of_end;
  int* d_smallptr = nullptr;
  i64* d_eaptr = nullptr;
  i64* d_lvslot = nullptr;
  int launches_per_factor() const;
  int launches_per_solve() const;
  void release();
};
