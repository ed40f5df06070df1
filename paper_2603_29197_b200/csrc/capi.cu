// C ABI of libqsocp_cuda.so (include/qsocp_cuda.h): handle, setup, the
// per-kernel entry points and the device-resident IPM phases.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/qsocp_cuda.h"
#include "cone_kernels.h"
#include "devmem.h"
#include "host_setup.h"
#include "kkt_kernels.h"
#include "ldl.h"
#include "ruiz_kernels.h"
#include "spmv_kernels.h"

thread_local int qs_tls_batch = 1;  // common.cuh: instances per launch of this thread (qs_batch_* calls raise it)

// ------------------------------------------------------------ device memory (devmem.h)
namespace {
// Batched mode: while a thread works on a batch, every device allocation is a bump allocation inside slot 0 of the
// batch's arena (so that the whole handle has the same layout in every slot); frees of arena pointers are no-ops.
struct QsArena {
  char* base = nullptr;
  size_t slot_bytes = 0, used = 0;
  int slots = 0;
};
thread_local QsArena* qs_tls_arena = nullptr;
struct DevMem {
  std::mutex mu;
  bool ready[64] = {false};
  bool pooled[64] = {false};
  cudaStream_t stream[64] = {nullptr};
  std::unordered_set<void*> from_pool;  // pointers handed out by cudaMallocAsync
  std::vector<std::pair<char*, size_t>> arenas;  // live batch arenas (base, total bytes)
  struct CachedArena {
    int dev;
    char* base;
    size_t bytes;
  };
  std::vector<CachedArena> arena_cache;  // released arenas kept for the next batch (at most 2 per process)
};
DevMem g_devmem;
}  // namespace

cudaError_t qs_dev_malloc(void** p, size_t bytes) {
  if (QsArena* a = qs_tls_arena) {
    const size_t at = (a->used + 255) & ~size_t(255);
    if (at + bytes > a->slot_bytes) return cudaErrorMemoryAllocation;  // the instance does not fit one slot
    *p = a->base + at;
    a->used = at + bytes;
    return cudaSuccess;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaMalloc(p, bytes);
  {
    std::lock_guard<std::mutex> lk(g_devmem.mu);
    if (!g_devmem.ready[dev]) {
      g_devmem.ready[dev] = true;
      int supported = 0;
      cudaDeviceGetAttribute(&supported, cudaDevAttrMemoryPoolsSupported, dev);
      cudaMemPool_t pool = nullptr;
      if (supported && !getenv("QS_NO_MEMPOOL") && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
          cudaStreamCreateWithFlags(&g_devmem.stream[dev], cudaStreamNonBlocking) == cudaSuccess) {
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        g_devmem.pooled[dev] = true;
      }
      cudaGetLastError();
    }
  }
  if (!g_devmem.pooled[dev]) return cudaMalloc(p, bytes);
  cudaError_t e = cudaMallocAsync(p, bytes, g_devmem.stream[dev]);
  if (e != cudaSuccess) {  // pool exhausted or fragmented: hand the cached blocks back to the driver and retry once
    cudaGetLastError();
    cudaMemPool_t pool = nullptr;
    cudaStreamSynchronize(g_devmem.stream[dev]);
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(p, bytes, g_devmem.stream[dev]);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cudaMalloc(p, bytes);
    }
  }
  cudaStreamSynchronize(g_devmem.stream[dev]);  // the block may now be used on any stream
  std::lock_guard<std::mutex> lk(g_devmem.mu);
  g_devmem.from_pool.insert(*p);
  return cudaSuccess;
}

void qs_dev_free(void* p) {
  if (!p) return;
  bool pooled = false;
  {
    std::lock_guard<std::mutex> lk(g_devmem.mu);
    for (const auto& a : g_devmem.arenas)
      if ((char*)p >= a.first && (char*)p < a.first + a.second) return;  // lives and dies with its batch arena
    pooled = g_devmem.from_pool.erase(p) > 0;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (pooled && dev >= 0 && dev < 64 && g_devmem.stream[dev])
    cudaFreeAsync(p, g_devmem.stream[dev]);
  else
    cudaFree(p);
}


namespace {

thread_local std::string g_error;

enum TimerCat { T_CONE = 0, T_KKT, T_RESID, T_FACTOR, T_SOLVE, T_REFINE, T_ANALYSIS, T_H2D, T_COUNT };

struct DevPool {
  std::vector<void*> ptrs;
  size_t bytes = 0;
  size_t uploaded = 0;  // host -> device bytes copied through this pool
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    const size_t sz = std::max<size_t>(count, 1) * sizeof(T);
    if (qs_dev_malloc(&p, sz) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    ptrs.push_back(p);
    bytes += sz;
    return (T*)p;
  }
  template <class T>
  T* upload(const T* src, size_t count, cudaStream_t st) {
    T* d = alloc<T>(count);
    if (d && count) cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, st);
    if (d) uploaded += count * sizeof(T);
    return d;
  }
  void release() {
    for (void* p : ptrs) qs_dev_free(p);
    ptrs.clear();
    bytes = 0;
  }
};

struct PhaseTimer {
  struct Span {
    cudaEvent_t a, b;
    int cat;
  };
  std::vector<Span> open_spans;
  std::vector<cudaEvent_t> pool;
  double total[T_COUNT] = {0};
  bool enabled = true;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void begin(int cat, cudaStream_t st) {
    if (!enabled) return;
    Span s{get(), get(), cat};
    cudaEventRecord(s.a, st);
    open_spans.push_back(s);
  }
  void end(cudaStream_t st) {
    if (!enabled) return;
    cudaEventRecord(open_spans.back().b, st);
  }
  void collect() {  // call after a stream sync
    for (auto& s : open_spans) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, s.a, s.b) == cudaSuccess) total[s.cat] += ms * 1e-3;
      pool.push_back(s.a);
      pool.push_back(s.b);
    }
    open_spans.clear();
  }
  void release() {
    collect();
    for (auto e : pool) cudaEventDestroy(e);
    pool.clear();
  }
};

}  // namespace

struct qs_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  std::string err;
  DevPool cone_pool, prob_pool;
  PhaseTimer tm;
  i64 launches = 0;

  // ---- cone layout
  bool have_cones = false;
  ConeLayout L{};
  WtwPlan wp{};
  std::vector<i64> q_host;
  std::vector<int> soc_ptr_host;
  i64 S = 0;            // scaling slots
  i64* d_slot_start = nullptr;
  double* cone_tmp = nullptr;  // [m] scratch of the unit entry points
  double deg = 0.0;

  // reduction scratch + scalars
  GridRed gr{};
  double* scalars = nullptr;       // device [SC_COUNT]
  double* scalars_host = nullptr;  // pinned [SC_COUNT]

  // ---- problem
  bool have_problem = false;
  i64 n = 0, p = 0, m = 0, N = 0;
  qs_settings st{};
  Csr Pf{}, At{}, Gt{}, Ar{}, Gr{}, Pu{};
  Csr Dt{};            // fused dual-range matrix [Pf | A' | G'] with tagged indices (spmv_kernels.h), or ptr == nullptr
  double* seg_partial = nullptr;  // [p * QS_ROW_SEGS] when the equality rows are long (spmv_kernels.h)
  int* dt_map = nullptr;  // Dt.val[k] = {Pf, At, Gt}.val[dt_map[k] & mask] by tag
  i64 nnzDt = 0;
  // value maps for qs_update_values: Ar.val[k] = Ax[ar_map[k]], Gr.val[k] = Gx[gr_map[k]], Pf.val[k] = Px[pf_map[k]]
  int *ar_map = nullptr, *gr_map = nullptr, *pf_map = nullptr;
  double *c = nullptr, *b = nullptr, *hv = nullptr;
  double norm_c = 0, norm_b = 0, norm_h = 0;
  // KKT
  i64 knnz = 0;
  i64 nnzP = 0, nnzPf = 0, nnzA = 0, nnzG = 0;
  i64 d2h_bytes = 0, h2d_extra = 0;  // transfer accounting (qs_get_transfer_bytes)
  std::vector<i64> Kp_h;  // host copy of the KKT column pointers (the entries live on the device only)
  i64* d_Kp = nullptr;
  int* d_Ki = nullptr;
  double* d_Kx = nullptr;
  i64* d_pos = nullptr;
  bool direct_ok = false;
  LinSys ls;
  bool factored = false;
  i64 n_factor = 0, n_solve = 0;
  // ---- state
  double *x = nullptr, *y = nullptr, *z = nullptr, *s = nullptr;
  double *x2 = nullptr, *y2 = nullptr, *z2 = nullptr, *s2 = nullptr;  // next iterate; swapped in when the step is good
  double *w = nullptr, *eta = nullptr, *wbar = nullptr, *lam = nullptr, *lam_sq = nullptr;
  double *d = nullptr, *dcomp = nullptr, *wdz = nullptr, *ds = nullptr, *r_cone = nullptr, *w2vz = nullptr;
  double *rhs = nullptr, *sol = nullptr, *xa = nullptr, *xb = nullptr, *ra = nullptr, *rb = nullptr, *dx = nullptr;
  double* tmp_m = nullptr;
  // Ruiz scalings (null when ruiz_iters == 0)
  double *rD = nullptr, *rE = nullptr, *rF = nullptr;
};

namespace {

#define CK(h, call)                                                      \
  do {                                                                   \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) {                                             \
      (h)->err = std::string(#call) + ": " + cudaGetErrorString(e_);     \
      return QS_E_CUDA;                                                  \
    }                                                                    \
  } while (0)

int fail(qs_handle* h, int code, const std::string& msg) {
  h->err = msg;
  return code;
}

int check_launch(qs_handle* h, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, QS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return QS_OK;
}

// Pinned host mirrors of the scalar block are recycled across handles: cudaMallocHost / cudaFreeHost synchronise the
// device and showed up as 10-230 ms of handle teardown.
std::mutex g_pinned_mu;
std::vector<double*> g_pinned_free;

double* pinned_scalars_get() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      double* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  double* p = nullptr;
  if (cudaMallocHost((void**)&p, SC_COUNT * sizeof(double)) != cudaSuccess) return nullptr;
  return p;
}

void pinned_scalars_put(double* p) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}

bool ensure_scratch(qs_handle* h) {
  if (h->scalars) return true;
  if (qs_dev_malloc((void**)&h->scalars, SC_COUNT * sizeof(double)) != cudaSuccess) return false;
  cudaMemsetAsync(h->scalars, 0, SC_COUNT * sizeof(double), h->stream);
  h->scalars_host = pinned_scalars_get();
  if (!h->scalars_host) return false;
  if (qs_dev_malloc((void**)&h->gr.partial, (size_t)QS_MAX_GRID * QS_RED_MAXK * sizeof(double)) != cudaSuccess)
    return false;
  if (qs_dev_malloc((void**)&h->gr.counter, sizeof(unsigned)) != cudaSuccess) return false;
  cudaMemsetAsync(h->gr.counter, 0, sizeof(unsigned), h->stream);
  return true;
}

int fetch_scalars(qs_handle* h) {
  h->d2h_bytes += SC_COUNT * sizeof(double);
  CK(h, cudaMemcpyAsync(h->scalars_host, h->scalars, SC_COUNT * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  h->tm.collect();
  return QS_OK;
}

i64 flags_of(const double* sc) {
  i64 f = 0;
  if (sc[SC_FLAG_NOT_INTERIOR] != 0.0) f |= 1;
  if (sc[SC_FLAG_NONFINITE] != 0.0) f |= 2;
  if (sc[SC_FLAG_BAD_STEP] != 0.0) f |= 4;
  if (sc[SC_PIVOT_NONFINITE] != 0.0) f |= 8;
  return f;
}

void clear_flags(qs_handle* h) {
  // SC_FLAG_NOT_INTERIOR .. SC_FLAG_BAD_STEP are contiguous
  qs_memset_b(h->scalars + SC_FLAG_NOT_INTERIOR, 0, 3 * sizeof(double), h->stream);
  qs_memset_b(h->scalars + SC_PIVOT_BUMPS, 0, 2 * sizeof(double), h->stream);
}

template <class T>
std::vector<int> to_i32(const T* src, size_t count) {
  std::vector<int> out(count);
  for (size_t k = 0; k < count; ++k) out[k] = (int)src[k];
  return out;
}

bool make_csr(qs_handle* h, Csr* M, i64 rows, i64 cols, const i64* ptr, const i64* idx, const double* val) {
  const i64 nnz = ptr[rows];
  std::vector<int> p32 = to_i32(ptr, rows + 1), i32 = to_i32(idx, nnz);
  M->rows = (int)rows;
  M->cols = (int)cols;
  M->ptr = h->prob_pool.upload(p32.data(), p32.size(), h->stream);
  M->idx = h->prob_pool.upload(i32.data(), i32.size(), h->stream);
  M->val = h->prob_pool.upload(val, nnz, h->stream);
  M->tpr = qsk_pick_tpr(nnz, rows);
  M->exact1 = nnz == rows && rows > 0;
  for (i64 r = 0; r < rows && M->exact1; ++r) M->exact1 = ptr[r] == r;
  cudaStreamSynchronize(h->stream);  // the int32 staging vectors die here
  return M->ptr && M->idx && M->val;
}

int scatter_scaling(qs_handle* h, const double* w, const double* eta, const double* wbar, bool have_consts = false) {
  h->tm.begin(T_KKT, h->stream);
  qsk_neg_wtw(h->wp, h->direct_ok ? 2 : 1, w, eta, wbar, h->d_pos, h->d_Kx, h->stream, have_consts);
  h->launches += have_consts ? 1 : 2;
  h->tm.end(h->stream);
  return check_launch(h, "neg_wtw scatter");
}

// solve_refine (ldl.py:135-166) on the device: result in h->sol.
int solve_refined(qs_handle* h, const double* rhs) {
  const i64 N = h->N;
  cudaStream_t st = h->stream;
  auto backsolve = [&](const double* r, double* out) {
    h->tm.begin(T_SOLVE, st);
    h->ls.solve(r, out, st);
    h->tm.end(st);
    h->launches += h->ls.launches_per_solve();
  };
  auto residual = [&](const double* v, double* r, int slot) {
    h->tm.begin(T_REFINE, st);
    if (h->st.kkt_literal) {
      // r = rhs - sym(K) v over the stored entries (the reference's form)
      cudaMemsetAsync(r, 0, N * sizeof(double), st);
      qsk_spmv_sym_upper_csc((int)N, h->d_Kp, h->d_Ki, h->d_Kx, v, r, st);
      qsk_axpby(N, 1.0, rhs, -1.0, r, r, st);
      qsk_absmax(N, r, h->scalars + slot, nullptr, h->gr, st);
      h->launches += 3;
    } else {
      qsk_apply_w2(h->L, h->w, h->eta, h->wbar, v + h->n + h->p, h->w2vz, st);
      KktResidualArgs A{(int)h->n, (int)h->p, (int)h->m, h->Pf, h->At, h->Gt, h->Ar, h->Gr, h->Dt, h->seg_partial,
                        v,         rhs,       h->w2vz,   r,     h->scalars, slot, h->gr};
      qsk_kkt_residual(A, st);
      h->launches += 2;
    }
    h->tm.end(st);
  };
  double* x = h->xa;
  double* xn = h->xb;
  double* r = h->ra;
  double* r2 = h->rb;
  backsolve(rhs, x);
  if (h->st.refine_iters > 0) {
    qsk_absmax(N, rhs, h->scalars + SC_TMP0, nullptr, h->gr, st);
    residual(x, r, SC_TMP1);
    h->launches += 1;
    int rc = fetch_scalars(h);
    if (rc) return rc;
    const double stop = 1e-12 * (1.0 + h->scalars_host[SC_TMP0]);  // ldl.py:19,151
    double rn = h->scalars_host[SC_TMP1];
    if (!(fabs(rn) <= DBL_MAX)) return fail(h, QS_E_NUMERICAL, "non-finite triangular solve result");
    for (i64 it = 0; it < h->st.refine_iters; ++it) {
      if (rn <= stop) break;
      backsolve(r, h->dx);
      qsk_axpby(N, 1.0, x, 1.0, h->dx, xn, st);
      residual(xn, r2, SC_TMP2);
      h->launches += 1;
      rc = fetch_scalars(h);
      if (rc) return rc;
      const double rn2 = h->scalars_host[SC_TMP2];
      if (!(fabs(rn2) <= DBL_MAX)) return fail(h, QS_E_NUMERICAL, "non-finite refinement residual");
      if (rn2 >= rn) break;
      std::swap(x, xn);
      std::swap(r, r2);
      rn = rn2;
    }
  }
  h->sol = x;
  h->n_solve++;
  return check_launch(h, "linear solve");
}

int do_factor(qs_handle* h) {
  h->tm.begin(T_FACTOR, h->stream);
  h->ls.factor(h->d_Kx, h->scalars, h->stream);
  h->tm.end(h->stream);
  h->launches += h->ls.launches_per_factor();
  h->n_factor++;
  h->factored = true;
  return check_launch(h, "factor");
}

void fill_residual_info(qs_handle* h, qs_residual_info* o) {
  const double* sc = h->scalars_host;
  o->norm_r_dual = sc[SC_NORM_RDUAL];
  o->norm_r_eq = sc[SC_NORM_REQ];
  o->norm_r_cone = sc[SC_NORM_RCONE];
  o->gap = sc[SC_GAP];
  o->objective = sc[SC_OBJ];
  o->norm_Px = sc[SC_NORM_PX];
  o->norm_Aty = sc[SC_NORM_ATY];
  o->norm_Gtz = sc[SC_NORM_GTZ];
  o->norm_c = h->norm_c;
  o->norm_Ax = sc[SC_NORM_AX];
  o->norm_b = h->norm_b;
  o->norm_Gx = sc[SC_NORM_GX];
  o->norm_h = h->norm_h;
  o->norm_s = sc[SC_NORM_S];
  o->mu = sc[SC_MU];
  o->flags = flags_of(sc);
}

double inf_norm(const double* v, i64 n) {
  double t = 0.0;
  for (i64 k = 0; k < n; ++k) {
    const double a = fabs(v[k]);
    if (a > t || a != a) t = a;
  }
  return t;
}

}  // namespace

// =============================================================== C ABI ======
extern "C" {

int qs_version(void) { return 100; }

int qs_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

const char* qs_global_error(void) { return g_error.c_str(); }

qs_handle* qs_create(int device) {
  int cnt = qs_device_count();
  if (device < 0 || device >= cnt) {
    g_error = "no CUDA device " + std::to_string(device) + " (visible devices: " + std::to_string(cnt) + ")";
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    g_error = "cudaSetDevice failed";
    return nullptr;
  }
  qs_handle* h = new qs_handle();
  h->device = device;
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess || !ensure_scratch(h)) {
    g_error = std::string("stream/scratch creation failed: ") + cudaGetErrorString(cudaGetLastError());
    delete h;
    return nullptr;
  }
  return h;
}

void qs_destroy(qs_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  const bool verbose = getenv("QS_VERBOSE") != nullptr;
  auto t_mark = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (verbose) {
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[qs destroy] %-28s %8.3f s\n", what, std::chrono::duration<double>(now - t_mark).count());
      t_mark = now;
    }
  };
  h->tm.release();
  lap("timers");
  h->ls.release();
  lap("LDL' (graphs + storage)");
  h->cone_pool.release();
  h->prob_pool.release();
  lap("problem + cone pools");
  if (h->scalars) qs_dev_free(h->scalars);
  if (h->scalars_host) pinned_scalars_put(h->scalars_host);
  if (h->gr.partial) qs_dev_free(h->gr.partial);
  if (h->gr.counter) qs_dev_free(h->gr.counter);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  lap("scratch + stream");
  delete h;
  lap("host vectors");
}

const char* qs_last_error(qs_handle* h) { return h ? h->err.c_str() : g_error.c_str(); }

int qs_set_stream(qs_handle* h, void* cuda_stream) {
  if (!h) return QS_E_INVALID;
  cudaStreamSynchronize(h->stream);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  h->stream = (cudaStream_t)cuda_stream;
  h->own_stream = false;
  return QS_OK;
}

// Page-lock caller memory (e.g. a mapped problem file) so host -> device copies skip the driver's staging buffer.
int qs_host_register(const void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return QS_E_INVALID;
  cudaError_t e = cudaHostRegister(const_cast<void*>(ptr), (size_t)bytes, cudaHostRegisterReadOnly | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    e = cudaHostRegister(const_cast<void*>(ptr), (size_t)bytes, cudaHostRegisterPortable);
  }
  if (e != cudaSuccess) {
    g_error = std::string("cudaHostRegister: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return QS_E_CUDA;
  }
  return QS_OK;
}

int qs_host_unregister(const void* ptr) {
  if (!ptr) return QS_E_INVALID;
  if (cudaHostUnregister(const_cast<void*>(ptr)) != cudaSuccess) {
    cudaGetLastError();
    return QS_E_CUDA;
  }
  return QS_OK;
}

int qs_sync(qs_handle* h) {
  if (!h) return QS_E_INVALID;
  CK(h, cudaStreamSynchronize(h->stream));
  h->tm.collect();
  return QS_OK;
}

// ---------------------------------------------------------------- host-side
int64_t qs_kkt_nnz(int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q, const int64_t* Pp,
                   const int64_t* Pi, int64_t nnzA, int64_t nnzG) {
  KktDims d{n, p, m, l, nsoc, (const i64*)q};
  return hs_kkt_nnz(d, (const i64*)Pp, (const i64*)Pi, nnzA, nnzG);
}

int64_t qs_kkt_slot_count(int64_t l, int64_t nsoc, const int64_t* q) {
  KktDims d{0, 0, 0, l, nsoc, (const i64*)q};
  return hs_slot_count(d);
}

int qs_kkt_assemble(int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q, const int64_t* Pp,
                    const int64_t* Pi, const double* Px, const int64_t* Ap, const int64_t* Ai, const double* Ax,
                    const int64_t* Gp, const int64_t* Gi, const double* Gx, int64_t* Kp, int64_t* Ki, double* Kx,
                    int64_t* nt_entry_positions, int64_t* nt_slot_offsets, int64_t* soc_slot_starts) {
  i64 msum = l;
  for (i64 k = 0; k < nsoc; ++k) msum += q[k];
  if (msum != m) return QS_E_DIMENSION;
  KktDims d{n, p, m, l, nsoc, (const i64*)q};
  const i64 nnzA = Ap[n], nnzG = Gp[n];
  std::vector<i64> Arp(p + 1), Ari(nnzA), Grp(m + 1), Gri(nnzG);
  std::vector<double> Arx(nnzA), Grx(nnzG);
  hs_transpose(p, n, (const i64*)Ap, (const i64*)Ai, Ax, Arp.data(), Ari.data(), Arx.data());
  hs_transpose(m, n, (const i64*)Gp, (const i64*)Gi, Gx, Grp.data(), Gri.data(), Grx.data());
  hs_kkt_assemble(d, (const i64*)Pp, (const i64*)Pi, Px, Arp.data(), Ari.data(), Arx.data(), Grp.data(), Gri.data(),
                  Grx.data(), (i64*)Kp, (i64*)Ki, Kx, (i64*)nt_entry_positions, (i64*)nt_slot_offsets,
                  (i64*)soc_slot_starts);
  return QS_OK;
}

int qs_symbolic_stats(int64_t N, const int64_t* Kp, const int64_t* Ki, int64_t ordering, const int64_t* user_perm,
                      int64_t ncliques, const int64_t* clique_start, const int64_t* clique_size, int64_t* out_perm,
                      double* stats6) {
  Symbolic S;
  std::string err = hs_symbolic_cliques(N, (const i64*)Kp, (const i64*)Ki, (int)ordering, (const i64*)user_perm,
                                        ncliques, (const i64*)clique_start, (const i64*)clique_size, &S);
  if (!err.empty()) {
    g_error = err;
    return QS_E_INVALID;
  }
  if (out_perm)
    for (i64 k = 0; k < N; ++k) out_perm[k] = S.perm[k];
  if (stats6) {
    stats6[0] = S.nsup;
    stats6[1] = S.nlevels;
    stats6[2] = (double)S.lnz;
    stats6[3] = S.flops;
    stats6[4] = S.max_nr;
    stats6[5] = S.max_ns;
  }
  return QS_OK;
}

// --------------------------------------------------------------- cone layout
int qs_set_cones(qs_handle* h, int64_t l, int64_t nsoc, const int64_t* q, int64_t big_threshold) {
  if (!h) return QS_E_INVALID;
  if (l < 0 || nsoc < 0) return fail(h, QS_E_INVALID, "negative cone dimension");
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  h->cone_pool.release();
  if (big_threshold <= 0) big_threshold = 2048;
  i64 m = l;
  std::vector<int> ptr(nsoc + 1);
  std::vector<int> small_ids, big_ids;
  ptr[0] = (int)l;
  // Lane-group width G from the mean size of the cones a warp could hold (dim <= 256): smallest power of two with
  // 8 G >= mean.  A cone is "small" (lane group, whole cone in registers) iff dim <= G * R; the rest get a CTA.
  double mean = 0.0;
  i64 cnt = 0;
  for (i64 k = 0; k < nsoc; ++k) {
    if (q[k] < 1) return fail(h, QS_E_INVALID, "every SOC dimension must be >= 1");
    if (q[k] <= 256) {
      mean += (double)q[k];
      ++cnt;
    }
  }
  mean = cnt ? mean / cnt : 256.0;
  int G = 1, single = -1;
  while (G < 32 && G * 8 < mean) G <<= 1;
  // experiment knobs (tests/gpu_cone_sweep.py): QS_CONE_G, QS_CONE_SINGLE
  if (const char* e = getenv("QS_CONE_G")) {
    G = 1;
    while (G < 32 && G < atoi(e)) G <<= 1;
  }
  if (const char* e = getenv("QS_CONE_SINGLE")) single = atoi(e) != 0;
  // register-resident ops need dim <= 8 G; when every op runs chunked (single == 0) a lane group takes any dim
  i64 small_cap = std::min<i64>(single == 0 ? big_threshold : (i64)G * 8, big_threshold);
  if (const char* e = getenv("QS_CONE_SMALLCAP")) small_cap = std::max(1, atoi(e));
  for (i64 k = 0; k < nsoc; ++k) {
    m += q[k];
    if (m >= ((i64)1 << 31)) return fail(h, QS_E_DIMENSION, "m exceeds 2^31");
    ptr[k + 1] = (int)m;
    (q[k] > small_cap ? big_ids : small_ids).push_back((int)k);
  }
  h->q_host.assign(q, q + nsoc);
  h->soc_ptr_host = ptr;
  ConeLayout& L = h->L;
  L.m = (int)m;
  L.l = (int)l;
  L.nsoc = (int)nsoc;
  L.soc_ptr = h->cone_pool.upload(ptr.data(), ptr.size(), h->stream);
  // small cones sorted by dimension, largest first: the lane groups of a CTA then work on cones of similar size
  // (no warp waits at the CTA's final barrier for a much longer neighbour, the per-size dispatch does not diverge)
  // and the shortest cones fill the tail of the persistent grid
  std::stable_sort(small_ids.begin(), small_ids.end(), [&](int a, int b) { return q[a] > q[b]; });
  if (getenv("QS_CONE_UNSORTED")) std::sort(small_ids.begin(), small_ids.end());
  L.nsmall = (int)small_ids.size();
  L.nbig = (int)big_ids.size();
  L.small_ids = small_ids.empty() ? nullptr : h->cone_pool.upload(small_ids.data(), small_ids.size(), h->stream);
  L.big_ids = big_ids.empty() ? nullptr : h->cone_pool.upload(big_ids.data(), big_ids.size(), h->stream);
  L.group = G;
  L.single = single;
  L.waves = 1;
  if (const char* e = getenv("QS_CONE_WAVES")) L.waves = std::max(1, atoi(e));
  h->deg = (double)(l + nsoc);
  // -W'W plan: column tiles of ~QS_WTW_TILE block entries
  WtwPlan& P = h->wp;
  P.l = (int)l;
  P.nsoc = (int)nsoc;
  P.m = (int)m;
  P.soc_ptr = L.soc_ptr;
  i64 wtw_tile = QS_WTW_TILE;
  if (const char* e = getenv("QS_WTW_TILE")) wtw_tile = std::max(256, atoi(e));  // tuning knob
  std::vector<int> cone_of_col(m - l), tile_ptr;
  std::vector<i64> slot_start(nsoc);
  i64 slot = l, acc = 0;
  tile_ptr.push_back((int)l);
  int max_cols = 1, max_window = 1, tile_first_cone_start = (int)l;
  auto close_tile = [&](int end_col) {
    max_cols = std::max(max_cols, end_col - tile_ptr.back());
    max_window = std::max(max_window, end_col - tile_first_cone_start);
    tile_ptr.push_back(end_col);
    acc = 0;
  };
  for (i64 k = 0; k < nsoc; ++k) {
    slot_start[k] = slot;
    slot += q[k] * (q[k] + 1) / 2;
    for (i64 j = 0; j < q[k]; ++j) {
      const int col = ptr[k] + (int)j;
      if (col == tile_ptr.back()) tile_first_cone_start = ptr[k];  // first column of a new tile
      cone_of_col[col - l] = (int)k;
      acc += j + 1;
      if (acc >= wtw_tile || col + 1 - tile_ptr.back() >= QS_WTW_MAXCOLS) close_tile(col + 1);
    }
  }
  if (tile_ptr.back() != (int)m) close_tile((int)m);
  P.max_tile_cols = max_cols;
  P.max_tile_window = max_window;
  h->S = slot;
  P.ntiles = (int)tile_ptr.size() - 1;
  P.cone_of_col = h->cone_pool.upload(cone_of_col.data(), cone_of_col.size(), h->stream);
  P.tile_ptr = h->cone_pool.upload(tile_ptr.data(), tile_ptr.size(), h->stream);
  h->d_slot_start = h->cone_pool.upload(slot_start.data(), slot_start.size(), h->stream);
  P.slot_start = h->d_slot_start;
  P.kp_conic = nullptr;
  P.g_ptr = nullptr;
  P.g_val = nullptr;
  // staged variant, dense-slot output: tiles of <= QS_WTW_STAGE packed slots
  std::vector<int> st_ptr;  // outlives the stream synchronisation below
  {
    st_ptr.push_back((int)l);
    i64 run = 0;
    for (i64 k = 0; k < nsoc; ++k)
      for (i64 j = 0; j < q[k]; ++j) {
        if (run + j + 1 > QS_WTW_STAGE || ptr[k] + (int)j - st_ptr.back() >= QS_WTW_SCOLS) {
          st_ptr.push_back(ptr[k] + (int)j);
          run = 0;
        }
        run += j + 1;
      }
    if (st_ptr.back() != (int)m) st_ptr.push_back((int)m);
    bool fits = true;  // a single column longer than the stage cannot be staged
    for (i64 k = 0; k < nsoc; ++k) fits = fits && q[k] <= QS_WTW_STAGE;
    P.n_stiles_slots = fits ? (int)st_ptr.size() - 1 : 0;
    P.stile_ptr = fits ? h->cone_pool.upload(st_ptr.data(), st_ptr.size(), h->stream) : nullptr;
    P.stile_ptr_direct = nullptr;
    P.n_stiles_direct = 0;
    P.kstart = nullptr;
  }
  P.c4 = h->cone_pool.alloc<double>(nsoc);
  P.e2 = h->cone_pool.alloc<double>(nsoc);
  h->cone_tmp = h->cone_pool.alloc<double>(m);
  CK(h, cudaStreamSynchronize(h->stream));
  if (!L.soc_ptr || !P.cone_of_col || !P.tile_ptr || !P.c4 || !P.e2 || !h->cone_tmp ||
      (!small_ids.empty() && !L.small_ids))
    return fail(h, QS_E_MEMORY, "cone layout alloc");
  h->have_cones = true;
  return QS_OK;
}

// ------------------------------------------------------- per-kernel entries
#define NEED_CONES(h)                                                       \
  if (!(h) || !(h)->have_cones) return (h) ? fail(h, QS_E_INVALID, "qs_set_cones first") : QS_E_INVALID; \
  cudaSetDevice((h)->device);

int qs_nt_scaling(qs_handle* h, const double* s, const double* z, double* w, double* eta, double* wbar, double* lam,
                  double* lam_sq, int* not_interior_host) {
  NEED_CONES(h)
  if (not_interior_host) cudaMemsetAsync(h->scalars + SC_FLAG_NOT_INTERIOR, 0, sizeof(double), h->stream);
  qsk_nt_scaling(h->L, s, z, w, eta, wbar, lam, lam_sq, nullptr, nullptr, nullptr, nullptr, nullptr, h->scalars,
                 h->stream);
  h->launches++;
  int rc = check_launch(h, "nt_scaling");
  if (rc || !not_interior_host) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  *not_interior_host = h->scalars_host[SC_FLAG_NOT_INTERIOR] != 0.0;
  return QS_OK;
}

int qs_apply_w(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* u, double* out,
               int inverse) {
  NEED_CONES(h)
  qsk_apply_w(h->L, w, eta, wbar, u, out, inverse, h->stream);
  h->launches++;
  return check_launch(h, "apply_w");
}

int qs_jordan_product(qs_handle* h, const double* u, const double* v, double* out) {
  NEED_CONES(h)
  qsk_jordan_product(h->L, u, v, out, h->stream);
  h->launches++;
  return check_launch(h, "jordan_product");
}

int qs_jordan_divide(qs_handle* h, const double* lam, const double* v, double* out) {
  NEED_CONES(h)
  qsk_jordan_divide(h->L, lam, v, out, h->stream);
  h->launches++;
  return check_launch(h, "jordan_divide");
}

int qs_max_step(qs_handle* h, const double* u, const double* du, double* step_host, double* violation_host) {
  NEED_CONES(h)
  qsk_max_step(h->L, u, du, h->scalars, SC_TMP0, SC_TMP1, h->gr, h->stream);
  h->launches++;
  int rc = check_launch(h, "max_step");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  if (step_host) *step_host = h->scalars_host[SC_TMP0];
  if (violation_host) *violation_host = h->scalars_host[SC_TMP1];
  return QS_OK;
}

int qs_bring_to_interior(qs_handle* h, const double* u, double scale, double* out, double* alpha_host) {
  NEED_CONES(h)
  // violation of scale*u, then the shift (cones.py:302-311)
  double* t = h->cone_tmp;
  qsk_axpby(h->L.m, scale, u, 0.0, nullptr, t, h->stream);
  qsk_max_step(h->L, t, nullptr, h->scalars, -1, SC_SHIFT, h->gr, h->stream);
  qsk_shift(h->L, t, out, h->scalars, SC_SHIFT, 1.0, h->stream);
  h->launches += 3;
  int rc = check_launch(h, "bring_to_interior");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (alpha_host) *alpha_host = h->scalars_host[SC_SHIFT];
  return rc;
}

int qs_compute_mu(qs_handle* h, const double* s, const double* z, double* mu_host) {
  NEED_CONES(h)
  qsk_dot(h->L.m, s, z, 1.0 / h->deg, h->scalars + SC_TMP0, h->gr, h->stream);
  h->launches++;
  int rc = check_launch(h, "compute_mu");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (mu_host) *mu_host = h->scalars_host[SC_TMP0];
  return rc;
}

int qs_neg_wtw(qs_handle* h, int mode, const double* w, const double* eta, const double* wbar,
               const int64_t* soc_slot_starts_dev, const int64_t* positions_dev, const int64_t* kp_conic_dev,
               double* out) {
  NEED_CONES(h)
  if (mode < 0 || mode > 2) return fail(h, QS_E_INVALID, "mode must be 0, 1 or 2");
  WtwPlan P = h->wp;
  if (soc_slot_starts_dev) P.slot_start = (const i64*)soc_slot_starts_dev;
  if (mode == 1 && !positions_dev) return fail(h, QS_E_INVALID, "mode 1 needs the positions map");
  if (mode == 2) {
    if (!kp_conic_dev) return fail(h, QS_E_INVALID, "mode 2 needs kp_conic");
    P.kp_conic = (const i64*)kp_conic_dev;
  }
  qsk_neg_wtw(P, mode, w, eta, wbar, (const i64*)positions_dev, out, h->stream);
  h->launches += 2;
  return check_launch(h, "neg_wtw");
}

// ---- the fused per-iteration kernels on caller-owned device vectors (vector-level parity tests, ncu)
// predictor_rhs: compute_nt_scaling + lam o lam + d = lam \ (-lam o lam) + rhs_z = -r_cone - W d
// (cones.py:159-184, ipm.py:180-184,191-192) -- the first cone kernel of qs_step.
int qs_predictor_rhs(qs_handle* h, const double* s, const double* z, const double* r_cone, double* w, double* eta,
                     double* wbar, double* lam, double* lam_sq, double* d, double* rhs_z, int* not_interior_host) {
  NEED_CONES(h)
  cudaMemsetAsync(h->scalars + SC_FLAG_NOT_INTERIOR, 0, sizeof(double), h->stream);
  qsk_nt_scaling(h->L, s, z, w, eta, wbar, lam, lam_sq, h->wp.c4, h->wp.e2, r_cone, d, rhs_z, h->scalars, h->stream);
  h->launches++;
  int rc = check_launch(h, "predictor_rhs");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  if (not_interior_host) *not_interior_host = h->scalars_host[SC_FLAG_NOT_INTERIOR] != 0.0;
  return QS_OK;
}

// corrector_rhs: d_comp = sigma mu e - lam o lam - (W^-1 ds_a) o (W dz_a), d = lam \ d_comp,
// rhs_z = -r_cone - W d (ipm.py:180-184,209-212).  dcomp may be null.
int qs_corrector_rhs(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* lam,
                     const double* lam_sq, const double* ds_a, const double* wdz_a, const double* r_cone, double sigma,
                     double mu, double* dcomp, double* d, double* rhs_z) {
  NEED_CONES(h)
  h->scalars_host[SC_SIGMA] = sigma;
  h->scalars_host[SC_MU] = mu;
  CK(h, cudaMemcpyAsync(h->scalars + SC_SIGMA, h->scalars_host + SC_SIGMA, sizeof(double), cudaMemcpyHostToDevice,
                        h->stream));
  CK(h, cudaMemcpyAsync(h->scalars + SC_MU, h->scalars_host + SC_MU, sizeof(double), cudaMemcpyHostToDevice, h->stream));
  qsk_corrector_rhs(h->L, w, eta, wbar, lam, lam_sq, ds_a, wdz_a, r_cone, dcomp, d, rhs_z, h->scalars, h->stream);
  h->launches++;
  CK(h, cudaStreamSynchronize(h->stream));  // the pinned mirror is reused by the next fetch
  return check_launch(h, "corrector_rhs");
}

// post_solve: wdz = W dz, ds = W (d - W dz), max_step_to_boundary of (s, ds) and (z, dz) with the interior
// pre-check; predictor (corrector = 0): alpha_aff, mu_aff, mu = s'z/deg, sigma; corrector: alpha
// (ipm.py:187-188,195-206,214-218).  out8 = {step_s, step_z, alpha_aff, alpha, mu, mu_aff, sigma, flags}.
int qs_post_solve(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* d,
                  const double* dz, const double* s, const double* z, int corrector, double step_fraction, double* wdz,
                  double* ds, double* out8_host) {
  NEED_CONES(h)
  clear_flags(h);
  qsk_post_solve(h->L, w, eta, wbar, d, dz, s, z, wdz, ds, h->scalars, corrector, step_fraction, h->deg, h->gr,
                 h->stream);
  h->launches++;
  int rc = check_launch(h, "post_solve");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  if (out8_host) {
    const double* sc = h->scalars_host;
    const double o[8] = {sc[SC_STEP_S], sc[SC_STEP_Z], sc[SC_ALPHA_AFF], sc[SC_ALPHA],
                         sc[SC_MU],     sc[SC_MU_AFF], sc[SC_SIGMA],     (double)flags_of(sc)};
    for (int k = 0; k < 8; ++k) out8_host[k] = o[k];
  }
  return QS_OK;
}

// update_iterate: (x, y, z, s) + alpha (dx, dy, dz, ds) with sol = (dx, dy, dz), the finite check and the new
// mu = s'z/deg (ipm.py:219-234).  out2 = {mu, flags}.
int qs_update_iterate(qs_handle* h, int64_t n, int64_t p, const double* x, const double* y, const double* z,
                      const double* s, const double* sol, const double* ds, double alpha, double* xo, double* yo,
                      double* zo, double* so, double* out2_host) {
  NEED_CONES(h)
  clear_flags(h);
  h->scalars_host[SC_ALPHA] = alpha;
  CK(h, cudaMemcpyAsync(h->scalars + SC_ALPHA, h->scalars_host + SC_ALPHA, sizeof(double), cudaMemcpyHostToDevice,
                        h->stream));
  qsk_update_iterate((int)n, (int)p, h->L.m, x, y, z, s, xo, yo, zo, so, sol, ds, h->deg, h->scalars, h->gr, h->stream);
  h->launches++;
  int rc = check_launch(h, "update_iterate");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  if (out2_host) {
    out2_host[0] = h->scalars_host[SC_MU];
    out2_host[1] = (double)flags_of(h->scalars_host);
  }
  return QS_OK;
}

int qs_spmv_csr(qs_handle* h, int64_t rows, int64_t cols, const int32_t* ptr, const int32_t* idx, const double* val,
                const double* x, double* y, int accumulate) {
  if (!h) return QS_E_INVALID;
  cudaSetDevice(h->device);
  int nnz_last = 0;
  CK(h, cudaMemcpyAsync(&nnz_last, ptr + rows, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  Csr M{(int)rows, (int)cols, ptr, idx, val, qsk_pick_tpr(nnz_last, rows), 0};
  qsk_spmv_csr(M, x, y, accumulate, h->stream);
  h->launches++;
  return check_launch(h, "spmv_csr");
}

int qs_spmv_sym_upper(qs_handle* h, int64_t ncols, const int64_t* colptr, const int32_t* rowidx, const double* val,
                      const double* x, double* out) {
  if (!h) return QS_E_INVALID;
  cudaSetDevice(h->device);
  qsk_spmv_sym_upper_csc((int)ncols, (const i64*)colptr, rowidx, val, x, out, h->stream);
  h->launches++;
  return check_launch(h, "spmv_sym_upper");
}

// ------------------------------------------------------------------- setup
int qs_setup(qs_handle* h, int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q,
             const int64_t* Pp, const int64_t* Pi, const double* Px, const int64_t* Ap, const int64_t* Ai,
             const double* Ax, const int64_t* Gp, const int64_t* Gi, const double* Gx, const double* c,
             const double* b, const double* hvec, const qs_settings* settings, const int64_t* user_perm) {
  if (!h || !settings) return QS_E_INVALID;
  if (h->have_problem) return fail(h, QS_E_INVALID, "handle already set up");
  cudaSetDevice(h->device);
  const auto t_begin = std::chrono::steady_clock::now();
  auto t_mark = t_begin;
  const bool verbose = getenv("QS_VERBOSE") != nullptr;
  auto lap = [&](const char* what) {
    if (verbose) {
      cudaStreamSynchronize(h->stream);
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[qs setup] %-32s %8.3f s\n", what, std::chrono::duration<double>(now - t_mark).count());
      t_mark = now;
    }
  };
  h->st = *settings;
  if (n < 1 || m < 1 || p < 0) return fail(h, QS_E_DIMENSION, "need n >= 1, m >= 1, p >= 0");
  int rc = qs_set_cones(h, l, nsoc, q, 0);
  if (rc) return rc;
  if (h->L.m != m) return fail(h, QS_E_DIMENSION, "cone dimensions do not sum to m");
  h->n = n;
  h->p = p;
  h->m = m;
  h->N = n + p + m;
  const i64 N = h->N;
  cudaStream_t st = h->stream;
  lap("cone layout + plans");
  // ---- row views
  const i64 nnzA = Ap[n], nnzG = Gp[n], nnzP = Pp[n];
  std::vector<i64> Arp(p + 1), Ari(nnzA), Grp(m + 1), Gri(nnzG);
  std::vector<double> Arx(nnzA), Grx(nnzG);
  // one transpose per matrix: the INDEX vector goes through it (where does every entry of the row view come from --
  // kept for value-only updates), the values follow by a gather
  std::vector<int> ar_map(nnzA), gr_map(nnzG);
  {
    std::vector<double> iota(std::max(nnzA, nnzG));
    for (size_t k = 0; k < iota.size(); ++k) iota[k] = (double)k;
    hs_transpose(p, n, (const i64*)Ap, (const i64*)Ai, iota.data(), Arp.data(), Ari.data(), Arx.data());
    for (i64 k = 0; k < nnzA; ++k) {
      ar_map[k] = (int)Arx[k];
      Arx[k] = Ax[ar_map[k]];
    }
    hs_transpose(m, n, (const i64*)Gp, (const i64*)Gi, iota.data(), Grp.data(), Gri.data(), Grx.data());
    for (i64 k = 0; k < nnzG; ++k) {
      gr_map[k] = (int)Grx[k];
      Grx[k] = Gx[gr_map[k]];
    }
  }
  // Pf = P + P' - diag(P), rows ascending
  std::vector<i64> Pfp(n + 1, 0);
  for (i64 j = 0; j < n; ++j)
    for (i64 k = Pp[j]; k < Pp[j + 1]; ++k) {
      const i64 i = Pi[k];
      if (i > j) return fail(h, QS_E_INVALID, "P has an entry below the diagonal");
      Pfp[i + 1]++;
      if (i != j) Pfp[j + 1]++;
    }
  for (i64 r = 0; r < n; ++r) Pfp[r + 1] += Pfp[r];
  std::vector<i64> Pfi(Pfp[n]);
  std::vector<double> Pfx(Pfp[n]);
  std::vector<int> pf_map(Pfp[n]);
  {
    std::vector<i64> next(Pfp.begin(), Pfp.end() - 1);
    for (i64 j = 0; j < n; ++j) {
      for (i64 k = Pp[j]; k < Pp[j + 1]; ++k) {  // row j receives its cols i < j (and the diagonal)
        const i64 i = Pi[k];
        Pfi[next[j]] = i;
        pf_map[next[j]] = (int)k;
        Pfx[next[j]++] = Px[k];
      }
      for (i64 k = Pp[j]; k < Pp[j + 1]; ++k) {  // rows i < j receive col j
        const i64 i = Pi[k];
        if (i == j) continue;
        Pfi[next[i]] = j;
        pf_map[next[i]] = (int)k;
        Pfx[next[i]++] = Px[k];
      }
    }
  }
  lap("row views + value maps (host)");
  h->nnzP = nnzP;
  h->nnzPf = Pfp[n];
  h->nnzA = nnzA;
  h->nnzG = nnzG;
  // ---- KKT system: column pointers + compact pattern on the host (O(N + nnz(P,A,G))); the 10^8 entries
  // themselves (row indices, initial values, slot -> position map) are written by the device (qsk_kkt_fill).
  // QS_HOST_ASSEMBLY=1 keeps the original host assembly + upload as the checked alternative.
  KktDims dims{n, p, m, l, nsoc, (const i64*)q};
  h->knnz = hs_kkt_nnz(dims, (const i64*)Pp, (const i64*)Pi, nnzA, nnzG);
  if (h->knnz >= ((i64)1 << 31)) return fail(h, QS_E_DIMENSION, "KKT nonzeros exceed 2^31");
  const bool host_assembly = getenv("QS_HOST_ASSEMBLY") != nullptr;
  h->Kp_h.resize(N + 1);
  std::vector<i64> Kcp, Kci;  // compact pattern for the analysis
  std::vector<i64> Ki_full, pos_full;
  std::vector<double> Kx_full;
  if (host_assembly) {
    Ki_full.resize(h->knnz);
    Kx_full.resize(h->knnz);
    pos_full.resize(h->S);
    std::vector<i64> soc_starts(nsoc), view_off(nsoc + 2);
    hs_kkt_assemble(dims, (const i64*)Pp, (const i64*)Pi, Px, Arp.data(), Ari.data(), Arx.data(), Grp.data(),
                    Gri.data(), Grx.data(), h->Kp_h.data(), Ki_full.data(), Kx_full.data(), pos_full.data(),
                    view_off.data(), soc_starts.data());
  } else {
    hs_kkt_pattern(dims, (const i64*)Pp, (const i64*)Pi, Arp.data(), Ari.data(), Grp.data(), Gri.data(),
                   h->Kp_h.data(), &Kcp, &Kci);
    if (h->Kp_h[N] != h->knnz) return fail(h, QS_E_INVALID, "internal: KKT column pointers disagree with the count");
  }
  lap("KKT column pointers + compact pattern");
  const auto t_h2d = std::chrono::steady_clock::now();
  bool ok = make_csr(h, &h->Pf, n, n, Pfp.data(), Pfi.data(), Pfx.data()) &&
            make_csr(h, &h->At, n, p, (const i64*)Ap, (const i64*)Ai, Ax) &&
            make_csr(h, &h->Gt, n, m, (const i64*)Gp, (const i64*)Gi, Gx) &&
            make_csr(h, &h->Ar, p, n, Arp.data(), Ari.data(), Arx.data()) &&
            make_csr(h, &h->Gr, m, n, Grp.data(), Gri.data(), Grx.data());
  if (!ok) return fail(h, QS_E_MEMORY, "out of device memory for the problem matrices");
  // one lane-group width for the whole dual range (three products per row)
  h->Pf.tpr = std::min(32, qsk_pick_tpr(std::max(std::max(nnzP * 2, nnzA), nnzG), n));  // no CTA-per-row mode here
  h->At.tpr = h->Gt.tpr = h->Pf.tpr;
  if (h->Ar.tpr >= 256 && p > 0) {  // CTA-per-row class: the residual's equality range uses the split product
    h->seg_partial = h->prob_pool.alloc<double>((size_t)p * QS_ROW_SEGS);
    if (!h->seg_partial) return fail(h, QS_E_MEMORY, "out of device memory for the row-segment partials");
  }
  if (h->Pf.tpr == 1 && n < (1 << QS_DT_TAG_SHIFT) && p < (1 << QS_DT_TAG_SHIFT) && m < (1 << QS_DT_TAG_SHIFT) &&
      Pfp[n] + nnzA + nnzG < ((i64)1 << 31) && std::max(std::max(Pfp[n], nnzA), nnzG) < (1 << QS_DT_TAG_SHIFT)) {
    // short rows: the dual range reads ONE matrix [Pf | A' | G'] (tagged indices) instead of three; built on the
    // device from the row views uploaded above
    const i64 nd = Pfp[n] + nnzA + nnzG;
    int* dp = h->prob_pool.alloc<int>(n + 1);
    int* di = h->prob_pool.alloc<int>(nd);
    double* dv = h->prob_pool.alloc<double>(nd);
    h->dt_map = h->prob_pool.alloc<int>(nd);
    h->Dt.rows = (int)n;
    h->Dt.cols = (int)(n + p + m);
    h->Dt.ptr = dp;
    h->Dt.idx = di;
    h->Dt.val = dv;
    h->Dt.tpr = 1;
    h->Dt.exact1 = 0;
    h->nnzDt = nd;
    if (dp && di && dv && h->dt_map) {
      qsk_build_dt((int)n, h->Pf, h->At, h->Gt, dp, di, dv, h->dt_map, st);
      h->launches++;
    }
    if (!h->Dt.ptr || !h->Dt.idx || !h->Dt.val || !h->dt_map) return fail(h, QS_E_MEMORY, "out of device memory for the fused dual-range matrix");
  }
  h->c = h->prob_pool.upload(c, n, st);
  h->b = h->prob_pool.upload(b, p, st);
  h->hv = h->prob_pool.upload(hvec, m, st);
  h->norm_c = inf_norm(c, n);
  h->norm_b = inf_norm(b, p);
  h->norm_h = inf_norm(hvec, m);
  h->d_Kp = h->prob_pool.upload(h->Kp_h.data(), h->Kp_h.size(), st);
  if (host_assembly) {
    std::vector<int> ki32 = to_i32(Ki_full.data(), Ki_full.size());
    h->d_Ki = h->prob_pool.upload(ki32.data(), ki32.size(), st);
    h->d_Kx = h->prob_pool.upload(Kx_full.data(), Kx_full.size(), st);
    h->d_pos = h->prob_pool.upload(pos_full.data(), pos_full.size(), st);
    CK(h, cudaStreamSynchronize(st));
  } else {
    Csr& Pu = h->Pu;
    if (!make_csr(h, &Pu, n, n, (const i64*)Pp, (const i64*)Pi, Px))  // CSC of upper(P) = CSR of its transpose
      return fail(h, QS_E_MEMORY, "out of device memory for P");
    h->ar_map = h->prob_pool.upload(ar_map.data(), ar_map.size(), st);
    h->gr_map = h->prob_pool.upload(gr_map.data(), gr_map.size(), st);
    h->pf_map = h->prob_pool.upload(pf_map.data(), pf_map.size(), st);
    if (!h->ar_map || !h->gr_map || !h->pf_map) return fail(h, QS_E_MEMORY, "out of device memory for the value maps");
    h->d_Ki = h->prob_pool.alloc<int>(h->knnz);
    h->d_Kx = h->prob_pool.alloc<double>(h->knnz);
    h->d_pos = h->prob_pool.alloc<i64>(h->S);
    if (h->d_Kp && h->d_Ki && h->d_Kx && h->d_pos) {
      WtwPlan plan = h->wp;
      plan.slot_start = h->d_slot_start;
      qsk_kkt_fill(plan, (int)n, (int)p, Pu, h->Ar, h->Gr, h->d_Kp, h->d_Ki, h->d_Kx, h->d_pos, st);
      h->launches++;
      CK(h, cudaStreamSynchronize(st));
    }
  }
  if (!h->c || !h->b || !h->hv || !h->d_Kp || !h->d_Ki || !h->d_Kx || !h->d_pos)
    return fail(h, QS_E_MEMORY, "out of device memory for the KKT system");
  h->wp.kp_conic = h->d_Kp + n + p + 1;
  h->wp.g_ptr = h->Gr.ptr;
  h->wp.g_val = h->Gr.val;
  // staged variant, in-place output: tiles of whole conic K columns (G' entries + block entries) whose run
  // [Kp[n+p+c0], Kp[n+p+c1]) fits the stage; only when every conic column is exactly that union
  {
    const i64* kp = h->Kp_h.data() + n + p;
    bool whole = true;
    std::vector<int> st_ptr;
    st_ptr.push_back((int)l);
    i64 run_begin = kp[l];
    for (i64 k = 0; k < nsoc && whole; ++k) {
      const i64 o = h->soc_ptr_host[k];
      for (i64 j = 0; j < q[k]; ++j) {
        const i64 c = o + j, len = kp[c + 1] - kp[c];
        if (len != (Grp[c + 1] - Grp[c]) + j + 1 || len > QS_WTW_STAGE) {
          whole = false;
          break;
        }
        if (kp[c + 1] - run_begin > QS_WTW_STAGE || c - st_ptr.back() >= QS_WTW_SCOLS) {
          st_ptr.push_back((int)c);
          run_begin = kp[c];
        }
      }
    }
    if (st_ptr.back() != (int)m) st_ptr.push_back((int)m);
    if (whole && nsoc > 0) {
      h->wp.stile_ptr_direct = h->prob_pool.upload(st_ptr.data(), st_ptr.size(), st);
      h->wp.n_stiles_direct = (int)st_ptr.size() - 1;
      h->wp.kstart = h->d_Kp + n + p;
      CK(h, cudaStreamSynchronize(st));
    }
  }
  lap("H2D of P/A/G views + device KKT fill");
  // closed-form map == explicit map?
  {
    int* flag = h->prob_pool.alloc<int>(1);
    cudaMemsetAsync(flag, 0, sizeof(int), st);
    qsk_check_direct_map(h->wp, h->d_pos, flag, st);
    int bad = 1;
    CK(h, cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    h->direct_ok = (bad == 0);
  }
  // ---- state vectors
  DevPool& P = h->prob_pool;
#define ALLOC(field, count)                  \
  h->field = P.alloc<double>(count);         \
  if (!h->field) return fail(h, QS_E_MEMORY, "out of device memory for the iterate");
  ALLOC(x, n) ALLOC(y, p) ALLOC(z, m) ALLOC(s, m)
  ALLOC(x2, n) ALLOC(y2, p) ALLOC(z2, m) ALLOC(s2, m)
  ALLOC(w, l) ALLOC(eta, nsoc) ALLOC(wbar, m) ALLOC(lam, m) ALLOC(lam_sq, m)
  ALLOC(d, m) ALLOC(dcomp, m) ALLOC(wdz, m) ALLOC(ds, m) ALLOC(r_cone, m) ALLOC(w2vz, m) ALLOC(tmp_m, m)
  ALLOC(rhs, N) ALLOC(xa, N) ALLOC(xb, N) ALLOC(ra, N) ALLOC(rb, N) ALLOC(dx, N)
#undef ALLOC
  cudaMemsetAsync(h->wbar, 0, m * sizeof(double), st);
  h->sol = h->xa;
  if (h->st.ruiz_iters > 0) {
    std::vector<double> ones(std::max<i64>(std::max<i64>(n, p), m), 1.0);
    h->rD = P.upload(ones.data(), n, st);
    h->rE = P.upload(ones.data(), p, st);
    h->rF = P.upload(ones.data(), m, st);
    if (!h->rD || !h->rE || !h->rF) return fail(h, QS_E_MEMORY, "out of device memory for the Ruiz scalings");
    RuizArgs R{(int)n, (int)p, (int)m, h->L.nsoc, h->L.soc_ptr, h->Pf, h->At, h->Gt, h->Ar, h->Gr, h->rD, h->rE, h->rF};
    qsk_ruiz(R, (int)h->st.ruiz_iters, h->xa, h->xa + n, h->xa + n + p, st);
    qsk_ruiz_apply(R, h->d_Kp, h->d_Ki, h->d_Kx, h->c, h->b, h->hv, st);
    if (h->Dt.ptr) qsk_gather3(h->nnzDt, h->Pf.val, h->At.val, h->Gt.val, h->dt_map, const_cast<double*>(h->Dt.val), st);
    // norms of the scaled data feed the termination test
    std::vector<double> hc(n), hb(p), hh(m);
    CK(h, cudaMemcpyAsync(hc.data(), h->c, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(h, cudaMemcpyAsync(hb.data(), h->b, p * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(h, cudaMemcpyAsync(hh.data(), h->hv, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    h->norm_c = inf_norm(hc.data(), n);
    h->norm_b = inf_norm(hb.data(), p);
    h->norm_h = inf_norm(hh.data(), m);
    h->launches += 6 * h->st.ruiz_iters + 9;
  }
  h->tm.total[T_H2D] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_h2d).count();
  lap("map check + state vectors (+ Ruiz)");
  // ---- factorisation analysis; the SOC blocks are cliques of the pattern
  std::vector<i64> cstart(nsoc), csize(nsoc);
  for (i64 k = 0; k < nsoc; ++k) {
    cstart[k] = n + p + h->soc_ptr_host[k];
    csize[k] = q[k];
  }
  const i64* an_p = host_assembly ? h->Kp_h.data() : Kcp.data();
  const i64* an_i = host_assembly ? Ki_full.data() : Kci.data();
  std::string err = h->ls.analyze(N, an_p, an_i, h->knnz, h->d_Kp, h->d_Ki, (int)h->st.ordering,
                                  (const i64*)user_perm, nsoc, cstart.data(), csize.data(), n, h->st.static_reg, st);
  if (!err.empty()) return fail(h, err.find("memory") != std::string::npos ? QS_E_MEMORY : QS_E_INVALID, err);
  if (h->direct_ok && nsoc > 0 && h->wp.kp_conic) {  // closed-form block positions hold: tiled K -> panel scatter
    err = h->ls.set_cone_blocks((int)(n + p), (int)l, (int)nsoc, (const i64*)q, h->L.soc_ptr, h->wp.kp_conic,
                                h->wp.cone_of_col, h->d_Kp, h->Kp_h[n + p + l], st);
    if (!err.empty()) return fail(h, QS_E_MEMORY, err);
  }
  h->tm.total[T_ANALYSIS] += h->ls.analysis_seconds;
  lap("ordering + symbolic + LDL' setup");
  h->have_problem = true;
  (void)t_begin;
  return QS_OK;
}

#define NEED_PROBLEM(h)                                                                                     \
  if (!(h) || !(h)->have_problem) return (h) ? fail(h, QS_E_INVALID, "qs_setup first") : QS_E_INVALID;       \
  cudaSetDevice((h)->device);

// Same sparsity pattern, new numbers (parametric re-solve).  Any pointer may be null (= unchanged).
// Keeps the row views' structure, the KKT pattern, the ordering, the symbolic analysis, the assembly lists and the
// captured launch graphs; re-uploads the values (host -> device: exactly the arrays given), regathers the row
// views on the device and rewrites the KKT values.  The next qs_initialize_iterate starts a fresh solve.
int qs_update_values(qs_handle* h, const double* Px, const double* Ax, const double* Gx, const double* c,
                     const double* b, const double* hvec) {
  NEED_PROBLEM(h)
  if (h->rD) return fail(h, QS_E_INVALID, "qs_update_values with ruiz_iters > 0 is not supported");
  if (!h->pf_map) return fail(h, QS_E_INVALID, "qs_update_values needs the device-assembled KKT path");
  cudaStream_t st = h->stream;
  const i64 n = h->n, p = h->p, m = h->m;
  auto up = [&](const double* src, const double* dst, i64 count) {
    if (count > 0) cudaMemcpyAsync(const_cast<double*>(dst), src, count * sizeof(double), cudaMemcpyHostToDevice, st);
    h->h2d_extra += count * (i64)sizeof(double);
  };
  if (Px) {
    i64 nnzP = 0, nnzPf = 0;
    nnzP = h->nnzP;
    nnzPf = h->nnzPf;
    up(Px, h->Pu.val, nnzP);
    qsk_gather(nnzPf, h->Pu.val, h->pf_map, const_cast<double*>(h->Pf.val), st);
  }
  if (Ax) {
    up(Ax, h->At.val, h->nnzA);
    qsk_gather(h->nnzA, h->At.val, h->ar_map, const_cast<double*>(h->Ar.val), st);
  }
  if (Gx) {
    up(Gx, h->Gt.val, h->nnzG);
    qsk_gather(h->nnzG, h->Gt.val, h->gr_map, const_cast<double*>(h->Gr.val), st);
  }
  if (c) {
    up(c, h->c, n);
    h->norm_c = inf_norm(c, n);
  }
  if (b) {
    up(b, h->b, p);
    h->norm_b = inf_norm(b, p);
  }
  if (hvec) {
    up(hvec, h->hv, m);
    h->norm_h = inf_norm(hvec, m);
  }
  if (Px || Ax || Gx) {
    WtwPlan plan = h->wp;
    plan.slot_start = h->d_slot_start;
    qsk_kkt_fill(plan, (int)n, (int)p, h->Pu, h->Ar, h->Gr, h->d_Kp, h->d_Ki, h->d_Kx, h->d_pos, st);
    if (h->Dt.ptr) qsk_gather3(h->nnzDt, h->Pf.val, h->At.val, h->Gt.val, h->dt_map, const_cast<double*>(h->Dt.val), st);
    h->launches += 5;
  }
  h->factored = false;
  CK(h, cudaStreamSynchronize(st));  // the caller's buffers may be released on return
  return check_launch(h, "update_values");
}

int64_t qs_kkt_size(qs_handle* h, int64_t* nnz, int64_t* slots) {
  if (!h || !h->have_problem) return -1;
  if (nnz) *nnz = h->knnz;
  if (slots) *slots = h->S;
  return h->N;
}

int qs_get_kkt(qs_handle* h, int64_t* Kp, int64_t* Ki, double* Kx, int64_t* positions) {
  NEED_PROBLEM(h)
  if (Kp) memcpy(Kp, h->Kp_h.data(), h->Kp_h.size() * sizeof(i64));
  if (Ki) {  // the device keeps int32 row indices; the reference contract is int64
    std::vector<int> ki32(h->knnz);
    CK(h, cudaMemcpyAsync(ki32.data(), h->d_Ki, h->knnz * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    for (i64 k = 0; k < h->knnz; ++k) Ki[k] = ki32[k];
  }
  if (positions) {
    CK(h, cudaMemcpyAsync(positions, h->d_pos, h->S * sizeof(i64), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
  }
  if (Kx) {  // current device values
    CK(h, cudaMemcpyAsync(Kx, h->d_Kx, h->knnz * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
  }
  return QS_OK;
}

int qs_linsys_update_identity(qs_handle* h) {
  NEED_PROBLEM(h)
  // identity_scaling (cones.py:146-156): w = 1, eta = 1, wbar = e on the SOC heads, lam = e
  std::vector<double> one(std::max<i64>(std::max<i64>(h->L.l, h->L.nsoc), 1), 1.0), e(h->m, 0.0);
  for (int k = 0; k < h->L.nsoc; ++k) e[h->soc_ptr_host[k]] = 1.0;
  CK(h, cudaMemcpyAsync(h->w, one.data(), h->L.l * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(h->eta, one.data(), h->L.nsoc * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(h->wbar, e.data(), h->m * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  for (int i = 0; i < h->L.l; ++i) e[i] = 1.0;
  CK(h, cudaMemcpyAsync(h->lam, e.data(), h->m * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  h->h2d_extra += (h->L.l + h->L.nsoc + 2 * h->m) * (i64)sizeof(double);
  int rc = scatter_scaling(h, h->w, h->eta, h->wbar);
  CK(h, cudaStreamSynchronize(h->stream));
  return rc;
}

int qs_linsys_update(qs_handle* h) {
  NEED_PROBLEM(h)
  return scatter_scaling(h, h->w, h->eta, h->wbar);
}

int qs_linsys_factor(qs_handle* h) {
  NEED_PROBLEM(h)
  return do_factor(h);
}

int qs_linsys_solve(qs_handle* h, const double* rhs_host, double* sol_host) {
  NEED_PROBLEM(h)
  if (!h->factored) return fail(h, QS_E_INVALID, "factor() must run before solve()");
  CK(h, cudaMemcpyAsync(h->rhs, rhs_host, h->N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  int rc = solve_refined(h, h->rhs);
  if (rc) return rc;
  CK(h, cudaMemcpyAsync(sol_host, h->sol, h->N * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  for (i64 k = 0; k < h->N; ++k)
    if (!(fabs(sol_host[k]) <= DBL_MAX)) return fail(h, QS_E_NUMERICAL, "non-finite linear-system solution");
  return QS_OK;
}

// initialize_iterate (ipm.py:135-156)
int qs_initialize_iterate(qs_handle* h, double* mu_host) {
  NEED_PROBLEM(h)
  cudaStream_t st = h->stream;
  const i64 n = h->n, p = h->p, m = h->m;
  clear_flags(h);
  int rc = qs_linsys_update_identity(h);
  if (rc) return rc;
  rc = do_factor(h);
  if (rc) return rc;
  // rhs = (-c, b, h)
  qsk_axpby(n, -1.0, h->c, 0.0, nullptr, h->rhs, st);
  CK(h, cudaMemcpyAsync(h->rhs + n, h->b, p * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(h, cudaMemcpyAsync(h->rhs + n + p, h->hv, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  rc = solve_refined(h, h->rhs);
  if (rc) return rc;
  CK(h, cudaMemcpyAsync(h->x, h->sol, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(h, cudaMemcpyAsync(h->y, h->sol + n, p * sizeof(double), cudaMemcpyDeviceToDevice, st));
  // s = bring_to_interior(-z~)
  h->tm.begin(T_CONE, st);
  qsk_axpby(m, -1.0, h->sol + n + p, 0.0, nullptr, h->tmp_m, st);
  qsk_max_step(h->L, h->tmp_m, nullptr, h->scalars, -1, SC_SHIFT, h->gr, st);
  qsk_shift(h->L, h->tmp_m, h->s, h->scalars, SC_SHIFT, 1.0, st);
  h->tm.end(st);
  // rhs = (-c, 0, 0)
  CK(h, cudaMemsetAsync(h->rhs + n, 0, (p + m) * sizeof(double), st));
  rc = solve_refined(h, h->rhs);
  if (rc) return rc;
  h->tm.begin(T_CONE, st);
  qsk_max_step(h->L, h->sol + n + p, nullptr, h->scalars, -1, SC_SHIFT, h->gr, st);
  qsk_shift(h->L, h->sol + n + p, h->z, h->scalars, SC_SHIFT, 1.0, st);
  qsk_dot((int)m, h->s, h->z, 1.0 / h->deg, h->scalars + SC_MU, h->gr, st);
  h->tm.end(st);
  h->launches += 7;
  rc = check_launch(h, "initialize_iterate");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  const double mu = h->scalars_host[SC_MU];
  if (mu_host) *mu_host = mu;
  if (!(fabs(mu) <= DBL_MAX)) return fail(h, QS_E_NUMERICAL, "non-finite initial iterate");
  if (h->scalars_host[SC_PIVOT_NONFINITE] != 0.0) return fail(h, QS_E_NUMERICAL, "non-finite pivot during LDL' factorization");
  return QS_OK;
}

// compute_residuals (ipm.py:70-103)
int qs_residuals(qs_handle* h, qs_residual_info* out) {
  NEED_PROBLEM(h)
  h->tm.begin(T_RESID, h->stream);
  ResidualArgs A{(int)h->n, (int)h->p, (int)h->m, h->Pf, h->At, h->Gt, h->Ar, h->Gr, h->Dt, h->seg_partial, h->x, h->y, h->z, h->s,
                 h->c,      h->b,      h->hv,     h->rhs, h->r_cone, h->scalars, h->gr};
  h->launches += qsk_residuals(A, h->stream);
  h->tm.end(h->stream);
  int rc = check_launch(h, "residuals");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  if (out) fill_residual_info(h, out);
  if (h->scalars_host[SC_FLAG_NONFINITE] != 0.0) return fail(h, QS_E_NUMERICAL, "non-finite residuals");
  return QS_OK;
}

// ipm_step (ipm.py:159-235).  qs_residuals must have run on the current iterate
// (rhs[0:n+p] and r_cone hold -r_dual, -r_eq, r_cone).
int qs_step(qs_handle* h, qs_step_info* out) {
  NEED_PROBLEM(h)
  cudaStream_t st = h->stream;
  const ConeLayout& L = h->L;
  const i64 n = h->n, p = h->p, m = h->m;
  clear_flags(h);
  // scaling, lam o lam, the -W'W constants and the predictor's third RHS block (d_comp = -lam o lam) in one pass
  h->tm.begin(T_CONE, st);
  qsk_nt_scaling(L, h->s, h->z, h->w, h->eta, h->wbar, h->lam, h->lam_sq, h->wp.c4, h->wp.e2, h->r_cone, h->d,
                 h->rhs + n + p, h->scalars, st);
  h->tm.end(st);
  int rc = scatter_scaling(h, h->w, h->eta, h->wbar, /*have_consts=*/L.nsoc > 0);
  if (rc) return rc;
  rc = do_factor(h);
  if (rc) return rc;
  rc = solve_refined(h, h->rhs);
  if (rc) {
    // a point outside the cone poisons the scaling and with it the solve: report what the reference would have
    // raised first (compute_nt_scaling -> NotInterior, cones.py:169-170,182-183); the scalars were fetched by the solve
    if (rc == QS_E_NUMERICAL && h->scalars_host[SC_FLAG_NOT_INTERIOR] != 0.0)
      return fail(h, QS_E_NOT_INTERIOR, "point is not strictly inside the cone");
    return rc;
  }
  h->tm.begin(T_CONE, st);
  // predictor: ds_a, W dz_a, both steps, alpha_aff, mu_aff, sigma
  qsk_post_solve(L, h->w, h->eta, h->wbar, h->d, h->sol + n + p, h->s, h->z, h->wdz, h->ds, h->scalars, 0,
                 h->st.step_fraction, h->deg, h->gr, st);
  // corrector: d_comp = sigma mu e - lam o lam - (W^-1 ds_a) o (W dz_a), d = lam \ d_comp, rhs_z = -r_cone - W d
  qsk_corrector_rhs(L, h->w, h->eta, h->wbar, h->lam, h->lam_sq, h->ds, h->wdz, h->r_cone, nullptr, h->d,
                    h->rhs + n + p, h->scalars, st);
  h->tm.end(st);
  rc = solve_refined(h, h->rhs);
  if (rc) return rc;
  h->tm.begin(T_CONE, st);
  qsk_post_solve(L, h->w, h->eta, h->wbar, h->d, h->sol + n + p, h->s, h->z, nullptr, h->ds, h->scalars, 1,
                 h->st.step_fraction, h->deg, h->gr, st);
  qsk_update_iterate((int)n, (int)p, (int)m, h->x, h->y, h->z, h->s, h->x2, h->y2, h->z2, h->s2, h->sol, h->ds, h->deg,
                     h->scalars, h->gr, st);
  h->tm.end(st);
  h->launches += 5;
  rc = check_launch(h, "ipm_step");
  if (rc) return rc;
  rc = fetch_scalars(h);
  if (rc) return rc;
  const double* sc = h->scalars_host;
  // the new iterate replaces the old one only when the step raised nothing (the reference assigns `it = nxt` after
  // ipm_step returned, ipm.py:219-235,286): a NumericalError result carries the last good iterate
  if (flags_of(sc) == 0) {
    std::swap(h->x, h->x2);
    std::swap(h->y, h->y2);
    std::swap(h->z, h->z2);
    std::swap(h->s, h->s2);
  }
  if (out) {
    out->alpha = sc[SC_ALPHA];
    out->alpha_affine = sc[SC_ALPHA_AFF];
    out->sigma = sc[SC_SIGMA];
    out->mu_affine = sc[SC_MU_AFF];
    out->mu = sc[SC_MU];
    out->step_s = sc[SC_STEP_S];
    out->step_z = sc[SC_STEP_Z];
    out->flags = flags_of(sc);
  }
  if (sc[SC_FLAG_NOT_INTERIOR] != 0.0) return fail(h, QS_E_NOT_INTERIOR, "point is not strictly inside the cone");
  if (sc[SC_PIVOT_NONFINITE] != 0.0) return fail(h, QS_E_NUMERICAL, "non-finite pivot during LDL' factorization");
  if (sc[SC_FLAG_BAD_STEP] != 0.0) return fail(h, QS_E_NUMERICAL, "non-positive or non-finite step length");
  if (sc[SC_FLAG_NONFINITE] != 0.0) return fail(h, QS_E_NUMERICAL, "non-finite iterate");
  return QS_OK;
}

int qs_get_iterate(qs_handle* h, double* x, double* y, double* z, double* s) {
  NEED_PROBLEM(h)
  cudaStream_t st = h->stream;
  const double *sx = h->x, *sy = h->y, *sz = h->z, *ss = h->s;
  if (h->rD) {  // back to the caller's scaling: x = D x^, y = E y^, z = F z^, s = s^ / F
    double* t = h->dx;  // scratch of length n + p + m
    CK(h, cudaMemcpyAsync(t, h->x, h->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CK(h, cudaMemcpyAsync(t + h->n, h->y, h->p * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CK(h, cudaMemcpyAsync(t + h->n + h->p, h->z, h->m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CK(h, cudaMemcpyAsync(h->tmp_m, h->s, h->m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    qsk_vec_scale((int)h->n, t, h->rD, 0, st);
    qsk_vec_scale((int)h->p, t + h->n, h->rE, 0, st);
    qsk_vec_scale((int)h->m, t + h->n + h->p, h->rF, 0, st);
    qsk_vec_scale((int)h->m, h->tmp_m, h->rF, 1, st);
    sx = t;
    sy = t + h->n;
    sz = t + h->n + h->p;
    ss = h->tmp_m;
  }
  h->d2h_bytes += ((x ? h->n : 0) + (y ? h->p : 0) + (z ? h->m : 0) + (s ? h->m : 0)) * (i64)sizeof(double);
  if (x) CK(h, cudaMemcpyAsync(x, sx, h->n * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (y) CK(h, cudaMemcpyAsync(y, sy, h->p * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (z) CK(h, cudaMemcpyAsync(z, sz, h->m * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (s) CK(h, cudaMemcpyAsync(s, ss, h->m * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  return QS_OK;
}

int qs_get_ruiz(qs_handle* h, double* D, double* E, double* F) {
  NEED_PROBLEM(h)
  if (!h->rD) return fail(h, QS_E_INVALID, "ruiz_iters is 0: the problem is not equilibrated");
  cudaStream_t st = h->stream;
  if (D) CK(h, cudaMemcpyAsync(D, h->rD, h->n * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (E) CK(h, cudaMemcpyAsync(E, h->rE, h->p * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (F) CK(h, cudaMemcpyAsync(F, h->rF, h->m * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  return QS_OK;
}

int qs_set_iterate(qs_handle* h, const double* x, const double* y, const double* z, const double* s) {
  NEED_PROBLEM(h)
  cudaStream_t st = h->stream;
  if (x) CK(h, cudaMemcpyAsync(h->x, x, h->n * sizeof(double), cudaMemcpyHostToDevice, st));
  if (y) CK(h, cudaMemcpyAsync(h->y, y, h->p * sizeof(double), cudaMemcpyHostToDevice, st));
  if (z) CK(h, cudaMemcpyAsync(h->z, z, h->m * sizeof(double), cudaMemcpyHostToDevice, st));
  if (s) CK(h, cudaMemcpyAsync(h->s, s, h->m * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(h, cudaStreamSynchronize(st));
  return QS_OK;
}

int qs_get_scaling(qs_handle* h, double* w, double* eta, double* wbar, double* lam) {
  NEED_PROBLEM(h)
  cudaStream_t st = h->stream;
  if (w) CK(h, cudaMemcpyAsync(w, h->w, h->L.l * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (eta) CK(h, cudaMemcpyAsync(eta, h->eta, h->L.nsoc * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (wbar) CK(h, cudaMemcpyAsync(wbar, h->wbar, h->m * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (lam) CK(h, cudaMemcpyAsync(lam, h->lam, h->m * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  return QS_OK;
}

int qs_set_scaling(qs_handle* h, const double* w, const double* eta, const double* wbar, const double* lam) {
  NEED_PROBLEM(h)
  cudaStream_t st = h->stream;
  if (w) CK(h, cudaMemcpyAsync(h->w, w, h->L.l * sizeof(double), cudaMemcpyHostToDevice, st));
  if (eta) CK(h, cudaMemcpyAsync(h->eta, eta, h->L.nsoc * sizeof(double), cudaMemcpyHostToDevice, st));
  if (wbar) CK(h, cudaMemcpyAsync(h->wbar, wbar, h->m * sizeof(double), cudaMemcpyHostToDevice, st));
  if (lam) CK(h, cudaMemcpyAsync(h->lam, lam, h->m * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(h, cudaStreamSynchronize(st));
  return QS_OK;
}

int qs_get_counters(qs_handle* h, int64_t* n_factor, int64_t* n_solve, int64_t* n_launches) {
  if (!h) return QS_E_INVALID;
  if (n_factor) *n_factor = h->n_factor;
  if (n_solve) *n_solve = h->n_solve;
  if (n_launches) *n_launches = h->launches;
  return QS_OK;
}

int qs_get_transfer_bytes(qs_handle* h, int64_t* h2d, int64_t* d2h) {
  if (!h) return QS_E_INVALID;
  if (h2d) *h2d = (int64_t)(h->cone_pool.uploaded + h->prob_pool.uploaded + h->ls.h2d_bytes) + h->h2d_extra;
  if (d2h) *d2h = h->d2h_bytes;
  return QS_OK;
}

int qs_get_timers(qs_handle* h, double* timers8) {
  if (!h) return QS_E_INVALID;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  h->tm.collect();
  for (int k = 0; k < T_COUNT; ++k) timers8[k] = h->tm.total[k];
  return QS_OK;
}

int qs_get_graph_stats(qs_handle* h, int64_t* replays, int64_t* direct) {
  if (!h) return QS_E_INVALID;
  if (replays) *replays = h->ls.graph_counts[0];
  if (direct) *direct = h->ls.graph_counts[1];
  return QS_OK;
}

int qs_get_factor_stats(qs_handle* h, double* s8) {
  NEED_PROBLEM(h)
  const Symbolic& S = h->ls.S;
  s8[0] = S.nsup;
  s8[1] = S.nlevels;
  s8[2] = (double)S.lnz;
  s8[3] = S.flops;
  s8[4] = S.max_nr;
  s8[5] = S.max_ns;
  s8[6] = (double)h->ls.device_bytes;
  s8[7] = h->direct_ok ? 1.0 : 0.0;
  return QS_OK;
}

static int time_kernel_impl(qs_handle* h, int kernel_id, int reps, int cold, double* ms_host);

int qs_time_kernel(qs_handle* h, int kernel_id, int reps, double* ms_host) {
  return time_kernel_impl(h, kernel_id, reps, 0, ms_host);
}

int qs_time_kernel_cold(qs_handle* h, int kernel_id, int reps, double* ms_host) {
  return time_kernel_impl(h, kernel_id, reps, 1, ms_host);
}

static int time_kernel_impl(qs_handle* h, int kernel_id, int reps, int cold, double* ms_host) {
  NEED_PROBLEM(h)
  if (reps < 1) reps = 1;
  cudaStream_t st = h->stream;
  const ConeLayout& L = h->L;
  const i64 n = h->n, p = h->p, m = h->m;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&]() {
    switch (kernel_id) {
      case 0: qsk_nt_scaling(L, h->s, h->z, h->w, h->eta, h->wbar, h->lam, h->lam_sq, h->wp.c4, h->wp.e2, h->r_cone, h->d,
                             h->rhs + n + p, h->scalars, st); break;
      case 1: qsk_neg_wtw(h->wp, 2, h->w, h->eta, h->wbar, h->d_pos, h->d_Kx, st, L.nsoc > 0); break;
      case 2: qsk_neg_wtw(h->wp, 1, h->w, h->eta, h->wbar, h->d_pos, h->d_Kx, st, L.nsoc > 0); break;
      case 3: qsk_nt_scaling(L, h->s, h->z, h->w, h->eta, h->wbar, h->lam, h->lam_sq, nullptr, nullptr, nullptr, nullptr,
                             nullptr, h->scalars, st); break;  // scaling + lam o lam alone
      case 4: qsk_post_solve(L, h->w, h->eta, h->wbar, h->d, h->sol + n + p, h->s, h->z, h->wdz, h->ds, h->scalars, 0,
                             h->st.step_fraction, h->deg, h->gr, st); break;
      case 5: qsk_post_solve(L, h->w, h->eta, h->wbar, h->d, h->sol + n + p, h->s, h->z, nullptr, h->tmp_m, h->scalars, 1,
                             h->st.step_fraction, h->deg, h->gr, st); break;
      case 6: qsk_corrector_rhs(L, h->w, h->eta, h->wbar, h->lam, h->lam_sq, h->ds, h->wdz, h->r_cone, nullptr, h->tmp_m,
                                h->w2vz, h->scalars, st); break;
      case 7: {
        ResidualArgs A{(int)n, (int)p, (int)m, h->Pf, h->At, h->Gt, h->Ar, h->Gr, h->Dt, h->seg_partial, h->x, h->y, h->z, h->s,
                       h->c,   h->b,   h->hv,  h->rhs, h->r_cone, h->scalars, h->gr};
        qsk_residuals(A, st);
        break;
      }
      case 8: qsk_apply_w(L, h->w, h->eta, h->wbar, h->ds, h->tmp_m, 0, st); break;
      case 9: qsk_jordan_product(L, h->lam, h->lam, h->tmp_m, st); break;
      case 10: qsk_jordan_divide(L, h->lam, h->lam_sq, h->tmp_m, st); break;
      case 11: qsk_max_step(L, h->s, h->ds, h->scalars, SC_TMP0, SC_TMP1, h->gr, st); break;
      case 12: h->ls.factor(h->d_Kx, h->scalars, st); break;
      case 13: h->ls.solve(h->rhs, h->dx, st); break;
      case 14: {
        qsk_apply_w2(L, h->w, h->eta, h->wbar, h->sol + n + p, h->w2vz, st);
        KktResidualArgs A{(int)n, (int)p, (int)m, h->Pf, h->At, h->Gt, h->Ar, h->Gr, h->Dt, h->seg_partial,
                          h->sol, h->rhs, h->w2vz, h->rb, h->scalars, SC_TMP3, h->gr};
        qsk_kkt_residual(A, st);
        break;
      }
      case 15: qsk_update_iterate((int)n, (int)p, (int)m, h->x, h->y, h->z, h->s, h->x2, h->y2, h->z2, h->s2, h->sol, h->ds,
                                  h->deg, h->scalars, h->gr, st); break;
      default: break;
    }
  };
  if (kernel_id < 0 || kernel_id > 15) return fail(h, QS_E_INVALID, "unknown kernel id");
  run();  // warm-up
  float ms = 0.f;
  if (!cold) {
    CK(h, cudaEventRecord(a, st));
    for (int r = 0; r < reps; ++r) run();
    CK(h, cudaEventRecord(b, st));
    CK(h, cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
  } else {
    // cold: every timed launch starts with an L2 that holds none of its operands (256 MiB > 126 MB L2 rewritten
    // in between), as inside a solve, where a 5.7 GB factorisation runs between two cone phases
    const size_t flush_bytes = (size_t)256 << 20;
    void* flush = nullptr;
    if (cudaMalloc(&flush, flush_bytes) != cudaSuccess) return fail(h, QS_E_MEMORY, "L2 flush buffer");
    cudaMemsetAsync(flush, 0, flush_bytes, st);
    for (int r = 0; r < reps; ++r) {
      // read-only sweep: the L2 ends up full of CLEAN lines of the flush buffer (a memset would leave dirty lines
      // whose write-back would be billed to the timed kernel)
      qsk_absmax((i64)(flush_bytes / sizeof(double)), (const double*)flush, h->scalars + SC_TMP2, nullptr, h->gr, st);
      cudaEventRecord(a, st);
      run();
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float one = 0.f;
      cudaEventElapsedTime(&one, a, b);
      ms += one;
    }
    cudaFree(flush);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (ms_host) *ms_host = (double)ms / reps;
  return check_launch(h, "time_kernel");
}

// ===================================================== batched small-problem mode ======
// B instances with ONE sparsity pattern, solved in lockstep: every launch of the ordinary solver carries
// gridDim.z = B (common.cuh), one host synchronisation serves all instances, and the analysis, index maps and
// launch graphs are built once.  Per-instance decisions (termination, refinement accept / reject, step flags) are
// taken on the host from the B scalar blocks and handed back as one flag per instance; an instance that has
// finished keeps its iterate frozen (its share of later launches is wasted work, nothing else).
}  // extern "C"

struct qs_batch {
  int device = 0;
  int B = 0;
  QsArena arena;
  size_t arena_bytes = 0;       // allocated size (>= slots * stride when the arena was taken from the cache)
  qs_handle* h = nullptr;       // the handle of slot 0; every device pointer in it is valid in every slot + b * stride
  double* sc_host = nullptr;    // pinned [B][SC_COUNT]
  double* flag_host = nullptr;  // pinned [B]
  std::vector<double> norm_c, norm_b, norm_h;
  bool values_dirty = false;
  std::string err;
  double solve_seconds = 0.0;
  i64 launches = 0, syncs = 0;
};

namespace {

struct BatchScope {
  explicit BatchScope(qs_batch* b, bool batched_launches = true) {
    cudaSetDevice(b->device);
    qs_tls_arena = &b->arena;
    qs_tls_batch = batched_launches ? b->B : 1;
  }
  ~BatchScope() {
    qs_tls_arena = nullptr;
    qs_tls_batch = 1;
  }
};

int bfail(qs_batch* bt, int code, const std::string& msg) {
  bt->err = msg;
  return code;
}

#define BCK(bt, call)                                                                 \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return bfail(bt, QS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// all B scalar blocks -> pinned host mirror (one synchronisation for the whole batch)
int fetch_b(qs_batch* bt) {
  qs_handle* h = bt->h;
  BCK(bt, cudaMemcpy2DAsync(bt->sc_host, SC_COUNT * sizeof(double), h->scalars, QS_BSTRIDE, SC_COUNT * sizeof(double),
                            (size_t)bt->B, cudaMemcpyDeviceToHost, h->stream));
  BCK(bt, cudaStreamSynchronize(h->stream));
  h->tm.collect();
  bt->syncs++;
  return QS_OK;
}

// flag_host[b] -> scalars[slot] of instance b
int upload_flags(qs_batch* bt, int slot) {
  qs_handle* h = bt->h;
  BCK(bt, cudaMemcpy2DAsync(h->scalars + slot, QS_BSTRIDE, bt->flag_host, sizeof(double), sizeof(double), (size_t)bt->B,
                            cudaMemcpyHostToDevice, h->stream));
  return QS_OK;
}

inline const double* sc_of(const qs_batch* bt, int b) { return bt->sc_host + (size_t)b * SC_COUNT; }

enum { BS_RUNNING = 0, BS_SOLVED = 1, BS_MAX_ITERS = 2, BS_TIME_LIMIT = 3, BS_NUMERICAL = 4, BS_NOT_INTERIOR = 5 };

// solve_refine (ldl.py:135-166) for every live instance; result in h->xa (= h->sol).  `live` instances whose
// residual is not finite are marked BS_NUMERICAL.
int solve_refined_b(qs_batch* bt, const double* rhs, std::vector<int>& status) {
  qs_handle* h = bt->h;
  const i64 N = h->N;
  const int B = bt->B;
  cudaStream_t st = h->stream;
  double *x = h->xa, *xn = h->xb, *r = h->ra, *r2 = h->rb;
  auto backsolve = [&](const double* rr, double* out) {
    h->tm.begin(T_SOLVE, st);
    h->ls.solve(rr, out, st);
    h->tm.end(st);
    bt->launches += h->ls.launches_per_solve();
  };
  auto residual = [&](const double* v, double* rr, int slot) {
    h->tm.begin(T_REFINE, st);
    qsk_apply_w2(h->L, h->w, h->eta, h->wbar, v + h->n + h->p, h->w2vz, st);
    KktResidualArgs A{(int)h->n, (int)h->p, (int)h->m, h->Pf, h->At, h->Gt, h->Ar, h->Gr, h->Dt, h->seg_partial,
                      v,         rhs,       h->w2vz,   rr,    h->scalars, slot, h->gr};
    qsk_kkt_residual(A, st);
    h->tm.end(st);
    bt->launches += 2;
  };
  backsolve(rhs, x);
  h->sol = x;
  h->n_solve++;
  if (h->st.refine_iters <= 0) return check_launch(h, "linear solve") ? bfail(bt, QS_E_CUDA, h->err) : QS_OK;
  qsk_absmax(N, rhs, h->scalars + SC_TMP0, nullptr, h->gr, st);
  residual(x, r, SC_TMP1);
  bt->launches += 1;
  int rc = fetch_b(bt);
  if (rc) return rc;
  std::vector<double> stop(B), rn(B);
  std::vector<char> active(B, 0);
  int nactive = 0;
  for (int b = 0; b < B; ++b) {
    const double* sc = sc_of(bt, b);
    stop[b] = 1e-12 * (1.0 + sc[SC_TMP0]);  // ldl.py:19,151
    rn[b] = sc[SC_TMP1];
    if (status[b] != BS_RUNNING) continue;
    if (!(fabs(rn[b]) <= DBL_MAX)) {  // non-finite triangular solve result (a point outside the cone poisons it)
      status[b] = sc[SC_FLAG_NOT_INTERIOR] != 0.0 ? BS_NOT_INTERIOR : BS_NUMERICAL;
      continue;
    }
    active[b] = rn[b] > stop[b];
    nactive += active[b];
  }
  for (i64 it = 0; it < h->st.refine_iters && nactive > 0; ++it) {
    backsolve(r, h->dx);
    qsk_axpby(N, 1.0, x, 1.0, h->dx, xn, st);
    residual(xn, r2, SC_TMP2);
    bt->launches += 1;
    rc = fetch_b(bt);
    if (rc) return rc;
    nactive = 0;
    for (int b = 0; b < B; ++b) {
      bt->flag_host[b] = 0.0;
      if (!active[b]) continue;
      const double rn2 = sc_of(bt, b)[SC_TMP2];
      if (!(fabs(rn2) <= DBL_MAX)) {
        status[b] = BS_NUMERICAL;  // non-finite refinement residual
        active[b] = 0;
      } else if (rn2 >= rn[b]) {
        active[b] = 0;  // no decrease: keep the previous solution (ldl.py:161-162)
      } else {
        bt->flag_host[b] = 1.0;
        rn[b] = rn2;
        active[b] = rn2 > stop[b];
        nactive += active[b];
      }
    }
    rc = upload_flags(bt, SC_TMP3);
    if (rc) return rc;
    qsk_copy_if(N, h->scalars + SC_TMP3, xn, x, st);
    qsk_copy_if(N, h->scalars + SC_TMP3, r2, r, st);
    bt->launches += 2;
    // the pinned flags are read by the copy above: do not overwrite them before it ran
    BCK(bt, cudaStreamSynchronize(st));
  }
  return check_launch(h, "linear solve") ? bfail(bt, QS_E_CUDA, h->err) : QS_OK;
}

}  // namespace

extern "C" {

qs_batch* qs_batch_create(int device, int64_t count) {
  int cnt = qs_device_count();
  if (device < 0 || device >= cnt || count < 1 || count > 65535) {
    g_error = "qs_batch_create: bad device or instance count (1..65535)";
    return nullptr;
  }
  cudaSetDevice(device);
  qs_batch* bt = new qs_batch();
  bt->device = device;
  bt->B = (int)count;
  bt->arena.slot_bytes = QS_BSTRIDE;
  bt->arena.slots = (int)count;
  const size_t total = (size_t)count * QS_BSTRIDE;
  // The arena: a released one of this device that is large enough (kept in a small cache by qs_batch_destroy, zeroed
  // here: 2.5 ms for 16 GB), else plain cudaMalloc (10-50 ms for 16 GB, but now and then 0.5 s when the driver has to
  // map again what a cudaFree just gave back -- every third bench run showed it).  The stream-ordered memory pool
  // was tried for this: the second batch is free, the first pays 0.6-0.9 s of pool growth.
  {
    std::lock_guard<std::mutex> lk(g_devmem.mu);
    int best = -1;
    for (size_t k = 0; k < g_devmem.arena_cache.size(); ++k) {
      const auto& c = g_devmem.arena_cache[k];
      if (c.dev == device && c.bytes >= total && (best < 0 || c.bytes < g_devmem.arena_cache[best].bytes)) best = (int)k;
    }
    if (best >= 0) {
      bt->arena.base = g_devmem.arena_cache[best].base;
      bt->arena_bytes = g_devmem.arena_cache[best].bytes;
      g_devmem.arena_cache.erase(g_devmem.arena_cache.begin() + best);
    }
  }
  if (bt->arena.base) {
    cudaMemset(bt->arena.base, 0, total);
  } else {
    bt->arena_bytes = total;
    if (cudaMalloc((void**)&bt->arena.base, total) != cudaSuccess) bt->arena.base = nullptr;
  }
  if (!bt->arena.base ||
      cudaMallocHost((void**)&bt->sc_host, (size_t)count * SC_COUNT * sizeof(double)) != cudaSuccess ||
      cudaMallocHost((void**)&bt->flag_host, (size_t)count * sizeof(double)) != cudaSuccess) {
    g_error = std::string("qs_batch_create: ") + cudaGetErrorString(cudaGetLastError());
    if (bt->arena.base) cudaFree(bt->arena.base);
    if (bt->sc_host) cudaFreeHost(bt->sc_host);
    delete bt;
    return nullptr;
  }
  {
    std::lock_guard<std::mutex> lk(g_devmem.mu);
    g_devmem.arenas.emplace_back(bt->arena.base, total);
  }
  {
    BatchScope sc(bt, false);
    bt->h = qs_create(device);
  }
  if (!bt->h) {
    qs_batch_destroy(bt);
    return nullptr;
  }
  bt->norm_c.assign(count, 0.0);
  bt->norm_b.assign(count, 0.0);
  bt->norm_h.assign(count, 0.0);
  return bt;
}

void qs_batch_destroy(qs_batch* bt) {
  if (!bt) return;
  cudaSetDevice(bt->device);
  if (bt->h) {
    BatchScope sc(bt, false);
    qs_destroy(bt->h);  // frees of arena pointers are no-ops
  }
  {
    std::lock_guard<std::mutex> lk(g_devmem.mu);
    auto& v = g_devmem.arenas;
    v.erase(std::remove_if(v.begin(), v.end(), [&](const std::pair<char*, size_t>& a) { return a.first == bt->arena.base; }),
            v.end());
  }
  if (bt->arena.base) {
    cudaDeviceSynchronize();  // nothing of this batch is in flight any more
    bool kept = false;
    {
      std::lock_guard<std::mutex> lk(g_devmem.mu);
      if (g_devmem.arena_cache.size() < 2) {
        g_devmem.arena_cache.push_back(DevMem::CachedArena{bt->device, bt->arena.base, bt->arena_bytes});
        kept = true;
      }
    }
    if (!kept) cudaFree(bt->arena.base);
  }
  cudaFreeHost(bt->sc_host);
  cudaFreeHost(bt->flag_host);
  delete bt;
}

const char* qs_batch_last_error(qs_batch* bt) {
  if (!bt) return g_error.c_str();
  if (!bt->err.empty()) return bt->err.c_str();
  return bt->h ? bt->h->err.c_str() : "";
}

// The shared pattern and the numbers of instance 0 (same arguments as qs_setup); every slot starts as a copy of it.
int qs_batch_setup(qs_batch* bt, int64_t n, int64_t m, int64_t p, int64_t l, int64_t nsoc, const int64_t* q,
                   const int64_t* Pp, const int64_t* Pi, const double* Px, const int64_t* Ap, const int64_t* Ai,
                   const double* Ax, const int64_t* Gp, const int64_t* Gi, const double* Gx, const double* c,
                   const double* b, const double* hvec, const qs_settings* settings) {
  if (!bt || !bt->h) return QS_E_INVALID;
  if (settings && settings->ruiz_iters > 0) return bfail(bt, QS_E_INVALID, "batched mode does not equilibrate");
  int rc;
  {
    BatchScope sc(bt, false);  // slot 0 is set up as an ordinary handle whose memory comes from the arena
    rc = qs_setup(bt->h, n, m, p, l, nsoc, q, Pp, Pi, Px, Ap, Ai, Ax, Gp, Gi, Gx, c, b, hvec, settings, nullptr);
  }
  if (rc) return bfail(bt, rc, bt->h->err.empty() ? "qs_setup failed" : bt->h->err +
                                  " (batched mode: one instance must fit a 32 MiB slot)");
  if (!bt->h->pf_map) return bfail(bt, QS_E_INVALID, "batched mode needs the device-assembled KKT path");
  qs_handle* h = bt->h;
  // replicate slot 0 (patterns, analysis, values of instance 0, zeroed scratch) into every slot
  qsk_broadcast((i64)((bt->arena.used + 7) / 8), bt->arena.base, bt->B, h->stream);
  BCK(bt, cudaStreamSynchronize(h->stream));
  for (int k = 0; k < bt->B; ++k) {
    bt->norm_c[k] = h->norm_c;
    bt->norm_b[k] = h->norm_b;
    bt->norm_h[k] = h->norm_h;
  }
  bt->values_dirty = false;
  return QS_OK;
}

// Numbers of all instances at once: each array is [count][len] row-major (len = nnz(P), nnz(A), nnz(G), n, p, m)
// or null (= every instance keeps the numbers given at setup).
int qs_batch_set_values(qs_batch* bt, const double* Px, const double* Ax, const double* Gx, const double* c,
                        const double* b, const double* hvec) {
  if (!bt || !bt->h || !bt->h->have_problem) return QS_E_INVALID;
  cudaSetDevice(bt->device);
  qs_handle* h = bt->h;
  cudaStream_t st = h->stream;
  const size_t B = (size_t)bt->B;
  auto up = [&](const double* src, const double* dst, i64 len) -> cudaError_t {
    if (!src || len <= 0) return cudaSuccess;
    h->h2d_extra += (i64)B * len * (i64)sizeof(double);
    return cudaMemcpy2DAsync(const_cast<double*>(dst), QS_BSTRIDE, src, len * sizeof(double), len * sizeof(double), B,
                             cudaMemcpyHostToDevice, st);
  };
  BCK(bt, up(Px, h->Pu.val, h->nnzP));
  BCK(bt, up(Ax, h->At.val, h->nnzA));
  BCK(bt, up(Gx, h->Gt.val, h->nnzG));
  BCK(bt, up(c, h->c, h->n));
  BCK(bt, up(b, h->b, h->p));
  BCK(bt, up(hvec, h->hv, h->m));
  for (size_t k = 0; k < B; ++k) {
    if (c) bt->norm_c[k] = inf_norm(c + k * h->n, h->n);
    if (b) bt->norm_b[k] = inf_norm(b + k * h->p, h->p);
    if (hvec) bt->norm_h[k] = inf_norm(hvec + k * h->m, h->m);
  }
  if (Px || Ax || Gx) bt->values_dirty = true;
  BCK(bt, cudaStreamSynchronize(st));  // the caller's buffers may be released on return
  return QS_OK;
}

// Lockstep interior-point solve of every instance (the loop of ipm.py:259-297 per instance).  Outputs, all [count]
// or [count][len]: status (1 Solved, 2 MaxIters, 3 TimeLimit, 4 NumericalError, 5 NotInterior), iterations, and the
// final iterates x [n], y [p], z [m], s [m].
int qs_batch_solve(qs_batch* bt, int64_t* status_out, int64_t* iterations_out, double* x, double* y, double* z,
                   double* s) {
  if (!bt || !bt->h || !bt->h->have_problem) return QS_E_INVALID;
  BatchScope scope(bt);
  qs_handle* h = bt->h;
  cudaStream_t st = h->stream;
  const int B = bt->B;
  const i64 n = h->n, p = h->p, m = h->m, N = h->N;
  const ConeLayout& L = h->L;
  const auto t_begin = std::chrono::steady_clock::now();
  auto elapsed = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_begin).count(); };
  int rc;
#define BRC(call)                                                          \
  do {                                                                     \
    rc = (call);                                                           \
    if (rc) return bt->err.empty() ? bfail(bt, rc, h->err) : rc;           \
  } while (0)
  if (bt->values_dirty) {  // row views and KKT values of every instance from its raw numbers (qs_update_values)
    qsk_gather(h->nnzPf, h->Pu.val, h->pf_map, const_cast<double*>(h->Pf.val), st);
    qsk_gather(h->nnzA, h->At.val, h->ar_map, const_cast<double*>(h->Ar.val), st);
    qsk_gather(h->nnzG, h->Gt.val, h->gr_map, const_cast<double*>(h->Gr.val), st);
    WtwPlan plan = h->wp;
    plan.slot_start = h->d_slot_start;
    qsk_kkt_fill(plan, (int)n, (int)p, h->Pu, h->Ar, h->Gr, h->d_Kp, h->d_Ki, h->d_Kx, h->d_pos, st);
    if (h->Dt.ptr) qsk_gather3(h->nnzDt, h->Pf.val, h->At.val, h->Gt.val, h->dt_map, const_cast<double*>(h->Dt.val), st);
    bt->launches += 5;
    bt->values_dirty = false;
  }
  std::vector<int> status(B, BS_RUNNING), iters(B, 0), stalls(B, 0);
  // ---- initialize_iterate (ipm.py:135-156)
  clear_flags(h);
  {
    // identity_scaling (cones.py:146-156) written to slot 0, then copied to every slot
    std::vector<double> one(std::max<i64>(std::max<i64>(L.l, L.nsoc), 1), 1.0), e(m, 0.0);
    for (int k = 0; k < L.nsoc; ++k) e[h->soc_ptr_host[k]] = 1.0;
    BCK(bt, cudaMemcpyAsync(h->w, one.data(), L.l * sizeof(double), cudaMemcpyHostToDevice, st));
    BCK(bt, cudaMemcpyAsync(h->eta, one.data(), L.nsoc * sizeof(double), cudaMemcpyHostToDevice, st));
    BCK(bt, cudaMemcpyAsync(h->wbar, e.data(), m * sizeof(double), cudaMemcpyHostToDevice, st));
    BCK(bt, cudaStreamSynchronize(st));  // `e` is rewritten below
    for (int i = 0; i < L.l; ++i) e[i] = 1.0;
    BCK(bt, cudaMemcpyAsync(h->lam, e.data(), m * sizeof(double), cudaMemcpyHostToDevice, st));
    qsk_broadcast(L.l, h->w, B, st);
    qsk_broadcast(L.nsoc, h->eta, B, st);
    qsk_broadcast(m, h->wbar, B, st);
    qsk_broadcast(m, h->lam, B, st);
    BCK(bt, cudaStreamSynchronize(st));
  }
  BRC(scatter_scaling(h, h->w, h->eta, h->wbar));
  BRC(do_factor(h));
  qsk_axpby(n, -1.0, h->c, 0.0, nullptr, h->rhs, st);
  BCK(bt, qs_copy_b(h->rhs + n, h->b, p * sizeof(double), st));
  BCK(bt, qs_copy_b(h->rhs + n + p, h->hv, m * sizeof(double), st));
  BRC(solve_refined_b(bt, h->rhs, status));
  BCK(bt, qs_copy_b(h->x, h->sol, n * sizeof(double), st));
  BCK(bt, qs_copy_b(h->y, h->sol + n, p * sizeof(double), st));
  qsk_axpby(m, -1.0, h->sol + n + p, 0.0, nullptr, h->tmp_m, st);
  qsk_max_step(L, h->tmp_m, nullptr, h->scalars, -1, SC_SHIFT, h->gr, st);
  qsk_shift(L, h->tmp_m, h->s, h->scalars, SC_SHIFT, 1.0, st);
  BCK(bt, qs_memset_b(h->rhs + n, 0, (p + m) * sizeof(double), st));
  BRC(solve_refined_b(bt, h->rhs, status));
  qsk_max_step(L, h->sol + n + p, nullptr, h->scalars, -1, SC_SHIFT, h->gr, st);
  qsk_shift(L, h->sol + n + p, h->z, h->scalars, SC_SHIFT, 1.0, st);
  qsk_dot((int)m, h->s, h->z, 1.0 / h->deg, h->scalars + SC_MU, h->gr, st);
  bt->launches += 8;
  BRC(fetch_b(bt));
  for (int b = 0; b < B; ++b) {
    const double* sc = sc_of(bt, b);
    if (status[b] == BS_RUNNING && (!(fabs(sc[SC_MU]) <= DBL_MAX) || sc[SC_PIVOT_NONFINITE] != 0.0))
      status[b] = BS_NUMERICAL;
  }
  // ---- the loop
  const double ea = h->st.eps_abs, er = h->st.eps_rel;
  for (;;) {
    // compute_residuals (ipm.py:70-103) + check_termination (ipm.py:106-119)
    h->tm.begin(T_RESID, st);
    ResidualArgs A{(int)n, (int)p, (int)m, h->Pf, h->At, h->Gt, h->Ar, h->Gr, h->Dt, h->seg_partial, h->x, h->y, h->z, h->s,
                   h->c,   h->b,   h->hv,  h->rhs, h->r_cone, h->scalars, h->gr};
    bt->launches += qsk_residuals(A, st);
    h->tm.end(st);
    BRC(fetch_b(bt));
    int running = 0;
    const bool out_of_time = elapsed() > h->st.time_limit_seconds;
    for (int b = 0; b < B; ++b) {
      if (status[b] != BS_RUNNING) continue;
      const double* sc = sc_of(bt, b);
      if (sc[SC_FLAG_NONFINITE] != 0.0) {
        status[b] = BS_NUMERICAL;
        continue;
      }
      const bool dual_ok = sc[SC_NORM_RDUAL] <=
                           ea + er * std::max(std::max(sc[SC_NORM_PX], sc[SC_NORM_ATY]), std::max(sc[SC_NORM_GTZ], bt->norm_c[b]));
      const bool eq_ok = sc[SC_NORM_REQ] <= ea + er * std::max(sc[SC_NORM_AX], bt->norm_b[b]);
      const bool cone_ok = sc[SC_NORM_RCONE] <= ea + er * std::max(std::max(sc[SC_NORM_GX], sc[SC_NORM_S]), bt->norm_h[b]);
      const bool gap_ok = sc[SC_GAP] <= ea + er * std::max(fabs(sc[SC_OBJ]), 1.0);
      if (dual_ok && eq_ok && cone_ok && gap_ok) status[b] = BS_SOLVED;
      else if (iters[b] >= h->st.max_iters) status[b] = BS_MAX_ITERS;
      else if (out_of_time) status[b] = BS_TIME_LIMIT;
      else ++running;
    }
    if (running == 0) break;
    // ---- ipm_step (ipm.py:159-235) for every instance; finished ones keep their iterate
    clear_flags(h);
    h->tm.begin(T_CONE, st);
    qsk_nt_scaling(L, h->s, h->z, h->w, h->eta, h->wbar, h->lam, h->lam_sq, h->wp.c4, h->wp.e2, h->r_cone, h->d,
                   h->rhs + n + p, h->scalars, st);
    h->tm.end(st);
    BRC(scatter_scaling(h, h->w, h->eta, h->wbar, /*have_consts=*/L.nsoc > 0));
    BRC(do_factor(h));
    BRC(solve_refined_b(bt, h->rhs, status));
    h->tm.begin(T_CONE, st);
    qsk_post_solve(L, h->w, h->eta, h->wbar, h->d, h->sol + n + p, h->s, h->z, h->wdz, h->ds, h->scalars, 0,
                   h->st.step_fraction, h->deg, h->gr, st);
    qsk_corrector_rhs(L, h->w, h->eta, h->wbar, h->lam, h->lam_sq, h->ds, h->wdz, h->r_cone, nullptr, h->d,
                      h->rhs + n + p, h->scalars, st);
    h->tm.end(st);
    BRC(solve_refined_b(bt, h->rhs, status));
    h->tm.begin(T_CONE, st);
    qsk_post_solve(L, h->w, h->eta, h->wbar, h->d, h->sol + n + p, h->s, h->z, nullptr, h->ds, h->scalars, 1,
                   h->st.step_fraction, h->deg, h->gr, st);
    qsk_update_iterate((int)n, (int)p, (int)m, h->x, h->y, h->z, h->s, h->x2, h->y2, h->z2, h->s2, h->sol, h->ds, h->deg,
                       h->scalars, h->gr, st);
    h->tm.end(st);
    bt->launches += 5;
    BRC(fetch_b(bt));
    for (int b = 0; b < B; ++b) {
      bt->flag_host[b] = 0.0;
      if (status[b] != BS_RUNNING) continue;
      const double* sc = sc_of(bt, b);
      const i64 fl = flags_of(sc);
      if (fl) {  // the step raised: the last good iterate stays (ipm.py:219-235,292-293)
        status[b] = (fl & 1) ? BS_NOT_INTERIOR : BS_NUMERICAL;
        continue;
      }
      bt->flag_host[b] = 1.0;
      iters[b]++;
      if (sc[SC_ALPHA] < 1e-10) {  // TINY_STEP, MAX_CONSECUTIVE_STALLS (ipm.py:24-25,287-291)
        if (++stalls[b] >= 3) status[b] = BS_NUMERICAL;
      } else {
        stalls[b] = 0;
      }
    }
    BRC(upload_flags(bt, SC_TMP3));
    qsk_copy_if(n, h->scalars + SC_TMP3, h->x2, h->x, st);
    qsk_copy_if(p, h->scalars + SC_TMP3, h->y2, h->y, st);
    qsk_copy_if(m, h->scalars + SC_TMP3, h->z2, h->z, st);
    qsk_copy_if(m, h->scalars + SC_TMP3, h->s2, h->s, st);
    bt->launches += 4;
    BCK(bt, cudaStreamSynchronize(st));  // flag_host is rewritten by the next refinement round
  }
  // ---- results
  auto down = [&](double* dst, const double* src, i64 len) -> cudaError_t {
    if (!dst || len <= 0) return cudaSuccess;
    h->d2h_bytes += (i64)B * len * (i64)sizeof(double);
    return cudaMemcpy2DAsync(dst, len * sizeof(double), src, QS_BSTRIDE, len * sizeof(double), (size_t)B,
                             cudaMemcpyDeviceToHost, st);
  };
  BCK(bt, down(x, h->x, n));
  BCK(bt, down(y, h->y, p));
  BCK(bt, down(z, h->z, m));
  BCK(bt, down(s, h->s, m));
  BCK(bt, cudaStreamSynchronize(st));
  for (int b = 0; b < B; ++b) {
    if (status_out) status_out[b] = status[b];
    if (iterations_out) iterations_out[b] = iters[b];
  }
  bt->solve_seconds = elapsed();
  (void)N;
#undef BRC
  return QS_OK;
}

// launches issued, host synchronisations, seconds of the last qs_batch_solve, bytes of one slot in use
int qs_batch_stats(qs_batch* bt, double* out4) {
  if (!bt || !out4) return QS_E_INVALID;
  out4[0] = (double)(bt->launches + (bt->h ? bt->h->launches : 0));
  out4[1] = (double)bt->syncs;
  out4[2] = bt->solve_seconds;
  out4[3] = (double)bt->arena.used;
  return QS_OK;
}

}  // extern "C"
