// Host-side structure building (see host_setup.h).  Plain C++17, no CUDA.
#include "host_setup.h"

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstring>
#include <numeric>
#include <chrono>
#include <cstdio>
#include <cstdlib>

static double hs_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static bool hs_verbose() { return getenv("QS_VERBOSE") != nullptr; }

// ------------------------------------------------------------------ transpose
void hs_transpose(i64 rows, i64 cols, const i64* p, const i64* idx, const double* x, i64* tp, i64* ti, double* tx) {
  const i64 nnz = p[cols];
  std::fill(tp, tp + rows + 1, 0);
  for (i64 k = 0; k < nnz; ++k) tp[idx[k] + 1]++;
  for (i64 r = 0; r < rows; ++r) tp[r + 1] += tp[r];
  std::vector<i64> next(tp, tp + rows);
  for (i64 j = 0; j < cols; ++j)
    for (i64 k = p[j]; k < p[j + 1]; ++k) {
      const i64 dst = next[idx[k]]++;
      ti[dst] = j;
      if (tx) tx[dst] = x[k];
    }
}

// --------------------------------------------------------------- KKT assembly
// Column structure of the upper triangle of [P A' G'; . 0 0; . . -W'W], written
// directly (no triplet sort):
//   col j < n        : P(:, j) rows <= j, then the diagonal if P has none there
//   col n + r        : columns of A with an entry in row r (ascending), diagonal
//   col n + p + i    : columns of G with an entry in row i (ascending), then the
//                      scaling-block rows n+p+o .. n+p+i of i's cone
// which is exactly what the reference's lexsorted triplet build produces
// (kkt.py:59-104, sparse.py:83-116: duplicates summed in input order, explicit
// zeros kept).
static inline bool p_has_diag(const i64* Pp, const i64* Pi, i64 j) {
  return Pp[j + 1] > Pp[j] && Pi[Pp[j + 1] - 1] == j;
}

i64 hs_slot_count(const KktDims& d) {
  i64 s = d.l;
  for (i64 k = 0; k < d.nsoc; ++k) s += d.q[k] * (d.q[k] + 1) / 2;
  return s;
}

i64 hs_kkt_nnz(const KktDims& d, const i64* Pp, const i64* Pi, i64 nnzA, i64 nnzG) {
  i64 nnz = Pp[d.n];
  for (i64 j = 0; j < d.n; ++j)
    if (!p_has_diag(Pp, Pi, j)) nnz++;
  return nnz + nnzA + d.p + nnzG + hs_slot_count(d);
}

void hs_kkt_assemble(const KktDims& d, const i64* Pp, const i64* Pi, const double* Px, const i64* Arp, const i64* Ari,
                     const double* Arx, const i64* Grp, const i64* Gri, const double* Grx, i64* Kp, i64* Ki,
                     double* Kx, i64* positions, i64* slot_offsets, i64* soc_slot_starts) {
  const i64 n = d.n, p = d.p, l = d.l;
  i64 at = 0;
  Kp[0] = 0;
  for (i64 j = 0; j < n; ++j) {
    for (i64 k = Pp[j]; k < Pp[j + 1]; ++k) {
      Ki[at] = Pi[k];
      Kx[at] = (Pi[k] == j) ? Px[k] + 0.0 : Px[k];  // the explicit 0.0 diagonal is summed onto P_jj
      ++at;
    }
    if (!p_has_diag(Pp, Pi, j)) {
      Ki[at] = j;
      Kx[at] = 0.0;
      ++at;
    }
    Kp[j + 1] = at;
  }
  for (i64 r = 0; r < p; ++r) {
    for (i64 k = Arp[r]; k < Arp[r + 1]; ++k) {
      Ki[at] = Ari[k];
      Kx[at] = Arx[k];
      ++at;
    }
    Ki[at] = n + r;
    Kx[at] = 0.0;
    ++at;
    Kp[n + r + 1] = at;
  }
  const i64 base = n + p;
  i64 slot = 0, view = 0;
  if (slot_offsets) slot_offsets[0] = 0;
  auto g_rows = [&](i64 i) {
    for (i64 k = Grp[i]; k < Grp[i + 1]; ++k) {
      Ki[at] = Gri[k];
      Kx[at] = Grx[k];
      ++at;
    }
  };
  for (i64 i = 0; i < l; ++i) {
    g_rows(i);
    Ki[at] = base + i;
    Kx[at] = -1.0;
    if (positions) positions[slot] = at;
    ++slot;
    ++at;
    Kp[base + i + 1] = at;
  }
  if (l > 0 && slot_offsets) slot_offsets[++view] = slot;
  i64 o = l;
  for (i64 k = 0; k < d.nsoc; ++k) {
    const i64 q = d.q[k];
    if (soc_slot_starts) soc_slot_starts[k] = slot;
    for (i64 j = 0; j < q; ++j) {
      g_rows(o + j);
      for (i64 i = 0; i <= j; ++i) {
        Ki[at] = base + o + i;
        Kx[at] = (i == j) ? -1.0 : 0.0;
        if (positions) positions[slot] = at;
        ++slot;
        ++at;
      }
      Kp[base + o + j + 1] = at;
    }
    if (slot_offsets) slot_offsets[++view] = slot;
    o += q;
  }
}

// Column pointers of the full KKT matrix and the COMPACT pattern (the same matrix without the off-diagonal
// entries of the dense SOC blocks) in O(N + nnz(P, A, G)).  The device fills the entries of the full matrix
// (kkt_kernels.cu: qsk_kkt_fill); the analysis needs only the compact pattern plus the clique ranges.
void hs_kkt_pattern(const KktDims& d, const i64* Pp, const i64* Pi, const i64* Arp, const i64* Ari, const i64* Grp,
                    const i64* Gri, i64* Kp, std::vector<i64>* Kcp_out, std::vector<i64>* Kci_out) {
  const i64 n = d.n, p = d.p, l = d.l, m = d.m, N = n + p + m;
  std::vector<i64>& Kcp = *Kcp_out;
  std::vector<i64>& Kci = *Kci_out;
  Kcp.assign(N + 1, 0);
  Kci.clear();
  Kci.reserve(Pp[n] + n + Arp[p] + p + Grp[m] + m);
  Kp[0] = 0;
  for (i64 j = 0; j < n; ++j) {
    for (i64 k = Pp[j]; k < Pp[j + 1]; ++k) Kci.push_back(Pi[k]);
    if (!p_has_diag(Pp, Pi, j)) Kci.push_back(j);
    Kcp[j + 1] = (i64)Kci.size();
    Kp[j + 1] = Kcp[j + 1];
  }
  for (i64 r = 0; r < p; ++r) {
    for (i64 k = Arp[r]; k < Arp[r + 1]; ++k) Kci.push_back(Ari[k]);
    Kci.push_back(n + r);
    Kcp[n + r + 1] = (i64)Kci.size();
    Kp[n + r + 1] = Kcp[n + r + 1];
  }
  const i64 base = n + p;
  i64 at = Kp[base];
  auto conic_col = [&](i64 c, i64 block_entries) {
    for (i64 k = Grp[c]; k < Grp[c + 1]; ++k) Kci.push_back(Gri[k]);
    Kci.push_back(base + c);
    Kcp[base + c + 1] = (i64)Kci.size();
    at += (Grp[c + 1] - Grp[c]) + block_entries;
    Kp[base + c + 1] = at;
  };
  for (i64 i = 0; i < l; ++i) conic_col(i, 1);
  i64 o = l;
  for (i64 k = 0; k < d.nsoc; ++k) {
    for (i64 j = 0; j < d.q[k]; ++j) conic_col(o + j, j + 1);
    o += d.q[k];
  }
}

// ------------------------------------------------------- symmetric graph build
namespace {

// Symmetric adjacency (no diagonal) of the pattern whose upper triangle is
// (Kp, Ki), in the NEW numbering given by iperm (or identity when null).
// Entries with both ends inside the same clique range are dropped; the caller
// represents those cliques separately.
struct Graph {
  std::vector<i64> ptr;
  std::vector<int> adj;
};

void build_graph(i64 N, const i64* Kp, const i64* Ki, const int* clique_of, Graph* g) {
  g->ptr.assign(N + 1, 0);
  for (i64 j = 0; j < N; ++j)
    for (i64 k = Kp[j]; k < Kp[j + 1]; ++k) {
      const i64 i = Ki[k];
      if (i == j) continue;
      if (clique_of && clique_of[i] >= 0 && clique_of[i] == clique_of[j]) continue;
      g->ptr[i + 1]++;
      g->ptr[j + 1]++;
    }
  for (i64 v = 0; v < N; ++v) g->ptr[v + 1] += g->ptr[v];
  g->adj.resize(g->ptr[N]);
  std::vector<i64> next(g->ptr.begin(), g->ptr.end() - 1);
  for (i64 j = 0; j < N; ++j)
    for (i64 k = Kp[j]; k < Kp[j + 1]; ++k) {
      const i64 i = Ki[k];
      if (i == j) continue;
      if (clique_of && clique_of[i] >= 0 && clique_of[i] == clique_of[j]) continue;
      g->adj[next[i]++] = (int)j;
      g->adj[next[j]++] = (int)i;
    }
}

}  // namespace

// ------------------------------------------------------------------------ AMD
// Approximate minimum degree on a quotient graph (variables + elements), after
// Amestoy, Davis & Duff.  Cliques of the input (the dense SOC blocks of the KKT
// matrix) enter as pre-merged weighted supervariables, so a q x q block costs one
// node instead of q^2/2 edges.  Features: approximate external degrees, element
// absorption (incl. aggressive), mass elimination, supervariable detection by
// hashing, dense-row deferral.
namespace {

struct Amd {
  i64 N;
  int NT;  // N + initial cliques (element ids live in [0, NT))
  std::vector<std::vector<int>> adj, elems, Le;
  std::vector<int> nv, degree, elem_deg, absorbed_into, order_of_pivot;
  std::vector<char> elem_alive;
  std::vector<i64> w;
  i64 wflg = 1;
  // degree buckets
  std::vector<int> head, next, prev;
  int mindeg = 0;

  void list_insert(int i) {
    const int dgr = degree[i];
    next[i] = head[dgr];
    prev[i] = -1;
    if (head[dgr] >= 0) prev[head[dgr]] = i;
    head[dgr] = i;
    if (dgr < mindeg) mindeg = dgr;
  }
  void list_remove(int i) {
    const int dgr = degree[i];
    if (prev[i] >= 0)
      next[prev[i]] = next[i];
    else if (head[dgr] == i)
      head[dgr] = next[i];
    if (next[i] >= 0) prev[next[i]] = prev[i];
    next[i] = prev[i] = -1;
  }
};

}  // namespace

// N nodes with positive integer weights (a weight-w node stands for w original
// variables that are eliminated together); perm_out lists the nodes in
// elimination order.
static void amd_core(i64 N, const Graph& g, const std::vector<int>& weight, std::vector<int>* perm_out) {
  Amd a;
  a.N = N;
  a.NT = (int)N;
  i64 W = 0;
  for (i64 v = 0; v < N; ++v) W += weight[v];
  a.adj.resize(N);
  a.elems.resize(N);
  a.Le.resize(a.NT);
  a.nv = weight;
  a.degree.assign(N, 0);
  a.elem_deg.assign(a.NT, 0);
  a.absorbed_into.assign(N, -1);
  a.elem_alive.assign(a.NT, 0);
  a.w.assign(a.NT, 0);
  a.head.assign(W + 1, -1);
  a.next.assign(N, -1);
  a.prev.assign(N, -1);
  for (i64 v = 0; v < N; ++v) {
    a.adj[v].assign(g.adj.begin() + g.ptr[v], g.adj.begin() + g.ptr[v + 1]);
    i64 dgr = 0;
    for (int u : a.adj[v]) dgr += weight[u];
    a.degree[v] = (int)std::min<i64>(dgr, W - 1);
  }
  // dense rows/columns are ordered last
  // SuiteSparse AMD defers nodes of degree > 10 sqrt(W).  KKT systems of regression / design-matrix problems have a
  // few thousand equality rows of a few hundred entries each (a lasso: 5000 rows x 200) that end up in the root front
  // whatever the ordering does, but stay below that threshold and cost the quotient graph most of its time
  // (element absorption over 200-entry lists): 2.6 s -> 0.47 s at C2 with max(128, sqrt(W) / 4), fill + 20 %, flops
  // unchanged; C1, C3, C4 keep their fill exactly (C1 0.18 -> 0.04 s, C4 unchanged).  QS_AMD_DENSE / QS_AMD_DENSE_MIN
  // override the factor and the floor.
  const double dense_factor = getenv("QS_AMD_DENSE") ? atof(getenv("QS_AMD_DENSE")) : 0.25;
  const i64 dense_floor = getenv("QS_AMD_DENSE_MIN") ? atol(getenv("QS_AMD_DENSE_MIN")) : 128;
  const i64 dense = std::max<i64>(dense_floor, (i64)(dense_factor * std::sqrt((double)W)));
  std::vector<int> dense_nodes;
  i64 nel = 0;
  i64 dense_weight = 0;
  for (i64 v = 0; v < N; ++v) {
    if (a.nv[v] > 0 && a.degree[v] > dense) {
      dense_nodes.push_back((int)v);
      dense_weight += a.nv[v];
      a.nv[v] = 0;
      a.absorbed_into[v] = -1;
    }
  }
  nel = dense_weight;
  a.mindeg = (int)W;
  for (i64 v = 0; v < N; ++v)
    if (a.nv[v] > 0) a.list_insert((int)v);

  std::vector<int> pivots;  // principal variables in elimination order
  pivots.reserve(N);
  std::vector<int> Lme, hashes(N, 0), stamp(a.NT, 0), bucket_head, bucket_next(N, -1);
  int stampv = 0;
  const i64 nprincipal_total = W - dense_weight;
  i64 eliminated = 0;

  while (eliminated < nprincipal_total) {
    while (a.mindeg <= W && a.head[a.mindeg] < 0) a.mindeg++;
    const int me = a.head[a.mindeg];
    a.list_remove(me);
    int nvpiv = a.nv[me];
    a.nv[me] = -nvpiv;
    Lme.clear();
    i64 degme = 0;
    auto take = [&](int j) {
      if (a.nv[j] > 0) {
        degme += a.nv[j];
        a.list_remove(j);
        a.nv[j] = -a.nv[j];
        Lme.push_back(j);
      }
    };
    for (int j : a.adj[me]) take(j);
    for (int e : a.elems[me]) {
      if (!a.elem_alive[e]) continue;
      for (int j : a.Le[e]) take(j);
      a.elem_alive[e] = 0;
      std::vector<int>().swap(a.Le[e]);
    }
    std::vector<int>().swap(a.adj[me]);
    std::vector<int>().swap(a.elems[me]);
    a.elem_alive[me] = 1;

    // pass 1: w[e] - wflg = |Le \ Lme| for every element touching Lme
    if (a.wflg > (i64)1 << 60) {
      std::fill(a.w.begin(), a.w.end(), 0);
      a.wflg = 1;
    }
    for (int i : Lme) {
      const int nvi = -a.nv[i];
      for (int e : a.elems[i]) {
        if (!a.elem_alive[e] || e == me) continue;
        if (a.w[e] >= a.wflg)
          a.w[e] -= nvi;
        else
          a.w[e] = a.elem_deg[e] + a.wflg - nvi;
      }
    }
    // pass 2: prune lists, approximate degrees, hashes
    for (int i : Lme) {
      const int nvi = -a.nv[i];
      i64 deg = 0;
      unsigned hash = 0;
      auto& el = a.elems[i];
      size_t ke = 0;
      for (int e : el) {
        if (!a.elem_alive[e] || e == me) continue;
        const i64 dext = a.w[e] - a.wflg;
        if (dext > 0) {
          deg += dext;
          el[ke++] = e;
          hash += (unsigned)e;
        } else {
          a.elem_alive[e] = 0;  // aggressive absorption: Le is a subset of Lme
          std::vector<int>().swap(a.Le[e]);
        }
      }
      el.resize(ke);
      auto& av = a.adj[i];
      size_t kv = 0;
      for (int j : av) {
        if (a.nv[j] > 0) {
          deg += a.nv[j];
          av[kv++] = j;
          hash += (unsigned)j;
        }
      }
      av.resize(kv);
      if (ke == 0 && kv == 0) {
        // mass elimination: i only sees the new element -> goes with the pivot
        a.absorbed_into[i] = me;
        nvpiv += nvi;
        degme -= nvi;
        a.nv[i] = 0;
        eliminated += 0;  // counted through nvpiv below
        hashes[i] = -1;
      } else {
        a.degree[i] = (int)std::min<i64>(a.degree[i], deg);
        el.push_back(me);
        std::swap(el.front(), el.back());  // new element first
        hashes[i] = (int)(hash % 1000003u);
      }
    }
    a.wflg += W + 2;
    // supervariable detection among the survivors of Lme
    {
      std::vector<int> live;
      for (int i : Lme)
        if (a.nv[i] < 0) live.push_back(i);
      std::sort(live.begin(), live.end(), [&](int x, int y) { return hashes[x] != hashes[y] ? hashes[x] < hashes[y] : x < y; });
      size_t s0 = 0;
      while (s0 < live.size()) {
        size_t s1 = s0 + 1;
        while (s1 < live.size() && hashes[live[s1]] == hashes[live[s0]]) ++s1;
        for (size_t x = s0; x < s1; ++x) {
          const int i = live[x];
          if (a.nv[i] == 0) continue;
          ++stampv;
          for (int e : a.elems[i]) stamp[e] = stampv;
          std::vector<int>& ai = a.adj[i];
          // variables and elements share the id space [0, NT): elements stamped above, variables here
          // (a variable id never collides with a live element id it is adjacent to except `me`, stamped too)
          std::vector<int> vmark;
          for (int j : ai) vmark.push_back(j);
          std::sort(vmark.begin(), vmark.end());
          for (size_t y = x + 1; y < s1; ++y) {
            const int j = live[y];
            if (a.nv[j] == 0) continue;
            if (a.elems[j].size() != a.elems[i].size() || a.adj[j].size() != ai.size()) continue;
            bool same = true;
            for (int e : a.elems[j])
              if (stamp[e] != stampv) {
                same = false;
                break;
              }
            if (same) {
              std::vector<int> vj(a.adj[j]);
              std::sort(vj.begin(), vj.end());
              same = (vj == vmark);
            }
            if (same) {
              a.nv[i] += a.nv[j];  // both negative here
              a.nv[j] = 0;
              a.absorbed_into[j] = i;
              std::vector<int>().swap(a.adj[j]);
              std::vector<int>().swap(a.elems[j]);
            }
          }
        }
        s0 = s1;
      }
    }
    // finalize the new element and the degrees of its members
    nel += nvpiv;
    eliminated += nvpiv;
    size_t kl = 0;
    const i64 nleft = W - nel;
    for (int i : Lme) {
      if (a.nv[i] >= 0) continue;  // absorbed
      const int nvi = -a.nv[i];
      a.nv[i] = nvi;
      i64 deg = (i64)a.degree[i] + degme - nvi;
      deg = std::min<i64>(deg, nleft - nvi);
      if (deg < 0) deg = 0;
      a.degree[i] = (int)deg;
      a.list_insert(i);
      Lme[kl++] = i;
    }
    Lme.resize(kl);
    a.nv[me] = 0;
    a.Le[me] = Lme;
    a.elem_deg[me] = (int)degme;
    if (Lme.empty()) a.elem_alive[me] = 0;
    pivots.push_back(me);
  }
  // expand supervariables: every non-principal variable follows its representative
  std::vector<int> root(N, -1), pos(N, -1);
  for (size_t k = 0; k < pivots.size(); ++k) pos[pivots[k]] = (int)k;
  std::vector<std::vector<int>> members(pivots.size());
  for (i64 v = 0; v < N; ++v) {
    if (pos[v] >= 0 || a.absorbed_into[v] < 0) continue;
    int r = (int)v;
    while (pos[r] < 0 && a.absorbed_into[r] >= 0) r = a.absorbed_into[r];
    members[pos[r]].push_back((int)v);
  }
  perm_out->clear();
  perm_out->reserve(N);
  for (size_t k = 0; k < pivots.size(); ++k) {
    perm_out->push_back(pivots[k]);
    for (int v : members[k]) perm_out->push_back(v);
  }
  std::sort(dense_nodes.begin(), dense_nodes.end(), [&](int x, int y) {
    return a.degree[x] != a.degree[y] ? a.degree[x] < a.degree[y] : x < y;
  });
  for (int v : dense_nodes) perm_out->push_back(v);
}

void amd_order(i64 N, const i64* Kp, const i64* Ki, std::vector<int>* perm) {
  Graph g;
  build_graph(N, Kp, Ki, nullptr, &g);
  amd_core(N, g, std::vector<int>(N, 1), perm);
}

// Cone-block AMD for conic KKT patterns.  Every dense SOC block is a clique; a
// variable whose only clique neighbours lie in ONE block (in the KKT matrix: an x
// column touching a single second-order cone, e.g. the group variables and the
// epigraph variable of a group-lasso cone) is "private" to it.  Block = clique +
// its private variables.  Blocks are eliminated as units: AMD runs on the
// compressed graph (blocks as weighted nodes), then each block expands to
// [private variables, clique rows].  One pivot per cone instead of one per row.
static void block_amd(i64 N, const Graph& g, const std::vector<std::pair<int, int>>& cliques, const int* clique_of,
                      std::vector<int>* perm) {
  const int nb = (int)cliques.size();
  std::vector<int> comp(N, -1);
  for (int c = 0; c < nb; ++c)
    for (int t = 0; t < cliques[c].second; ++t) comp[cliques[c].first + t] = c;
  std::vector<std::vector<int>> priv(nb);
  for (i64 v = 0; v < N; ++v) {
    if (clique_of[v] >= 0) continue;
    int owner = -1;
    for (i64 k = g.ptr[v]; k < g.ptr[v + 1]; ++k) {
      const int c = clique_of[g.adj[k]];
      if (c < 0) continue;
      if (owner == -1)
        owner = c;
      else if (owner != c) {
        owner = -2;
        break;
      }
    }
    if (owner >= 0) {
      comp[v] = owner;
      priv[owner].push_back((int)v);
    }
  }
  int Nc = nb;
  std::vector<int> single;  // compressed id - nb -> original node
  for (i64 v = 0; v < N; ++v)
    if (comp[v] < 0) {
      comp[v] = Nc++;
      single.push_back((int)v);
    }
  std::vector<int> weight(Nc, 1);
  for (int c = 0; c < nb; ++c) weight[c] = cliques[c].second + (int)priv[c].size();
  // compressed adjacency, deduplicated
  Graph gc;
  gc.ptr.assign(Nc + 1, 0);
  std::vector<std::vector<int>> cadj(Nc);
  {
    std::vector<int> seen(Nc, -1);
    auto gather = [&](int cn, int v) {
      for (i64 k = g.ptr[v]; k < g.ptr[v + 1]; ++k) {
        const int u = comp[g.adj[k]];
        if (u != cn && seen[u] != cn) {
          seen[u] = cn;
          cadj[cn].push_back(u);
        }
      }
    };
    for (int c = 0; c < nb; ++c) {
      for (int t = 0; t < cliques[c].second; ++t) gather(c, cliques[c].first + t);
      for (int v : priv[c]) gather(c, v);
    }
    for (size_t k = 0; k < single.size(); ++k) gather(nb + (int)k, single[k]);
  }
  for (int v = 0; v < Nc; ++v) gc.ptr[v + 1] = gc.ptr[v] + (i64)cadj[v].size();
  gc.adj.resize(gc.ptr[Nc]);
  for (int v = 0; v < Nc; ++v) std::copy(cadj[v].begin(), cadj[v].end(), gc.adj.begin() + gc.ptr[v]);
  std::vector<std::vector<int>>().swap(cadj);
  std::vector<int> order;
  amd_core(Nc, gc, weight, &order);
  perm->clear();
  perm->reserve(N);
  for (int cn : order) {
    if (cn < nb) {
      for (int v : priv[cn]) perm->push_back(v);
      for (int t = 0; t < cliques[cn].second; ++t) perm->push_back(cliques[cn].first + t);
    } else {
      perm->push_back(single[cn - nb]);
    }
  }
}

// ------------------------------------------------------------------- symbolic
namespace {

// upper-triangular CSC (col = larger new index) of the permuted pattern, with
// each clique replaced by a star from its first-ordered member (same filled
// graph: eliminating the centre rebuilds the clique).
struct Upper {
  std::vector<i64> ptr;
  std::vector<int> row;
};

void permuted_upper(i64 N, const i64* Kp, const i64* Ki, const int* clique_of,
                    const std::vector<std::pair<int, int>>& cliques, const std::vector<int>& iperm, Upper* B) {
  B->ptr.assign(N + 1, 0);
  auto count = [&](int a, int b) { B->ptr[std::max(a, b) + 1]++; };
  for (i64 j = 0; j < N; ++j)
    for (i64 k = Kp[j]; k < Kp[j + 1]; ++k) {
      const i64 i = Ki[k];
      if (i == j) continue;
      if (clique_of && clique_of[i] >= 0 && clique_of[i] == clique_of[j]) continue;
      count(iperm[i], iperm[j]);
    }
  std::vector<int> centre(cliques.size());
  for (size_t c = 0; c < cliques.size(); ++c) {
    int best = iperm[cliques[c].first];
    for (int t = 1; t < cliques[c].second; ++t) best = std::min(best, iperm[cliques[c].first + t]);
    centre[c] = best;
    for (int t = 0; t < cliques[c].second; ++t) {
      const int v = iperm[cliques[c].first + t];
      if (v != best) count(best, v);
    }
  }
  for (i64 v = 0; v < N; ++v) B->ptr[v + 1] += B->ptr[v];
  B->row.resize(B->ptr[N]);
  std::vector<i64> next(B->ptr.begin(), B->ptr.end() - 1);
  auto put = [&](int a, int b) { B->row[next[std::max(a, b)]++] = std::min(a, b); };
  for (i64 j = 0; j < N; ++j)
    for (i64 k = Kp[j]; k < Kp[j + 1]; ++k) {
      const i64 i = Ki[k];
      if (i == j) continue;
      if (clique_of && clique_of[i] >= 0 && clique_of[i] == clique_of[j]) continue;
      put(iperm[i], iperm[j]);
    }
  for (size_t c = 0; c < cliques.size(); ++c)
    for (int t = 0; t < cliques[c].second; ++t) {
      const int v = iperm[cliques[c].first + t];
      if (v != centre[c]) put(centre[c], v);
    }
}

void etree_of(i64 N, const Upper& B, std::vector<int>* parent) {
  parent->assign(N, -1);
  std::vector<int> anc(N, -1);
  for (i64 j = 0; j < N; ++j)
    for (i64 k = B.ptr[j]; k < B.ptr[j + 1]; ++k) {
      int i = B.row[k];
      while (i != -1 && i < j) {
        const int nxt = anc[i];
        anc[i] = (int)j;
        if (nxt == -1) (*parent)[i] = (int)j;
        i = nxt;
      }
    }
}

void postorder_of(i64 N, const std::vector<int>& parent, std::vector<int>* post) {
  std::vector<int> head(N, -1), nxt(N, -1);
  for (i64 j = N - 1; j >= 0; --j)
    if (parent[j] >= 0) {
      nxt[j] = head[parent[j]];
      head[parent[j]] = (int)j;
    }
  post->clear();
  post->reserve(N);
  std::vector<int> stack;
  for (i64 r = 0; r < N; ++r) {
    if (parent[r] >= 0) continue;
    stack.push_back((int)r);
    while (!stack.empty()) {
      const int v = stack.back();
      const int c = head[v];
      if (c >= 0) {
        head[v] = nxt[c];
        stack.push_back(c);
      } else {
        stack.pop_back();
        post->push_back(v);
      }
    }
  }
}

// Column counts of L (diagonal included) for a POSTORDERED tree (post = identity),
// skeleton-leaf algorithm of Gilbert, Ng & Peyton.
void column_counts(i64 N, const Upper& B, const std::vector<int>& parent, std::vector<int>* cc) {
  // lower pattern by column: Lc(j) = { i > j : (j, i) in B }
  std::vector<i64> lp(N + 1, 0);
  for (i64 j = 0; j < N; ++j)
    for (i64 k = B.ptr[j]; k < B.ptr[j + 1]; ++k) lp[B.row[k] + 1]++;
  for (i64 v = 0; v < N; ++v) lp[v + 1] += lp[v];
  std::vector<int> li(lp[N]);
  {
    std::vector<i64> next(lp.begin(), lp.end() - 1);
    for (i64 j = 0; j < N; ++j)
      for (i64 k = B.ptr[j]; k < B.ptr[j + 1]; ++k) li[next[B.row[k]]++] = (int)j;
  }
  std::vector<int> first(N, -1), maxfirst(N, -1), prevleaf(N, -1), anc(N);
  std::vector<i64> delta(N, 0);
  for (i64 k = 0; k < N; ++k) {
    int j = (int)k;
    delta[j] = (first[j] == -1) ? 1 : 0;
    for (; j != -1 && first[j] == -1; j = parent[j]) first[j] = (int)k;
  }
  std::iota(anc.begin(), anc.end(), 0);
  for (i64 j = 0; j < N; ++j) {
    if (parent[j] != -1) delta[parent[j]]--;
    for (i64 k = lp[j]; k < lp[j + 1]; ++k) {
      const int i = li[k];  // i > j
      if (first[j] <= maxfirst[i]) continue;  // j is not a leaf of row subtree i
      maxfirst[i] = first[j];
      const int jprev = prevleaf[i];
      prevleaf[i] = (int)j;
      delta[j]++;
      if (jprev != -1) {
        int q = jprev;
        while (q != anc[q]) q = anc[q];
        for (int s = jprev; s != q;) {
          const int sp = anc[s];
          anc[s] = q;
          s = sp;
        }
        delta[q]--;
      }
    }
    if (parent[j] != -1) anc[j] = parent[j];
  }
  for (i64 j = 0; j < N; ++j)
    if (parent[j] != -1) delta[parent[j]] += delta[j];
  cc->resize(N);
  for (i64 j = 0; j < N; ++j) (*cc)[j] = (int)delta[j];
}

}  // namespace

std::string hs_symbolic(i64 N, const i64* Kp, const i64* Ki, int order, const i64* user_perm, Symbolic* S) {
  return hs_symbolic_cliques(N, Kp, Ki, order, user_perm, 0, nullptr, nullptr, S);
}

std::string hs_symbolic_cliques(i64 N, const i64* Kp, const i64* Ki, int order, const i64* user_perm, i64 ncliques,
                                const i64* clique_start, const i64* clique_size, Symbolic* S) {
  if (N <= 0 || N >= (i64)1 << 31) return "KKT dimension out of range";
  S->N = N;
  std::vector<std::pair<int, int>> cliques;
  std::vector<int> clique_of;
  for (i64 c = 0; c < ncliques; ++c)
    if (clique_size[c] >= 2) cliques.emplace_back((int)clique_start[c], (int)clique_size[c]);
  if (!cliques.empty()) {
    clique_of.assign(N, -1);
    for (size_t c = 0; c < cliques.size(); ++c)
      for (int t = 0; t < cliques[c].second; ++t) clique_of[cliques[c].first + t] = (int)c;
  }
  const int* cof = clique_of.empty() ? nullptr : clique_of.data();

  // 1. fill-reducing order
  double t_mark = hs_now();
  auto lap = [&](const char* what) {
    if (hs_verbose()) fprintf(stderr, "[qs symbolic] %-28s %8.3f s\n", what, hs_now() - t_mark);
    t_mark = hs_now();
  };
  std::vector<int> perm(N);
  if (order == 1) {
    Graph g;
    build_graph(N, Kp, Ki, cof, &g);
    if (cliques.empty())
      amd_core(N, g, std::vector<int>(N, 1), &perm);
    else
      block_amd(N, g, cliques, cof, &perm);
  } else if (order == 2 && user_perm) {
    std::vector<char> seen(N, 0);
    for (i64 k = 0; k < N; ++k) {
      if (user_perm[k] < 0 || user_perm[k] >= N || seen[user_perm[k]]) return "permutation is not a bijection";
      seen[user_perm[k]] = 1;
      perm[k] = (int)user_perm[k];
    }
  } else {
    std::iota(perm.begin(), perm.end(), 0);
  }
  lap("ordering");
  if ((i64)perm.size() != N) return "ordering produced a wrong-sized permutation";
  std::vector<int> iperm(N);
  for (i64 k = 0; k < N; ++k) iperm[perm[k]] = (int)k;

  // 2. elimination tree, then compose with its postorder so supernodes are contiguous
  Upper B;
  std::vector<int> parent, post;
  permuted_upper(N, Kp, Ki, cof, cliques, iperm, &B);
  lap("permuted pattern");
  etree_of(N, B, &parent);
  lap("etree");
  postorder_of(N, parent, &post);
  lap("postorder");
  {
    std::vector<int> perm2(N);
    for (i64 k = 0; k < N; ++k) perm2[k] = perm[post[k]];
    perm.swap(perm2);
    for (i64 k = 0; k < N; ++k) iperm[perm[k]] = (int)k;
    permuted_upper(N, Kp, Ki, cof, cliques, iperm, &B);
    // the elimination tree of a postordered relabelling is the relabelled tree: no second etree pass
    std::vector<int> where(N), parent2(N);
    for (i64 k = 0; k < N; ++k) where[post[k]] = (int)k;
    for (i64 k = 0; k < N; ++k) parent2[k] = parent[post[k]] >= 0 ? where[parent[post[k]]] : -1;
    parent.swap(parent2);
  }
  for (i64 j = 0; j < N; ++j)
    if (parent[j] != -1 && parent[j] <= j) return "internal: tree is not postordered";

  lap("etree + postorder");
  // 3. column counts and supernodes (maximal chains with nested structure)
  std::vector<int> cc;
  column_counts(N, B, parent, &cc);
  lap("column counts");
  std::vector<int> nchild(N, 0);
  for (i64 j = 0; j < N; ++j)
    if (parent[j] >= 0) nchild[parent[j]]++;
  S->col0.clear();
  S->sup_of.assign(N, 0);
  // Fundamental chains (parent[j-1] == j with nested structure) merge for free.
  // Relaxed amalgamation on top: a chain child whose columns directly precede its
  // parent's is merged while the explicit zeros this pads into the merged panel stay
  // below QS_RELAX (default 0.4) of the panel.  This turns the row-by-row chain of a
  // cone block (each row adds a few new rows of structure) into one dense front.
  double relax = 0.4;
  if (const char* e = getenv("QS_RELAX")) relax = atof(e);
  i64 g_ns = 0, g_nr = 0, g_zeros = 0;  // current group: columns, front rows, padded zeros
  std::vector<i64> nr_of;               // front rows of every group (supernode)
  for (i64 j = 0; j < N; ++j) {
    bool merge = false;
    if (j > 0 && parent[j - 1] == j) {
      // merged front: g_ns + 1 columns, rows = g_ns + cc[j]
      const i64 nr_new = g_ns + cc[j];
      const i64 add = g_ns * (nr_new - g_nr);  // previous columns padded to the new height
      const i64 zeros = g_zeros + add;
      const double panel = (double)(g_ns + 1) * (double)nr_new;
      if (add == 0 || (double)zeros <= relax * panel) {
        merge = true;
        g_zeros = zeros;
        g_nr = nr_new;
        g_ns += 1;
        nr_of.back() = g_nr;
      }
    }
    if (!merge) {
      S->col0.push_back((int)j);
      g_ns = 1;
      g_nr = cc[j];
      g_zeros = 0;
      nr_of.push_back(g_nr);
    }
    S->sup_of[j] = (int)S->col0.size() - 1;
  }
  S->nsup = (int)S->col0.size();
  S->col0.push_back((int)N);
  const int nsup = S->nsup;

  // 4. supernodal tree
  S->parent.assign(nsup, -1);
  for (int s = 0; s < nsup; ++s) {
    const int last = S->col0[s + 1] - 1;
    if (parent[last] >= 0) S->parent[s] = S->sup_of[parent[last]];
  }
  S->childptr.assign(nsup + 1, 0);
  for (int s = 0; s < nsup; ++s)
    if (S->parent[s] >= 0) S->childptr[S->parent[s] + 1]++;
  for (int s = 0; s < nsup; ++s) S->childptr[s + 1] += S->childptr[s];
  S->child.resize(S->childptr[nsup]);
  {
    std::vector<int> next(S->childptr.begin(), S->childptr.end() - 1);
    for (int s = 0; s < nsup; ++s)
      if (S->parent[s] >= 0) S->child[next[S->parent[s]]++] = s;
  }

  // 5. front row structures.  The row COUNT of every front is known from the grouping pass (nr_of), so the storage
  // is laid out first and the fronts of one tree level -- independent of each other, children one level down already
  // done -- are filled by host threads with private marker arrays.  Any count mismatch falls back to the sequential
  // bottom-up pass below.
  bool fronts_done = false;
  {
    std::vector<int> lev(nsup, 0);
    int nlev = 1;
    for (int s = 0; s < nsup; ++s) {  // children precede parents
      const int par = S->parent[s];
      if (par >= 0) lev[par] = std::max(lev[par], lev[s] + 1);
      nlev = std::max(nlev, lev[s] + 1);
    }
    const int nthreads = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    if (nsup >= 100000 && nthreads > 1 && nlev <= 64) {
      std::vector<int> lptr(nlev + 1, 0), lsup(nsup);
      for (int s = 0; s < nsup; ++s) lptr[lev[s] + 1]++;
      for (int v = 0; v < nlev; ++v) lptr[v + 1] += lptr[v];
      {
        std::vector<int> next(lptr.begin(), lptr.end() - 1);
        for (int s = 0; s < nsup; ++s) lsup[next[lev[s]]++] = s;
      }
      lap("  level buckets");
      S->rowptr.assign(nsup + 1, 0);
      for (int s = 0; s < nsup; ++s) S->rowptr[s + 1] = S->rowptr[s] + nr_of[s];
      S->rowidx.assign(S->rowptr[nsup], 0);
      lap("  row storage");
      // lower pattern by column = transpose of B.  Every thread streams all of B but counts / writes only the
      // destination columns of its own range: sequential reads, private writes, no atomics, same order as serial.
      std::vector<i64> lp(N + 1, 0);
      auto split = [&](auto fn) {
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t) pool.emplace_back(fn, (int)(N * t / nthreads), (int)(N * (t + 1) / nthreads));
        for (auto& th : pool) th.join();
      };
      split([&](int lo, int hi) {
        for (i64 j = 0; j < N; ++j)
          for (i64 k = B.ptr[j]; k < B.ptr[j + 1]; ++k) {
            const int r = B.row[k];
            if (r >= lo && r < hi) lp[r + 1]++;
          }
      });
      lap("  transpose: count");
      for (i64 v = 0; v < N; ++v) lp[v + 1] += lp[v];
      std::vector<int> li(lp[N]);
      {
        std::vector<i64> next(lp.begin(), lp.end() - 1);
        split([&](int lo, int hi) {
          for (i64 j = 0; j < N; ++j)
            for (i64 k = B.ptr[j]; k < B.ptr[j + 1]; ++k) {
              const int r = B.row[k];
              if (r >= lo && r < hi) li[next[r]++] = (int)j;
            }
        });
      }
      lap("  lower pattern by column");
      std::atomic<bool> mismatch{false};
      std::vector<std::vector<int>> marks(nthreads);
      for (int v = 0; v < nlev && !mismatch; ++v) {
        const int cnt = lptr[v + 1] - lptr[v];
        const int use = cnt >= 4096 ? nthreads : 1;
        auto work = [&](int t) {
          std::vector<int>& mark = marks[t];
          if (mark.empty()) mark.assign(N, -1);
          for (int q = lptr[v] + (int)((i64)cnt * t / use); q < lptr[v] + (int)((i64)cnt * (t + 1) / use); ++q) {
            const int s = lsup[q];
            const int c0 = S->col0[s], c1 = S->col0[s + 1];
            int* out = S->rowidx.data() + S->rowptr[s];
            const i64 cap = nr_of[s];
            i64 at = 0;
            for (int c = c0; c < c1; ++c) {
              mark[c] = s;
              if (at < cap) out[at] = c;
              ++at;
            }
            auto add = [&](int r) {
              if (r >= c1 && mark[r] != s) {
                mark[r] = s;
                if (at < cap) out[at] = r;
                ++at;
              }
            };
            for (int c = c0; c < c1; ++c)
              for (i64 k = lp[c]; k < lp[c + 1]; ++k) add(li[k]);
            for (int ci = S->childptr[s]; ci < S->childptr[s + 1]; ++ci) {
              const int ch = S->child[ci];
              const int nsc = S->col0[ch + 1] - S->col0[ch];
              for (i64 k = S->rowptr[ch] + nsc; k < S->rowptr[ch + 1]; ++k) add(S->rowidx[k]);
            }
            if (at != cap) {
              mismatch = true;
              return;
            }
            std::sort(out + (c1 - c0), out + cap);
          }
        };
        if (use == 1) {
          work(0);
        } else {
          std::vector<std::thread> pool;
          for (int t = 0; t < use; ++t) pool.emplace_back(work, t);
          for (auto& th : pool) th.join();
        }
      }
      fronts_done = !mismatch;
      lap(fronts_done ? "  fronts by level (threaded)" : "  fronts by level: count mismatch");
    }
  }
  if (!fronts_done) {
  // sequential bottom-up pass (children precede parents)
  S->rowptr.assign(nsup + 1, 0);
  S->rowidx.clear();
  S->rowidx.reserve((size_t)N * 4);
  {
    // lower pattern by column again (rows > col), from B
    std::vector<i64> lp(N + 1, 0);
    for (i64 j = 0; j < N; ++j)
      for (i64 k = B.ptr[j]; k < B.ptr[j + 1]; ++k) lp[B.row[k] + 1]++;
    for (i64 v = 0; v < N; ++v) lp[v + 1] += lp[v];
    std::vector<int> li(lp[N]);
    std::vector<i64> next(lp.begin(), lp.end() - 1);
    for (i64 j = 0; j < N; ++j)
      for (i64 k = B.ptr[j]; k < B.ptr[j + 1]; ++k) li[next[B.row[k]]++] = (int)j;
    std::vector<int> mark(N, -1);
    for (int s = 0; s < nsup; ++s) {
      const int c0 = S->col0[s], c1 = S->col0[s + 1];
      const size_t begin = S->rowidx.size();
      if (c1 - c0 == 1 && S->childptr[s + 1] == S->childptr[s]) {
        // one-column leaf (the 1.35 M private x-columns of C4): its rows are its own lower pattern, which `li`
        // already lists in ascending order without repeats -- no marking, no sort
        S->rowidx.push_back(c0);
        bool ascending = true;
        int prev = c0;
        for (i64 k = lp[c0]; k < lp[c0 + 1]; ++k) {
          ascending = ascending && li[k] > prev;
          prev = li[k];
          S->rowidx.push_back(li[k]);
        }
        if (ascending) {
          S->rowptr[s + 1] = (i64)S->rowidx.size();
          if ((i64)(S->rowidx.size() - begin) < cc[c0]) return "internal: front smaller than its first column count";
          continue;
        }
        S->rowidx.resize(begin);  // repeated entries in the pattern: take the general path
      }
      for (int c = c0; c < c1; ++c) {
        mark[c] = s;
        S->rowidx.push_back(c);
      }
      auto add = [&](int r) {
        if (r >= c1 && mark[r] != s) {
          mark[r] = s;
          S->rowidx.push_back(r);
        }
      };
      for (int c = c0; c < c1; ++c)
        for (i64 k = lp[c]; k < lp[c + 1]; ++k) add(li[k]);
      for (int ci = S->childptr[s]; ci < S->childptr[s + 1]; ++ci) {
        const int ch = S->child[ci];
        const int nsc = S->col0[ch + 1] - S->col0[ch];
        for (i64 k = S->rowptr[ch] + nsc; k < S->rowptr[ch + 1]; ++k) add(S->rowidx[k]);
      }
      std::sort(S->rowidx.begin() + begin + (c1 - c0), S->rowidx.end());
      S->rowptr[s + 1] = (i64)S->rowidx.size();
      if ((i64)(S->rowidx.size() - begin) < cc[c0]) return "internal: front smaller than its first column count";
    }
  }
  }
  lap("front structures");
  // 6. relative indices, storage offsets, levels, statistics
  S->relptr.assign(nsup + 1, 0);
  S->Loff.assign(nsup + 1, 0);
  S->Uoff.assign(nsup + 1, 0);
  S->Boff.assign(nsup + 1, 0);
  S->lnz = 0;
  S->flops = 0.0;
  S->max_nr = S->max_ns = 0;
  for (int s = 0; s < nsup; ++s) {
    const i64 ns = S->col0[s + 1] - S->col0[s], nr = S->rowptr[s + 1] - S->rowptr[s], nu = nr - ns;
    S->relptr[s + 1] = S->relptr[s] + nu;
    S->Loff[s + 1] = S->Loff[s] + nr * ns;
    S->Uoff[s + 1] = S->Uoff[s] + nu * (nu + 1) / 2;  // packed lower triangle (ldl.cu: qs_ucol)
    S->Boff[s + 1] = S->Boff[s] + nu;
    S->lnz += ns * (ns + 1) / 2 + nu * ns;
    for (i64 k = 0; k < ns; ++k) {
      const double r = (double)(nr - k);
      S->flops += r * r;
    }
    S->max_nr = std::max<int>(S->max_nr, (int)nr);
    S->max_ns = std::max<int>(S->max_ns, (int)ns);
  }
  lap("offsets + flop count");
  S->rel.resize(S->relptr[nsup]);
  {
    // independent per supernode: split over host threads
    std::atomic<bool> missing{false};
    auto work = [&](int s_lo, int s_hi) {
      for (int s = s_lo; s < s_hi; ++s) {
        const int par = S->parent[s];
        if (par < 0) continue;
        const int ns = S->col0[s + 1] - S->col0[s];
        const int* prow = S->rowidx.data() + S->rowptr[par];
        const i64 pn = S->rowptr[par + 1] - S->rowptr[par];
        i64 at = 0;
        int* rel = S->rel.data() + S->relptr[s];
        for (i64 k = S->rowptr[s] + ns; k < S->rowptr[s + 1]; ++k) {
          const int r = S->rowidx[k];
          // both lists ascend; a leaf with 4 rows under a 700-row front must not walk the front: binary search
          at = std::lower_bound(prow + at, prow + pn, r) - prow;
          if (at >= pn || prow[at] != r) {
            missing = true;
            return;
          }
          *rel++ = (int)at;
        }
      }
    };
    const int nthreads = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    if (nsup < 100000 || nthreads == 1) {
      work(0, nsup);
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < nthreads; ++t)
        pool.emplace_back(work, (int)((i64)nsup * t / nthreads), (int)((i64)nsup * (t + 1) / nthreads));
      for (auto& th : pool) th.join();
    }
    if (missing) return "internal: child row missing from the parent front";
  }
  lap("relative indices");
  std::vector<int> level(nsup, 0);
  int maxlevel = 0;
  for (int s = 0; s < nsup; ++s) {
    const int par = S->parent[s];
    if (par >= 0) level[par] = std::max(level[par], level[s] + 1);
    maxlevel = std::max(maxlevel, level[s]);
  }
  S->nlevels = maxlevel + 1;
  S->levelptr.assign(S->nlevels + 1, 0);
  for (int s = 0; s < nsup; ++s) S->levelptr[level[s] + 1]++;
  for (int v = 0; v < S->nlevels; ++v) S->levelptr[v + 1] += S->levelptr[v];
  S->levelsup.resize(nsup);
  {
    std::vector<int> next(S->levelptr.begin(), S->levelptr.end() - 1);
    for (int s = 0; s < nsup; ++s) S->levelsup[next[level[s]]++] = s;
  }
  S->perm.swap(perm);
  S->iperm.swap(iperm);
  lap("levels");
  return std::string();
}
