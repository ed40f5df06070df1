/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain-C restatement of the reference's fill-reducing ordering
 * (/root/reference/pkg/src/qsocp/_amd.py:97-390, `_amd_kernel`): approximate
 * minimum degree on a quotient graph with element absorption, mass
 * elimination, supervariable detection by hashing, in-place compaction of the
 * adjacency store, and a lazy binary heap keyed by degree*(n+1)+vertex so that
 * ties go to the smallest vertex index.  The oracle needs its own ordering so
 * that neither the parity checker nor the CPU baseline touches the product
 * library (libqsocp_cuda.so).
 *
 * Parity status: PINNED -- tests/test_oracle_pinned.py compares the returned
 * permutation element by element with the reference's `amd_order` (imported
 * from /root/reference when present) and with the `amd_perm` arrays stored in
 * tests/golden/*.npz by oracle/gen_golden.py.
 *
 * The sequence of pivots depends only on the multiset of live heap keys, so
 * the heap capacity (the reference allocates 4*cnz+4n+64 words) may be smaller
 * here without changing the result: a full heap is compacted to its live
 * entries exactly as in _amd.py:57-83.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

typedef int64_t i64;

#define FLIP(i) (-(i) - 2) /* _amd.py:13-18 */

static void sift_down(i64 *heap, i64 size, i64 i) {
  for (;;) {
    i64 l = 2 * i + 1, r = l + 1, small = i;
    if (l < size && heap[l] < heap[small]) small = l;
    if (r < size && heap[r] < heap[small]) small = r;
    if (small == i) return;
    i64 t = heap[small];
    heap[small] = heap[i];
    heap[i] = t;
    i = small;
  }
}

/* _amd.py:21-31 */
static i64 heap_push(i64 *heap, i64 size, i64 key) {
  i64 i = size;
  heap[i] = key;
  while (i > 0) {
    i64 parent = (i - 1) >> 1;
    if (heap[parent] <= heap[i]) break;
    i64 t = heap[parent];
    heap[parent] = heap[i];
    heap[i] = t;
    i = parent;
  }
  return size + 1;
}

/* _amd.py:34-53 */
static i64 heap_pop(i64 *heap, i64 *size) {
  i64 top = heap[0];
  *size -= 1;
  if (*size > 0) {
    heap[0] = heap[*size];
    sift_down(heap, *size, 0);
  }
  return top;
}

/* _amd.py:56-83 : keep one live entry per vertex whose key still carries the
 * vertex's current degree, then re-heapify bottom-up. */
static i64 heap_compact(i64 *heap, i64 size, i64 stride, const i64 *degree,
                        const i64 *elen, const i64 *nv, i64 *seen, i64 stamp) {
  i64 out = 0;
  for (i64 i = 0; i < size; ++i) {
    i64 key = heap[i], v = key % stride, d = key / stride;
    if (elen[v] >= 0 && nv[v] > 0 && degree[v] == d && seen[v] != stamp) {
      seen[v] = stamp;
      heap[out++] = key;
    }
  }
  for (i64 start = (out - 2) >> 1; start >= 0; --start) sift_down(heap, out, start);
  return out;
}

/* _amd.py:86-93 */
static i64 wclear(i64 mark, i64 lemax, i64 *w, i64 n) {
  if (mark < 2 || mark + lemax < 0) {
    for (i64 k = 0; k < n; ++k)
      if (w[k] != 0) w[k] = 1;
    mark = 2;
  }
  return mark;
}

/* _amd.py:96-390.  Cp[n+2] / Ci[nzmax] hold the symmetric adjacency without the
 * diagonal (first cnz words used); heap[heap_cap], seen[n+1] are workspace.
 * Writes the postordered permutation to order[n]; returns n, or 0 when the
 * heap runs dry before every vertex is eliminated (the reference returns an
 * empty array there), or -1 if workspace allocation fails. */
i64 orc_amd_kernel(i64 n, i64 *Cp, i64 *Ci, i64 nzmax, i64 cnz, i64 *heap,
                   i64 heap_cap, i64 *seen, i64 *order) {
  const i64 stride = n + 1;
  i64 *ws = (i64 *)malloc((size_t)(9 * (n + 1)) * sizeof(i64));
  if (!ws) return -1;
  i64 *lenv = ws, *elen = lenv + (n + 1), *nv = elen + (n + 1),
      *degree = nv + (n + 1), *w = degree + (n + 1), *hhead = w + (n + 1),
      *next_ = hhead + (n + 1), *last = next_ + (n + 1), *post = last + (n + 1);
  for (i64 i = 0; i <= n; ++i) {
    elen[i] = 0;
    nv[i] = 1;
    w[i] = 1;
    hhead[i] = next_[i] = last[i] = -1;
  }

  i64 dense = 10 * (i64)sqrt((double)n); /* _amd.py:110-113 */
  if (dense < 16) dense = 16;
  if (dense > n - 2) dense = n - 2;
  if (dense < 0) dense = 0;

  for (i64 i = 0; i < n; ++i) degree[i] = lenv[i] = Cp[i + 1] - Cp[i];
  lenv[n] = degree[n] = 0;
  elen[n] = -2;
  w[n] = 0;
  i64 nel = 0, lemax = 0, hsize = 0, stamp = 1;
  i64 mark = wclear(0, 0, w, n);
  Cp[n] = -1;

  for (i64 i = 0; i < n; ++i) { /* _amd.py:131-145 */
    i64 d = degree[i];
    if (d == 0) { /* isolated vertex: already an (empty) element */
      elen[i] = -2;
      ++nel;
      Cp[i] = -1;
      w[i] = 0;
    } else if (d > dense) { /* dense row: deferred to the end */
      nv[i] = 0;
      elen[i] = -1;
      ++nel;
      Cp[i] = FLIP(n);
      ++nv[n];
    } else {
      hsize = heap_push(heap, hsize, d * stride + i);
    }
  }

  while (nel < n) {
    i64 k;
    for (;;) { /* _amd.py:149-156 : smallest live key */
      if (hsize == 0) {
        free(ws);
        return 0;
      }
      i64 key = heap_pop(heap, &hsize);
      k = key % stride;
      if (elen[k] >= 0 && nv[k] > 0 && degree[k] == key / stride) break;
    }
    const i64 elenk = elen[k];
    i64 nvk = nv[k];
    nel += nvk;

    if (elenk > 0 && cnz + degree[k] >= nzmax) { /* _amd.py:162-181 */
      for (i64 j = 0; j < n; ++j) {
        i64 p = Cp[j];
        if (p >= 0) {
          Cp[j] = Ci[p];
          Ci[p] = FLIP(j);
        }
      }
      i64 q = 0, p = 0;
      while (p < cnz) {
        i64 j = FLIP(Ci[p]);
        ++p;
        if (j >= 0) {
          Ci[q] = Cp[j];
          Cp[j] = q++;
          for (i64 k3 = 0; k3 < lenv[j] - 1; ++k3) Ci[q++] = Ci[p++];
        }
      }
      cnz = q;
    }

    /* _amd.py:184-217 : the new element = union of k's variables and of the
     * variables of every element adjacent to k */
    i64 dk = 0;
    nv[k] = -nvk;
    i64 p = Cp[k];
    const i64 pk1 = (elenk == 0) ? p : cnz;
    i64 pk2 = pk1;
    for (i64 k1 = 1; k1 <= elenk + 1; ++k1) {
      i64 e, pj, ln;
      if (k1 > elenk) {
        e = k;
        pj = p;
        ln = lenv[k] - elenk;
      } else {
        e = Ci[p++];
        pj = Cp[e];
        ln = lenv[e];
      }
      for (i64 k2 = 0; k2 < ln; ++k2) {
        i64 i = Ci[pj++];
        i64 nvi = nv[i];
        if (nvi <= 0) continue;
        dk += nvi;
        nv[i] = -nvi;
        Ci[pk2++] = i;
      }
      if (e != k) {
        Cp[e] = FLIP(k);
        w[e] = 0;
      }
    }
    if (elenk != 0) cnz = pk2;
    degree[k] = dk;
    Cp[k] = pk1;
    lenv[k] = pk2 - pk1;
    elen[k] = -2;

    /* _amd.py:220-233 : |Le \ Lk| for every element touching the new one */
    mark = wclear(mark, lemax, w, n);
    for (i64 pk = pk1; pk < pk2; ++pk) {
      i64 i = Ci[pk], eln = elen[i];
      if (eln <= 0) continue;
      i64 nvi = -nv[i], wnvi = mark - nvi;
      for (i64 q = Cp[i]; q < Cp[i] + eln; ++q) {
        i64 e = Ci[q];
        if (w[e] >= mark)
          w[e] -= nvi;
        else if (w[e] != 0)
          w[e] = degree[e] + wnvi;
      }
    }

    /* _amd.py:236-286 : prune, approximate degree, absorb, hash */
    for (i64 pk = pk1; pk < pk2; ++pk) {
      i64 i = Ci[pk];
      i64 p1 = Cp[i], p2 = p1 + elen[i] - 1, pn = p1, h = 0, d = 0;
      for (i64 q = p1; q <= p2; ++q) {
        i64 e = Ci[q];
        if (w[e] != 0) {
          i64 dext = w[e] - mark;
          if (dext > 0) {
            d += dext;
            Ci[pn++] = e;
            h += e;
          } else { /* aggressive absorption */
            Cp[e] = FLIP(k);
            w[e] = 0;
          }
        }
      }
      elen[i] = pn - p1 + 1;
      i64 p3 = pn, p4 = p1 + lenv[i];
      for (i64 q = p2 + 1; q < p4; ++q) {
        i64 j = Ci[q], nvj = nv[j];
        if (nvj <= 0) continue;
        d += nvj;
        Ci[pn++] = j;
        h += j;
      }
      if (d == 0) { /* mass elimination */
        Cp[i] = FLIP(k);
        i64 nvi = -nv[i];
        dk -= nvi;
        nvk += nvi;
        nel += nvi;
        nv[i] = 0;
        elen[i] = -1;
      } else {
        if (d < degree[i]) degree[i] = d;
        Ci[pn] = Ci[p3];
        Ci[p3] = Ci[p1];
        Ci[p1] = k;
        lenv[i] = pn - p1 + 1;
        h = h % n;
        next_[i] = hhead[h];
        hhead[h] = i;
        last[i] = h;
      }
    }
    degree[k] = dk;
    if (dk > lemax) lemax = dk;
    mark = wclear(mark + lemax, lemax, w, n);

    /* _amd.py:292-324 : indistinguishable variables inside one hash bucket */
    for (i64 pk = pk1; pk < pk2; ++pk) {
      i64 i = Ci[pk];
      if (nv[i] >= 0) continue;
      i64 h = last[i];
      i = hhead[h];
      hhead[h] = -1;
      while (i != -1 && next_[i] != -1) {
        i64 ln = lenv[i], eln = elen[i];
        for (i64 q = Cp[i] + 1; q < Cp[i] + ln; ++q) w[Ci[q]] = mark;
        i64 jlast = i, j = next_[i];
        while (j != -1) {
          int same = (lenv[j] == ln && elen[j] == eln);
          for (i64 q = Cp[j] + 1; same && q < Cp[j] + ln; ++q)
            if (w[Ci[q]] != mark) same = 0;
          if (same) {
            Cp[j] = FLIP(i);
            nv[i] += nv[j];
            nv[j] = 0;
            elen[j] = -1;
            j = next_[j];
            next_[jlast] = j;
          } else {
            jlast = j;
            j = next_[j];
          }
        }
        i = next_[i];
        ++mark;
      }
    }

    /* _amd.py:327-353 : final degrees, requeue what is left of the front */
    p = pk1;
    for (i64 pk = pk1; pk < pk2; ++pk) {
      i64 i = Ci[pk], nvi = -nv[i];
      if (nvi <= 0) continue;
      nv[i] = nvi;
      i64 d = degree[i] + dk - nvi, dcap = n - nel - nvi;
      if (dcap < d) d = dcap;
      if (d < 0) d = 0;
      degree[i] = d;
      if (hsize + 1 > heap_cap) {
        ++stamp;
        hsize = heap_compact(heap, hsize, stride, degree, elen, nv, seen, stamp);
        if (hsize + 1 > heap_cap) { /* cannot happen with heap_cap >= n+1 */
          free(ws);
          return -1;
        }
      }
      hsize = heap_push(heap, hsize, d * stride + i);
      Ci[p++] = i;
    }
    nv[k] = nvk;
    lenv[k] = p - pk1;
    if (lenv[k] == 0) {
      Cp[k] = -1;
      w[k] = 0;
    }
    if (elenk != 0) cnz = p;
  }

  /* _amd.py:356-390 : assembly-tree postorder */
  for (i64 i = 0; i <= n; ++i) Cp[i] = FLIP(Cp[i]);
  for (i64 j = 0; j <= n; ++j) hhead[j] = -1;
  for (i64 j = n; j >= 0; --j) {
    if (nv[j] > 0) continue;
    next_[j] = hhead[Cp[j]];
    hhead[Cp[j]] = j;
  }
  for (i64 e = n; e >= 0; --e) {
    if (nv[e] <= 0) continue;
    if (Cp[e] != -1) {
      next_[e] = hhead[Cp[e]];
      hhead[Cp[e]] = e;
    }
  }
  i64 *stack = last, kout = 0;
  for (i64 root = 0; root <= n; ++root) {
    if (Cp[root] != -1) continue;
    i64 top = 0;
    stack[0] = root;
    while (top >= 0) {
      i64 node = stack[top], child = hhead[node];
      if (child == -1) {
        --top;
        post[kout++] = node;
      } else {
        hhead[node] = next_[child];
        stack[++top] = child;
      }
    }
  }
  for (i64 i = 0; i < n; ++i) order[i] = post[i];
  free(ws);
  return n;
}
