/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain-C, single-threaded CPU restatement of the reference solver's numeric
 * kernels (the reference is Python + numba; nothing here is shipped or called
 * by paper_2603_29197_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * Parity status: PINNED.  tests/test_oracle_pinned.py compares every function
 * below with the unmodified reference imported from /root/reference (when that
 * tree is present) and with fixtures under tests/golden/ that were generated
 * by the reference itself (oracle/gen_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared  (no FMA contraction, so the
 * floating-point sequence equals the reference's numba loops operation for
 * operation).
 *
 * Each function names the reference lines it follows.  All indices int64, all
 * values float64, exactly like the reference (sparse.py:18-19).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
#define UNBOUNDED DBL_MAX /* _cone_kernels.py:13 */

/* ------------------------------------------------------------------ cones */

/* _cone_kernels.py:16-53 : NT scaling of every SOC; returns 1 if some cone is
 * not strictly interior. */
int orc_soc_nt_scaling(const double *s, const double *z, const i64 *starts,
                       const i64 *dims, i64 nsoc, double *eta, double *wbar,
                       double *lam) {
  for (i64 k = 0; k < nsoc; ++k) {
    const i64 o = starts[k], e = o + dims[k];
    const double s0 = s[o], z0 = z[o];
    double sres = s0 * s0, zres = z0 * z0;
    for (i64 t = o + 1; t < e; ++t) {
      sres -= s[t] * s[t];
      zres -= z[t] * z[t];
    }
    if (s0 <= 0.0 || z0 <= 0.0 || sres <= 0.0 || zres <= 0.0) return 1;
    const double sa = sqrt(sres), za = sqrt(zres);
    double sz = 0.0;
    for (i64 t = o; t < e; ++t) sz += s[t] * z[t];
    const double gamma = sqrt((1.0 + sz / (sa * za)) / 2.0);
    const double nt0 = (s0 / sa + z0 / za) / (2.0 * gamma);
    const double den = sqrt(2.0 * (1.0 + nt0)); /* Jordan square root, :40-44 */
    wbar[o] = (nt0 + 1.0) / den;
    for (i64 t = o + 1; t < e; ++t)
      wbar[t] = (s[t] / sa - z[t] / za) / (2.0 * gamma) / den;
    const double ek = sqrt(sa / za);
    eta[k] = ek;
    double wz = 0.0;
    for (i64 t = o; t < e; ++t) wz += wbar[t] * z[t];
    lam[o] = ek * (2.0 * wbar[o] * wz - z0);
    for (i64 t = o + 1; t < e; ++t) lam[t] = ek * (2.0 * wbar[t] * wz + z[t]);
  }
  return 0;
}

/* _cone_kernels.py:56-74 : out = W u, or W^{-1} u when inverse != 0. */
void orc_soc_apply_w(const double *eta, const double *wbar, const i64 *starts,
                     const i64 *dims, i64 nsoc, const double *u, double *out,
                     int inverse) {
  for (i64 k = 0; k < nsoc; ++k) {
    const i64 o = starts[k], e = o + dims[k];
    const double scale = inverse ? 1.0 / eta[k] : eta[k];
    const double sgn = inverse ? -1.0 : 1.0;
    double dot = wbar[o] * u[o];
    for (i64 t = o + 1; t < e; ++t) dot += sgn * wbar[t] * u[t];
    out[o] = scale * (2.0 * wbar[o] * dot - u[o]);
    for (i64 t = o + 1; t < e; ++t)
      out[t] = scale * (2.0 * sgn * wbar[t] * dot + u[t]);
  }
}

/* _cone_kernels.py:77-89 */
void orc_soc_jordan(const double *u, const double *v, double *out,
                    const i64 *starts, const i64 *dims, i64 nsoc) {
  for (i64 k = 0; k < nsoc; ++k) {
    const i64 o = starts[k], e = o + dims[k];
    double dot = 0.0;
    for (i64 t = o; t < e; ++t) dot += u[t] * v[t];
    const double u0 = u[o], v0 = v[o];
    out[o] = dot;
    for (i64 t = o + 1; t < e; ++t) out[t] = u0 * v[t] + v0 * u[t];
  }
}

/* _cone_kernels.py:92-106 : solve lam o x = v. */
void orc_soc_jordan_div(const double *lam, const double *v, double *out,
                        const i64 *starts, const i64 *dims, i64 nsoc) {
  for (i64 k = 0; k < nsoc; ++k) {
    const i64 o = starts[k], e = o + dims[k];
    const double a = lam[o];
    double den = a * a, cross = 0.0;
    for (i64 t = o + 1; t < e; ++t) {
      den -= lam[t] * lam[t];
      cross += lam[t] * v[t];
    }
    const double u0 = (a * v[o] - cross) / den;
    out[o] = u0;
    for (i64 t = o + 1; t < e; ++t) out[t] = (v[t] - u0 * lam[t]) / a;
  }
}

/* _cone_kernels.py:109-146 : smallest boundary-exit step over all SOCs. */
double orc_soc_max_step(const double *u, const double *du, const i64 *starts,
                        const i64 *dims, i64 nsoc) {
  double best = UNBOUNDED;
  for (i64 k = 0; k < nsoc; ++k) {
    const i64 o = starts[k], e = o + dims[k];
    double a = du[o] * du[o], b = u[o] * du[o], c = u[o] * u[o];
    for (i64 t = o + 1; t < e; ++t) {
      a -= du[t] * du[t];
      b -= u[t] * du[t];
      c -= u[t] * u[t];
    }
    b *= 2.0;
    double step;
    if (a == 0.0) {
      step = (b < 0.0) ? -c / b : UNBOUNDED;
    } else {
      const double disc = b * b - 4.0 * a * c;
      if (a > 0.0 && disc < 0.0) {
        step = UNBOUNDED;
      } else {
        const double sq = sqrt(disc);
        double r1, den;
        if (b >= 0.0) {
          r1 = (-b - sq) / (2.0 * a);
          den = -b - sq;
        } else {
          r1 = (-b + sq) / (2.0 * a);
          den = -b + sq;
        }
        const double r2 = (den != 0.0) ? 2.0 * c / den : UNBOUNDED;
        step = UNBOUNDED;
        if (0.0 < r1 && r1 < step) step = r1;
        if (0.0 < r2 && r2 < step) step = r2;
      }
    }
    if (step < best) best = step;
  }
  return best;
}

/* _cone_kernels.py:149-162 : max_k |u_tail| - u_head (-inf with no cones). */
double orc_soc_violation(const double *u, const i64 *starts, const i64 *dims,
                         i64 nsoc) {
  double worst = -INFINITY;
  for (i64 k = 0; k < nsoc; ++k) {
    const i64 o = starts[k], e = o + dims[k];
    double nrm = 0.0;
    for (i64 t = o + 1; t < e; ++t) nrm += u[t] * u[t];
    const double v = sqrt(nrm) - u[o];
    if (v > worst) worst = v;
  }
  return worst;
}

/* _cone_kernels.py:165-186 : -W'W, packed upper triangle, column-major. */
void orc_soc_neg_wtw(const double *eta, const double *wbar, const i64 *starts,
                     const i64 *dims, i64 nsoc, const i64 *slot_starts,
                     double *out) {
  for (i64 k = 0; k < nsoc; ++k) {
    const i64 o = starts[k], d = dims[k];
    const double e2 = eta[k] * eta[k];
    double c = 0.0;
    for (i64 t = o; t < o + d; ++t) c += wbar[t] * wbar[t];
    i64 slot = slot_starts[k];
    for (i64 j = 0; j < d; ++j) {
      const double wj = wbar[o + j];
      const double jj = (j == 0) ? wj : -wj;
      for (i64 i = 0; i <= j; ++i) {
        const double wi = wbar[o + i];
        const double ji = (i == 0) ? wi : -wi;
        double v = 4.0 * c * wi * wj - 2.0 * wi * jj - 2.0 * ji * wj;
        if (i == j) v += 1.0;
        out[slot++] = -e2 * v;
      }
    }
  }
}

/* ------------------------------------------------------------------- spmv */

/* _kernels.py:13-20 : out += M x (column scatter; skips x_j == 0). */
void orc_csc_matvec(i64 ncols, const i64 *cp, const i64 *ri, const double *vx,
                    const double *x, double *out) {
  for (i64 j = 0; j < ncols; ++j) {
    const double xj = x[j];
    if (xj != 0.0)
      for (i64 p = cp[j]; p < cp[j + 1]; ++p) out[ri[p]] += vx[p] * xj;
  }
}

/* _kernels.py:23-30 : out += M' x (column gather-dot). */
void orc_csc_matvec_t(i64 ncols, const i64 *cp, const i64 *ri, const double *vx,
                      const double *x, double *out) {
  for (i64 j = 0; j < ncols; ++j) {
    double acc = 0.0;
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) acc += vx[p] * x[ri[p]];
    out[j] += acc;
  }
}

/* _kernels.py:33-43 : out += sym(M) x, M stored as its upper triangle. */
void orc_csc_sym_upper_matvec(i64 ncols, const i64 *cp, const i64 *ri,
                              const double *vx, const double *x, double *out) {
  for (i64 j = 0; j < ncols; ++j) {
    const double xj = x[j];
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) {
      const i64 i = ri[p];
      const double v = vx[p];
      out[i] += v * xj;
      if (i != j) out[j] += v * x[i];
    }
  }
}

/* -------------------------------------------------------------- sparse LDL */

/* _kernels.py:46-71 : elimination tree + column counts of L for an
 * upper-triangular pattern.  -1 if an entry lies below the diagonal. */
int orc_etree_and_counts(i64 n, const i64 *Ap, const i64 *Ai, i64 *parent,
                         i64 *lnz, i64 *work) {
  for (i64 i = 0; i < n; ++i) {
    parent[i] = -1;
    lnz[i] = 0;
    work[i] = -1;
  }
  for (i64 j = 0; j < n; ++j) {
    work[j] = j;
    for (i64 p = Ap[j]; p < Ap[j + 1]; ++p) {
      i64 i = Ai[p];
      if (i > j) return -1;
      while (work[i] != j) {
        if (parent[i] == -1) parent[i] = j;
        lnz[i] += 1;
        work[i] = j;
        i = parent[i];
      }
    }
  }
  return 0;
}

/* _kernels.py:74-99 : row indices of L in the order the numeric pass appends. */
void orc_ldl_pattern(i64 n, const i64 *Ap, const i64 *Ai, const i64 *parent,
                     const i64 *Lp, i64 *Li, i64 *next_pos, i64 *marker,
                     i64 *chain) {
  for (i64 i = 0; i < n; ++i) {
    next_pos[i] = Lp[i];
    marker[i] = -1;
  }
  for (i64 k = 0; k < n; ++k) {
    marker[k] = k;
    for (i64 p = Ap[k]; p < Ap[k + 1]; ++p) {
      const i64 i = Ai[p];
      if (i == k) continue;
      i64 nxt = i, nchain = 0;
      while (nxt != -1 && nxt < k && marker[nxt] != k) {
        marker[nxt] = k;
        chain[nchain++] = nxt;
        nxt = parent[nxt];
      }
      for (i64 q = 0; q < nchain; ++q) {
        const i64 c = chain[q];
        Li[next_pos[c]++] = k;
      }
    }
  }
}

/* _kernels.py:102-168 : up-looking LDL' with sign-matched static diagonal and
 * dynamic pivot floor.  Returns #dynamic bumps, or -1 on a non-finite pivot. */
i64 orc_ldl_factor(i64 n, const i64 *Ap, const i64 *Ai, const double *Ax,
                   const i64 *parent, const i64 *Lp, const i64 *Li, double *Lx,
                   double *D, const double *static_diag, double dyn_eps,
                   const i64 *sign_hint, double *yvals, i64 *yidx, i64 *chain,
                   i64 *next_pos, i64 *marker) {
  i64 bumps = 0;
  for (i64 i = 0; i < n; ++i) {
    next_pos[i] = Lp[i];
    marker[i] = -1;
    yvals[i] = 0.0;
  }
  for (i64 k = 0; k < n; ++k) {
    marker[k] = k;
    double dk = static_diag[k];
    i64 nnz_y = 0;
    for (i64 p = Ap[k]; p < Ap[k + 1]; ++p) {
      const i64 i = Ai[p];
      if (i == k) {
        dk += Ax[p];
        continue;
      }
      yvals[i] = Ax[p];
      i64 nxt = i, nchain = 0;
      while (nxt != -1 && nxt < k && marker[nxt] != k) {
        marker[nxt] = k;
        chain[nchain++] = nxt;
        nxt = parent[nxt];
      }
      for (i64 q = nchain - 1; q >= 0; --q) yidx[nnz_y++] = chain[q];
    }
    for (i64 q = nnz_y - 1; q >= 0; --q) {
      const i64 c = yidx[q];
      const double yc = yvals[c];
      const i64 top = next_pos[c];
      for (i64 r = Lp[c]; r < top; ++r) yvals[Li[r]] -= Lx[r] * yc;
      const double lkc = yc / D[c];
      Lx[top] = lkc;
      dk -= yc * lkc;
      next_pos[c] = top + 1;
      yvals[c] = 0.0;
    }
    if (!isfinite(dk)) return -1;
    if (fabs(dk) < dyn_eps) {
      dk = (sign_hint[k] >= 0) ? dyn_eps : -dyn_eps;
      bumps += 1;
    }
    D[k] = dk;
  }
  return bumps;
}

/* _kernels.py:171-184 : x <- (L D L')^{-1} x. */
void orc_ldl_solve_inplace(i64 n, const i64 *Lp, const i64 *Li,
                           const double *Lx, const double *D, double *x) {
  for (i64 j = 0; j < n; ++j) {
    const double xj = x[j];
    if (xj != 0.0)
      for (i64 p = Lp[j]; p < Lp[j + 1]; ++p) x[Li[p]] -= Lx[p] * xj;
  }
  for (i64 j = 0; j < n; ++j) x[j] /= D[j];
  for (i64 j = n - 1; j >= 0; --j) {
    double acc = x[j];
    for (i64 p = Lp[j]; p < Lp[j + 1]; ++p) acc -= Lx[p] * x[Li[p]];
    x[j] = acc;
  }
}

/* ------------------------------------------------------------ KKT position */

/* kkt.py:107-143 : slot -> position map.  For column `col` the wanted row is
 * found by binary search in that column, exactly as _entry_position does.
 * rows_of_slot / cols_of_slot are produced by the Python driver in the
 * reference's slot order.  Returns -1 if an entry is missing. */
int orc_entry_positions(const i64 *cp, const i64 *ri, i64 nslots,
                        const i64 *slot_row, const i64 *slot_col, i64 *pos) {
  for (i64 s = 0; s < nslots; ++s) {
    i64 lo = cp[slot_col[s]], hi = cp[slot_col[s] + 1];
    const i64 end = hi, want = slot_row[s];
    while (lo < hi) { /* np.searchsorted(side="left") */
      const i64 mid = lo + (hi - lo) / 2;
      if (ri[mid] < want) lo = mid + 1; else hi = mid;
    }
    if (lo >= end || ri[lo] != want) return -1;
    pos[s] = lo;
  }
  return 0;
}
