/*
 * CPU ORACLE — test infrastructure only.
 *
 * A plain-C restatement of the reference algorithm for the ILU / stri / spmv
 * hot path of the Javelin reference package (`ilukit`, Python + numba, under
 * /root/reference/pkg/src/ilukit).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (paper_1812_06160_b200) never calls it.
 *
 * Pinning: every function here is checked against golden vectors produced by
 * running the reference itself (tests/golden/make_golden.py) — see
 * tests/test_oracle_golden.py.
 *
 * Arithmetic contract (reference _kernels.py:1-9): IEEE binary64, no FMA
 * contraction (built with -ffp-contract=off), per-position updates applied in
 * ascending pivot order, inf/nan allowed to flow.
 *
 * Index arrays are int64 (the reference's layout), values double.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <sched.h>

typedef int64_t i64;

/* reference: _kernels.py:28-34 (spmv_kernel) */
void or_spmv(i64 n, const i64* rs, const i64* col, const double* val,
             const double* x, double* y) {
  for (i64 r = 0; r < n; ++r) {
    double s = 0.0;
    for (i64 p = rs[r]; p < rs[r + 1]; ++p) s += val[p] * x[col[p]];
    y[r] = s;
  }
}

/* reference: _kernels.py:37-48 (levels_forward_kernel). The dependency
 * pattern is strictly lower: level[r] = 1 + max level of its columns. */
void or_levels_forward(i64 n, const i64* rs, const i64* col, i64* level_of) {
  for (i64 r = 0; r < n; ++r) {
    i64 m = -1;
    for (i64 p = rs[r]; p < rs[r + 1]; ++p) {
      i64 lc = level_of[col[p]];
      if (lc > m) m = lc;
    }
    level_of[r] = m + 1;
  }
}

/* reference: _kernels.py:51-62 (levels_backward_kernel); only columns j > r
 * count, sweep runs from the last row down. */
void or_levels_backward(i64 n, const i64* rs, const i64* col, i64* level_of) {
  for (i64 r = n - 1; r >= 0; --r) {
    i64 m = -1;
    for (i64 p = rs[r]; p < rs[r + 1]; ++p) {
      i64 j = col[p];
      if (j > r && level_of[j] > m) m = level_of[j];
    }
    level_of[r] = m + 1;
  }
}

/* reference: _kernels.py:165-194 (_factor_row). Up-looking elimination of
 * row r over pivot columns clo <= c < chi, in ascending column order. */
static void factor_row(const i64* rs, const i64* col, double* val,
                       const i64* diag, double row_norm, double tau, int milu,
                       i64 r, i64 clo, i64 chi) {
  i64 re = rs[r + 1];
  i64 dpos = diag[r];
  for (i64 p = rs[r]; p < re; ++p) {
    i64 c = col[p];
    if (c >= chi || c >= r) break;
    if (c < clo) continue;
    double l = val[p] / val[diag[c]];
    if (tau > 0.0 && fabs(l) < tau * row_norm) {
      val[p] = 0.0;
      if (milu)
        for (i64 q = diag[c] + 1; q < rs[c + 1]; ++q) val[dpos] -= l * val[q];
      continue;
    }
    val[p] = l;
    i64 w = p + 1;
    for (i64 q = diag[c] + 1; q < rs[c + 1]; ++q) {
      i64 j = col[q];
      while (w < re && col[w] < j) ++w;
      if (w < re && col[w] == j) val[w] -= l * val[q];
      else if (milu) val[dpos] -= l * val[q];
    }
  }
}

/* reference: _kernels.py:197-204 (factor_serial_kernel); returns the first
 * row whose post-elimination diagonal is exactly zero, or -1. */
i64 or_factor_serial(i64 n, const i64* rs, const i64* col, double* val,
                     const i64* diag, const double* norms, double tau, int milu) {
  for (i64 r = 0; r < n; ++r) {
    factor_row(rs, col, val, diag, norms[r], tau, milu, r, 0, r);
    if (val[diag[r]] == 0.0) return r;
  }
  return -1;
}

/* reference: _kernels.py:221-228 + :231-240 (ER tail then serial corner);
 * rows [r0, r1) restricted to pivots [clo, chi) */
void or_factor_rows(const i64* rs, const i64* col, double* val, const i64* diag,
                    const double* norms, double tau, int milu, i64 r0, i64 r1,
                    i64 clo, i64 chi) {
  for (i64 r = r0; r < r1; ++r)
    factor_row(rs, col, val, diag, norms[r], tau, milu, r, clo, chi < r ? chi : r);
}

/* reference: factor.py:25-34 (row_inf_norms) — zeros unless tau > 0;
 * np.maximum.at semantics: a NaN, once seen, sticks */
void or_row_inf_norms(i64 n, const i64* rs, const double* val, double tau, double* norms) {
  for (i64 r = 0; r < n; ++r) {
    double m = 0.0;
    if (tau > 0.0)
      for (i64 p = rs[r]; p < rs[r + 1]; ++p) {
        double a = fabs(val[p]);
        if (isnan(m)) break;
        if (isnan(a) || a > m) m = a;
      }
    norms[r] = m;
  }
}

/* reference: _kernels.py:348-357 (solve_forward_serial_kernel), unit L */
void or_solve_forward(i64 n, const i64* rs, const i64* col, const double* val, double* y) {
  for (i64 r = 0; r < n; ++r) {
    double s = y[r];
    for (i64 p = rs[r]; p < rs[r + 1]; ++p) {
      i64 c = col[p];
      if (c >= r) break;
      s -= val[p] * y[c];
    }
    y[r] = s;
  }
}

/* reference: _kernels.py:360-366 (solve_backward_serial_kernel) */
void or_solve_backward(i64 n, const i64* rs, const i64* col, const double* val,
                       const i64* diag, double* x) {
  for (i64 r = n - 1; r >= 0; --r) {
    double s = x[r];
    for (i64 p = diag[r] + 1; p < rs[r + 1]; ++p) s -= val[p] * x[col[p]];
    x[r] = s / val[diag[r]];
  }
}

/* reference: trisolve.py:54-57 (_check_diagonals): smallest zero diagonal */
i64 or_first_zero_diag(i64 n, const double* val, const i64* diag) {
  for (i64 r = 0; r < n; ++r)
    if (val[diag[r]] == 0.0) return r;
  return -1;
}

/* ------------------------------------------------------------------------
 * Level-of-fill symbolic ILU(k).  reference: symbolic.py:86-138
 * (iluk_pattern).  The reference pops pivot columns m < i from a heap in
 * ascending order and merges the finalized upper rows; fill candidates are
 * always > m, so an ordered linked list over the row's columns visits the
 * same sequence.  Output: malloc'd row_start/col/level; caller frees via
 * or_free.  Returns nnz or -1 on allocation failure.  The caller has already
 * checked the diagonal (symbolic.py:70-75).
 * ---------------------------------------------------------------------- */
i64 or_iluk_pattern(i64 n, const i64* rs, const i64* col, i64 k,
                    i64** out_rs, i64** out_col, i64** out_lev) {
  i64 cap = rs[n] * 2 + 16, nnz = 0;
  i64* orow = (i64*)malloc(sizeof(i64) * (n + 1));
  i64* ocol = (i64*)malloc(sizeof(i64) * cap);
  i64* olev = (i64*)malloc(sizeof(i64) * cap);
  i64* ustart = (i64*)malloc(sizeof(i64) * (n + 1)); /* first upper pos per row */
  i64* lev = (i64*)malloc(sizeof(i64) * (n + 1));
  i64* next = (i64*)malloc(sizeof(i64) * (n + 1));
  i64* mark = (i64*)malloc(sizeof(i64) * (n + 1));
  if (!orow || !ocol || !olev || !ustart || !lev || !next || !mark) return -1;
  for (i64 j = 0; j < n; ++j) mark[j] = -1;
  const i64 HEAD = n; /* sentinel list head */
  orow[0] = 0;
  for (i64 i = 0; i < n; ++i) {
    /* sorted singly linked list of this row's columns */
    next[HEAD] = -1;
    i64 tail = HEAD;
    for (i64 p = rs[i]; p < rs[i + 1]; ++p) {
      i64 j = col[p];
      mark[j] = i; lev[j] = 0;
      next[tail] = j; next[j] = -1; tail = j;
    }
    /* walk lower columns in ascending order; insertions land after m */
    i64 m = next[HEAD];
    while (m != -1 && m < i) {
      i64 lim = lev[m];
      if (lim <= k) {
        i64 prev = m; /* insertion cursor: columns only grow */
        for (i64 q = ustart[m]; q < orow[m + 1]; ++q) {
          i64 j = ocol[q];
          i64 cand = lim + olev[q] + 1;
          if (mark[j] == i) {
            if (cand < lev[j]) lev[j] = cand;
            while (next[prev] != -1 && next[prev] <= j) prev = next[prev];
          } else if (cand <= k) {
            while (next[prev] != -1 && next[prev] < j) prev = next[prev];
            mark[j] = i; lev[j] = cand;
            next[j] = next[prev]; next[prev] = j; prev = j;
          }
        }
      }
      m = next[m];
    }
    /* emit */
    for (i64 j = next[HEAD]; j != -1; j = next[j]) {
      if (lev[j] > k) continue;
      if (nnz == cap) {
        cap *= 2;
        ocol = (i64*)realloc(ocol, sizeof(i64) * cap);
        olev = (i64*)realloc(olev, sizeof(i64) * cap);
        if (!ocol || !olev) return -1;
      }
      ocol[nnz] = j; olev[nnz] = lev[j]; ++nnz;
    }
    orow[i + 1] = nnz;
    ustart[i] = orow[i + 1];
    for (i64 q = orow[i]; q < orow[i + 1]; ++q)
      if (ocol[q] > i) { ustart[i] = q; break; }
  }
  free(ustart); free(lev); free(next); free(mark);
  *out_rs = orow; *out_col = ocol; *out_lev = olev;
  return nnz;
}

void or_free(void* p) { free(p); }

/* ------------------------------------------------------------------------
 * Reference rcm_order restated (ordering.py:199-266): components rooted at
 * the minimum-degree unvisited vertex (ties by index), George-Liu
 * pseudo-peripheral refinement (pick the minimum (degree, index) vertex of
 * the last BFS tier, keep it while eccentricity strictly grows), then
 * Cuthill-McKee BFS with fresh neighbours sorted by (degree, index); the
 * full order is reversed.  Input: symmetrized pattern (self loops allowed).
 * ---------------------------------------------------------------------- */
static const i64* g_deg;
static int cmp_deg_idx(const void* a, const void* b) {
  i64 x = *(const i64*)a, y = *(const i64*)b;
  if (g_deg[x] != g_deg[y]) return g_deg[x] < g_deg[y] ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* BFS tiers from start over vertices with seen==0 (seen is scratch, stamp
 * marks); returns number of tiers, last tier in [*lo, *hi) of queue */
static i64 bfs_tiers(i64 start, const i64* rs, const i64* col, const char* visited,
                     i64* stamp, i64 st, i64* queue, i64* last_lo, i64* last_hi) {
  i64 head = 0, tail = 0, tiers = 0;
  queue[tail++] = start; stamp[start] = st;
  i64 tier_lo = 0, tier_hi = 1;
  while (1) {
    ++tiers;
    *last_lo = tier_lo; *last_hi = tier_hi;
    for (head = tier_lo; head < tier_hi; ++head) {
      i64 v = queue[head];
      for (i64 p = rs[v]; p < rs[v + 1]; ++p) {
        i64 w = col[p];
        if (w == v || visited[w] || stamp[w] == st) continue;
        stamp[w] = st; queue[tail++] = w;
      }
    }
    if (tail == tier_hi) return tiers;
    tier_lo = tier_hi; tier_hi = tail;
  }
}

i64 or_rcm(i64 n, const i64* rs, const i64* col, i64* perm_out) {
  i64* deg = (i64*)malloc(sizeof(i64) * (n ? n : 1));
  i64* bymin = (i64*)malloc(sizeof(i64) * (n ? n : 1));
  i64* queue = (i64*)malloc(sizeof(i64) * (n ? n : 1));
  i64* stamp = (i64*)malloc(sizeof(i64) * (n ? n : 1));
  i64* fresh = (i64*)malloc(sizeof(i64) * (n ? n : 1));
  char* visited = (char*)calloc(n ? n : 1, 1);
  for (i64 i = 0; i < n; ++i) {
    i64 d = rs[i + 1] - rs[i];
    for (i64 p = rs[i]; p < rs[i + 1]; ++p) if (col[p] == i) { --d; break; }
    deg[i] = d; bymin[i] = i; stamp[i] = -1;
  }
  g_deg = deg;
  qsort(bymin, n, sizeof(i64), cmp_deg_idx);
  i64 out = 0, st = 0;
  for (i64 ci = 0; ci < n; ++ci) {
    i64 cand = bymin[ci];
    if (visited[cand]) continue;
    i64 lo, hi;
    i64 ecc = bfs_tiers(cand, rs, col, visited, stamp, st++, queue, &lo, &hi);
    i64 root = cand;
    while (1) {
      i64 pick = queue[lo];
      for (i64 t = lo + 1; t < hi; ++t) {
        i64 v = queue[t];
        if (deg[v] < deg[pick] || (deg[v] == deg[pick] && v < pick)) pick = v;
      }
      i64 e2 = bfs_tiers(pick, rs, col, visited, stamp, st++, queue, &lo, &hi);
      if (e2 > ecc) { root = pick; ecc = e2; } else break;
    }
    /* Cuthill-McKee traversal */
    i64 head = out;
    visited[root] = 1; perm_out[out++] = root;
    while (head < out) {
      i64 v = perm_out[head++];
      i64 nf = 0;
      for (i64 p = rs[v]; p < rs[v + 1]; ++p) {
        i64 w = col[p];
        if (w != v && !visited[w]) fresh[nf++] = w;
      }
      qsort(fresh, nf, sizeof(i64), cmp_deg_idx);
      for (i64 t = 0; t < nf; ++t) {
        /* neighbours are unique in a deduplicated pattern */
        visited[fresh[t]] = 1; perm_out[out++] = fresh[t];
      }
    }
  }
  for (i64 i = 0; i < n / 2; ++i) { i64 t = perm_out[i]; perm_out[i] = perm_out[n - 1 - i]; perm_out[n - 1 - i] = t; }
  free(deg); free(bymin); free(queue); free(stamp); free(fresh); free(visited);
  return out;
}

/* ------------------------------------------------------------------------
 * Threaded CPU baseline: the reference's parallel upper-stage factor
 * (factor_p2p_kernel, _kernels.py:207-218) and p2p solves (:404-433), with
 * rows dealt round-robin in level order (sync.py:639-647) and every
 * structural dependency awaited through acquire/release flags
 * (_atomics.py:27-53).  Waits are not pruned (sync.py:59-98 is a CPU
 * optimisation that does not change results); results are bitwise equal to
 * the serial kernels.  Used as bench.py's --impl reference arm on the host.
 * ---------------------------------------------------------------------- */
typedef struct {
  int wid, nthreads, kind; /* kind 0 factor, 1 fwd, 2 bwd */
  i64 n; const i64 *rs, *col, *diag, *order; double* val; const double* norms;
  double tau; int milu; double* vec; _Atomic int64_t* done; i64 epoch;
  i64* errflag;
} p2p_arg;

static void await_row(_Atomic int64_t* done, i64 c, i64 epoch) {
  int spins = 0;
  while (atomic_load_explicit(done + c, memory_order_acquire) != epoch) {
    if (++spins > 64) { sched_yield(); spins = 0; }
  }
}

static void* p2p_worker(void* vp) {
  p2p_arg* a = (p2p_arg*)vp;
  for (i64 k = a->wid; k < a->n; k += a->nthreads) {
    i64 r = a->order ? a->order[k] : k;
    if (a->kind == 2) r = a->n - 1 - k;
    if (a->kind == 0) {
      for (i64 p = a->rs[r]; p < a->rs[r + 1] && a->col[p] < r; ++p)
        await_row(a->done, a->col[p], a->epoch);
      factor_row(a->rs, a->col, a->val, a->diag, a->norms[r], a->tau, a->milu, r, 0, r);
      if (a->val[a->diag[r]] == 0.0) a->errflag[r] = 1;
    } else if (a->kind == 1) {
      double s = a->vec[r];
      for (i64 p = a->rs[r]; p < a->rs[r + 1]; ++p) {
        i64 c = a->col[p];
        if (c >= r) break;
        await_row(a->done, c, a->epoch);
        s -= a->val[p] * a->vec[c];
      }
      a->vec[r] = s;
    } else {
      double s = a->vec[r];
      for (i64 p = a->diag[r] + 1; p < a->rs[r + 1]; ++p) {
        await_row(a->done, a->col[p], a->epoch);
        s -= a->val[p] * a->vec[a->col[p]];
      }
      a->vec[r] = s / a->val[a->diag[r]];
    }
    atomic_store_explicit(a->done + r, a->epoch, memory_order_release);
  }
  return NULL;
}

/* kind: 0 factor (returns first zero-pivot row or -1), 1 forward, 2 backward.
 * Rows are taken in index order, which is a topological order for all three
 * (the matrix is level-ordered or not, it does not matter: deps point to
 * smaller indices forward and larger indices backward). */
i64 or_p2p(int kind, int nthreads, i64 n, const i64* rs, const i64* col, double* val,
           const i64* diag, const double* norms, double tau, int milu, double* vec) {
  if (nthreads < 1) nthreads = 1;
  _Atomic int64_t* done = (_Atomic int64_t*)calloc(n ? n : 1, sizeof(int64_t));
  i64* err = kind == 0 ? (i64*)calloc(n ? n : 1, sizeof(i64)) : NULL;
  pthread_t th[256];
  p2p_arg args[256];
  if (nthreads > 256) nthreads = 256;
  for (int w = 0; w < nthreads; ++w) {
    p2p_arg a = {w, nthreads, kind, n, rs, col, diag, NULL, val, norms, tau, milu, vec, done, 1, err};
    args[w] = a;
  }
  for (int w = 1; w < nthreads; ++w) pthread_create(&th[w], NULL, p2p_worker, &args[w]);
  p2p_worker(&args[0]);
  for (int w = 1; w < nthreads; ++w) pthread_join(th[w], NULL);
  i64 bad = -1;
  if (err) { for (i64 r = 0; r < n; ++r) if (err[r]) { bad = r; break; } free(err); }
  free((void*)done);
  return bad;
}
