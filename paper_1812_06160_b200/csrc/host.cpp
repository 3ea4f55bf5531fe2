// Host-side setup helpers of libjv (C++).  Neither is on the timed path:
//  * jv_rcm_host — the config-2 base ordering, bit-exact with the reference
//    rcm_order (ordering.py:199-266).  The device version is the next item
//    (SURVEY.md §8f #2).
//  * jv_iluk_host — level-of-fill symbolic ILU(k) for k >= 2
//    (symbolic.py:86-138); k = 1 runs on the device (jv_iluk1_pattern).
#include "../../include/jv.h"

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

namespace {

struct RcmState {
  const int32_t* rs;
  const int32_t* col;
  std::vector<int32_t> deg;
  std::vector<char> visited;
  std::vector<int64_t> stamp;
  std::vector<int32_t> queue;
  int64_t st = 0;
};

bool less_deg(const RcmState& S, int32_t a, int32_t b) {
  return S.deg[a] != S.deg[b] ? S.deg[a] < S.deg[b] : a < b;
}

// BFS tiers from `start` over unvisited vertices; returns the tier count and
// the last tier's range in S.queue
int64_t bfs_tiers(RcmState& S, int32_t start, size_t& lo, size_t& hi) {
  const int64_t st = ++S.st;
  S.queue.clear();
  S.queue.push_back(start);
  S.stamp[start] = st;
  size_t tlo = 0, thi = 1;
  int64_t tiers = 0;
  for (;;) {
    ++tiers;
    lo = tlo;
    hi = thi;
    for (size_t h = tlo; h < thi; ++h) {
      const int32_t v = S.queue[h];
      for (int32_t p = S.rs[v]; p < S.rs[v + 1]; ++p) {
        const int32_t w = S.col[p];
        if (w == v || S.visited[w] || S.stamp[w] == st) continue;
        S.stamp[w] = st;
        S.queue.push_back(w);
      }
    }
    if (S.queue.size() == thi) return tiers;
    tlo = thi;
    thi = S.queue.size();
  }
}

}  // namespace

extern "C" int jv_rcm_host(int32_t n, const int32_t* rs, const int32_t* col, int32_t* perm) {
  if (n < 0) return JV_EINVAL;
  RcmState S;
  S.rs = rs;
  S.col = col;
  S.deg.resize(n);
  S.visited.assign(n, 0);
  S.stamp.assign(n, 0);
  for (int32_t i = 0; i < n; ++i) {
    int32_t d = rs[i + 1] - rs[i];
    for (int32_t p = rs[i]; p < rs[i + 1]; ++p)
      if (col[p] == i) { --d; break; }
    S.deg[i] = d;
  }
  std::vector<int32_t> bymin(n);
  for (int32_t i = 0; i < n; ++i) bymin[i] = i;
  std::stable_sort(bymin.begin(), bymin.end(),
                   [&](int32_t a, int32_t b) { return less_deg(S, a, b); });
  int32_t out = 0;
  std::vector<int32_t> fresh;
  for (int32_t cand : bymin) {
    if (S.visited[cand]) continue;
    size_t lo, hi;
    int64_t ecc = bfs_tiers(S, cand, lo, hi);
    int32_t root = cand;
    for (;;) {
      int32_t pick = S.queue[lo];
      for (size_t t = lo + 1; t < hi; ++t)
        if (less_deg(S, S.queue[t], pick)) pick = S.queue[t];
      const int64_t e2 = bfs_tiers(S, pick, lo, hi);
      if (e2 > ecc) { root = pick; ecc = e2; } else break;
    }
    int32_t head = out;
    S.visited[root] = 1;
    perm[out++] = root;
    while (head < out) {
      const int32_t v = perm[head++];
      fresh.clear();
      for (int32_t p = rs[v]; p < rs[v + 1]; ++p) {
        const int32_t w = col[p];
        if (w != v && !S.visited[w]) fresh.push_back(w);
      }
      std::sort(fresh.begin(), fresh.end(), [&](int32_t a, int32_t b) { return less_deg(S, a, b); });
      for (int32_t w : fresh) {
        S.visited[w] = 1;
        perm[out++] = w;
      }
    }
  }
  std::reverse(perm, perm + n);
  return JV_OK;
}

// Level-of-fill ILU(k): row i walks its lower columns m in ascending order
// over an ordered linked list, merging the finalized upper part of row m
// (fill candidates are > m, so insertions never precede the cursor).
// Outputs are malloc'd; free with jv_free_host.  Returns nnz or < 0.
extern "C" int64_t jv_iluk_host(int32_t n, const int32_t* rs, const int32_t* col, int32_t k,
                                int32_t** out_rs, int32_t** out_col, int32_t** out_lev) {
  std::vector<int32_t> orow(n + 1, 0), ocol, olev, ustart(n, 0), lev(n + 1), nxt(n + 1),
      mark(n + 1, -1);
  ocol.reserve((size_t)rs[n] * 2);
  olev.reserve((size_t)rs[n] * 2);
  const int32_t HEAD = n;
  for (int32_t i = 0; i < n; ++i) {
    nxt[HEAD] = -1;
    int32_t tail = HEAD;
    for (int32_t p = rs[i]; p < rs[i + 1]; ++p) {
      const int32_t j = col[p];
      mark[j] = i;
      lev[j] = 0;
      nxt[tail] = j;
      nxt[j] = -1;
      tail = j;
    }
    for (int32_t m = nxt[HEAD]; m != -1 && m < i; m = nxt[m]) {
      const int32_t lim = lev[m];
      if (lim > k) continue;
      int32_t prev = m;
      for (int32_t q = ustart[m]; q < orow[m + 1]; ++q) {
        const int32_t j = ocol[q];
        const int32_t cand = lim + olev[q] + 1;
        if (mark[j] == i) {
          if (cand < lev[j]) lev[j] = cand;
          while (nxt[prev] != -1 && nxt[prev] <= j) prev = nxt[prev];
        } else if (cand <= k) {
          while (nxt[prev] != -1 && nxt[prev] < j) prev = nxt[prev];
          mark[j] = i;
          lev[j] = cand;
          nxt[j] = nxt[prev];
          nxt[prev] = j;
          prev = j;
        }
      }
    }
    for (int32_t j = nxt[HEAD]; j != -1; j = nxt[j]) {
      if (lev[j] > k) continue;
      ocol.push_back(j);
      olev.push_back(lev[j]);
    }
    orow[i + 1] = (int32_t)ocol.size();
    ustart[i] = orow[i + 1];
    for (int32_t q = orow[i]; q < orow[i + 1]; ++q)
      if (ocol[q] > i) { ustart[i] = q; break; }
  }
  const size_t nnz = ocol.size();
  *out_rs = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  *out_col = (int32_t*)malloc(sizeof(int32_t) * (nnz ? nnz : 1));
  *out_lev = (int32_t*)malloc(sizeof(int32_t) * (nnz ? nnz : 1));
  if (!*out_rs || !*out_col || !*out_lev) return JV_ENOMEM;
  std::copy(orow.begin(), orow.end(), *out_rs);
  std::copy(ocol.begin(), ocol.end(), *out_col);
  std::copy(olev.begin(), olev.end(), *out_lev);
  return (int64_t)nnz;
}

extern "C" void jv_free_host(void* p) { free(p); }

// ---------------------------------------------------------------------------
// Hub-row gather plan (setup, host): the target-parallel schedule of one
// heavy row's elimination, so the numeric kernel folds many positions at
// once instead of walking the pivots one by one.
//
// Input: the row's elimination list in pivot order (jv_elim_lists): pivot j
// owns ops [piv_ptr[j], piv_ptr[j+1]) = (q, w): subtract l_j * u_q from
// position w.  For every position w the updates must be applied in
// ascending j (the order of _factor_row, _kernels.py:165-194), and l_w
// (w < nL) = (a_w - its updates) / d_w is available to later updates.
//
//   depth(w) = 1 + max depth(j) over w's updaters (0 without any), w < nL;
//   an update (j -> w) can run in phase depth(j) + 1, and not before the
//   previous update of w  ->  each position's updates split into runs, one
//   per phase; an L position w is finalised (divided) in phase depth(w).
//   Phases run in order; inside a phase, runs of different positions are
//   independent and are dealt to 32 lanes longest-first (LPT), lanes sorted
//   by load, and the stream is step-major (step t: entry t of every lane
//   with more than t entries), so lanes t < active(t) are a prefix.  The
//   phase's divisions follow as a block of their own (32 per step), after
//   every update of the phase: no division diverges inside an update step.
//
// Stream entry (int2): x = q (update) or d_slot | 1<<31 (finalise: divide by
// the pivot diagonal, mailbox slot d_slot); y = j | w << 16 (j unused for a
// finalise).  Meta: nphases, then per phase 32 lane loads (descending) and
// the number of divisions.
// Returns 0, or -1 when a row does not fit (len > 65535).
extern "C" int jv_hub_plan_host(int32_t len, int32_t nL, const int64_t* piv_ptr,
                                const int32_t* op_q, const int32_t* op_w, const int32_t* dslot,
                                int32_t* stream, int64_t* nstream, int32_t* meta, int64_t* nmeta) {
  if (len > 65535 || nL > len) return -1;
  const int64_t nops = piv_ptr[nL] - piv_ptr[0];
  const int64_t base = piv_ptr[0];
  for (int64_t o = 0; o < nops; ++o)
    if (op_w[o] < 0 || op_w[o] >= len) return -1;   // e.g. MILU out-of-pattern targets
  // 1. updates grouped by target, ascending pivot (counting sort, stable)
  std::vector<int32_t> cnt(len + 1, 0);
  for (int64_t o = 0; o < nops; ++o) cnt[op_w[o] + 1]++;
  for (int w = 0; w < len; ++w) cnt[w + 1] += cnt[w];
  std::vector<int32_t> gj(nops), gq(nops), fill(cnt.begin(), cnt.end() - 1);
  for (int j = 0; j < nL; ++j)
    for (int64_t o = piv_ptr[j] - base; o < piv_ptr[j + 1] - base; ++o) {
      const int w = op_w[o];
      gj[fill[w]] = j;
      gq[fill[w]] = op_q[o];
      fill[w]++;
    }
  // 2. in-row depth of the L positions
  std::vector<int32_t> depth(nL, 0);
  int D = -1;
  for (int k = 0; k < nL; ++k) {
    int d = -1;
    for (int i = cnt[k]; i < cnt[k + 1]; ++i) d = std::max(d, depth[gj[i]]);
    depth[k] = d + 1;
    D = std::max(D, depth[k]);
  }
  const int P = D + 2;   // U positions may take updates up to phase D + 1
  // 3. runs per phase: (w, first update, count, finalise)
  struct Run { int32_t w, first, count; };
  std::vector<std::vector<Run>> runs(P);
  std::vector<std::vector<int32_t>> fins(P);
  for (int w = 0; w < len; ++w) {
    int ph = 0, start = cnt[w];
    for (int i = cnt[w]; i < cnt[w + 1]; ++i) {
      const int p = std::max(ph, depth[gj[i]] + 1);
      if (p != ph && i > start) {
        runs[ph].push_back({w, start, i - start});
        start = i;
      }
      ph = p;
    }
    if (cnt[w + 1] > start) runs[ph].push_back({w, start, cnt[w + 1] - start});
    // the last run sits in phase depth(w) (its newest updater has depth
    // depth(w) - 1); the division follows in that phase's finalise block
    if (w < nL) fins[depth[w]].push_back(w);
  }
  // 4. per phase: LPT over 32 lanes, lanes by load, step-major stream
  int64_t ns = 0, nm = 0;
  meta[nm++] = P;
  std::vector<int32_t> order;
  for (int p = 0; p < P; ++p) {
    auto& rp = runs[p];
    order.resize(rp.size());
    for (size_t i = 0; i < rp.size(); ++i) order[i] = (int32_t)i;
    auto cost = [&](const Run& r) { return r.count; };
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return cost(rp[a]) > cost(rp[b]); });
    std::vector<std::vector<int32_t>> lane(32);
    int64_t load[32] = {0};
    for (int32_t i : order) {
      int best = 0;
      for (int l = 1; l < 32; ++l)
        if (load[l] < load[best]) best = l;
      lane[best].push_back(i);
      load[best] += cost(rp[i]);
    }
    int perm[32];
    for (int l = 0; l < 32; ++l) perm[l] = l;
    std::stable_sort(perm, perm + 32, [&](int a, int b) { return load[a] > load[b]; });
    // each lane's entry sequence
    std::vector<std::vector<int64_t>> seq(32);   // packed (x << 32 | y)
    for (int l = 0; l < 32; ++l) {
      auto& s = seq[l];
      for (int32_t i : lane[perm[l]]) {
        const Run& r = rp[i];
        for (int t = 0; t < r.count; ++t) {
          const int g = r.first + t;
          const uint32_t x = (uint32_t)gq[g];
          const uint32_t y = (uint32_t)gj[g] | ((uint32_t)r.w << 16);
          s.push_back((int64_t)(((uint64_t)x << 32) | y));
        }
      }
      meta[nm++] = (int32_t)s.size();
    }
    const size_t steps = seq[0].size();
    for (size_t t = 0; t < steps; ++t)
      for (int l = 0; l < 32 && t < seq[l].size(); ++l) {
        const uint64_t e = (uint64_t)seq[l][t];
        stream[2 * ns] = (int32_t)(uint32_t)(e >> 32);
        stream[2 * ns + 1] = (int32_t)(uint32_t)e;
        ++ns;
      }
    // finalise block: the divisions of the phase, 32 per step
    meta[nm++] = (int32_t)fins[p].size();
    for (int32_t w : fins[p]) {
      stream[2 * ns] = (int32_t)((uint32_t)dslot[w] | 0x80000000u);
      stream[2 * ns + 1] = (int32_t)((uint32_t)w << 16);
      ++ns;
    }
  }
  *nstream = ns;
  *nmeta = nm;
  return 0;
}
