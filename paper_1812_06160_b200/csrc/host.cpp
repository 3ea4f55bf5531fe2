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
