// Region plans (setup, host C++) for the CTA-resident region kernels
// (region.cu): one co-resident CTA per region walks its rows level by level,
// in-region dependencies through shared memory, cross-region ones through
// the 16-byte mailboxes.
//
// 1. Partition (jv_region_partition_host).  A region pipeline is only fast
//    when the quotient graph of the regions is ACYCLIC: then every region
//    lags its upstream neighbours by one mailbox hop and runs its levels at
//    CTA-barrier speed, instead of paying a hop per level.  Any topological
//    order tau of the DAG gives an acyclic partition by contiguous ranges;
//    lexicographic refinement by further topological orders keeps it acyclic
//    (cells (a, b, c) in lexicographic order are a topological order of the
//    cells).  The orders come from depth-first Kahn sorts (LIFO ready stack)
//    whose successor lists are rotated by t = 0, 1, 2: on a stencil DAG each
//    rotation sweeps a different grid axis slowest (measured on config 2:
//    |corr(position, axis)| = 1.0 for one axis each), so the cells come out
//    as boxes — a domain decomposition found from the pattern alone.
// 2. Wave streams (jv_rstream_build / _export).  Per direction (factor,
//    forward, backward): rows of each region in (level, row) order = local
//    slots; consecutive rows of one level in waves of <= threads rows; every
//    wave is a 16-byte aligned block of int32 words
//        [cnt, slot0, K, NP | rec[cnt] | xref[K - 4][cnt] | pslot[NP]]
//    with one 32-byte record per row,
//        rec = {ref0, ref1, ref2, ref3, p0, row, meta, me},
//    K = most dependencies of a row in the wave, meta = ndep | pub << 6 |
//    umask << 7 (factor).  A ref is the BYTE OFFSET in the CTA's shared
//    memory of the dependency's value: a slot of the region's value ring, an
//    entry of the wave's decoded remote values (written by the prober warp
//    from the mailbox packets pslot[j]), or the constant 1.0 for the unused
//    refs of a row with fewer than 4 dependencies — the kernel reads every
//    ref with one load and no case distinction.  `me` is the offset of the
//    row's own ring slot.  Dependencies beyond the fourth are in xref.
//    The factor's u(c_k, r) come with the packed values.  The wave's dynamic
//    block holds vals[NV][cnt] (matrix values), the per-call vector and the
//    NP remote values (doubles the prober warps read from the mailboxes).  Static blocks are
//    bulk-copied (TMA) S waves ahead into a shared-memory ring, dynamic
//    blocks D waves ahead; ring offsets are placed here by simulating both
//    FIFO rings, and the remote refs are patched once the rings are placed.
#include "../../include/jv.h"

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace {

// successor lists of the lower DAG (edge c -> r for every strictly-lower
// entry (r, c)), each list ascending
void lower_successors(int32_t n, const int32_t* rs, const int32_t* col, const int32_t* diag,
                      std::vector<int64_t>& sptr, std::vector<int32_t>& succ,
                      std::vector<int32_t>& indeg) {
  sptr.assign(n + 1, 0);
  indeg.assign(n, 0);
  for (int32_t r = 0; r < n; ++r)
    for (int32_t p = rs[r]; p < diag[r]; ++p) {
      ++sptr[col[p] + 1];
      ++indeg[r];
    }
  for (int32_t i = 0; i < n; ++i) sptr[i + 1] += sptr[i];
  succ.resize(sptr[n]);
  std::vector<int64_t> fill(sptr.begin(), sptr.end() - 1);
  for (int32_t r = 0; r < n; ++r)
    for (int32_t p = rs[r]; p < diag[r]; ++p) succ[fill[col[p]]++] = r;
}

// depth-first Kahn order, successor lists rotated by t; pos[v] = position
void lifo_order(int32_t n, const std::vector<int64_t>& sptr, const std::vector<int32_t>& succ,
                std::vector<int32_t> indeg, int t, std::vector<int32_t>& pos) {
  std::vector<int32_t> stack;
  stack.reserve(n);
  for (int32_t v = n - 1; v >= 0; --v)
    if (indeg[v] == 0) stack.push_back(v);
  pos.assign(n, -1);
  int32_t k = 0;
  while (!stack.empty()) {
    const int32_t v = stack.back();
    stack.pop_back();
    pos[v] = k++;
    const int64_t a = sptr[v], len = sptr[v + 1] - a;
    if (len == 0) continue;
    const int64_t rot = t % len;
    for (int64_t i = 0; i < len; ++i) {
      const int32_t w = succ[a + (i + rot) % len];
      if (--indeg[w] == 0) stack.push_back(w);
    }
  }
}

}  // namespace

// Acyclic region partition of the lower DAG of a combined L|U pattern.
// nreg_max regions at most (one CTA per SM), each <= max_rows rows, refined
// by at most dims_max (1-3; 0 = 3) orders: 3 gives boxes, 2 pencils.
// region_of[r] receives the region id; returns the number of regions, or
// -1 when the rows do not fit (n > nreg * max_rows).
extern "C" int32_t jv_region_partition_host(int32_t n, const int32_t* rs, const int32_t* col,
                                            const int32_t* diag, int32_t nreg_max,
                                            int32_t max_rows, int32_t dims_max,
                                            int32_t* region_of) {
  if (n <= 0 || nreg_max < 1) return -1;
  std::vector<int64_t> sptr;
  std::vector<int32_t> succ, indeg;
  lower_successors(n, rs, col, diag, sptr, succ, indeg);
  int64_t maxs = 0;
  for (int32_t v = 0; v < n; ++v) maxs = std::max(maxs, sptr[v + 1] - sptr[v]);
  const int dims = (int)std::max<int64_t>(
      1, std::min<int64_t>(dims_max > 0 ? std::min(dims_max, 3) : 3, maxs));
  // balanced factorisation of <= nreg_max parts into `dims` factors
  int best[3] = {nreg_max, 1, 1};
  int64_t bprod = dims == 1 ? nreg_max : 0;
  double bratio = 1e30;
  if (dims > 1) {
    for (int a = 1; a <= nreg_max; ++a)
      for (int b = 1; b <= a && (int64_t)a * b <= nreg_max; ++b) {
        int c = 1;
        if (dims == 3) {
          c = nreg_max / (a * b);
          c = std::min(c, b);
          if (c < 1) continue;
        }
        const int64_t prod = (int64_t)a * b * c;
        const double ratio = (double)a / (dims == 3 ? c : b);
        if (ratio > 1.6) continue;
        if (prod > bprod || (prod == bprod && ratio < bratio)) {
          bprod = prod;
          bratio = ratio;
          best[0] = a;
          best[1] = b;
          best[2] = dims == 3 ? c : 1;
        }
      }
  }
  int64_t nparts = (int64_t)best[0] * best[1] * best[2];
  while (nparts > 1 && (int64_t)n < nparts) {   // tiny matrices: fewer regions
    for (int d = 0; d < 3; ++d)
      if (best[d] > 1) { --best[d]; break; }
    nparts = (int64_t)best[0] * best[1] * best[2];
  }
  if ((n + nparts - 1) / nparts > max_rows) return -1;
  std::vector<int32_t> reg(n, 0), pos, idx(n), next(n);
  int32_t ngroups = 1;
  for (int d = 0; d < dims; ++d) {
    const int p = best[d];
    lifo_order(n, sptr, succ, indeg, d, pos);
    for (int32_t i = 0; i < n; ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
      return reg[a] != reg[b] ? reg[a] < reg[b] : pos[a] < pos[b];
    });
    int32_t i = 0;
    while (i < n) {
      int32_t e = i;
      const int32_t g = reg[idx[i]];
      while (e < n && reg[idx[e]] == g) ++e;
      const int64_t cnt = e - i;
      for (int32_t k = i; k < e; ++k) next[idx[k]] = g * p + (int32_t)(((int64_t)(k - i) * p) / cnt);
      i = e;
    }
    reg.swap(next);
    ngroups *= p;
  }
  // compact ids (empty cells are possible only for tiny inputs)
  std::vector<int32_t> remap(ngroups, -1);
  int32_t nreg = 0;
  for (int32_t r = 0; r < n; ++r)
    if (remap[reg[r]] < 0) remap[reg[r]] = 0;
  for (int32_t g = 0; g < ngroups; ++g)
    if (remap[g] == 0) remap[g] = nreg++;
  for (int32_t r = 0; r < n; ++r) region_of[r] = remap[reg[r]];
  return nreg;
}

namespace {

struct RStream {
  int kind = 0;
  int32_t nreg = 0, max_region = 0, max_waves = 0;
  int32_t S = 0, D = 0, CS = 0, CD = 0, SC = 0;
  std::vector<int32_t> words;     // static stream (16-byte aligned blocks)
  std::vector<int32_t> table;     // 8 ints per wave {goff16, bytes, soff, doff, voff16, vbytes, 0, 0}
  std::vector<int32_t> sidx;      // packed value -> source position in val (-1: padding)
  std::vector<int32_t> vidx;      // packed per-call vector -> row (-1: padding)
  std::vector<int32_t> reg_wave;  // nreg + 1
  int64_t nrows_remote = 0, ndeps_remote = 0;
};

std::mutex g_rs_mu;
std::map<int64_t, std::unique_ptr<RStream>> g_rs;
int64_t g_rs_next = 1;

// FIFO ring placement: block w may not overlap blocks w-window .. w-1
bool ring_place(const std::vector<int32_t>& sz, int32_t cap, int window,
                std::vector<int32_t>& off) {
  off.assign(sz.size(), 0);
  int64_t head = 0;
  for (size_t w = 0; w < sz.size(); ++w) {
    const int64_t s = sz[w];
    if (s > cap) return false;
    int64_t o = head;
    if (o + s > cap) o = 0;
    for (size_t v = w > (size_t)window ? w - window : 0; v < w; ++v) {
      const int64_t a = off[v], b = a + sz[v];
      if (s > 0 && sz[v] > 0 && o < b && a < o + s) return false;
    }
    off[w] = (int32_t)o;
    head = o + s;
  }
  return true;
}

int32_t min_cap(const std::vector<std::vector<int32_t>>& per_region, int window, int32_t budget) {
  // smallest capacity (16-byte steps) that places every region's blocks
  int32_t lo = 16;
  for (auto& v : per_region)
    for (int32_t s : v) lo = std::max(lo, s);
  std::vector<int32_t> off;
  auto fits = [&](int32_t cap) {
    for (auto& v : per_region)
      if (!ring_place(v, cap, window, off)) return false;
    return true;
  };
  if (lo > budget || !fits(budget)) return -1;
  int32_t hi = budget;   // fits(hi); binary search in 16-byte steps
  lo = (lo + 15) & ~15;
  while (lo < hi) {
    const int32_t mid = ((lo + (hi - lo) / 2) + 15) & ~15;
    if (mid >= hi) break;
    if (fits(mid)) hi = mid;
    else lo = mid + 16;
  }
  return fits(lo) ? lo : hi;
}

}  // namespace

// Build a wave stream.  kind 0: factorization (stencil-class rows only:
// <= 4 pivots, every pivot's U row meets the row only at its diagonal),
// 1: forward solve (unit L), 2: backward solve.  threads = rows per wave,
// smem_budget = shared memory the kernel may use (bytes), tau_norms = the
// factor gathers each row's norm (tau > 0).  sizes[0..11] receive
// {static bytes, total waves, nreg, slot ring, max_waves, S, D, CS, CD,
// remote-dependency count, packed values, packed vector, most rows in a wave}.  Returns a handle > 0, or
// -1 (a row does not qualify), -2 (does not fit in shared memory).
extern "C" int64_t jv_rstream_build(int32_t kind, int32_t n, const int32_t* rs, const int32_t* col,
                                    const int32_t* diag, const int32_t* region_of, int32_t nreg,
                                    int32_t threads, int64_t smem_budget, int32_t tau_norms,
                                    int64_t* sizes) {
  if (n <= 0 || nreg < 1 || threads < 32) return -1;
  auto R = std::make_unique<RStream>();
  R->kind = kind;
  R->nreg = nreg;
  const bool fwd = kind != 2;
  // dependencies of row r (ascending column): fwd/factor = strict lower,
  // bwd = strict upper
  auto dep_lo = [&](int32_t r) { return fwd ? rs[r] : diag[r] + 1; };
  auto dep_hi = [&](int32_t r) { return fwd ? diag[r] : rs[r + 1]; };
  // levels of this direction's DAG
  std::vector<int32_t> lev(n, 0);
  if (fwd) {
    for (int32_t r = 0; r < n; ++r) {
      int32_t l = 0;
      for (int32_t p = dep_lo(r); p < dep_hi(r); ++p) l = std::max(l, lev[col[p]] + 1);
      lev[r] = l;
    }
  } else {
    for (int32_t r = n - 1; r >= 0; --r) {
      int32_t l = 0;
      for (int32_t p = dep_lo(r); p < dep_hi(r); ++p) l = std::max(l, lev[col[p]] + 1);
      lev[r] = l;
    }
  }
  // qualification (factor: stencil class) and per-row u positions
  std::vector<int32_t> us;
  std::vector<int32_t> umask;
  if (kind == 0) {
    us.assign((size_t)4 * n, 0);
    umask.assign(n, 0);
    std::vector<int32_t> mark(n, -1);
    for (int32_t r = 0; r < n; ++r) {
      const int32_t nL = diag[r] - rs[r];
      if (nL > 4) return -1;
      for (int32_t p = rs[r]; p < rs[r + 1]; ++p) mark[col[p]] = r;
      for (int32_t k = 0; k < nL; ++k) {
        const int32_t c = col[rs[r] + k];
        for (int32_t q = diag[c] + 1; q < rs[c + 1]; ++q) {
          const int32_t j = col[q];
          if (j == r) {
            us[(size_t)4 * r + k] = q;
            umask[r] |= 1 << k;
          } else if (mark[j] == r) {
            return -1;   // the pivot's U row meets row r off the diagonal
          }
        }
      }
    }
  } else {
    for (int32_t r = 0; r < n; ++r)
      if (dep_hi(r) - dep_lo(r) > 32) return -1;
  }
  // slots: rows of each region in (level, row) order
  std::vector<int32_t> reg_ptr(nreg + 1, 0);
  for (int32_t r = 0; r < n; ++r) {
    if (region_of[r] < 0 || region_of[r] >= nreg) return -1;
    ++reg_ptr[region_of[r] + 1];
  }
  for (int32_t g = 0; g < nreg; ++g) reg_ptr[g + 1] += reg_ptr[g];
  std::vector<int32_t> slot_row(n), slot_of(n);
  {
    std::vector<int32_t> fill(reg_ptr.begin(), reg_ptr.end() - 1);
    for (int32_t r = 0; r < n; ++r) slot_row[fill[region_of[r]]++] = r;
    for (int32_t g = 0; g < nreg; ++g)
      std::stable_sort(slot_row.begin() + reg_ptr[g], slot_row.begin() + reg_ptr[g + 1],
                       [&](int32_t a, int32_t b) { return lev[a] < lev[b]; });
    for (int32_t i = 0; i < n; ++i) slot_of[slot_row[i]] = i;
  }
  // waves: consecutive rows of one level, <= threads rows
  std::vector<int32_t> wave_first, wave_cnt, wave_of_slot(n);
  R->reg_wave.assign(nreg + 1, 0);
  for (int32_t g = 0; g < nreg; ++g) {
    R->max_region = std::max(R->max_region, reg_ptr[g + 1] - reg_ptr[g]);
    int32_t i = reg_ptr[g];
    while (i < reg_ptr[g + 1]) {
      const int32_t l = lev[slot_row[i]];
      int32_t e = i;
      while (e < reg_ptr[g + 1] && lev[slot_row[e]] == l && e - i < threads) ++e;
      for (int32_t k = i; k < e; ++k) wave_of_slot[k] = (int32_t)wave_first.size();
      wave_first.push_back(i);
      wave_cnt.push_back(e - i);
      i = e;
    }
    R->reg_wave[g + 1] = (int32_t)wave_first.size();
    R->max_waves = std::max(R->max_waves, R->reg_wave[g + 1] - R->reg_wave[g]);
  }
  const int64_t nw = (int64_t)wave_first.size();
  // In-region dependency values live in a ring of SC slots (slot i at
  // i % SC): a dependency is read from it when the slot cannot have been
  // overwritten — (last slot of the reading wave) - slot(c) < SC — and
  // through the mailbox otherwise, like a remote one.
  int64_t need = 1;
  for (int32_t r = 0; r < n; ++r) {
    const int32_t wv = wave_of_slot[slot_of[r]];
    const int32_t last = wave_first[wv] + wave_cnt[wv] - 1;
    for (int32_t p = dep_lo(r); p < dep_hi(r); ++p)
      if (region_of[col[p]] == region_of[r]) need = std::max<int64_t>(need, last - slot_of[col[p]] + 1);
  }
  int64_t sc_need = 64;
  while (sc_need < need) sc_need <<= 1;
  std::vector<char> pub(n, 0);
  std::vector<int32_t> goff(nw), sbytes(nw), dbytes(nw), voff(nw), vbytes(nw);
  std::vector<int32_t>& sidx = R->sidx;
  std::vector<int32_t>& vidx = R->vidx;
  std::vector<int32_t> coff(nw), cbytes(nw), npk(nw);
  int64_t vtot = 0, ctot = 0;
  std::vector<std::vector<int32_t>> ssz(nreg), dsz(nreg);
  std::vector<int32_t>& W = R->words;
  auto local = [&](int32_t r, int32_t c, int32_t SC) {
    if (region_of[c] != region_of[r]) return false;
    const int32_t wv = wave_of_slot[slot_of[r]];
    return wave_first[wv] + wave_cnt[wv] - 1 - slot_of[c] < SC;
  };
  // shared-memory byte offsets the refs point to (region.cu's layout)
  const int32_t kOneOff = 144;                             // the constant 1.0
  const int32_t slot_base = 256 + 16 * R->max_waves;       // value ring
  auto emit = [&](int32_t SC) {
    std::fill(pub.begin(), pub.end(), 0);
    for (int32_t r = 0; r < n; ++r)
      for (int32_t p = dep_lo(r); p < dep_hi(r); ++p)
        if (!local(r, col[p], SC)) pub[col[p]] = 1;
    W.clear();
    R->ndeps_remote = R->nrows_remote = 0;
    int32_t g = 0;
    for (int32_t gg = 0; gg < nreg; ++gg) { ssz[gg].clear(); dsz[gg].clear(); }
    std::vector<int32_t> ref, pslot;
    sidx.clear();
    vidx.clear();
    vtot = 0;
    ctot = 0;
    for (int64_t w = 0; w < nw; ++w) {
      while (w >= R->reg_wave[g + 1]) ++g;
      const int32_t s0 = wave_first[w], cnt = wave_cnt[w];
      int32_t K = 0;
      for (int32_t i = 0; i < cnt; ++i) {
        const int32_t r = slot_row[s0 + i];
        K = std::max(K, dep_hi(r) - dep_lo(r));
      }
      // block: header, 32-byte records, xref[K - 4][], pslot[]
      const int32_t KX = std::max(K - 4, 0);
      ref.assign((size_t)KX * cnt, kOneOff);
      pslot.clear();
      const size_t base = W.size();
      goff[w] = (int32_t)(base / 4);
      W.resize(base + 4 + (size_t)8 * cnt, 0);
      for (int32_t i = 0; i < cnt; ++i) {
        const int32_t r = slot_row[s0 + i];
        const int32_t lo = dep_lo(r), hi = dep_hi(r), nd = hi - lo;
        int32_t nrem = 0;
        int32_t* rec = &W[base + 4 + (size_t)8 * i];
        for (int32_t k = 0; k < 4; ++k) rec[k] = kOneOff;
        for (int32_t p = lo; p < hi; ++p) {
          const int32_t c = col[p];
          int32_t v;
          if (local(r, c, SC)) {
            v = slot_base + 8 * ((slot_of[c] - reg_ptr[g]) % SC);
          } else {
            v = -(1 + (int32_t)pslot.size());   // patched after ring placement
            pslot.push_back(c);   // mailbox slot = row (dense: 8 packets per 128-byte line)
            ++nrem;
          }
          if (p - lo < 4) rec[p - lo] = v;
          else ref[(size_t)(p - lo - 4) * cnt + i] = v;
        }
        R->ndeps_remote += nrem;
        R->nrows_remote += nrem > 0;
        rec[4] = kind == 2 ? diag[r] : rs[r];
        rec[5] = r;
        rec[6] = nd | (pub[r] ? 1 << 6 : 0) | (kind == 0 ? umask[r] << 7 : 0);
        rec[7] = slot_base + 8 * ((s0 - reg_ptr[g] + i) % SC);
      }
      W[base + 0] = cnt;
      W[base + 1] = s0 - reg_ptr[g];
      W[base + 2] = K;
      W[base + 3] = (int32_t)pslot.size();
      W.insert(W.end(), ref.begin(), ref.end());
      W.insert(W.end(), pslot.begin(), pslot.end());
      while ((W.size() - base) % 4) W.push_back(0);
      // values of the wave, packed once per factorization into a global
      // array in wave order (vals[NVm][cnt], jv_pack_values with sidx) and
      // bulk-copied: factor: a_k (k < K), a_rr, u_k (k < K);  fwd: l_k;
      // bwd: u_rr, u_k.  The per-call vector (fwd b, bwd y; factor norms
      // when tau > 0) is gathered per row behind them, then the packets.
      const int32_t NVm = kind == 0 ? 2 * K + 1 : (kind == 1 ? K : K + 1);
      const bool vec = kind != 0 || tau_norms;
      const int32_t vb = (8 * NVm * cnt + 15) & ~15;
      voff[w] = vtot / 16;
      vbytes[w] = vb;
      vtot += vb;
      const size_t s0x = sidx.size();
      sidx.resize(s0x + vb / 8, -1);
      for (int32_t i = 0; i < cnt; ++i) {
        const int32_t r = slot_row[s0 + i];
        const int32_t nd = dep_hi(r) - dep_lo(r);
        auto put = [&](int32_t k, int32_t src) { sidx[s0x + (size_t)k * cnt + i] = src; };
        if (kind == 0) {
          for (int32_t k = 0; k < nd; ++k) put(k, rs[r] + k);
          put(K, rs[r] + nd);
          for (int32_t k = 0; k < nd; ++k) put(K + 1 + k, us[(size_t)4 * r + k]);
        } else if (kind == 1) {
          for (int32_t k = 0; k < nd; ++k) put(k, rs[r] + k);
        } else {
          for (int32_t k = 0; k <= nd; ++k) put(k, diag[r] + k);
        }
      }
      // the per-call vector in wave order (jv_pack_values with vidx)
      const int32_t cb = vec ? (8 * cnt + 15) & ~15 : 0;
      coff[w] = ctot / 16;
      cbytes[w] = cb;
      ctot += cb;
      if (vec) {
        const size_t c0 = vidx.size();
        vidx.resize(c0 + cb / 8, -1);
        for (int32_t i = 0; i < cnt; ++i) vidx[c0 + i] = slot_row[s0 + i];
      }
      // then the wave's remote values (8 bytes each, written by the prober warps)
      sbytes[w] = (int32_t)(4 * (W.size() - base));
      dbytes[w] = vb + cb + ((8 * (int32_t)pslot.size() + 15) & ~15);
      npk[w] = (int32_t)pslot.size();
      ssz[g].push_back(sbytes[w]);
      dsz[g].push_back(dbytes[w]);
    }
  };
  // slot ring and ring buffers: the largest prefetch distance D that fits,
  // then the largest slot ring for it (a smaller ring sends far-back
  // in-region dependencies through the mailbox, where the D-wave prefetch
  // finds them long published)
  auto fit = [&](int64_t SC, int32_t& D_, int32_t& cs_, int32_t& cd_) {
    const int64_t fixed = 512 + 16 * (int64_t)R->max_waves + 8 * SC;
    const int64_t ring = (smem_budget - fixed) & ~(int64_t)15;
    if (ring < 1024) return false;
    for (int D = 8; D >= 2; --D) {   // (the kernel's producer needs two waves of slack)
      const int32_t cd = min_cap(dsz, D, (int32_t)ring);
      if (cd < 0) continue;
      const int32_t cs = min_cap(ssz, D, (int32_t)(ring - cd));
      if (cs < 0) continue;
      D_ = D;
      cs_ = cs;
      cd_ = cd;
      return true;
    }
    return false;
  };
  int64_t bestSC = 0;
  int32_t bestD = 0;
  for (int64_t SC = std::min<int64_t>(sc_need, 8192); SC >= 64; SC >>= 1) {
    emit((int32_t)SC);
    int32_t D = 0, cs = 0, cd = 0;
    if (fit(SC, D, cs, cd) && D > bestD) {
      bestD = D;
      bestSC = SC;
    }
    if (std::getenv("JV_RS_DEBUG")) {
      int32_t ms = 0, md = 0;
      for (auto& v : ssz) for (int32_t x : v) ms = std::max(ms, x);
      for (auto& v : dsz) for (int32_t x : v) md = std::max(md, x);
      std::fprintf(stderr, "rstream kind %d threads %d SC %lld: max static block %d, max dynamic block %d, "
                   "max_waves %d, budget %lld -> D %d\n", kind, threads, (long long)SC, ms, md,
                   R->max_waves, (long long)smem_budget, D);
    }
    if (bestD >= 6) break;
  }
  if (bestD == 0) return -2;
  emit((int32_t)bestSC);
  {
    int32_t D = 0, cs = 0, cd = 0;
    fit(bestSC, D, cs, cd);
    R->S = D;
    R->D = D;
    R->CS = cs;
    R->CD = cd;
    R->SC = (int32_t)bestSC;
  }
  R->table.assign((size_t)8 * nw, 0);
  std::vector<int32_t> so, dof;
  for (int32_t gg = 0; gg < nreg; ++gg) {
    ring_place(ssz[gg], R->CS, R->S, so);
    ring_place(dsz[gg], R->CD, R->D, dof);
    for (int32_t k = 0; k < R->reg_wave[gg + 1] - R->reg_wave[gg]; ++k) {
      const int64_t w = R->reg_wave[gg] + k;
      R->table[8 * w + 0] = goff[w];   // 16-byte units
      R->table[8 * w + 1] = sbytes[w];
      R->table[8 * w + 2] = so[k];
      R->table[8 * w + 3] = dof[k];
      R->table[8 * w + 4] = voff[w];   // 16-byte units
      R->table[8 * w + 5] = vbytes[w];
      R->table[8 * w + 6] = coff[w];   // 16-byte units
      R->table[8 * w + 7] = cbytes[w] | (npk[w] << 16);   // | remote packets of the wave
      // remote refs -> offsets of the wave's decoded values (behind its
      // packed values, vector and packets in the dynamic ring)
      const int32_t rem = slot_base + 8 * R->SC + R->CS + dof[k] + vbytes[w] + cbytes[w];
      int32_t* blk = &W[(size_t)goff[w] * 4];
      const int32_t cnt = blk[0], K = blk[2];
      for (int32_t i = 0; i < cnt; ++i)
        for (int32_t q = 0; q < 4; ++q) {
          int32_t& v = blk[4 + 8 * i + q];
          if (v < 0) v = rem + 8 * (-1 - v);
        }
      for (int32_t q = 0; q < std::max(K - 4, 0) * cnt; ++q) {
        int32_t& v = blk[4 + 8 * cnt + q];
        if (v < 0) v = rem + 8 * (-1 - v);
      }
    }
  }
  sizes[0] = 4 * (int64_t)W.size();
  sizes[1] = nw;
  sizes[2] = nreg;
  sizes[3] = R->SC;
  sizes[4] = R->max_waves;
  sizes[5] = R->S;
  sizes[6] = R->D;
  sizes[7] = R->CS;
  sizes[8] = R->CD;
  sizes[9] = R->ndeps_remote;
  sizes[10] = (int64_t)R->sidx.size();
  sizes[11] = (int64_t)R->vidx.size();
  {
    int64_t mr = 0;
    for (int64_t w = 0; w < nw; ++w) mr = std::max<int64_t>(mr, wave_cnt[w]);
    sizes[12] = mr;
  }
  std::lock_guard<std::mutex> lk(g_rs_mu);
  const int64_t h = g_rs_next++;
  g_rs[h] = std::move(R);
  return h;
}

// Copy a built stream out (host buffers sized from jv_rstream_build's
// sizes) and release it.
extern "C" int jv_rstream_export(int64_t handle, int32_t* words, int32_t* table,
                                 int32_t* reg_wave, int32_t* sidx, int32_t* vidx) {
  std::unique_ptr<RStream> R;
  {
    std::lock_guard<std::mutex> lk(g_rs_mu);
    auto it = g_rs.find(handle);
    if (it == g_rs.end()) return JV_EINVAL;
    R = std::move(it->second);
    g_rs.erase(it);
  }
  std::memcpy(words, R->words.data(), 4 * R->words.size());
  std::memcpy(table, R->table.data(), 4 * R->table.size());
  std::memcpy(reg_wave, R->reg_wave.data(), 4 * R->reg_wave.size());
  std::memcpy(sidx, R->sidx.data(), 4 * R->sidx.size());
  std::memcpy(vidx, R->vidx.data(), 4 * R->vidx.size());
  return JV_OK;
}
