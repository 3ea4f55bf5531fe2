// Sync-free numeric ILU(k, tau) factorization for sm_100a.
//
// Reference semantics: _kernels.py:165-204 (_factor_row, factor_serial_kernel).
// Row r is eliminated up-looking over its strictly-lower pivots c in
// ascending column order:   l = a_rc / u_cc ; tau drop ; a_rj -= l * u_cj.
// Every operation is an explicitly rounded binary64 op (no FMA), and per
// stored position the updates arrive in ascending pivot order, so the result
// is bitwise equal to factor_serial for ANY schedule that respects the
// dependencies.
//
// Schedule (jv_build_schedule): rows in level order of the factor DAG; inside
// a level, "short" rows (<= kR entries, <= kP pivots, <= kU upper entries per
// pivot, no MILU — every stencil row of configs 1-2) come in batches of 32
// (lane = row), every other row is a batch of its own (warp = row).  Warp w
// of a persistent co-resident (cooperative) grid takes batches w, w+W, ...;
// batch b depends only on batches < b, so the lowest unfinished batch always
// progresses: deadlock-free.
//
// Communication: a finished row publishes its U part (diagonal + upper
// entries) as 16-byte mailbox packets {value, epoch} (common.cuh); consumers
// probe exactly the packets they need.  A warp first waits at a gate — one
// lane polls the newest pivot row of the batch with __nanosleep backoff —
// so the ~10^5 rows resident ahead of the dependency frontier do not flood
// L2 with probes; then all lanes probe their packets back to back.
//
// Thread path: the whole row, its pivots' U rows and the gathered values
// live in registers (compile-time caps, fully unrolled).  Divisions of
// pivots whose value no earlier pivot touches are issued together; the
// dependent chain per hop is then one division plus the per-position
// update sequence.
// Warp path: row cached in shared memory, pivots in chunks of 32 (lane k =
// pivot k: its diagonal position and U range), the matching U entries found
// by parallel binary searches and compacted into a shared op list, gathered
// in one parallel probe round, then applied pivot by pivot (lanes over the
// pivot's updates, which hit distinct positions).
#include "common.cuh"
#include "../../include/jv.h"

namespace {

// JV_HEAVY_PROFILE (diagnostic builds only): per-phase clock64 sums of the
// warp / heavy row paths, written to the batch trace (tools/trace.py)
#ifdef JV_HEAVY_PROFILE
#define HP_T0(v) long long v = clock64()
#define HP_ADD(acc, v) acc += clock64() - v
#else
#define HP_T0(v)
#define HP_ADD(acc, v)
#endif

constexpr int kR = 8;       // thread path: row entries
constexpr int kP = 4;       // thread path: pivots (strict-lower entries)
constexpr int kU = 4;       // thread path: strict-upper entries per pivot row
constexpr int kWarpRow = 128;   // warp path: row entries cached in smem
constexpr int kWarpOps = 256;   // warp path: op list capacity per chunk
#ifndef JV_FACTOR_WARPS
#define JV_FACTOR_WARPS 8
#endif
constexpr int kFactorWarps = JV_FACTOR_WARPS; // warps per CTA (one CTA per SM)
constexpr int kOut = 1 << 30;   // op target flag: out-of-pattern (MILU -> diagonal)

struct FactorArgs {
  const int32_t* row_start;
  const int32_t* col;
  double* val;
  const int32_t* diag;
  const double* norms;
  double tau;
  int milu;
  const int32_t* order;
  const int32_t* batch_ptr;
  int32_t nbatch;
  int32_t ready_below;
  uint64_t* mbox;
  uint32_t epoch;
  int32_t* err;
  int* ticket;
  const int8_t* heavy;        // nullable: rows with an elimination list
  const int64_t* elim_ptr;    // [nnz+1]: ops of L entry p = [elim_ptr[p], elim_ptr[p+1])
  const int2* elim;           // op = (q: U entry of the pivot row, w: target position | kOut)
  const int8_t* bclass;       // nullable: batch class (0 thread rows, 1 row pair, 2 single row)
  const int2* hub_stream;     // nullable: hub-row gather plans (jv_hub_plan_host)
  const int64_t* hub_sptr;    // per row: first stream entry (rows with flag 4)
  const int32_t* hub_meta;
  const int64_t* hub_mptr;    // per row: offset of [nphases, 32 lane loads per phase]
};

struct WarpArena {
  double val[kWarpRow];
  int col[kWarpRow];
  int opq[kWarpOps];
  int opw[kWarpOps];
  double opv[kWarpOps];
  int opend[32];
  int pivc[32];
};

// lower_bound of key in arr[lo, hi)
JV_INLINE int lower_bound(const int32_t* arr, int lo, int hi, int key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (arr[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// raw probe: issue the load now, check the tag later (no compiler barrier, so
// consecutive probes are in flight together)
struct Probe {
  unsigned long long w0, w1;
};
JV_INLINE Probe probe_issue(const uint64_t* box, int64_t slot) {
  Probe p;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
               : "=l"(p.w0), "=l"(p.w1) : "l"(box + 2 * slot));
  return p;
}
JV_INLINE bool probe_ok(const Probe& p, uint32_t epoch) {
  return (uint32_t)(p.w0 >> 32) == epoch && (uint32_t)(p.w1 >> 32) == epoch;
}
JV_INLINE double probe_val(const Probe& p) {
  return __longlong_as_double((long long)((p.w0 & 0xffffffffull) | (p.w1 << 32)));
}

// value of U entry q of pivot row c (final in val[] below ready_below)
JV_INLINE double pivot_value(const FactorArgs& A, int c, int q) {
  if (c < A.ready_below) return __ldcg(A.val + q);
  return jv::mbox_wait(A.mbox, q, A.epoch);
}

// ---------------------------------------------------------------- thread path
//
// Per-thread state lives in a shared-memory slice (slot-major, so a warp's
// accesses to one slot are contiguous): compact loops instead of unrolled
// register code keep the hot path inside the instruction cache — a fully
// unrolled first version (64 KB of SASS) spent ~5 us per batch on
// instruction fetch.

constexpr int kSlotsI = kR + 2 * kP + kP * kU;    // cj | dq | ulen | op list
constexpr int kSlotsD = kR + kP + kP * kU + kP;   // a | dv | uv | lspec
constexpr int kThreads = kFactorWarps * 32;
// The warp arena of a warp-path row lives in the warp's own slice block
// (a warp runs one batch at a time: thread-path slices, warp-path arena and
// heavy-row ring never coexist), so the slab is slices + the heavy buffer.
constexpr size_t kArenaBytes = 0;
static_assert(sizeof(WarpArena) <= 32 * kSlotsD * sizeof(double), "arena must fit a slice block");

extern __shared__ __align__(16) unsigned char jv_factor_smem[];

// Per-thread slice of the shared slab: warp-major blocks (warp w owns a
// contiguous 32-lane x slots block, so an idle warp can reuse its block as
// plain scratch — the heavy-row ring), slot-major inside a block, one column
// per lane.  Addressed through the kernel's extern __shared__ array so every
// access compiles to LDS/STS.
JV_INLINE int* slice_ints(int warp) {
  return reinterpret_cast<int*>(jv_factor_smem + kArenaBytes + (size_t)kThreads * kSlotsD * 8) +
         warp * (32 * kSlotsI);
}
JV_INLINE double* slice_doubles(int warp) {
  return reinterpret_cast<double*>(jv_factor_smem + kArenaBytes) + warp * (32 * kSlotsD);
}
struct Slice {
  int tid;
  JV_INLINE int* ib() const { return slice_ints(tid >> 5) + (tid & 31); }
  JV_INLINE double* db() const { return slice_doubles(tid >> 5) + (tid & 31); }
  JV_INLINE int& cj(int k) const { return ib()[k * 32]; }
  JV_INLINE int& dq(int k) const { return ib()[(kR + k) * 32]; }
  JV_INLINE int& ul(int k) const { return ib()[(kR + kP + k) * 32]; }
  // update op o: (k << 16) | (t << 8) | target entry
  JV_INLINE int& op(int o) const { return ib()[(kR + 2 * kP + o) * 32]; }
  JV_INLINE double& a(int k) const { return db()[k * 32]; }
  JV_INLINE double& dv(int k) const { return db()[(kR + k) * 32]; }
  JV_INLINE double& uv(int k, int t) const { return db()[(kR + kP + k * kU + t) * 32]; }
  JV_INLINE double& ls(int k) const { return db()[(kR + kP + kP * kU + k) * 32]; }
};

struct ShortRow {
  int rs, len, nL;
  unsigned miss;      // gather slots still to be awaited (bit k*(kU+1)+u)
  unsigned opend;     // 5-bit end offset of pivot k's ops at bit 5k
  double thresh;      // tau * row norm (0 when tau == 0)
  unsigned touched;   // bit k: a[k] receives an update from an earlier pivot
  int gate, gate_q;
};

// structure of a short row (no waiting).  false: caps exceeded.
JV_INLINE bool short_structure(const FactorArgs& A, int r, ShortRow& R, Slice S) {
  R.rs = __ldg(A.row_start + r);
  R.len = __ldg(A.row_start + r + 1) - R.rs;
  R.nL = __ldg(A.diag + r) - R.rs;
  R.gate = -1;
  R.gate_q = 0;
  R.touched = 0;
  R.thresh = 0.0;
  if (R.len > kR || R.nL > kP || A.milu) return false;
  if (A.tau > 0.0) R.thresh = jv::dmul(A.tau, __ldg(A.norms + r));
  // every round of loads is issued as one batch (registers), then spilled to
  // the slice: 4 dependent memory rounds per row instead of one per entry
  int cj[kR];
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    if (i < R.len) {
      cj[i] = __ldg(A.col + R.rs + i);
      S.a(i) = __ldcs(A.val + R.rs + i);
    } else {
      cj[i] = -1;
    }
  }
  int dq[kP], ce[kP];
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    S.cj(k) = cj[k];
    if (k < R.nL) {
      dq[k] = __ldg(A.diag + cj[k]);
      ce[k] = __ldg(A.row_start + cj[k] + 1);
    } else {
      dq[k] = 0;
      ce[k] = 1;
    }
  }
#pragma unroll
  for (int i = kP; i < kR; ++i) S.cj(i) = cj[i];
  bool ok = true;
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    S.dq(k) = dq[k];
    S.ul(k) = ce[k] - dq[k] - 1;
    ok &= ce[k] - dq[k] - 1 <= kU;
  }
  if (!ok) return false;
  R.miss = 0;
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    if (k < R.nL) {
      const int ul = ce[k] - dq[k] - 1;
      if (cj[k] < A.ready_below) {
        // factored by an earlier call: final in val[]
        S.dv(k) = __ldcg(A.val + dq[k]);
#pragma unroll
        for (int t = 0; t < kU; ++t)
          if (t < ul) S.uv(k, t) = __ldcg(A.val + dq[k] + 1 + t);
      } else {
        R.miss |= ((2u << ul) - 1u) << (k * (kU + 1));
      }
    }
  }
  if (R.nL > 0) {
    // pivots ascend: the last one is the newest row
    const int c = S.cj(R.nL - 1);
    // the pivot row publishes its U packets in position order: poll the last
    if (c >= A.ready_below) { R.gate = c; R.gate_q = S.dq(R.nL - 1) + S.ul(R.nL - 1); }
  }
  int uc[kP][kU];
#pragma unroll
  for (int k = 0; k < kP; ++k)
#pragma unroll
    for (int t = 0; t < kU; ++t)
      uc[k][t] = (t < ce[k] - dq[k] - 1) ? __ldg(A.col + dq[k] + 1 + t) : -1;
  int nops = 0;
  R.opend = 0;
  for (int k = 0; k < R.nL; ++k) {
    for (int t = 0; t < kU; ++t) {
      int j = -1;
#pragma unroll
      for (int kk = 0; kk < kP; ++kk)
#pragma unroll
        for (int tt = 0; tt < kU; ++tt)
          if (kk == k && tt == t) j = uc[kk][tt];
      if (j < 0) continue;
      for (int i = k + 1; i < R.len; ++i) {
        if (S.cj(i) == j) {
          S.op(nops++) = (k << 16) | (t << 8) | i;
          if (i < R.nL) R.touched |= 1u << i;
          break;
        }
      }
    }
    R.opend |= (unsigned)nops << (5 * k);
  }
  return true;
}

// Gather of a short row's pivot values.  The wait is warp-converged: every
// lane re-probes only its still-missing packets, then the warp votes; lanes
// never spin on their own (divergent per-lane spin loops inside one warp
// were measured to stretch a hop to ~20 us on config 2).
JV_INLINE unsigned short_gather(const FactorArgs& A, const ShortRow& R, Slice S, unsigned mask) {
  constexpr int kSlots = kP * (kU + 1);
  // slot (k, u): u = 0 the pivot's diagonal, u > 0 its u-th upper entry;
  // R.miss was prepared before the gate (pivots factored by an earlier call
  // were read there already)
  unsigned miss = R.miss;
  int dq[kP];
#pragma unroll
  for (int k = 0; k < kP; ++k) dq[k] = S.dq(k);
  unsigned ns = 0, spins = 0, rounds = 0;
  while (__any_sync(mask, miss)) {
    ++rounds;
    Probe p[kSlots];
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl)
      if (miss & (1u << sl)) p[sl] = probe_issue(A.mbox, dq[sl / (kU + 1)] + sl % (kU + 1));
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      if ((miss & (1u << sl)) && probe_ok(p[sl], A.epoch)) {
        const int k = sl / (kU + 1), u = sl % (kU + 1);
        if (u == 0) S.dv(k) = probe_val(p[sl]); else S.uv(k, u - 1) = probe_val(p[sl]);
        miss &= ~(1u << sl);
      }
    }
    if (__any_sync(mask, miss)) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(2 * ns, jv::g_poll_cap) : 16u;
      if (++spins == jv::g_spin_limit) {
        atomicExch(&jv::g_hang, 1);
        break;
      }
    }
  }
  return rounds;
}

JV_INLINE void short_finish(const FactorArgs& A, int r, const ShortRow& R, Slice S,
                            unsigned mask, int cur_batch, const jv::Trace& T) {
  const unsigned rounds = short_gather(A, R, S, mask);
  if ((threadIdx.x & 31) == __ffs(mask) - 1) {
    jv::trace_mark(T, cur_batch, 7);
    jv::trace_word(T, cur_batch, 8, rounds);
  }
  // divisions of untouched pivots: independent, issued together
  double ls[kP];
#pragma unroll
  for (int k = 0; k < kP; ++k) ls[k] = (k < R.nL) ? jv::ddiv(S.a(k), S.dv(k)) : 0.0;
  const double thresh = R.thresh;
  int o = 0;
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    if (k < R.nL) {
      const double l = (R.touched & (1u << k)) ? jv::ddiv(S.a(k), S.dv(k)) : ls[k];
      const bool drop = A.tau > 0.0 && fabs(l) < thresh;
      S.a(k) = drop ? 0.0 : l;
      const int oe = (R.opend >> (5 * k)) & 31;
      if (!drop) {
        for (; o < oe; ++o) {
          const int op = S.op(o);
          const int w = op & 0xff, t = (op >> 8) & 0xff;
          S.a(w) = jv::dsub(S.a(w), jv::dmul(l, S.uv(k, t)));
        }
      }
      o = oe;
    }
  }
  if ((threadIdx.x & 31) == __ffs(mask) - 1) jv::trace_mark2(T, cur_batch);
  for (int i = 0; i < R.len; ++i) {
    const double v = S.a(i);
    __stcg(A.val + R.rs + i, v);
    if (i >= R.nL) jv::mbox_put(A.mbox, R.rs + i, v, A.epoch);
  }
  if (S.a(R.nL) == 0.0) atomicMin(A.err, r);
}

// ------------------------------------------------------ stencil fast path
//
// A short row whose pivots' U rows meet the row ONLY at its diagonal (every
// 5/7-point stencil row under ILU(0): the grid graph has no triangles) has
// independent pivots and a single update target.  Its strictly-upper
// entries are final from the start, so they are published before the gate;
// after the gate the row needs 2 packets per pivot, one division per pivot
// (all independent) and the diagonal's subtraction chain — everything in
// registers.

struct SfpRow {
  int rs, nL, dp;
  double aL[kP];      // strict-lower values
  double adiag;
  int dq[kP];         // pivot diagonal positions
  int us[kP];         // position of u(c_k, r) (-1: none)
  double dv[kP], uv[kP];   // values of pivots factored by an earlier call
  unsigned old;       // bit k: pivot k read from val[] (ready_below)
  double thresh;
  int gate, gate_q;
};

JV_INLINE bool sfp_structure(const FactorArgs& A, int r, SfpRow& F) {
  F.rs = __ldg(A.row_start + r);
  const int len = __ldg(A.row_start + r + 1) - F.rs;
  F.dp = __ldg(A.diag + r);
  F.nL = F.dp - F.rs;
  F.gate = -1;
  F.gate_q = 0;
  F.old = 0;
  if (len > kR || F.nL > kP || A.milu) return false;
  int cj[kR];
  double a[kR];
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    cj[i] = (i < len) ? __ldg(A.col + F.rs + i) : -1;
    a[i] = (i < len) ? __ldcs(A.val + F.rs + i) : 0.0;
  }
  int ce[kP];
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    F.dq[k] = (k < F.nL) ? __ldg(A.diag + cj[k]) : 0;
    ce[k] = (k < F.nL) ? __ldg(A.row_start + cj[k] + 1) : 1;
  }
  bool ok = true;
#pragma unroll
  for (int k = 0; k < kP; ++k) ok &= ce[k] - F.dq[k] - 1 <= kU;
  if (!ok) return false;
  int uc[kP][kU];
#pragma unroll
  for (int k = 0; k < kP; ++k)
#pragma unroll
    for (int t = 0; t < kU; ++t)
      uc[k][t] = (k < F.nL && t < ce[k] - F.dq[k] - 1) ? __ldg(A.col + F.dq[k] + 1 + t) : -2;
  // every U entry of every pivot must miss the row, except at column r
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    F.us[k] = -1;
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const int j = uc[k][t];
      if (j == r) F.us[k] = F.dq[k] + 1 + t;
#pragma unroll
      for (int i = 0; i < kR; ++i) ok &= !(j >= 0 && j != r && cj[i] == j);
    }
  }
  if (!ok) return false;
#pragma unroll
  for (int k = 0; k < kP; ++k) F.aL[k] = a[k];
  F.adiag = 0.0;
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    if (i == F.nL) F.adiag = a[i];
    // strictly-upper entries are final: publish them now
    if (i > F.nL && i < len) jv::mbox_put(A.mbox, F.rs + i, a[i], A.epoch);
  }
  F.thresh = (A.tau > 0.0) ? jv::dmul(A.tau, __ldg(A.norms + r)) : 0.0;
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    if (k < F.nL && cj[k] < A.ready_below) {
      F.old |= 1u << k;
      F.dv[k] = __ldcg(A.val + F.dq[k]);
      F.uv[k] = F.us[k] >= 0 ? __ldcg(A.val + F.us[k]) : 0.0;
    }
  }
  if (F.nL > 0) {
    int c = -1, q = 0;
#pragma unroll
    for (int k = 0; k < kP; ++k)
      if (k < F.nL) { c = cj[k]; q = F.dq[k]; }
    if (c >= A.ready_below) { F.gate = c; F.gate_q = q; }
  }
  return true;
}

// finishing a row once all its inputs are in: parallel divisions, the
// diagonal chain, stores and the diagonal's packet
JV_INLINE void sfp_compute(const FactorArgs& A, int r, SfpRow& F) {
  double l[kP];
  jv::ddiv_batch<kP>(F.aL, F.dv, l, F.nL);
  double d = F.adiag;
#pragma unroll
  for (int k = 0; k < kP; ++k) {
    if (k < F.nL) {
      const bool drop = A.tau > 0.0 && fabs(l[k]) < F.thresh;
      if (drop) l[k] = 0.0;
      else if (F.us[k] >= 0) d = jv::dsub(d, jv::dmul(l[k], F.uv[k]));
    }
  }
  jv::mbox_put(A.mbox, F.dp, d, A.epoch);
#pragma unroll
  for (int k = 0; k < kP; ++k)
    if (k < F.nL) __stcg(A.val + F.rs + k, l[k]);
  __stcg(A.val + F.dp, d);
  if (d == 0.0) atomicMin(A.err, r);
}

// Gather of the pivots' diagonals and u(c_k, r), warp-converged (no lane
// spins alone), then the row is finished.  (Finishing each lane inside the
// loop as soon as its own inputs arrive was measured slower on config 2:
// the divergent compute inside the polling loop costs more than the
// coupling it removes.)
JV_INLINE void sfp_finish(const FactorArgs& A, int r, SfpRow& F, unsigned mask, int cur_batch,
                          const jv::Trace& T) {
  unsigned miss = 0;
#pragma unroll
  for (int k = 0; k < kP; ++k)
    if (k < F.nL && !(F.old & (1u << k))) miss |= (F.us[k] >= 0 ? 3u : 1u) << (2 * k);
  unsigned ns = 0, spins = 0;
  while (__any_sync(mask, miss)) {
    Probe p[2 * kP];
#pragma unroll
    for (int k = 0; k < kP; ++k) {
      if (miss & (1u << (2 * k))) p[2 * k] = probe_issue(A.mbox, F.dq[k]);
      if (miss & (2u << (2 * k))) p[2 * k + 1] = probe_issue(A.mbox, F.us[k]);
    }
#pragma unroll
    for (int k = 0; k < kP; ++k) {
      if ((miss & (1u << (2 * k))) && probe_ok(p[2 * k], A.epoch)) {
        F.dv[k] = probe_val(p[2 * k]);
        miss &= ~(1u << (2 * k));
      }
      if ((miss & (2u << (2 * k))) && probe_ok(p[2 * k + 1], A.epoch)) {
        F.uv[k] = probe_val(p[2 * k + 1]);
        miss &= ~(2u << (2 * k));
      }
    }
    if (__any_sync(mask, miss)) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(2 * ns, jv::g_poll_cap) : 16u;
      if (++spins == jv::g_spin_limit) {
        atomicExch(&jv::g_hang, 1);
        break;
      }
    }
  }
  if ((threadIdx.x & 31) == __ffs(mask) - 1) {
    jv::trace_mark(T, cur_batch, 7);
#ifdef JV_HEAVY_PROFILE
    jv::trace_word(T, cur_batch, 13, spins);
#endif
  }
  sfp_compute(A, r, F);
}

// ------------------------------------------------------------------ warp path

// Warp-converged wait for one packet per lane (lanes with need == false
// just vote): no lane ever spins alone.
JV_INLINE double warp_value(const FactorArgs& A, bool need, int c, int q) {
  double v = 0.0;
  bool miss = need;
  if (need && c < A.ready_below) {
    v = __ldcg(A.val + q);
    miss = false;
  }
  unsigned ns = 0, spins = 0;
  while (__any_sync(0xffffffffu, miss)) {
    if (miss) {
      const Probe p = probe_issue(A.mbox, q);
      if (probe_ok(p, A.epoch)) {
        v = probe_val(p);
        miss = false;
      }
    }
    if (__any_sync(0xffffffffu, miss)) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(2 * ns, jv::g_poll_cap) : 16u;
      if (++spins == jv::g_spin_limit) {
        atomicExch(&jv::g_hang, 1);
        break;
      }
    }
  }
  return v;
}

// ------------------------------------------------------------ pair path
//
// Two listed warp-path rows of the same level (so independent) in one warp,
// a half-warp each: the memory latency of one row's phases overlaps the
// other's, doubling warp-row throughput (configs 3/4 are bound by warp
// time per row).  Rows qualify at setup (jv_elim_lists flag 1): cached
// length <= kPairRow, every pivot's ops <= kPairOps.
constexpr int kPairRow = 64;
constexpr int kPairOps = 160;

struct HalfArena {
  double val[kPairRow];
  double opv[kPairOps];
  int col[kPairRow];
  int opq[kPairOps];
  int opw[kPairOps];
  int opend[16];
  int pivc[16];
};

// converged wait inside one half-warp (mask = that half's lanes)
JV_INLINE double half_value(const FactorArgs& A, bool need, int q, unsigned mask) {
  double v = 0.0;
  bool miss = need;
  unsigned ns = 0, spins = 0;
  while (__any_sync(mask, miss)) {
    if (miss) {
      const Probe p = probe_issue(A.mbox, q);
      if (probe_ok(p, A.epoch)) {
        v = probe_val(p);
        miss = false;
      }
    }
    if (__any_sync(mask, miss)) {
      if (ns) __nanosleep(ns);
      ns = ns ? min(2 * ns, jv::g_poll_cap) : 16u;
      if (++spins == jv::g_spin_limit) {
        atomicExch(&jv::g_hang, 1);
        break;
      }
    }
  }
  return v;
}

JV_INLINE void pair_row(const FactorArgs& A, int r, int hl, unsigned hmask, HalfArena& H) {
  const int rs = A.row_start[r], re = A.row_start[r + 1];
  const int len = re - rs;
  const int nL = A.diag[r] - rs;
  double* av = H.val;
  for (int i = hl; i < len; i += 16) {
    H.col[i] = A.col[rs + i];
    H.val[i] = __ldcs(A.val + rs + i);
  }
  __syncwarp(hmask);
  const double thresh = A.tau > 0.0 ? jv::dmul(A.tau, A.norms[r]) : 0.0;
  constexpr int kSlots = kPairOps / 16;

  for (int k0 = 0; k0 < nL;) {
    const int kc0 = min(16, nL - k0);
    const long long E0 = A.elim_ptr[rs + k0];
    int c = 0, d = 0;
    long long e1 = 0;
    if (hl < kc0) {
      c = H.col[k0 + hl];
      d = A.diag[c];
      e1 = A.elim_ptr[rs + k0 + hl + 1];
    }
    // the chunk: the leading pivots whose ops fit the half's list
    const bool fit = hl < kc0 && e1 - E0 <= kPairOps;
    const int kc = __popc(__ballot_sync(hmask, fit));
    if (hl < kc) {
      H.opend[hl] = (int)(e1 - E0);
      H.pivc[hl] = c;
    }
    const int nops = (int)(__shfl_sync(hmask, e1, kc - 1, 16) - E0);
    for (int o = hl; o < nops; o += 16) {
      const int2 op = __ldg(A.elim + E0 + o);
      H.opq[o] = op.x;
      H.opw[o] = op.y;
    }
    __syncwarp(hmask);
    // every probe of the chunk in flight before any is checked
    double dv = 0.0;
    bool dmiss = false;
    {
      Probe pd{0, 0};
      const bool have = hl < kc;
      if (have && c < A.ready_below) dv = __ldcg(A.val + d);
      else if (have) pd = probe_issue(A.mbox, d);
      Probe po[kSlots];
      bool old[kSlots];
#pragma unroll
      for (int i = 0; i < kSlots; ++i) {
        const int o = i * 16 + hl;
        po[i] = Probe{0, 0};
        old[i] = false;
        if (o < nops) {
          if (A.ready_below > 0) {
            int lo = 0, hi = kc - 1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (H.opend[mid] > o) hi = mid; else lo = mid + 1;
            }
            old[i] = H.pivc[lo] < A.ready_below;
          }
          if (old[i]) H.opv[o] = __ldcg(A.val + H.opq[o]);
          else po[i] = probe_issue(A.mbox, H.opq[o]);
        }
      }
      if (have && c >= A.ready_below) {
        if (probe_ok(pd, A.epoch)) dv = probe_val(pd);
        else dmiss = true;
      }
      unsigned omiss = 0;
#pragma unroll
      for (int i = 0; i < kSlots; ++i) {
        const int o = i * 16 + hl;
        if (o < nops && !old[i]) {
          if (probe_ok(po[i], A.epoch)) H.opv[o] = probe_val(po[i]);
          else omiss |= 1u << i;
        }
      }
      if (__any_sync(hmask, dmiss)) {
        const double v = half_value(A, dmiss, d, hmask);
        if (dmiss) dv = v;
      }
      if (__any_sync(hmask, omiss != 0)) {
        for (int i = 0; i < kSlots; ++i) {
          const bool m = (omiss >> i) & 1;
          const double v = half_value(A, m, m ? H.opq[i * 16 + hl] : 0, hmask);
          if (m) H.opv[i * 16 + hl] = v;
        }
      }
    }
    __syncwarp(hmask);
    // elimination, pivot by pivot
    for (int kk = 0, o0 = 0; kk < kc; ++kk) {
      const int k = k0 + kk;
      const int o1 = H.opend[kk];
      const double dk = __shfl_sync(hmask, dv, kk, 16);
      double l = 0.0;
      int drop = 0;
      if (hl == 0) {
        bool slow;
        const double a = av[k];
        l = jv::ddiv_fast(a, dk, slow);
        if (slow) l = __ddiv_rn(a, dk);
        drop = A.tau > 0.0 && fabs(l) < thresh;
        av[k] = drop ? 0.0 : l;
      }
      l = __shfl_sync(hmask, l, 0, 16);
      drop = __shfl_sync(hmask, drop, 0, 16);
      if (A.milu) {
        if (hl == 0)
          for (int o = o0; o < o1; ++o) {
            const int t = (drop || (H.opw[o] & kOut)) ? nL : H.opw[o];
            av[t] = jv::dsub(av[t], jv::dmul(l, H.opv[o]));
          }
      } else if (!drop) {
        for (int o = o0 + hl; o < o1; o += 16) {
          const int t = H.opw[o];
          av[t] = jv::dsub(av[t], jv::dmul(l, H.opv[o]));
        }
      }
      o0 = o1;
      __syncwarp(hmask);
    }
    k0 += kc;
  }
  for (int i = hl; i < len; i += 16) {
    const double v = av[i];
    __stcg(A.val + rs + i, v);
    if (i >= nL) jv::mbox_put(A.mbox, rs + i, v, A.epoch);
  }
  if (hl == 0 && av[nL] == 0.0) atomicMin(A.err, r);
  __syncwarp(hmask);
}

// Apply all pivots of row r with the whole warp.
JV_INLINE void warp_row(const FactorArgs& A, int r, int lane, WarpArena& W, const jv::Trace& T,
                        int bt) {
  [[maybe_unused]] long long wp_load = 0, wp_struct = 0, wp_gate = 0, wp_gather = 0, wp_elim = 0;
  HP_T0(wp_start);
  const unsigned full = 0xffffffffu;
  const int rs = A.row_start[r], re = A.row_start[r + 1];
  const int len = re - rs;
  const int dloc = A.diag[r] - rs;
  const int nL = dloc;
  const bool cached = len <= kWarpRow;
  const bool listed = A.heavy != nullptr && (A.heavy[r] == 1 || A.heavy[r] == 3);
  double* av = cached ? W.val : A.val + rs;
  const int* ac = cached ? W.col : A.col + rs;
  if (cached) {
    for (int i = lane; i < len; i += 32) {
      W.col[i] = A.col[rs + i];
      W.val[i] = __ldcs(A.val + rs + i);
    }
    __syncwarp();
  }
  const double thresh = A.tau > 0.0 ? jv::dmul(A.tau, A.norms[r]) : 0.0;
  HP_ADD(wp_load, wp_start);

  for (int k0 = 0; k0 < nL;) {
    HP_T0(t_struct);
    const int kc = min(32, nL - k0);
    int c = -1, d = 0, ce = 0;
    long long e1 = 0;
    if (lane < kc) {
      c = ac[k0 + lane];
      d = A.diag[c];
      if (listed) e1 = A.elim_ptr[rs + k0 + lane + 1];
      else ce = A.row_start[c + 1];
      W.pivc[lane] = c;
    }
    // ---- structure of the chunk: op list (q, target) per pivot
    int nops = 0, kdone = 0;
    bool direct = false;
    if (listed) {
      // precomputed (jv_elim_lists): the chunk's ops are one contiguous run
      // (a listed row has <= kWarpOps candidates in total)
      const long long E0 = A.elim_ptr[rs + k0];
      if (lane < kc) W.opend[lane] = (int)(e1 - E0);
      nops = (int)(__shfl_sync(full, e1, kc - 1) - E0);
      for (int o = lane; o < nops; o += 32) {
        const int2 op = __ldg(A.elim + E0 + o);
        W.opq[o] = op.x;
        W.opw[o] = op.y;
      }
      kdone = kc;
    }
    for (int kk = 0; kk < kc && !listed; ++kk) {
      const int k = k0 + kk;
      const int dk = __shfl_sync(full, d, kk), cek = __shfl_sync(full, ce, kk);
      const int ulen = cek - dk - 1, rem = len - k - 1;
      const int cand = A.milu ? ulen : min(ulen, rem);
      if (nops + cand > kWarpOps) {
        if (kk == 0) direct = true;   // a single pivot larger than the list
        break;
      }
      if (A.milu || ulen <= rem) {
        // lanes over U(c), each searched in the rest of this row
        for (int base = dk + 1; base < cek; base += 32) {
          const int q = base + lane;
          int w = -1;
          if (q < cek) {
            const int j = A.col[q];
            const int p = lower_bound(ac, k + 1, len, j);
            if (p < len && ac[p] == j) w = p;
            else if (A.milu) w = dloc | kOut;
          }
          const unsigned m = __ballot_sync(full, w >= 0);
          if (w >= 0) {
            const int pos = nops + __popc(m & ((1u << lane) - 1));
            W.opq[pos] = q;
            W.opw[pos] = w;
          }
          nops += __popc(m);
        }
      } else {
        // long pivot row: lanes over this row's rest, each searched in U(c)
        for (int base = k + 1; base < len; base += 32) {
          const int w = base + lane;
          int q = -1;
          if (w < len) {
            const int p = lower_bound(A.col, dk + 1, cek, ac[w]);
            if (p < cek && A.col[p] == ac[w]) q = p;
          }
          const unsigned m = __ballot_sync(full, q >= 0);
          if (q >= 0) {
            const int pos = nops + __popc(m & ((1u << lane) - 1));
            W.opq[pos] = q;
            W.opw[pos] = w;
          }
          nops += __popc(m);
        }
      }
      if (lane == 0) W.opend[kk] = nops;
      kdone = kk + 1;
    }
    __syncwarp();

    if (direct) {
      // one pivot whose updates exceed the op list: stream it in blocks of 32
      const int k = k0;
      const int dk = __shfl_sync(full, d, 0), cek = __shfl_sync(full, ce, 0);
      const int ck = __shfl_sync(full, c, 0);
      const double piv = warp_value(A, lane == 0, ck, dk);
      double l = 0.0;
      int drop = 0;
      if (lane == 0) {
        l = jv::ddiv(av[k], piv);
        drop = A.tau > 0.0 && fabs(l) < thresh;
        av[k] = drop ? 0.0 : l;
      }
      l = __shfl_sync(full, l, 0);
      drop = __shfl_sync(full, drop, 0);
      __syncwarp();
      const int ulen = cek - dk - 1, rem = len - k - 1;
      if (A.milu) {
        // diagonal contributions in q order: lane 0 folds each block in order
        for (int base = dk + 1; base < cek; base += 32) {
          const int q = base + lane;
          int w = dloc;
          if (q < cek && !drop) {
            const int j = A.col[q];
            const int p = lower_bound(ac, k + 1, len, j);
            if (p < len && ac[p] == j) w = p;
          }
          const double u = warp_value(A, q < cek, ck, q);
          const double prod = jv::dmul(l, u);
          for (int t = 0; t < 32 && base + t < cek; ++t) {
            const double pt = __shfl_sync(full, prod, t);
            const int wt = __shfl_sync(full, w, t);
            if (lane == 0) av[wt] = jv::dsub(av[wt], pt);
          }
          __syncwarp();
        }
      } else if (!drop) {
        if (ulen > rem) {
          for (int base = k + 1; base < len; base += 32) {
            const int w = base + lane;
            int p = -1;
            if (w < len) {
              const int pp = lower_bound(A.col, dk + 1, cek, ac[w]);
              if (pp < cek && A.col[pp] == ac[w]) p = pp;
            }
            const double u = warp_value(A, p >= 0, ck, p);
            if (p >= 0) av[w] = jv::dsub(av[w], jv::dmul(l, u));
          }
        } else {
          for (int base = dk + 1; base < cek; base += 32) {
            const int q = base + lane;
            int p = -1;
            if (q < cek) {
              const int j = A.col[q];
              const int pp = lower_bound(ac, k + 1, len, j);
              if (pp < len && ac[pp] == j) p = pp;
            }
            const double u = warp_value(A, p >= 0, ck, q);
            if (p >= 0) av[p] = jv::dsub(av[p], jv::dmul(l, u));
          }
        }
      }
      __syncwarp();
      k0 += 1;
      continue;
    }

    // ---- gate on the newest pivot of the chunk, then one converged gather
    HP_ADD(wp_struct, t_struct);
    HP_T0(t_gate);
    int g = (lane < kdone && c >= A.ready_below) ? c : -1, gq = d;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int og = __shfl_xor_sync(full, g, o), oq = __shfl_xor_sync(full, gq, o);
      if (og > g) { g = og; gq = oq; }
    }
    if (lane == 0 && g >= 0 && (jv::g_gate & 1)) jv::mbox_gate(A.mbox, gq, A.epoch);
    __syncwarp();
    HP_ADD(wp_gate, t_gate);
    HP_T0(t_gather);
    // every probe of the chunk (pivot diagonals + up to kWarpOps op values)
    // is issued before any is checked: one memory round trip, then
    // converged waits only for the packets that were not there yet
    constexpr int kSlots = kWarpOps / 32;
    double dv = 0.0;
    bool dmiss = false;
    {
      const bool have = lane < kdone;
      Probe pd{0, 0};
      if (have && c < A.ready_below) dv = __ldcg(A.val + d);
      else if (have) pd = probe_issue(A.mbox, d);
      Probe po[kSlots];
      int pk[kSlots];
#pragma unroll
      for (int i = 0; i < kSlots; ++i) {
        const int o = i * 32 + lane;
        pk[i] = 0;
        po[i] = Probe{0, 0};
        if (o < nops) {
          int ck = 0;
          if (A.ready_below > 0) {
            // pivot of op o: first kk with opend[kk] > o
            int lo = 0, hi = kdone - 1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (W.opend[mid] > o) hi = mid; else lo = mid + 1;
            }
            ck = W.pivc[lo];
          }
          pk[i] = ck;
          if (ck < A.ready_below) W.opv[o] = __ldcg(A.val + W.opq[o]);
          else po[i] = probe_issue(A.mbox, W.opq[o]);
        }
      }
      if (have && c >= A.ready_below) {
        if (probe_ok(pd, A.epoch)) dv = probe_val(pd);
        else dmiss = true;
      }
      unsigned omiss = 0;
#pragma unroll
      for (int i = 0; i < kSlots; ++i) {
        const int o = i * 32 + lane;
        if (o < nops && pk[i] >= A.ready_below) {
          if (probe_ok(po[i], A.epoch)) W.opv[o] = probe_val(po[i]);
          else omiss |= 1u << i;
        }
      }
      if (__any_sync(full, dmiss)) {
        const double v = warp_value(A, dmiss, c, d);
        if (dmiss) dv = v;
      }
      if (__any_sync(full, omiss != 0)) {
        for (int i = 0; i < kSlots; ++i) {
          const bool m = (omiss >> i) & 1;
          const int o = i * 32 + lane;
          const double v = warp_value(A, m, pk[i], m ? W.opq[o] : 0);
          if (m) W.opv[o] = v;
        }
      }
    }
    __syncwarp();
    HP_ADD(wp_gather, t_gather);
    HP_T0(t_elim);

    // ---- elimination, pivot by pivot
    for (int kk = 0, o0 = 0; kk < kdone; ++kk) {
      const int k = k0 + kk;
      const int o1 = W.opend[kk];
      const double dk = __shfl_sync(full, dv, kk);
      double l = 0.0;
      int drop = 0;
      if (lane == 0) {
        bool slow;
        const double a = av[k];
        l = jv::ddiv_fast(a, dk, slow);
        if (slow) l = __ddiv_rn(a, dk);
        drop = A.tau > 0.0 && fabs(l) < thresh;
        av[k] = drop ? 0.0 : l;
      }
      l = __shfl_sync(full, l, 0);
      drop = __shfl_sync(full, drop, 0);
      if (A.milu) {
        // the diagonal accumulates in q order: one lane
        if (lane == 0)
          for (int o = o0; o < o1; ++o) {
            const int t = (drop || (W.opw[o] & kOut)) ? dloc : W.opw[o];
            av[t] = jv::dsub(av[t], jv::dmul(l, W.opv[o]));
          }
      } else if (!drop) {
        for (int o = o0 + lane; o < o1; o += 32) {
          const int t = W.opw[o];
          av[t] = jv::dsub(av[t], jv::dmul(l, W.opv[o]));
        }
      }
      o0 = o1;
      __syncwarp();
    }
    HP_ADD(wp_elim, t_elim);
    k0 += kdone;
  }

  // ---- publish
  for (int i = lane; i < len; i += 32) {
    const double v = av[i];
    if (cached) __stcg(A.val + rs + i, v);
    if (i >= nL) jv::mbox_put(A.mbox, rs + i, v, A.epoch);
  }
  if (lane == 0 && av[dloc] == 0.0) atomicMin(A.err, r);
  __syncwarp();
#ifdef JV_HEAVY_PROFILE
  if (lane == 0) {
    jv::trace_word(T, bt, 7, ((unsigned long long)wp_load << 32) | (unsigned)wp_struct);
    jv::trace_word(T, bt, 13, wp_gate);
    jv::trace_word(T, bt, 14, ((unsigned long long)wp_gather << 32) | (unsigned)wp_elim);
    jv::trace_word(T, bt, 15, clock64() - wp_start);
  }
#else
  (void)T; (void)bt;
#endif
}

// Heavy rows (power-law hubs: thousands of pivots whose U rows hold
// thousands of entries) use the elimination list built once per pattern by
// jv_elim_lists — the structural matches (q, w) of every pivot, in ascending
// column order — so the numeric pass does no searching.  The row is then a
// chain of nL steps (one division, a parallel scatter of the pivot's
// updates); everything that does not depend on the chain is streamed ahead:
//  * the op pairs and the mailbox packets of the pivots' U entries flow
//    through a 512-entry per-warp ring in shared memory (the warp's idle
//    thread-path slices), filled by cp.async five windows (64 ops each)
//    ahead for the ops and three ahead for the packets;
//  * the row's values live in a CTA-wide shared buffer (one heavy row per
//    CTA at a time, try-lock; rows that do not fit or find it taken stay in
//    HBM), so the per-step read-modify-writes are shared-memory latency.
constexpr int kRing = 512;          // ops per warp ring
constexpr int kWin = 64;            // ops per window (2 per lane)
// row entries in the CTA heavy buffer: what the slices leave of the SM's
// shared memory (two halves)
constexpr int kHeavyCap =
    (int)(((232448 - 1024 - (size_t)kThreads * (kSlotsI * 4 + kSlotsD * 8)) / sizeof(double)) & ~63);
constexpr size_t kSliceBytes = (size_t)kThreads * (kSlotsI * 4 + kSlotsD * 8);
static_assert(kSlotsI * 32 >= 2 * kRing && kSlotsD * 32 >= 2 * kRing, "ring must fit the slices");

JV_INLINE unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
JV_INLINE void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
JV_INLINE void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
JV_INLINE void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
JV_INLINE void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
JV_INLINE void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct Ring {
  int2* ops;        // kRing (q, w) pairs
  uint64_t* pkts;   // kRing mailbox packets (2 words each)
  JV_INLINE int2* op(int e) const { return ops + (e & (kRing - 1)); }
  JV_INLINE uint64_t* pkt(int e) const { return pkts + 2 * (e & (kRing - 1)); }
};

struct HeavyStream {
  const int2* elim;
  const uint64_t* mbox;
  Ring R;
  long long O0;   // first op of the row
  int nops;       // ops of the row
  int lane;
  // window i: this lane's entries i*kWin + lane + {0, 32}
  JV_INLINE void issue_ops(int i) const {
#pragma unroll
    for (int h = 0; h < kWin; h += 32) {
      const int e = i * kWin + h + lane;
      if (e < nops) cp_async8(R.op(e), elim + O0 + e);
    }
    cp_commit();
  }
  JV_INLINE void issue_pkts(int i) const {
#pragma unroll
    for (int h = 0; h < kWin; h += 32) {
      const int e = i * kWin + h + lane;
      if (e < nops) cp_async16(R.pkt(e), mbox + 2 * (long long)(R.op(e)->x & 0x7fffffff));
    }
    cp_commit();
  }
  JV_INLINE void prologue() const {
    for (int i = 0; i < 5; ++i) issue_ops(i);
    cp_wait<0>();
    for (int i = 0; i < 3; ++i) issue_pkts(i);
    cp_wait<0>();
    __syncwarp();
  }
  // entering window i: its packets landed; windows i+5 (ops) / i+3 (packets) go out
  JV_INLINE void advance(int i) const {
    cp_wait<4>();
    __syncwarp();
    issue_ops(i + 5);
    cp_wait<4>();
    issue_pkts(i + 3);
  }
};

// u value of ring entry e (pivot row c); false when its packet is stale
JV_INLINE bool ring_value(const FactorArgs& A, const Ring& R, int e, int c, double& u) {
  if (c < A.ready_below) {
    u = __ldcg(A.val + R.op(e)->x);
    return true;
  }
  const uint64_t* pk = R.pkt(e);
  const Probe p{pk[0], pk[1]};
  if (!probe_ok(p, A.epoch)) return false;
  u = probe_val(p);
  return true;
}

constexpr int kGroup = 4;   // ops per lane per step (128 per warp)

JV_INLINE void heavy_row(const FactorArgs& A, int r, int lane, int* heavy_busy, double* hbuf,
                         const jv::Trace& T, int bt) {
  [[maybe_unused]] long long hp_adv = 0, hp_miss = 0, hp_div = 0, hp_piv = 0;
  HP_T0(hp_start);
  const unsigned full = 0xffffffffu;
  const int rs = A.row_start[r], re = A.row_start[r + 1];
  const int len = re - rs;
  const int nL = A.diag[r] - rs;
  const double thresh = A.tau > 0.0 ? jv::dmul(A.tau, A.norms[r]) : 0.0;
  const int wi = threadIdx.x >> 5;

  // row values: a slot of the CTA buffer (two halves; a long row takes both)
  int bits = 0;
  if (lane == 0 && len <= kHeavyCap) {
    for (int tries = 0; tries < 4 && !bits; ++tries) {
      const int st = *reinterpret_cast<volatile int*>(heavy_busy);
      int want = 0;
      if (len > kHeavyCap / 2) want = st == 0 ? 3 : 0;
      else if (!(st & 1)) want = 1;
      else if (!(st & 2)) want = 2;
      if (!want) break;
      if (atomicCAS(heavy_busy, st, st | want) == st) bits = want;
    }
  }
  bits = __shfl_sync(full, bits, 0);
  double* av = A.val + rs;
  if (bits) {
    av = hbuf + (bits == 2 ? kHeavyCap / 2 : 0);
    for (int i = lane; i < len; i += 32) av[i] = __ldcg(A.val + rs + i);
    __syncwarp();
  }

  HeavyStream H;
  H.elim = A.elim;
  H.mbox = A.mbox;
  H.R.ops = reinterpret_cast<int2*>(slice_ints(wi));
  H.R.pkts = reinterpret_cast<uint64_t*>(slice_doubles(wi));
  H.O0 = A.elim_ptr[rs];
  H.nops = (int)(A.elim_ptr[rs + nL] - H.O0);
  H.lane = lane;
  H.prologue();
  int cur = 0;
  H.advance(0);
  HP_ADD(hp_adv, hp_start);

  for (int k0 = 0; k0 < nL; k0 += 32) {
    const int kc = min(32, nL - k0);
    int c = 0, d = 0, e1 = 0;
    double dval = 0.0;
    int dready = 0;
    if (lane < kc) {
      c = A.col[rs + k0 + lane];
      d = A.diag[c];
      e1 = (int)(A.elim_ptr[rs + k0 + lane + 1] - H.O0);
      if (c < A.ready_below) {
        dval = __ldcg(A.val + d);
        dready = 1;
      } else {
        const Probe p = probe_issue(A.mbox, d);
        if (probe_ok(p, A.epoch)) { dval = probe_val(p); dready = 1; }
      }
    }
    int e0 = (int)(A.elim_ptr[rs + k0] - H.O0);
    for (int kk = 0; kk < kc; ++kk) {
      const int k = k0 + kk;
      const int ck = __shfl_sync(full, c, kk);
      const int r1 = __shfl_sync(full, e1, kk);
      const int r0 = e0;
      e0 = r1;
      double piv = __shfl_sync(full, dval, kk);
      HP_T0(t_piv);
      if (!__shfl_sync(full, dready, kk))
        piv = __shfl_sync(full, warp_value(A, lane == 0, ck, __shfl_sync(full, d, kk)), 0);
      HP_ADD(hp_piv, t_piv);

      if (A.milu) {
        // MILU: the diagonal accumulates in op order — lane 0 folds each
        // block of 32 in order (correctness path; no power-law MILU config)
        double l = 0.0;
        int drop = 0;
        if (lane == 0) {
          l = jv::ddiv(av[k], piv);
          drop = A.tau > 0.0 && fabs(l) < thresh;
          av[k] = drop ? 0.0 : l;
        }
        l = __shfl_sync(full, l, 0);
        drop = __shfl_sync(full, drop, 0);
        for (int b = r0; b < r1; b += 32) {
          const int need = (min(b + 32, r1) - 1) / kWin;
          while (cur < need) H.advance(++cur);
          const int e = b + lane;
          double u = 0.0;
          int w = 0;
          bool miss = false;
          if (e < r1) {
            w = H.R.op(e)->y;
            miss = !ring_value(A, H.R, e, ck, u);
          }
          if (__any_sync(full, miss)) {
            const double v = warp_value(A, miss, ck, miss ? H.R.op(e)->x : 0);
            if (miss) u = v;
          }
          const double prod = jv::dmul(l, u);
          const int wt0 = (drop || (w & kOut)) ? nL : w;
          for (int t = 0; t < 32 && b + t < r1; ++t) {
            const double pt = __shfl_sync(full, prod, t);
            const int wt = __shfl_sync(full, wt0, t);
            if (lane == 0) av[wt] = jv::dsub(av[wt], pt);
          }
        }
        __syncwarp();
        continue;
      }

      // groups of up to 32 * kGroup ops: the loads of a group (op, packet,
      // target value) are issued together, before the division they do not
      // depend on; every lane computes l itself (no broadcast)
      HP_T0(t_div);
      const bool direct = ck < A.ready_below;
      double l = 0.0;
      bool drop = false;
      for (int g0 = r0;; g0 += 32 * kGroup) {
        const int gend = min(g0 + 32 * kGroup, r1);
        if (g0 < gend) {
          HP_T0(t_adv);
          const int need = (gend - 1) / kWin;
          while (cur < need) H.advance(++cur);
          HP_ADD(hp_adv, t_adv);
        }
        int w[kGroup];
        double u[kGroup], tv[kGroup];
        unsigned missm = 0;
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
          const int e = g0 + 32 * j + lane;
          w[j] = -1;
          u[j] = 0.0;
          tv[j] = 0.0;
          if (e < gend) {
            const int2 op = *H.R.op(e);
            w[j] = op.y;
            if (direct) {
              u[j] = __ldcg(A.val + op.x);
            } else {
              const ulonglong2 pk = *reinterpret_cast<const ulonglong2*>(H.R.pkt(e));
              u[j] = __longlong_as_double((long long)((pk.x & 0xffffffffull) | (pk.y << 32)));
              if ((uint32_t)(pk.x >> 32) != A.epoch || (uint32_t)(pk.y >> 32) != A.epoch)
                missm |= 1u << j;
            }
            tv[j] = av[op.y];
          }
        }
        if (g0 == r0) {
          const double a = av[k];
          bool slow;
          l = jv::ddiv_fast(a, piv, slow);
          if (slow) l = __ddiv_rn(a, piv);
          drop = A.tau > 0.0 && fabs(l) < thresh;
          if (lane == 0) av[k] = drop ? 0.0 : l;
          HP_ADD(hp_div, t_div);
        }
        if (g0 >= gend || drop) break;
        if (__any_sync(full, missm != 0)) {
          HP_T0(t_miss);
#pragma unroll
          for (int j = 0; j < kGroup; ++j) {
            const int e = g0 + 32 * j + lane;
            const bool m = (missm >> j) & 1;
            const double v = warp_value(A, m, ck, m ? H.R.op(e)->x : 0);
            if (m) u[j] = v;
          }
          HP_ADD(hp_miss, t_miss);
        }
#pragma unroll
        for (int j = 0; j < kGroup; ++j)
          if (w[j] >= 0) av[w[j]] = jv::dsub(tv[j], jv::dmul(l, u[j]));
        if (gend >= r1) break;
      }
      __syncwarp();
    }
  }
  cp_wait<0>();
  __syncwarp();
  // ---- publish
  for (int i = lane; i < len; i += 32) {
    const double v = av[i];
    if (bits) __stcg(A.val + rs + i, v);
    if (i >= nL) jv::mbox_put(A.mbox, rs + i, v, A.epoch);
  }
  if (lane == 0 && av[nL] == 0.0) atomicMin(A.err, r);
  __syncwarp();
  if (bits && lane == 0) atomicAnd(heavy_busy, ~bits);
  __syncwarp();
#ifdef JV_HEAVY_PROFILE
  if (lane == 0) {
    // words 7, 13-15 (the batch marks use 0-6 and 8-12)
    jv::trace_word(T, bt, 7, ((unsigned long long)hp_piv << 1) | (bits != 0));
    jv::trace_word(T, bt, 13, hp_adv);
    jv::trace_word(T, bt, 14, hp_miss);
    jv::trace_word(T, bt, 15, ((unsigned long long)hp_div << 32) | (unsigned)(clock64() - hp_start));
  }
#else
  (void)T; (void)bt; (void)hp_adv; (void)hp_miss; (void)hp_div; (void)hp_piv;
#endif
}

// Hub rows with a gather plan (flag 4, jv_hub_plan_host): instead of the
// pivot-by-pivot walk, positions are folded in parallel — phase by phase
// (in-row dependency depth), each lane running its queue of (position,
// update run) items from a step-major stream that the same cp.async ring
// prefetches (update entries and their mailbox packets alike).  Bitwise
// equal to the pivot order: every position still receives its updates in
// ascending pivot order (tests/test_hubplan.py replays plans on the CPU).
// Needs the CTA row buffer; returns false (caller falls back to heavy_row)
// when the buffer is taken or the row does not fit.
JV_INLINE bool hub_row(const FactorArgs& A, int r, int lane, int* heavy_busy, double* hbuf,
                       const jv::Trace& T, int bt) {
  [[maybe_unused]] long long hp_adv = 0, hp_miss = 0, hp_divb = 0, hp_steps = 0;
  HP_T0(hp_start);
  const unsigned full = 0xffffffffu;
  const int rs = A.row_start[r], re = A.row_start[r + 1];
  const int len = re - rs;
  const int nL = A.diag[r] - rs;
  int bits = 0;
  if (lane == 0 && len <= kHeavyCap) {
    for (int tries = 0; tries < 4 && !bits; ++tries) {
      const int st = *reinterpret_cast<volatile int*>(heavy_busy);
      int want = 0;
      if (len > kHeavyCap / 2) want = st == 0 ? 3 : 0;
      else if (!(st & 1)) want = 1;
      else if (!(st & 2)) want = 2;
      if (!want) break;
      if (atomicCAS(heavy_busy, st, st | want) == st) bits = want;
    }
  }
  bits = __shfl_sync(full, bits, 0);
  if (!bits) return false;
  double* av = hbuf + (bits == 2 ? kHeavyCap / 2 : 0);
  for (int i = lane; i < len; i += 32) av[i] = __ldcg(A.val + rs + i);

  const long long s0 = A.hub_sptr[r];
  const int32_t* meta = A.hub_meta + A.hub_mptr[r];
  const int nph = meta[0];
  HeavyStream H;
  H.elim = A.hub_stream;
  H.mbox = A.mbox;
  H.R.ops = reinterpret_cast<int2*>(slice_ints(threadIdx.x >> 5));
  H.R.pkts = reinterpret_cast<uint64_t*>(slice_doubles(threadIdx.x >> 5));
  H.O0 = s0;
  H.lane = lane;
  // entries of the row: every phase's lane loads plus its divisions
  {
    long long tot = 0;
    for (int p = 0; p < nph; ++p) tot += meta[1 + 33 * p + lane] + (lane == 0 ? meta[33 * p + 33] : 0);
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(full, tot, o);
    H.nops = (int)tot;
  }
  __syncwarp();
  H.prologue();
  int cur = 0;
  H.advance(0);

  int qnext = nph > 0 ? meta[1 + lane] : 0;
  int fnext = nph > 0 ? meta[33] : 0;
  int base = 0;
  for (int p = 0; p < nph; ++p) {
    const int qlen = qnext, nfin = fnext;
    if (p + 1 < nph) {
      qnext = meta[1 + 33 * (p + 1) + lane];
      fnext = meta[33 * (p + 1) + 33];
    }
    const int maxq = __shfl_sync(full, qlen, 0);
    // ---- update block: runs of independent positions, one fold per lane,
    // four steps per round (their loads are independent: only the folds
    // chain), so a single warp keeps several shared-memory loads in flight
    int cw = -1;
    double acc = 0.0;
    constexpr int kU4 = 4;
    for (int t0 = 0; t0 < maxq; t0 += kU4) {
      int a[kU4], e[kU4];
      int tot = 0;
#pragma unroll
      for (int i = 0; i < kU4; ++i) {
        const bool act = t0 + i < qlen;
        a[i] = __popc(__ballot_sync(full, t0 + i < maxq ? act : false));
        e[i] = act ? base + tot + lane : -1;
        tot += a[i];
      }
      HP_T0(t_adv);
      if (tot > 0) {
        const int need = (base + tot - 1) / kWin;
        while (cur < need) H.advance(++cur);
      }
      HP_ADD(hp_adv, t_adv);
#ifdef JV_HEAVY_PROFILE
      hp_steps += kU4;
#endif
      int2 op[kU4];
      double u[kU4], lj[kU4];
      unsigned missm = 0;
#pragma unroll
      for (int i = 0; i < kU4; ++i) {
        op[i] = make_int2(0, 0);
        u[i] = 0.0;
        if (e[i] >= 0) {
          op[i] = *H.R.op(e[i]);
          const ulonglong2 pk = *reinterpret_cast<const ulonglong2*>(H.R.pkt(e[i]));
          u[i] = __longlong_as_double((long long)((pk.x & 0xffffffffull) | (pk.y << 32)));
          if ((uint32_t)(pk.x >> 32) != A.epoch || (uint32_t)(pk.y >> 32) != A.epoch)
            missm |= 1u << i;
        }
      }
#pragma unroll
      for (int i = 0; i < kU4; ++i) lj[i] = e[i] >= 0 ? av[op[i].y & 0xffff] : 0.0;
      if (__any_sync(full, missm != 0)) {
        HP_T0(t_miss);
        for (int i = 0; i < kU4; ++i) {
          const bool m = (missm >> i) & 1;
          const double v = warp_value(A, m, 0, op[i].x);
          if (m) u[i] = v;
        }
        HP_ADD(hp_miss, t_miss);
      }
#pragma unroll
      for (int i = 0; i < kU4; ++i) {
        if (e[i] >= 0) {
          const int w = (int)((unsigned)op[i].y >> 16);
          if (w != cw) {
            if (cw >= 0) av[cw] = acc;
            cw = w;
            acc = av[w];
          }
          acc = jv::dsub(acc, jv::dmul(lj[i], u[i]));
        }
      }
      base += tot;
    }
    if (cw >= 0) av[cw] = acc;
    __syncwarp();
    // ---- division block: the L positions of this depth
    HP_T0(t_divb);
    for (int f0 = 0; f0 < nfin; f0 += 32) {
      const int a = min(32, nfin - f0);
      const int need = (base + a - 1) / kWin;
      while (cur < need) H.advance(++cur);
      int w = 0, x = 0;
      double d = 1.0;
      bool miss = false;
      if (lane < a) {
        const int e = base + lane;
        const int2 op = *H.R.op(e);
        x = op.x & 0x7fffffff;
        w = (int)((unsigned)op.y >> 16);
        const ulonglong2 pk = *reinterpret_cast<const ulonglong2*>(H.R.pkt(e));
        d = __longlong_as_double((long long)((pk.x & 0xffffffffull) | (pk.y << 32)));
        miss = (uint32_t)(pk.x >> 32) != A.epoch || (uint32_t)(pk.y >> 32) != A.epoch;
      }
      if (__any_sync(full, miss)) {
        const double v = warp_value(A, miss, 0, x);
        if (miss) d = v;
      }
      if (lane < a) {
        const double num = av[w];
        bool slow;
        double l = jv::ddiv_fast(num, d, slow);
        if (slow) l = __ddiv_rn(num, d);
        av[w] = l;
      }
      base += a;
    }
    HP_ADD(hp_divb, t_divb);
    __syncwarp();
  }
  cp_wait<0>();
  __syncwarp();
  for (int i = lane; i < len; i += 32) {
    const double v = av[i];
    __stcg(A.val + rs + i, v);
    if (i >= nL) jv::mbox_put(A.mbox, rs + i, v, A.epoch);
  }
  if (lane == 0 && av[nL] == 0.0) atomicMin(A.err, r);
  __syncwarp();
  if (lane == 0) atomicAnd(heavy_busy, ~bits);
  __syncwarp();
#ifdef JV_HEAVY_PROFILE
  if (lane == 0) {
    jv::trace_word(T, bt, 7, ((unsigned long long)hp_steps << 1) | 1);
    jv::trace_word(T, bt, 13, hp_adv);
    jv::trace_word(T, bt, 14, hp_miss);
    jv::trace_word(T, bt, 15, ((unsigned long long)hp_divb << 32) | (unsigned)(clock64() - hp_start));
  }
#else
  (void)T; (void)bt;
#endif
  return true;
}

constexpr size_t kFactorSmem = kArenaBytes + kSliceBytes + sizeof(double) * kHeavyCap;
static_assert(kFactorSmem <= 232448 - 64, "factor kernel shared memory");

static_assert(2 * sizeof(HalfArena) <= 32 * kSlotsD * sizeof(double), "pair arenas must fit a slice block");

__global__ void __launch_bounds__(kThreads, 1) factor_kernel(FactorArgs A) {

  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  WarpArena& W = *reinterpret_cast<WarpArena*>(slice_doubles(threadIdx.x >> 5));
  const Slice S{(int)threadIdx.x};
  const jv::Trace T = jv::trace_begin();
  const int nw = (gridDim.x * blockDim.x) >> 5;
  __shared__ int heavy_busy;
  double* hbuf = reinterpret_cast<double*>(jv_factor_smem + kArenaBytes + kSliceBytes);
  if (threadIdx.x == 0) heavy_busy = 0;
  __syncthreads();
  for (;;) {
    const int b = jv::ticket_next(A.ticket, lane, T);
    if (b >= A.nbatch) break;
    const int lo = A.batch_ptr[b], hi = A.batch_ptr[b + 1];
    const int idx = lo + lane;
    const bool active = idx < hi;
    const int r = active ? A.order[idx] : -1;
    // batch class from the schedule (loaded alongside batch_ptr)
    const int bcls = A.bclass != nullptr ? A.bclass[b] : -1;
    SfpRow F;
    if (lane == 0) jv::trace_mark(T, b, 1);
    // row flags (jv_elim_lists): 0 thread path, 1 pairable listed warp row,
    // 2 heavy, 3 listed warp row
    const int flag = (bcls != 0 && A.heavy != nullptr && active) ? A.heavy[r] : 0;
    if (bcls == 1 && hi - lo == 2 && __shfl_sync(full, flag, 0) == 1 &&
        __shfl_sync(full, flag, 1) == 1) {
      const int half = lane >> 4;
      const unsigned hmask = 0xffffu << (16 * half);
      HalfArena* HA = reinterpret_cast<HalfArena*>(slice_doubles(threadIdx.x >> 5));
      pair_row(A, __shfl_sync(full, r, half), lane & 15, hmask, HA[half]);
      __syncwarp();
      if (lane == 0) jv::trace_mark(T, b, 4);
      continue;
    }
    ShortRow R;
    bool sfp = false, fits = false;
    if (active && flag == 0) {
      sfp = sfp_structure(A, r, F);
      if (!sfp) fits = short_structure(A, r, R, S);
    }
    __syncwarp();
    if (lane == 0) jv::trace_mark(T, b, 2);
    // warp gate on the newest pivot of the batch's thread-path rows
    int g = sfp ? F.gate : (fits ? R.gate : -1);
    int gq = sfp ? F.gate_q : (fits ? R.gate_q : 0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int og = __shfl_xor_sync(full, g, o), oq = __shfl_xor_sync(full, gq, o);
      if (og > g) { g = og; gq = oq; }
    }
    if (lane == 0 && g >= 0 && (jv::g_gate & 1)) jv::mbox_gate(A.mbox, gq, A.epoch);
    __syncwarp();
    if (lane == 0) jv::trace_mark(T, b, 3);
    const unsigned smask = __ballot_sync(full, sfp);
    if (sfp) {
      // lanes complete in groups of g_sfp_group (32: the whole warp waits
      // for its slowest row; smaller groups finish independently)
      const unsigned gs = jv::g_sfp_group;
      const unsigned gmask = gs >= 32 ? 0xffffffffu : (((1u << gs) - 1) << (lane & ~(gs - 1)));
      sfp_finish(A, r, F, smask & gmask, b, T);
    }
    const unsigned fmask = __ballot_sync(full, fits);
    if (fits) short_finish(A, r, R, S, fmask, b, T);
    unsigned pend = __ballot_sync(full, active && !fits && !sfp);
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1;
      const int rr = __shfl_sync(full, r, src);
      const int fl = A.heavy != nullptr ? A.heavy[rr] : 0;
      if (fl == 4 && A.ready_below == 0 && !A.milu && A.tau == 0.0 &&
          hub_row(A, rr, lane, &heavy_busy, hbuf, T, b)) {
      } else if (fl == 2 || fl == 4) heavy_row(A, rr, lane, &heavy_busy, hbuf, T, b);
      else warp_row(A, rr, lane, W, T, b);
    }
    __syncwarp();
    if (lane == 0) jv::trace_mark(T, b, 4);
  }
  jv::ticket_exit(A.ticket, lane, nw);
}

// row classes for the schedule: 0 = thread path, 1 = warp path
__global__ void classify_factor_kernel(int n, const int32_t* rs, const int32_t* diag, int milu,
                                       int32_t* cls) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int len = rs[r + 1] - rs[r];
    const int nL = diag[r] - rs[r];
    cls[r] = (!milu && len <= kR && nL <= kP) ? 0 : 1;
  }
}

__global__ void classify_factor_pivots_kernel(int n, const int32_t* rs, const int32_t* col,
                                              const int32_t* diag, int32_t* cls) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (cls[r]) continue;
    const int nL = diag[r] - rs[r];
    for (int k = 0; k < nL; ++k) {
      const int c = col[rs[r] + k];
      if (rs[c + 1] - diag[c] - 1 > kU) { cls[r] = 1; break; }
    }
  }
}

}  // namespace

extern "C" int jv_factor(int32_t n, const int32_t* row_start, const int32_t* col, double* val,
                         const int32_t* diag_pos, const double* norms, double tau, int milu,
                         const int32_t* order, const int32_t* batch_ptr, int32_t nbatch,
                         int32_t ready_below, uint64_t* mbox, uint32_t epoch, int32_t* err_row,
                         int32_t* ticket, const int8_t* heavy, const int64_t* elim_ptr,
                         const int32_t* elim, const int8_t* batch_class,
                         const int32_t* hub_stream, const int64_t* hub_sptr,
                         const int32_t* hub_meta, const int64_t* hub_mptr, void* stream) {
  if (n < 0 || nbatch < 0 || epoch == 0) {
    jvh::set_error("jv_factor: bad argument (n=%d nbatch=%d epoch=%u)", n, nbatch, epoch);
    return JV_EINVAL;
  }
  if (n == 0 || nbatch == 0) return JV_OK;
  FactorArgs A{row_start, col, val, diag_pos, norms, tau, milu, order, batch_ptr,
               nbatch, ready_below, mbox, epoch, err_row, ticket,
               elim != nullptr ? heavy : nullptr, elim_ptr, reinterpret_cast<const int2*>(elim),
               batch_class, reinterpret_cast<const int2*>(hub_stream), hub_sptr, hub_meta,
               hub_mptr};
  void* args[] = {&A};
  return jvh::persistent_launch(factor_kernel, kThreads, args, (cudaStream_t)stream, "jv_factor",
                                kFactorSmem);
}

extern "C" int jv_classify_factor(int32_t n, const int32_t* row_start, const int32_t* col,
                                  const int32_t* diag_pos, int milu, int32_t* cls, void* stream) {
  if (n <= 0) return JV_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = (n + 255) / 256;
  classify_factor_kernel<<<grid, 256, 0, s>>>(n, row_start, diag_pos, milu, cls);
  classify_factor_pivots_kernel<<<grid, 256, 0, s>>>(n, row_start, col, diag_pos, cls);
  JV_CHECK_LAUNCH("jv_classify_factor");
  return JV_OK;
}
