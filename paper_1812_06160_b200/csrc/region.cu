// CTA-resident region kernels (sm_100a): factorization of stencil-class
// matrices and forward / backward triangular solves of any matrix whose rows
// have <= 32 dependencies.
//
// The sync-free ticket kernels (factor.cu, solve.cu) pay a mailbox hop —
// an L2 round trip plus a warp's scheduling — on every level of the DAG
// (config 2: 382 levels, ~2 us each).  Here one co-resident CTA per region
// (an acyclic box-like partition found from the pattern, regions_host.cpp)
// walks its rows level by level:
//   * a dependency inside the region is read from shared memory (its value,
//     written by this CTA at an earlier wave; one __syncthreads per wave);
//   * a dependency in another region comes from the 16-byte mailbox
//     (common.cuh) — its packet is prefetched with the wave's values and
//     re-probed (warp-converged) only if it was not yet published;
//   * a row that another region reads publishes its value to the mailbox.
// The quotient graph of the regions is acyclic, so a region lags its
// upstream neighbours by about one hop and then runs at barrier speed.
//
// Data movement: every wave is a precomputed 16-byte aligned block of
// records (row, value positions, dependency slots) in HBM.  One thread
// bulk-copies (TMA, cp.async.bulk + mbarrier complete_tx) the block S waves
// ahead into a shared-memory ring; D waves ahead every thread gathers its
// row's values (matrix entries, right-hand side, mailbox packets) with
// cp.async into a second ring, so the DRAM latency of both dependent rounds
// overlaps the barrier-separated compute.  Ring offsets come from the plan.
//
// Arithmetic (explicitly rounded binary64, bitwise equal to the reference):
//   factor   (_kernels.py:165-204, stencil class): l_k = a_k / u_kk,
//            tau drop against tau * norm_r, u_rr = a_rr - sum_k l_k u_kr in
//            ascending k;
//   forward  (_kernels.py:348-357): y_r = b_r - sum_{c<r} l_rc y_c ascending;
//   backward (_kernels.py:360-366): x_r = (y_r - sum_{c>r} u_rc x_c) / u_rr.
//
// Deadlock freedom: each CTA processes its waves in level order and only
// waits on rows of lower levels; all CTAs are co-resident (cooperative
// launch), so the lowest pending level always progresses.
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "../../include/jv.h"

namespace jvr {

constexpr int kThreads = 512;   // rows per wave (compute threads)
constexpr int kNB = 16;   // static-block mbarriers in the ring (S + 1 <= kNB)
constexpr int kTab = 1;   // int4 entries per wave in the shared-memory table
constexpr int kL2 = 12;   // waves of L2 bulk prefetch ahead of the gathers (24 measured equal)

struct RArgs {
  const int4* words;   // static stream, 16-byte units
  const int4* table;   // 2 per wave: {block (16 B units), bytes, ring off, dyn off},
                       // {packed values (16 B units), bytes, 0, 0}
  const int32_t* reg_wave;
  int32_t SC, max_waves, S, D, CS, CD;   // SC: slot ring (power of 2)
  double* val;
  const double* pack;   // matrix values packed in wave order (jv_pack_values)
  const double* vpack;  // per-call vector packed in wave order
  double* out;
  const double* norms;
  double tau;
  uint64_t* mbox;
  uint32_t epoch;
  int32_t* err;
};

JV_INLINE uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

JV_INLINE void bar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
JV_INLINE void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes)
               : "memory");
}
JV_INLINE void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}
JV_INLINE void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "RW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra RW_%=;\n}" ::"r"(sa(b)), "r"(parity) : "memory");
}
// wave block view (regions_host.cpp): header, 32-byte row records
// {ref0..ref3, p0, row, meta, me}, xref[K - 4][cnt], pslot[NP]; refs and
// `me` are byte offsets into the CTA's shared memory
struct Wave {
  const int32_t* b;
  int cnt, slot0, K, NP;
  JV_INLINE Wave(const unsigned char* p) : b(reinterpret_cast<const int32_t*>(p)) {
    const int4 h = *reinterpret_cast<const int4*>(p);
    cnt = h.x;
    slot0 = h.y;
    K = h.z;
    NP = h.w;
  }
  JV_INLINE const int4* rec(int i) const { return reinterpret_cast<const int4*>(b + 4) + 2 * i; }
  JV_INLINE const int32_t* xref() const { return b + 4 + 8 * cnt; }
  JV_INLINE int pslot(int j) const { return b[4 + (8 + max(K - 4, 0)) * cnt + j]; }
};
#ifndef JV_RDIAG
#define JV_RDIAG 0   // diagnostic builds strip parts of the compute loop (wrong results)
#endif
constexpr int kOneOff = 144;   // shared-memory offset of the constant 1.0
constexpr int kCompute = 512;
// prober warps (warp p owns the waves w with w % P == p): 8, or 4 beside 512 compute threads
__host__ __device__ constexpr int probers_for(int nc) { return nc >= 512 ? 4 : 8; }
// threads beside the compute warps: a producer warp (one lane), a waiter warp, the prober warps
__host__ __device__ constexpr int extra_for(int nc) { return 64 + 32 * probers_for(nc); }
constexpr int kWin = 4;                 // prober window (waves; 16 and 2 measured slower on c2)

JV_INLINE void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(dst)), "l"(src) : "memory");
}
JV_INLINE bool bar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(sa(b)), "r"(parity) : "memory");
  return ok != 0;
}

JV_INLINE void l2_prefetch_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
JV_INLINE int ld_acquire_shared(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(sa(p)) : "memory");
  return v;
}
JV_INLINE int ld_volatile_shared(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(sa(p)) : "memory");
  return v;
}

// Warp-specialised CTA: warps 0..15 compute (one row per thread, a named
// barrier per wave); one lane of warp 16 produces.  Per wave the producer
// issues three bulk copies (TMA, cp.async.bulk + mbarrier complete_tx): the
// static block, the packed matrix values and the packed per-call vector,
// all addressed from the wave table alone, up to D waves ahead of the
// compute warps (whose progress it reads from a shared counter before
// reusing ring space), with L2 bulk prefetches kL2 waves further ahead.
template <int KIND, int NC, int KR, bool TAU>
__global__ void __launch_bounds__(NC + extra_for(NC), 1) region_kernel(RArgs A) {
  constexpr int kCompute = NC;
  constexpr int kProbers = probers_for(NC);   // compute threads: waves of at most NC rows
  extern __shared__ __align__(128) unsigned char rsm[];
  const unsigned full = 0xffffffffu;
  const int tid = threadIdx.x;
  uint64_t* bar = reinterpret_cast<uint64_t*>(rsm);            // wave full [kNB]
  int* done = reinterpret_cast<int*>(rsm + 8 * kNB);          // waves finished
  int* issued = done + 2;   // waves whose blocks the producer has issued
  int* probed = done + 8;   // [kProbers] per prober warp: its waves below this are released
  // per wave {static ring offset, dynamic ring offset, value bytes | vector
  // bytes << 18, rows | K << 10 | remote packets << 16}
  int4* tab = reinterpret_cast<int4*>(rsm + 256);
  unsigned char* sring = rsm + 256 + 16 * kTab * A.max_waves + 8 * A.SC;
  unsigned char* dring = sring + A.CS;
  const int w0 = A.reg_wave[blockIdx.x];
  const int nw = A.reg_wave[blockIdx.x + 1] - w0;
  for (int i = tid; i < nw; i += blockDim.x) {
    const int4 t = A.table[2 * (w0 + i)], v = A.table[2 * (w0 + i) + 1];
    const int4 hd = A.words[t.x];   // {cnt, slot0, K, NP}: read before the block lands
    tab[i] = make_int4(t.z, t.w, v.y | ((v.w & 0xffff) << 18), hd.x | (hd.z << 10) | (hd.w << 16));
  }
  if (tid == 0) {
    for (int b = 0; b < kNB; ++b) bar_init(&bar[b], 1);
    *done = 0;
    for (int p = 0; p < kProbers; ++p) probed[p] = 0;
    *issued = 0;
    *reinterpret_cast<double*>(rsm + kOneOff) = 1.0;   // the unused refs of short rows
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int D = A.D;
  constexpr bool tau = KIND == 0 && TAU;   // (the launch picks the instance from A.tau)
  const unsigned flags = jv::g_region_flags;

  if (tid >= kCompute + 64) {
    // -------------------------------------------------------------- prober
    // The prober warps fetch the remote dependencies of the coming waves
    // from the mailboxes and release each wave to the compute warps once
    // all of its values are in.  Warp p owns the waves w with
    // w % kProbers == p and has its own release counter, so four waves are
    // in flight and the warps' L2 round trips overlap (a single prober's
    // round took about as long as three waves of compute and paced every
    // region but the first: a stall every third wave in the trace).
    const int lane = tid & 31;
    const int pw = (tid - kCompute - 64) >> 5;
    constexpr int P = kProbers;
    int* const myprobed = probed + pw;
    auto pkts = [&](int x) -> unsigned char* {
      const int4 e = tab[x];
      return dring + e.y + (e.z & 0x3ffff) + (e.z >> 18);
    };
    auto np = [&](int x) { return (int)((unsigned)tab[x].w >> 16); };
    if (flags & 8) {   // diagnostic: no remote waits at all (wrong results)
      if (lane == 0)
        asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(sa(myprobed)), "r"(nw + P) : "memory");
      return;
    }
    // One wave at a time per warp, one packet per lane: direct 16-byte
    // relaxed loads from the mailbox (an L2 round trip each), repeated
    // warp-converged for the lanes whose packet is still stale; a fresh
    // value goes straight to the wave's decoded-values area.  A value
    // published upstream is seen within about one L2 round trip.
    bool hung = false;
#ifdef JV_REGION_TRACE
    const jv::Trace PT = jv::trace_begin();
#endif
    for (int x = pw; x < nw && !hung; x += P) {
#ifdef JV_REGION_TRACE
      if (lane == 0) jv::trace_word(PT, w0 + x, 3, clock64());   // prober turns to wave x
#endif
      if (np(x) > 0) {
        unsigned spins = 0;
        while (x >= ld_volatile_shared(issued) ||
               !bar_test(&bar[x % kNB], (uint32_t)((x / kNB) & 1))) {
          __nanosleep(32);
          if (++spins == jv::g_spin_limit) {
            hung = true;
            break;
          }
        }
        if (hung) break;
#ifdef JV_REGION_TRACE
        if (lane == 0) jv::trace_word(PT, w0 + x, 5, clock64());   // its block has landed
#endif
        const Wave X(sring + tab[x].x);
        double* rem = reinterpret_cast<double*>(pkts(x));   // the wave's remote values
        for (int j0 = 0; j0 < X.NP && !hung; j0 += 32) {
          const int j = j0 + lane;
          bool need = j < X.NP;
          const int64_t slot = need ? X.pslot(j) : 0;
          spins = 0;
          while (true) {
            double v;
            if (need && jv::mbox_try(A.mbox, slot, A.epoch, v)) {
              rem[j] = v;
              need = false;
            }
            if (!__any_sync(full, need)) break;
            if (++spins == jv::g_spin_limit) {
              hung = true;
              break;
            }
          }
        }
        if (hung) break;
        __syncwarp();
      }
#ifdef JV_REGION_TRACE
      if (lane == 0) jv::trace_word(PT, w0 + x, 6, clock64());   // all values in
#endif
      // release: the values written above are visible to whoever acquires
      if (lane == 0)
        asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(sa(myprobed)), "r"(x + P) : "memory");
    }
    if (hung) {
      atomicExch(&jv::g_hang, 1);
      if (lane == 0)
        asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(sa(myprobed)), "r"(nw + P) : "memory");
    }
    return;
  }
  if (tid >= kCompute + 32) {
    // -------------------------------------------------------------- waiter
    // Takes part in the compute warps' barrier so that they never touch an
    // mbarrier: in front of the barrier that ends wave w its lane 0 waits
    // for the blocks of wave w + 2 (when the compute warps start wave w + 1
    // and load the operands of wave w + 2, those have landed); behind it,
    // it publishes the progress counter the producer reads.
    const bool lead = tid == kCompute + 32;
    if (lead) {
      bar_wait(&bar[0], 0);
      if (nw > 1) bar_wait(&bar[1 % kNB], 0);
    }
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"n"(kCompute + 32) : "memory");
    for (int w = 0; w < nw; ++w) {
      if (lead && w + 2 < nw) bar_wait(&bar[(w + 2) % kNB], (uint32_t)(((w + 2) / kNB) & 1));
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"n"(kCompute + 32) : "memory");
      if (lead)
        asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(sa(done)), "r"(w + 1) : "memory");
    }
    return;
  }
  if (tid >= kCompute) {
    // ------------------------------------------------------------ producer
    if (tid != kCompute) return;
    // (the full table entries come from global memory, one wave ahead in
    // registers; shared memory keeps only what the other warps read)
    const int4* gt = A.table + 2 * (int64_t)w0;
    auto prefetch = [&](const int4& t2, const int4& v2) {
      l2_prefetch_bulk(A.words + t2.x, (uint32_t)t2.y);
      if (v2.y > 0) l2_prefetch_bulk(A.pack + 2 * (int64_t)v2.x, (uint32_t)v2.y);
      if (v2.w & 0xffff) l2_prefetch_bulk(A.vpack + 2 * (int64_t)v2.z, (uint32_t)(v2.w & 0xffff));
    };
    // (diagnostics: flags bits 8..15 override the L2 prefetch distance, 255 = none)
    const int kl2 = ((flags >> 8) & 255) == 255 ? 0 : ((flags >> 8) & 255) ? (int)((flags >> 8) & 255) : kL2;
    for (int x = 0; x < kl2 && x < nw; ++x) prefetch(gt[2 * x], gt[2 * x + 1]);
    int4 tn = gt[0], vn = gt[1];
    int4 ptn = make_int4(0, 0, 0, 0), pvn = ptn;
    if (kl2 && kl2 < nw) {
      ptn = gt[2 * kl2];
      pvn = gt[2 * kl2 + 1];
    }
    for (int x = 0; x < nw; ++x) {
      const int4 t = tn, v = vn, pt = ptn, pv = pvn;
      if (x + 1 < nw) {
        tn = gt[2 * (x + 1)];
        vn = gt[2 * (x + 1) + 1];
      }
      if (kl2 && x + 1 + kl2 < nw) {
        ptn = gt[2 * (x + 1 + kl2)];
        pvn = gt[2 * (x + 1 + kl2) + 1];
      }
      if (kl2 && x + kl2 < nw) prefetch(pt, pv);
      // ring blocks of wave x may overlap those of wave x - D - 1
      while (ld_volatile_shared(done) < x - D) __nanosleep(20);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint64_t* b = &bar[x % kNB];
      const bool skip = flags & 4;   // diagnostic: no value copies (wrong results)
      const int cb = v.w & 0xffff;
      bar_expect_tx(b, (uint32_t)(t.y + (skip ? 0 : v.y + cb)));
      bulk_g2s(sring + t.z, A.words + t.x, (uint32_t)t.y, b);
      unsigned char* blk = dring + t.w;
      if (!skip && v.y > 0) bulk_g2s(blk, A.pack + 2 * (int64_t)v.x, (uint32_t)v.y, b);
      if (!skip && cb > 0) bulk_g2s(blk + v.y, A.vpack + 2 * (int64_t)v.z, (uint32_t)cb, b);
      asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(sa(issued)), "r"(x + 1) : "memory");
    }
    return;
  }

  // -------------------------------------------------------------- compute
  // One row per thread, one warp per scheduler: nothing hides a stall, so
  // the wave loop is written as straight-line code — every shared-memory
  // access is an explicit ld/st.shared at a precomputed offset (program
  // order = issue order), a wave's operands (its 32-byte record, matrix
  // values, right-hand side) are loaded into registers while the wave
  // before it computes, the two operand sets ping-pong (no copies), threads
  // beyond a wave's rows redo its last row with their stores predicated
  // off, and the only branches are the remote-wave wait, the rare slow
  // division and the rare zero pivot.  Critical path per wave:
  //   barrier -> dependency loads -> arithmetic chain -> slot store -> barrier.
  constexpr int kR = KR;   // dependencies held in registers (every row's, for the factor)
  const uint32_t sb = sa(rsm);
  auto lds64 = [&](uint32_t off) -> double {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(sb + off));
    return v;
  };
  auto lds128 = [&](uint32_t off) -> int4 {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(sb + off));
    return v;
  };
  const uint32_t tab_off = 256, sring_off = (uint32_t)(sring - rsm), dring_off = (uint32_t)(dring - rsm);
  struct Ops {
    int cnt, K, np;
    int4 r0, r1;          // {ref0..3}, {p0, row, meta, me}
    double a[kR], u[kR], dg, rhs;
    const int32_t* xref;
    const double* vals;
  };
  struct Tab {            // a wave's table entries (static shared memory)
    int so, dof, vbytes, cnt, K, np;
  };
  auto load_tab = [&](int w, Tab& t) {
    const int4 e = lds128(tab_off + 16 * w);
    t.so = e.x;
    t.dof = e.y;
    t.vbytes = e.z & 0x3ffff;
    t.cnt = e.w & 1023;
    t.K = (e.w >> 10) & 63;
    t.np = (int)((unsigned)e.w >> 16);
  };
  // operands of a wave whose blocks have landed (the producer warp saw to
  // it before the last barrier): loads only, every address from registers
  auto fetch = [&](const Tab& t, Ops& s) {
    const uint32_t blk = sring_off + t.so;
    const int cnt = t.cnt, K = t.K;
    s.cnt = cnt;
    s.K = K;
    s.np = t.np;
    s.xref = reinterpret_cast<const int32_t*>(rsm + blk) + 4 + 8 * cnt;
    s.vals = reinterpret_cast<const double*>(rsm + dring_off + t.dof);
    // threads beyond the wave take its last row's operands
    const int i = min(tid, cnt - 1);
    s.r0 = lds128(blk + 16 + 32 * i);
    s.r1 = lds128(blk + 32 + 32 * i);
    const uint32_t vp = dring_off + t.dof + 8 * i;   // vals[k][i] at vp + 8 * k * cnt
    const uint32_t c8 = 8 * cnt;
    const uint32_t vec = dring_off + t.dof + t.vbytes + 8 * i;
    if (KIND == 0) {
      // a_k, a_rr, u_k in vals[2K + 1][cnt]; the pack holds +0.0 for the
      // entries of rows with fewer than K pivots
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        s.a[k] = lds64(vp + min(k, max(K, 1) - 1) * c8);
        s.u[k] = lds64(vp + (K + min(k + 1, K)) * c8);
      }
      s.dg = lds64(vp + K * c8);
      s.rhs = tau ? lds64(vec) : 0.0;   // the row's norm (no vector block without tau)
    } else {
      const int o = KIND == 1 ? 0 : 1;
#pragma unroll
      for (int k = 0; k < kR; ++k) s.a[k] = lds64(vp + (o + min(k, max(K, 1) - 1)) * c8);
      s.dg = lds64(vp);
      s.rhs = lds64(vec);
    }
  };
  double* const gval = A.val;
  double* const gout = A.out;
  uint64_t* const mbox = A.mbox;
  const uint32_t epoch = A.epoch;
  const double tauv = tau ? A.tau : 0.0;
#ifdef JV_REGION_TRACE
  const jv::Trace T = jv::trace_begin();
  const bool tracing = T.p != nullptr && tid == 0;
#endif
  int rel = 0;   // the release counter of the coming wave's prober, read a wave early
  auto step = [&](int w, const Ops& cur, Ops& nxt, const Tab& tn, Tab& tnn) {
    // the prober has released this wave's remote dependencies (a wave
    // without any passes straight through)
#ifdef JV_REGION_TRACE
    if (tracing) jv::trace_clock(T, w0 + w, 1);   // wave start
#endif
    // (its counter was read during the wave before: no load on the
    // critical path when the prober is ahead)
    if (cur.np > 0 && rel <= w) {
      const int* const pr = probed + (w % kProbers);
      while (ld_acquire_shared(pr) <= w) {
      }
    }
#ifdef JV_REGION_TRACE
    if (tracing) jv::trace_clock(T, w0 + w, 2);   // released by the prober
#endif
    double dv[kR];
    dv[0] = lds64(cur.r0.x);
    dv[1] = lds64(cur.r0.y);
    dv[2] = lds64(cur.r0.z);
    if (kR > 3) dv[kR - 1] = lds64(cur.r0.w);
    // the next wave's operands, in flight during this wave's arithmetic
    // (after the last wave: that wave again, its blocks are still there),
    // and the table entries of the wave after it
    fetch(tn, nxt);
    load_tab(min(w + 2, nw - 1), tnn);
    rel = ld_acquire_shared(probed + ((w + 1) % kProbers));
    const int cnt = cur.cnt, K = cur.K;
    const bool active = tid < cnt;
    const int meta = cur.r1.z, nd = meta & 63, row = cur.r1.y, p0 = cur.r1.x;
    const bool pub = active && (meta & 64);
    double res;
#if (JV_RDIAG & 2)
    res = cur.dg + dv[0] + dv[1] + dv[2] + dv[3] + cur.a[0] + cur.u[0] + cur.rhs;
    if (false) {
#else
    if (KIND == 0) {
#endif
      // pivots beyond the row's own: a = +0.0 (K > k >= nd) or a copy of an
      // earlier operand (k >= K), never used: umask and the stores are per nd
      double l[kR];
      jv::ddiv_batch<kR>(cur.a, dv, l, nd);   // (interleaved chains: the latency of one)
      const double thresh = tau ? jv::dmul(tauv, cur.rhs) : 0.0;
      double d = cur.dg;
      const int umask = (meta >> 7) & 15;
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        const bool drop = tau && fabs(l[k]) < thresh;
        const double dn = jv::dsub(d, jv::dmul(l[k], cur.u[k]));
        d = (!drop && (umask & (1 << k))) ? dn : d;
        l[k] = drop ? 0.0 : l[k];
      }
      res = d;
#if !(JV_RDIAG & 4)
#pragma unroll
      for (int k = 0; k < kR; ++k)
        if (active && k < nd) __stcg(gval + p0 + k, l[k]);
      if (active) __stcg(gval + p0 + nd, d);
      if (active && d == 0.0) atomicMin(A.err, row);
#endif
    } else {
      // unused refs read 1.0 against a packed +0.0 (or, beyond K, a copy of
      // an operand, masked here): s - 0 = s exactly
      const int o = KIND == 1 ? 0 : 1;
      double sacc = cur.rhs;
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        const double sn = jv::dsub(sacc, jv::dmul(cur.a[k], dv[k]));
        sacc = k < nd ? sn : sacc;
      }
      if (K > kR && active) {
        for (int k = kR; k < nd; ++k)
          sacc = jv::dsub(sacc, jv::dmul(cur.vals[(o + k) * cnt + tid],
                                         lds64((uint32_t)cur.xref[(k - kR) * cnt + tid])));
      }
      if (KIND == 2) sacc = jv::ddiv(sacc, cur.dg);
      res = sacc;
      if (active) __stcg(gout + row, sacc);
    }
    if (active) asm volatile("st.shared.f64 [%0], %1;" ::"r"(sb + (uint32_t)cur.r1.w), "d"(res) : "memory");
#if !(JV_RDIAG & 4)
    if (pub) jv::mbox_put(mbox, row, res, epoch);
#endif
#ifdef JV_REGION_TRACE
    if (tracing) jv::trace_clock(T, w0 + w, 4);   // computed, at the barrier
#endif
    asm volatile("bar.sync 1, %0;" ::"n"(kCompute + 32) : "memory");
#ifdef JV_REGION_TRACE
    if (tracing) {
      if (flags & 16) jv::trace_clock(T, w0 + w, 7);   // 16: clock only (no globaltimer read)
      else jv::trace_mark(T, w0 + w, 7);
    }
#endif
  };
  asm volatile("bar.sync 1, %0;" ::"n"(kCompute + 32) : "memory");   // blocks 0 and 1 have landed
  if (nw > 0) {
    Ops oa, ob;
    Tab ta, tb;
    load_tab(0, ta);
    load_tab(min(1, nw - 1), tb);
    fetch(ta, oa);
    int w = 0;
    for (; w + 1 < nw; w += 2) {
      step(w, oa, ob, tb, ta);       // consumes the entries of w + 1, loads those of w + 2
      step(w + 1, ob, oa, ta, tb);
    }
    if (w < nw) step(w, oa, ob, tb, ta);
  }
}

}  // namespace jvr

namespace jvr {
// Tiles of E * blockDim consecutive elements: each thread takes E
// of them blockDim apart (every load and store stays coalesced across the
// warp) and has all E gathers in flight together.
constexpr int kPackE = 4;
template <int E>
__device__ __forceinline__ void pack_tiles(int64_t m, const int32_t* __restrict__ sidx,
                                           const double* __restrict__ src,
                                           double* __restrict__ dst, int blk, int nblk) {
  const int64_t tile = (int64_t)E * blockDim.x;
  for (int64_t t0 = blk * tile; t0 < m; t0 += nblk * tile) {
    int k[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int64_t e = t0 + j * blockDim.x + threadIdx.x;
      k[j] = e < m ? __ldcs(sidx + e) : -1;
    }
    double x[E];
#pragma unroll
    for (int j = 0; j < E; ++j) x[j] = k[j] >= 0 ? __ldg(src + k[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int64_t e = t0 + j * blockDim.x + threadIdx.x;
      if (e < m) __stcs(dst + e, x[j]);
    }
  }
}
struct PackJob {
  int64_t m;
  const int32_t* sidx;
  const double* src;
  double* dst;
};
// two gathers in one launch (blocks [0, g1) do the first), and optionally
// an error-row slot reset: the launches in front of a region sweep
template <int E>
__global__ void pack_kernel(PackJob a, PackJob b, int g1, int32_t* reset) {
  if (reset && blockIdx.x == 0 && threadIdx.x == 0) *reset = jv::kNoRow;
  if ((int)blockIdx.x < g1) pack_tiles<E>(a.m, a.sidx, a.src, a.dst, blockIdx.x, g1);
  else pack_tiles<E>(b.m, b.sidx, b.src, b.dst, blockIdx.x - g1, gridDim.x - g1);
}
}  // namespace jvr

// dst[e] = src[sidx[e]] (0 where sidx < 0): the wave-ordered value arrays
// of the region kernels, refreshed once per factorization
extern "C" int jv_pack_values2(int64_t m1, const int32_t* sidx1, const double* src1, double* dst1,
                               int64_t m2, const int32_t* sidx2, const double* src2, double* dst2,
                               int32_t* reset_row, void* stream) {
  if (m1 < 0 || m2 < 0) {
    jvh::set_error("jv_pack_values2: negative length");
    return JV_EINVAL;
  }
  if (m1 == 0 && m2 == 0 && !reset_row) return JV_OK;
  // (measured at c2: 4 elements per thread, factor span 502 -> 487 us;
  // 1: 502, 2: 490, 8: 498; grid cap 4 / 8 / 16 blocks per SM: 494 / 487 / 489)
  const int64_t tile = jvr::kPackE * 256, cap = 8 * (int64_t)jvh::sm_count();
  int64_t g1 = (m1 + tile - 1) / tile, g2 = (m2 + tile - 1) / tile;
  if (g1 + g2 > cap) {   // share the cap in proportion, at least one block per job
    const int64_t c1 = m1 ? std::max<int64_t>(1, cap * m1 / (m1 + m2)) : 0;
    g2 = m2 ? std::max<int64_t>(1, std::min(g2, cap - c1)) : 0;
    g1 = std::min(g1, c1);
  }
  const int64_t grid = std::max<int64_t>(1, g1 + g2);
  jvr::pack_kernel<jvr::kPackE><<<(int)grid, 256, 0, (cudaStream_t)stream>>>(
      jvr::PackJob{m1, sidx1, src1, dst1}, jvr::PackJob{m2, sidx2, src2, dst2}, (int)g1,
      reset_row);
  JV_CHECK_LAUNCH("jv_pack_values2");
  return JV_OK;
}

extern "C" int jv_pack_values(int64_t m, const int32_t* sidx, const double* src, double* dst,
                              void* stream) {
  return jv_pack_values2(m, sidx, src, dst, 0, nullptr, nullptr, nullptr, nullptr, stream);
}

extern "C" int jv_region_threads(void) { return jvr::kThreads; }

extern "C" int jv_set_region_flags(unsigned flags) {
  cudaError_t e = cudaMemcpyToSymbol(jv::g_region_flags, &flags, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_region_flags");
  return JV_OK;
}

extern "C" int64_t jv_region_smem_fixed(int32_t slot_ring, int32_t max_waves) {
  return 256 + 16 * jvr::kTab * (int64_t)max_waves + 8 * (int64_t)slot_ring;
}

extern "C" int jv_region_run(int32_t kind, int32_t nreg, int32_t max_rows, const void* words,
                             const int32_t* table,
                             const int32_t* reg_wave, int32_t slot_ring, int32_t max_waves,
                             int32_t S, int32_t D, int32_t CS, int32_t CD, double* val,
                             const double* pack, const double* vpack, double* out, const double* norms, double tau,
                             uint64_t* mbox, uint32_t epoch, int32_t* err_row, void* stream) {
  if (kind < 0 || kind > 2 || nreg < 1 || epoch == 0 || D < 2 || D > 12 || S < D ||
      slot_ring < 1 || (slot_ring & (slot_ring - 1)) ||
      S + 1 > jvr::kNB) {
    jvh::set_error("jv_region_run: bad argument (kind=%d nreg=%d S=%d D=%d)", kind, nreg, S, D);
    return JV_EINVAL;
  }
  const size_t smem = (size_t)jv_region_smem_fixed(slot_ring, max_waves) + CS + CD;
  // waves of at most 256 (128) rows run on 8 (4) compute warps: a cheaper
  // barrier, no idle warps
  const int mr = max_rows & 0xffff;
  const int nc = mr > 0 && mr <= 128 ? 128 : mr > 0 && mr <= 256 ? 256 : jvr::kCompute;
  const int block = nc + jvr::extra_for(nc);
  const int kmax = max_rows >> 16;   // most dependencies of a row (0: unknown)
  if (kind == 0 && kmax > 4) {
    jvh::set_error("jv_region_run: factor rows with %d pivots", kmax);
    return JV_EINVAL;
  }
  const bool k3 = kmax > 0 && kmax <= 3;
  const bool tt = kind == 0 && tau > 0.0;
  const void* fn = nullptr;
#define JV_RK(K, N)                                                                           \
  (k3 ? (tt ? (const void*)jvr::region_kernel<K, N, 3, (K == 0)>                              \
            : (const void*)jvr::region_kernel<K, N, 3, false>)                                \
      : (tt ? (const void*)jvr::region_kernel<K, N, 4, (K == 0)>                              \
            : (const void*)jvr::region_kernel<K, N, 4, false>))
#define JV_RKN(K) (nc == 128 ? JV_RK(K, 128) : nc == 256 ? JV_RK(K, 256) : JV_RK(K, 512))
  fn = kind == 0 ? JV_RKN(0) : kind == 1 ? JV_RKN(1) : JV_RKN(2);
#undef JV_RKN
#undef JV_RK
  // attributes and residency are checked once per (instance, shared memory
  // size); the size attribute of an instance only ever grows
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> resident;
  static std::map<const void*, size_t> attr;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = resident.find({fn, smem});
    if (it != resident.end()) per_sm = it->second;
    if (per_sm == 0) {
      cudaError_t e = cudaSuccess;
      if (attr[fn] < smem) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return jvh::cuda_status(e, "jv_region_run attr");
        attr[fn] = smem;
      }
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem);
      if (e != cudaSuccess) return jvh::cuda_status(e, "jv_region_run occupancy");
      resident[{fn, smem}] = per_sm;
    }
  }
  if (per_sm * jvh::sm_count() < nreg) {
    jvh::set_error("jv_region_run: %d regions but only %d resident CTAs", nreg,
                   per_sm * jvh::sm_count());
    return JV_ECOOP;
  }
  jvr::RArgs A{reinterpret_cast<const int4*>(words), reinterpret_cast<const int4*>(table),
               reg_wave, slot_ring, max_waves, S, D, CS, CD, val, pack, vpack, out, norms, tau, mbox,
               epoch, err_row};
  void* args[] = {&A};
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(nreg), dim3(block), args, smem,
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_region_run");
  return JV_OK;
}
