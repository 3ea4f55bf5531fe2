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
#include "common.cuh"
#include "../../include/jv.h"

namespace jvr {

constexpr int kThreads = 512;   // rows per wave (compute threads)
constexpr int kNB = 16;   // static-block mbarriers in the ring (S + 1 <= kNB)

struct RArgs {
  const int4* words;   // static stream, 16-byte units
  const int4* table;   // per wave {block offset (16 B units), bytes, ring offset, dyn offset}
  const int32_t* reg_wave;
  int32_t SC, max_waves, S, D, CS, CD;   // SC: slot ring (power of 2)
  double* val;
  const double* in;
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
JV_INLINE void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(dst)), "l"(src) : "memory");
}
JV_INLINE void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(dst)), "l"(src) : "memory");
}
JV_INLINE void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
JV_INLINE void cp_wait_pending(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

// wave block view (regions_host.cpp): SoA arrays of cnt rows
struct Wave {
  const int32_t* b;
  int cnt, slot0, K, NP;
  JV_INLINE Wave(const unsigned char* p) : b(reinterpret_cast<const int32_t*>(p)) {
    cnt = b[0];
    slot0 = b[1];
    K = b[2];
    NP = b[3];
  }
  JV_INLINE int row(int i) const { return b[4 + i]; }
  JV_INLINE int p0(int i) const { return b[4 + cnt + i]; }
  JV_INLINE int meta(int i) const { return b[4 + 2 * cnt + i]; }
  JV_INLINE int ref(int k, int i) const { return b[4 + (3 + k) * cnt + i]; }
  JV_INLINE int us(int k, int i) const { return b[4 + (3 + K + k) * cnt + i]; }
  template <int KIND>
  JV_INLINE int pslot(int j) const { return b[4 + (3 + (KIND == 0 ? 2 * K : K)) * cnt + j]; }
};
// values per row in the dynamic block
template <int KIND>
JV_INLINE int nvals(int K, bool tau) {
  return KIND == 0 ? 2 * K + 1 + (tau ? 1 : 0) : (KIND == 1 ? K + 1 : K + 2);
}

constexpr int kCompute = 512;
constexpr int kProducers = 128;   // producer threads (4 warps)
constexpr int kBlock = kCompute + kProducers;

// Gathers of wave t by the producer warp: lane l fetches the values of rows
// l, l + 32, ... into column i of vals[NV][cnt] and the wave's mailbox
// packets; completion is signalled per lane with cp.async.mbarrier.arrive.
template <int KIND>
JV_INLINE void gather_wave(const RArgs& A, const int4& t, const unsigned char* sring,
                           unsigned char* dring, bool tau, int lane) {
  const Wave V(sring + t.z);
  double* vals = reinterpret_cast<double*>(dring + t.w);
  const int cnt = V.cnt, K = V.K;
  if (!(jv::g_region_flags & 4)) {
    for (int i = lane; i < cnt; i += kProducers) {
      const int p0 = V.p0(i);
      const int nd = V.meta(i) & 63;
      if (KIND == 0) {
        for (int k = 0; k < nd; ++k) cp8(vals + k * cnt + i, A.val + p0 + k);
        cp8(vals + K * cnt + i, A.val + p0 + nd);
        for (int k = 0; k < nd; ++k) cp8(vals + (K + 1 + k) * cnt + i, A.val + V.us(k, i));
        if (tau) cp8(vals + (2 * K + 1) * cnt + i, A.norms + V.row(i));
      } else if (KIND == 1) {
        cp8(vals + i, A.in + V.row(i));
        for (int k = 0; k < nd; ++k) cp8(vals + (1 + k) * cnt + i, A.val + p0 + k);
      } else {
        cp8(vals + i, A.in + V.row(i));
        for (int k = 0; k <= nd; ++k) cp8(vals + (1 + k) * cnt + i, A.val + p0 + k);
      }
    }
  }
  unsigned char* pk = dring + t.w + ((8 * nvals<KIND>(K, tau) * cnt + 15) & ~15);
  for (int j = lane; j < V.NP; j += kProducers)
    cp16(pk + 16 * j, A.mbox + 2 * (int64_t)V.pslot<KIND>(j));
}

JV_INLINE void cp_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(b)) : "memory");
}
JV_INLINE int ld_volatile_shared(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(sa(p)) : "memory");
  return v;
}

// Warp-specialised: warps 0..15 compute (one row per thread, a named
// barrier per wave), warp 16 produces — bulk copies of the static blocks
// (TMA, mbarrier complete_tx) and cp.async gathers of the values (mbarrier
// arrive per lane), running up to D waves ahead of the compute warps, whose
// progress it reads from a shared counter before reusing ring space.

template <int KIND>
__global__ void __launch_bounds__(kBlock, 1) region_kernel(RArgs A) {
  extern __shared__ __align__(128) unsigned char rsm[];
  const unsigned full = 0xffffffffu;
  const int tid = threadIdx.x;
  uint64_t* sbar = reinterpret_cast<uint64_t*>(rsm);          // static full [kNB]
  uint64_t* dbar = sbar + kNB;                                 // dynamic full [kNB]
  int* done = reinterpret_cast<int*>(rsm + 2 * 8 * kNB);      // waves finished
  int4* tab = reinterpret_cast<int4*>(rsm + 512);
  double* slot = reinterpret_cast<double*>(rsm + 512 + 16 * A.max_waves);
  unsigned char* sring = rsm + 512 + 16 * A.max_waves + 8 * A.SC;
  unsigned char* dring = sring + A.CS;
  const int w0 = A.reg_wave[blockIdx.x];
  const int nw = A.reg_wave[blockIdx.x + 1] - w0;
  for (int i = tid; i < nw; i += blockDim.x) tab[i] = A.table[w0 + i];
  if (tid == 0) {
    for (int b = 0; b < kNB; ++b) {
      bar_init(&sbar[b], 1);
      bar_init(&dbar[b], kProducers);
    }
    *done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int S = A.S, D = A.D;
  const bool tau = KIND == 0 && A.tau > 0.0;
  const unsigned flags = jv::g_region_flags;

  if (tid >= kCompute) {
    // ------------------------------------------------------------ producer
    const int lane = tid - kCompute;
    int sx = 0;   // next static block to issue
    for (int x = 0; x < nw; ++x) {
      // static blocks up to x + (S - D): block y may overlap block y - S - 1
      for (; sx < nw && sx <= x + (S - D); ++sx) {
        while (ld_volatile_shared(done) < sx - S) __nanosleep(32);
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          const int4 t = tab[sx];
          uint64_t* b = &sbar[sx % kNB];
          bar_expect_tx(b, (uint32_t)t.y);
          bulk_g2s(sring + t.z, A.words + t.x, (uint32_t)t.y, b);
        }
      }
      // dynamic block x may overlap block x - D - 1
      while (ld_volatile_shared(done) < x - D) __nanosleep(32);
      bar_wait(&sbar[x % kNB], (uint32_t)((x / kNB) & 1));
      gather_wave<KIND>(A, tab[x], sring, dring, tau, lane);
      cp_arrive(&dbar[x % kNB]);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }

  // -------------------------------------------------------------- compute
  const jv::Trace T = jv::trace_begin();
  for (int w = 0; w < nw; ++w) {
    if (tid == 0) jv::trace_mark(T, w0 + w, 1);
    bar_wait(&dbar[w % kNB], (uint32_t)((w / kNB) & 1));
    bar_wait(&sbar[w % kNB], (uint32_t)((w / kNB) & 1));
    const int4 t = tab[w];
    const Wave V(sring + t.z);
    const int cnt = V.cnt, K = V.K;
    const bool active = tid < cnt;
    const double* vals = reinterpret_cast<const double*>(dring + t.w);
    unsigned char* pk = dring + t.w + ((8 * nvals<KIND>(K, tau) * cnt + 15) & ~15);
    int nd = 0, meta = 0;
    unsigned miss = 0;   // bit k: dependency k still unpublished
    if (active) {
      meta = V.meta(tid);
      nd = meta & 63;
      for (int k = 0; k < nd; ++k) {
        const int ref = V.ref(k, tid);
        if (ref < 0) {
          const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(pk + 16 * (-1 - ref));
          if ((uint32_t)(p.x >> 32) != A.epoch || (uint32_t)(p.y >> 32) != A.epoch)
            miss |= 1u << k;
        }
      }
    }
    if (tid == 0) jv::trace_mark(T, w0 + w, 2);
    // dependencies not yet published when prefetched: warp-converged live
    // probes (no lane spins alone); a hit is written back into the packet
    if (flags & 8) miss = 0;   // diagnostic: no waiting (wrong results)
    if (__any_sync(full, miss)) {
      unsigned ns = 0, spins = 0;
      while (__any_sync(full, miss)) {
        unsigned m = miss;
        while (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1;
          const int j = -1 - V.ref(k, tid);
          unsigned long long x0, x1;
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(x0), "=l"(x1)
                       : "l"(A.mbox + 2 * (int64_t)V.pslot<KIND>(j)) : "memory");
          if ((uint32_t)(x0 >> 32) == A.epoch && (uint32_t)(x1 >> 32) == A.epoch) {
            *reinterpret_cast<ulonglong2*>(pk + 16 * j) = make_ulonglong2(x0, x1);
            miss &= ~(1u << k);
          }
        }
        if (__any_sync(full, miss)) {
          if (ns) __nanosleep(ns);
          ns = ns ? min(2 * ns, jv::g_poll_cap) : 16u;
          if (++spins == jv::g_spin_limit) {
            atomicExch(&jv::g_hang, 1);
            break;
          }
        }
      }
    }
    if (tid == 0) jv::trace_mark(T, w0 + w, 3);
    if (active) {
      const int me = (V.slot0 + tid) & (A.SC - 1);
      auto dep = [&](int k) -> double {
        const int ref = V.ref(k, tid);
        if (ref >= 0) return slot[ref];
        const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(pk + 16 * (-1 - ref));
        return __longlong_as_double((long long)((p.x & 0xffffffffull) | (p.y << 32)));
      };
      auto val = [&](int k) -> double { return vals[k * cnt + tid]; };
      const int p0 = V.p0(tid);
      if (KIND == 0) {
        double a[4], d4[4], u[4], l[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a[k] = k < nd ? val(k) : 0.0;
          d4[k] = k < nd ? dep(k) : 1.0;
          u[k] = k < nd ? val(K + 1 + k) : 0.0;
        }
        jv::ddiv_batch<4>(a, d4, l, nd);
        const double thresh = tau ? jv::dmul(A.tau, val(2 * K + 1)) : 0.0;
        double d = val(K);
        const int umask = (meta >> 7) & 15;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k < nd) {
            if (tau && fabs(l[k]) < thresh) l[k] = 0.0;
            else if (umask & (1 << k)) d = jv::dsub(d, jv::dmul(l[k], u[k]));
          }
        }
        slot[me] = d;
        if (meta & 64) jv::mbox_put(A.mbox, p0 + nd, d, A.epoch);
        if (!(flags & 16)) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < nd) __stcg(A.val + p0 + k, l[k]);
          __stcg(A.val + p0 + nd, d);
        }
        if (d == 0.0) atomicMin(A.err, V.row(tid));
      } else {
        const int o = KIND == 1 ? 1 : 2;
        double sacc = val(0);
        for (int k = 0; k < nd; ++k) sacc = jv::dsub(sacc, jv::dmul(val(o + k), dep(k)));
        if (KIND == 2) sacc = jv::ddiv(sacc, val(1));
        slot[me] = sacc;
        const int r = V.row(tid);
        if (meta & 64) jv::mbox_put(A.mbox, r, sacc, A.epoch);
        if (!(flags & 16)) __stcg(A.out + r, sacc);
      }
    }
    if (tid == 0) jv::trace_mark(T, w0 + w, 4);
    asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory");
    if (tid == 0) {
      asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(sa(done)), "r"(w + 1) : "memory");
      jv::trace_mark(T, w0 + w, 7);
    }
  }
}

}  // namespace jvr

extern "C" int jv_region_threads(void) { return jvr::kThreads; }

extern "C" int jv_set_region_flags(unsigned flags) {
  cudaError_t e = cudaMemcpyToSymbol(jv::g_region_flags, &flags, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_region_flags");
  return JV_OK;
}

extern "C" int64_t jv_region_smem_fixed(int32_t slot_ring, int32_t max_waves) {
  return 512 + 16 * (int64_t)max_waves + 8 * (int64_t)slot_ring;
}

extern "C" int jv_region_run(int32_t kind, int32_t nreg, const void* words, const int32_t* table,
                             const int32_t* reg_wave, int32_t slot_ring, int32_t max_waves,
                             int32_t S, int32_t D, int32_t CS, int32_t CD, double* val,
                             const double* in, double* out, const double* norms, double tau,
                             uint64_t* mbox, uint32_t epoch, int32_t* err_row, void* stream) {
  if (kind < 0 || kind > 2 || nreg < 1 || epoch == 0 || D < 1 || D > 4 || S < D ||
      slot_ring < 1 || (slot_ring & (slot_ring - 1)) ||
      S + 1 > jvr::kNB) {
    jvh::set_error("jv_region_run: bad argument (kind=%d nreg=%d S=%d D=%d)", kind, nreg, S, D);
    return JV_EINVAL;
  }
  const size_t smem = (size_t)jv_region_smem_fixed(slot_ring, max_waves) + CS + CD;
  const void* fn = kind == 0 ? (const void*)jvr::region_kernel<0>
                   : kind == 1 ? (const void*)jvr::region_kernel<1>
                               : (const void*)jvr::region_kernel<2>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_region_run attr");
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, jvr::kBlock, smem);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_region_run occupancy");
  if (per_sm * jvh::sm_count() < nreg) {
    jvh::set_error("jv_region_run: %d regions but only %d resident CTAs", nreg,
                   per_sm * jvh::sm_count());
    return JV_ECOOP;
  }
  jvr::RArgs A{reinterpret_cast<const int4*>(words), reinterpret_cast<const int4*>(table),
               reg_wave, slot_ring, max_waves, S, D, CS, CD, val, in, out, norms, tau, mbox,
               epoch, err_row};
  void* args[] = {&A};
  e = cudaLaunchCooperativeKernel(fn, dim3(nreg), dim3(jvr::kBlock), args, smem,
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_region_run");
  return JV_OK;
}
