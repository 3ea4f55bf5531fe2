// CTA-resident region factorization for stencil-class matrices (sm_100a).
//
// The sync-free ticket kernel (factor.cu) pays an L2 round trip plus a warp's
// scheduling on every one of the DAG's levels (config 2: 382 levels, ~2.4 us
// each).  Here every CTA owns one compact region of rows (BFS-grown, see
// jv_region_plan_host) and walks it level by level:
//   * a pivot inside the region is read from shared memory (its diagonal,
//     written by this CTA at an earlier level; __syncthreads between levels),
//   * a pivot in another region is read from the 16-byte mailbox (common.cuh),
//     with a warp-converged probe loop,
//   * rows whose diagonal another region reads publish it to the mailbox.
// A dependency chain crosses region boundaries only O(grid / region
// diameter) times, so most of the 382 hops cost a CTA barrier, not an L2
// round trip.
//
// Arithmetic is the stencil fast path of factor.cu (the only rows accepted
// by jv_region_desc_host): pivots are independent, the only update target is
// the diagonal, the strictly-upper entries are final from the start —
// l_k = a_k / u_kk, u_rr = a_rr - sum_k l_k u_kr in ascending k, explicitly
// rounded, bitwise equal to factor_serial (_kernels.py:165-204).
//
// Deadlock freedom: every CTA processes its levels in increasing order and
// only waits on rows of lower levels; all CTAs are co-resident (cooperative
// launch), so the lowest pending level always progresses.
#include "common.cuh"
#include "../../include/jv.h"

namespace {

constexpr int kRegThreads = 512;

struct RegionArgs {
  const int32_t* slot_row;
  const int32_t* info;
  const int32_t* drs;
  const int32_t* ref;   // [4][n]
  const int32_t* us;    // [4][n]
  int32_t n;
  double* val;
  const double* norms;
  double tau;
  const int32_t* reg_ptr;
  const int32_t* wave_ptr;
  const int32_t* wave_beg;
  uint64_t* mbox;
  uint32_t epoch;
  int32_t* err;
};

// One wave's per-thread state.  Descriptors (static structure) are loaded
// two waves ahead and the input values one wave ahead, so the DRAM/L2
// latency of both dependent rounds overlaps the barrier-separated compute of
// the current wave.
struct WaveDesc {
  int i;        // slot (or -1)
  int inf, rs;
  int ref[4], us[4];
};
struct WaveVals {
  double a[4], u[4], arr;
};

JV_INLINE WaveDesc load_desc(const RegionArgs& A, int w, int w1, int rend) {
  WaveDesc D;
  D.i = -1;
  D.inf = 0;
  D.rs = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) { D.ref[k] = 0; D.us[k] = 0; }
  if (w < w1) {
    const int s0 = A.wave_beg[w] & 0x7fffffff;
    const int s1 = (w + 1 < w1) ? (A.wave_beg[w + 1] & 0x7fffffff) : rend;
    const int i = s0 + threadIdx.x;
    if (i < s1) {
      D.i = i;
      D.inf = __ldg(A.info + i);
      D.rs = __ldg(A.drs + i);
      const int nL = D.inf & 7;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < nL) {
          D.ref[k] = __ldg(A.ref + (size_t)k * A.n + i);
          D.us[k] = __ldg(A.us + (size_t)k * A.n + i);
        }
      }
    }
  }
  return D;
}

JV_INLINE void l2_prefetch(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}

// L2 prefetch of wave w's descriptor lines (far ahead: the loads that use
// them come 3 waves later)
JV_INLINE void prefetch_desc(const RegionArgs& A, int w, int w1, int rend) {
  if (w >= w1) return;
  const int s0 = A.wave_beg[w] & 0x7fffffff;
  const int s1 = (w + 1 < w1) ? (A.wave_beg[w + 1] & 0x7fffffff) : rend;
  const int i = s0 + threadIdx.x;
  if (i < s1 && (threadIdx.x & 15) == 0) {   // one probe per 64-byte line of int32s
    l2_prefetch(A.info + i);
    l2_prefetch(A.drs + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      l2_prefetch(A.ref + (size_t)k * A.n + i);
      l2_prefetch(A.us + (size_t)k * A.n + i);
    }
  }
}

// L2 prefetch of the input values a wave will read
JV_INLINE void prefetch_vals(const RegionArgs& A, const WaveDesc& D) {
  if (D.i < 0) return;
  const int nL = D.inf & 7, umask = D.inf >> 4;
  l2_prefetch(A.val + D.rs);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < nL && (umask & (1 << k))) l2_prefetch(A.val + D.us[k]);
}

JV_INLINE WaveVals load_vals(const RegionArgs& A, const WaveDesc& D) {
  WaveVals V;
  const int nL = D.inf & 7, umask = D.inf >> 4;
  V.arr = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    V.a[k] = (D.i >= 0 && k < nL) ? __ldcs(A.val + D.rs + k) : 0.0;
    V.u[k] = (D.i >= 0 && k < nL && (umask & (1 << k))) ? __ldg(A.val + D.us[k]) : 0.0;
  }
  if (D.i >= 0) V.arr = __ldcs(A.val + D.rs + nL);
  return V;
}

__global__ void __launch_bounds__(kRegThreads, 1) region_factor_kernel(RegionArgs A) {
  extern __shared__ double dloc[];
  const int g = blockIdx.x;
  const int base = A.reg_ptr[g], rend = A.reg_ptr[g + 1];
  const int w0 = A.wave_ptr[g], w1 = A.wave_ptr[g + 1];
  const unsigned full = 0xffffffffu;
  const jv::Trace T = jv::trace_begin();
  // software pipeline: descriptors 3 waves ahead (L2-prefetched 6 ahead),
  // values L2-prefetched 2 ahead and loaded 1 ahead
  for (int w = w0; w < w0 + 6; ++w) prefetch_desc(A, w, w1, rend);
  WaveDesc cur = load_desc(A, w0, w1, rend);
  WaveDesc d1 = load_desc(A, w0 + 1, w1, rend);
  WaveDesc d2 = load_desc(A, w0 + 2, w1, rend);
  prefetch_vals(A, d1);
  prefetch_vals(A, d2);
  WaveVals cv = load_vals(A, cur);
  for (int w = w0; w < w1; ++w) {
    if (threadIdx.x == 0) jv::trace_mark(T, w, 1);
    prefetch_desc(A, w + 6, w1, rend);
    const WaveDesc d3 = load_desc(A, w + 3, w1, rend);
    prefetch_vals(A, d2);
    const WaveVals nv = load_vals(A, d1);
    const bool sync = A.wave_beg[w] < 0;
    const int i = cur.i;
    const bool active = i >= 0;
    const int nL = cur.inf & 7, pub = (cur.inf >> 3) & 1, umask = cur.inf >> 4;
    double dv[4];
    unsigned miss = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      dv[k] = 1.0;
      if (active && k < nL) {
        if (cur.ref[k] >= 0) dv[k] = dloc[cur.ref[k]];
        else miss |= 1u << k;
      }
    }
    if (threadIdx.x == 0) jv::trace_mark(T, w, 2);
    // remote pivots: warp-converged mailbox probes
    unsigned ns = 0, spins = 0;
    while (__any_sync(full, miss)) {
      unsigned long long p0[4], p1[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (miss & (1u << k))
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(p0[k]), "=l"(p1[k]) : "l"(A.mbox + 2 * (long long)(-1 - cur.ref[k])));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if ((miss & (1u << k)) && (uint32_t)(p0[k] >> 32) == A.epoch &&
            (uint32_t)(p1[k] >> 32) == A.epoch) {
          dv[k] = __longlong_as_double((long long)((p0[k] & 0xffffffffull) | (p1[k] << 32)));
          miss &= ~(1u << k);
        }
      }
      if (__any_sync(full, miss)) {
        if (ns) __nanosleep(ns);
        ns = ns ? min(2 * ns, 64u) : 16u;
        if (++spins == jv::g_spin_limit) {
          atomicExch(&jv::g_hang, 1);
          break;
        }
      }
    }
    if (threadIdx.x == 0) jv::trace_mark(T, w, 3);
    if (active) {
      const int row = (A.tau > 0.0) ? __ldg(A.slot_row + i) : 0;
      const double thresh = A.tau > 0.0 ? jv::dmul(A.tau, __ldg(A.norms + row)) : 0.0;
      double l[4];
      jv::ddiv_batch<4>(cv.a, dv, l, nL);
      double d = cv.arr;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < nL) {
          const bool drop = A.tau > 0.0 && fabs(l[k]) < thresh;
          if (drop) l[k] = 0.0;
          else if (umask & (1 << k)) d = jv::dsub(d, jv::dmul(l[k], cv.u[k]));
        }
      }
      dloc[i - base] = d;
      if (pub) jv::mbox_put(A.mbox, cur.rs + nL, d, A.epoch);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nL) __stcg(A.val + cur.rs + k, l[k]);
      __stcg(A.val + cur.rs + nL, d);
      if (d == 0.0) atomicMin(A.err, __ldg(A.slot_row + i));
    }
    if (threadIdx.x == 0) jv::trace_mark(T, w, 4);
    if (sync) __syncthreads();
    if (threadIdx.x == 0) jv::trace_mark(T, w, 7);
    cur = d1;
    cv = nv;
    d1 = d2;
    d2 = d3;
  }
}

}  // namespace

extern "C" int jv_factor_regions(int32_t n, int32_t nreg, const int32_t* slot_row,
                                 const int32_t* info, const int32_t* drs, const int32_t* ref,
                                 const int32_t* us, const int32_t* reg_ptr, const int32_t* wave_ptr,
                                 const int32_t* wave_beg, int32_t max_region, double* val,
                                 const double* norms, double tau, uint64_t* mbox, uint32_t epoch,
                                 int32_t* err_row, void* stream) {
  if (n < 0 || nreg < 1 || epoch == 0) {
    jvh::set_error("jv_factor_regions: bad argument");
    return JV_EINVAL;
  }
  if (n == 0) return JV_OK;
  const size_t smem = sizeof(double) * (size_t)max_region;
  if (smem > 220 * 1024) {
    jvh::set_error("jv_factor_regions: region of %d rows exceeds shared memory", max_region);
    return JV_ENOMEM;
  }
  cudaError_t e = cudaFuncSetAttribute((const void*)region_factor_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_factor_regions attr");
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, region_factor_kernel, kRegThreads, smem);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_factor_regions occupancy");
  if (per_sm * jvh::sm_count() < nreg) {
    jvh::set_error("jv_factor_regions: %d regions but only %d resident CTAs", nreg,
                   per_sm * jvh::sm_count());
    return JV_ECOOP;
  }
  RegionArgs A{slot_row, info, drs, ref, us, n, val, norms, tau, reg_ptr, wave_ptr, wave_beg,
               mbox, epoch, err_row};
  void* args[] = {&A};
  e = cudaLaunchCooperativeKernel((const void*)region_factor_kernel, dim3(nreg), dim3(kRegThreads),
                                  args, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_factor_regions");
  return JV_OK;
}

extern "C" int jv_region_threads(void) { return kRegThreads; }
