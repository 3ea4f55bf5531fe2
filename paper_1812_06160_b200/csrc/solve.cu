// Sync-free sparse triangular solves (stri) over the combined L|U storage.
//
// Reference semantics:
//   forward  (_kernels.py:348-357): y[r] = b[r] - sum_{c<r} l_rc y[c], unit L,
//            subtraction chain in ascending column order;
//   backward (_kernels.py:360-366): x[r] = (y[r] - sum_{c>r} u_rc x[c]) / u_rr.
// Every reference solve path (serial, CSR-LS, p2p, two-stage;
// trisolve.py:60-182) yields the same bits, and so does this kernel: each
// row's chain is evaluated in the reference order with explicitly rounded
// ops, dependencies awaited through mailbox packets (common.cuh).
//
// Schedule (jv_build_schedule): rows in level order of the solve's own DAG
// (forward: levels of lower(F); backward: reversed levels of upper(F)); rows
// with <= kThreadDeps dependencies come 32 to a batch (lane = row), longer
// rows (R-MAT hubs) one to a batch (warp = row: lanes gather 32 dependencies
// at a time, products formed in parallel, the subtraction chain kept in
// order by one lane).  Warp w of a co-resident grid takes batches w, w+W,
// ... (deadlock-free: batch b only waits on batches < b).  Each warp first
// waits at a gate (one lane, __nanosleep backoff) on the batch's newest
// dependency.
#include "common.cuh"
#include "../../include/jv.h"

namespace {

constexpr int kThreadDeps = 24;   // staging capacity; thread-path limit per direction below
// longer rows take the warp path: forward 24, backward 16 dependencies (swept
// 12-32 on configs 2-4: c4 forward prefers 24, c3/c4 backward 16)
constexpr int kThreadDepsFwd = 24;
constexpr int kThreadDepsBwd = 16;
constexpr int kProbe = 12;        // dependency values probed together per round (swept 8-16)
constexpr int kWarpBlock = 128;   // warp path: dependencies per prefetched block

struct SolveArgs {
  const int32_t* row_start;
  const int32_t* col;
  const double* val;
  const int32_t* diag;
  const int32_t* order;
  const int32_t* batch_ptr;
  int32_t nbatch;
  const double* in;
  double* out;
  uint64_t* mbox;
  uint32_t epoch;
  int* ticket;
};

// Converged wait: every lane re-probes its missing slots, the warp votes,
// nobody spins alone (divergent per-lane spin loops resolve slowly).
template <int N>
JV_INLINE void gather_conv(const SolveArgs& A, const int (&c)[N], double (&v)[N], unsigned miss,
                           unsigned mask) {
  unsigned ns = 0, spins = 0;
  while (__any_sync(mask, miss)) {
    unsigned long long w0[N], w1[N];
#pragma unroll
    for (int t = 0; t < N; ++t)
      if (miss & (1u << t))
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                     : "=l"(w0[t]), "=l"(w1[t]) : "l"(A.mbox + 2 * (long long)c[t]));
#pragma unroll
    for (int t = 0; t < N; ++t) {
      if ((miss & (1u << t)) && (uint32_t)(w0[t] >> 32) == A.epoch &&
          (uint32_t)(w1[t] >> 32) == A.epoch) {
        v[t] = __longlong_as_double((long long)((w0[t] & 0xffffffffull) | (w1[t] << 32)));
        miss &= ~(1u << t);
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
}

// thread path: s -= val[p] * v[col[p]] over p in [p0, p1), ascending, kProbe
// dependencies per round; `mask` = the lanes taking this path
JV_INLINE double fold_deps(const SolveArgs& A, int p0, int p1, double s, unsigned mask) {
  const int nch = (p1 - p0 + kProbe - 1) / kProbe;
  const int maxch = __reduce_max_sync(mask, (unsigned)nch);
  for (int ch = 0; ch < maxch; ++ch) {
    const int g = p0 + ch * kProbe;
    const int m = max(0, min(kProbe, p1 - g));
    int c[kProbe];
    double v[kProbe];
#pragma unroll
    for (int t = 0; t < kProbe; ++t) c[t] = (t < m) ? __ldg(A.col + g + t) : 0;
    gather_conv<kProbe>(A, c, v, m ? (1u << m) - 1 : 0u, mask);
#pragma unroll
    for (int t = 0; t < kProbe; ++t)
      if (t < m) s = jv::dsub(s, jv::dmul(__ldg(A.val + g + t), v[t]));
  }
  return s;
}

// thread path, staged: every dependency of the row (<= kThreadDeps) in two
// memory round trips — the column indices, then the values and the mailbox
// packets copied by cp.async into the warp's shared staging area (no
// registers held per dependency) — then the chain folded from shared
// memory in the reference order.  Stale packets are re-probed converged.
struct SolveStage {
  uint64_t* pk;   // [kThreadDeps][32] packets (2 words)
  double* v;      // [kThreadDeps][32] values
  int* c;         // [kThreadDeps][32] columns
};
constexpr size_t kSolveStageBytes = (size_t)kThreadDeps * 32 * (16 + 8 + 4);

JV_INLINE double fold_deps_staged(const SolveArgs& A, int p0, int p1, double s, unsigned mask,
                                  int lane, const SolveStage& St) {
  const int m = p1 - p0;
  for (int t = 0; t < m; ++t) {
    cp_async4(St.c + t * 32 + lane, A.col + p0 + t);
    cp_async8(St.v + t * 32 + lane, A.val + p0 + t);
  }
  cp_commit();
  cp_wait<0>();
  for (int t = 0; t < m; ++t)
    cp_async16(St.pk + 2 * (t * 32 + lane), A.mbox + 2 * (long long)St.c[t * 32 + lane]);
  cp_commit();
  cp_wait<0>();
  // stale packets: converged re-probes, one dependency slot at a time
  unsigned miss = 0;
  for (int t = 0; t < m; ++t) {
    const ulonglong2 pk = *reinterpret_cast<const ulonglong2*>(St.pk + 2 * (t * 32 + lane));
    if ((uint32_t)(pk.x >> 32) != A.epoch || (uint32_t)(pk.y >> 32) != A.epoch) miss |= 1u << t;
  }
  while (__any_sync(mask, miss != 0)) {
    const int t = miss ? __ffs(miss) - 1 : 0;
    int cc[1] = {St.c[t * 32 + lane]};
    double xv[1] = {0.0};
    gather_conv<1>(A, cc, xv, miss ? 1u : 0u, mask);
    if (miss) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(xv[0]);
      const unsigned long long tag = (unsigned long long)A.epoch << 32;
      St.pk[2 * (t * 32 + lane)] = tag | (b & 0xffffffffull);
      St.pk[2 * (t * 32 + lane) + 1] = tag | (b >> 32);
      miss &= miss - 1;
    }
  }
  for (int t = 0; t < m; ++t) {
    const ulonglong2 pk = *reinterpret_cast<const ulonglong2*>(St.pk + 2 * (t * 32 + lane));
    const double x = __longlong_as_double((long long)((pk.x & 0xffffffffull) | (pk.y << 32)));
    s = jv::dsub(s, jv::dmul(St.v[t * 32 + lane], x));
  }
  return s;
}

// warp path: same chain in blocks of 128 dependencies: the probes of block
// k+1 are issued before block k is folded (one L2 round trip hides behind
// the fold), products go to shared memory and one lane keeps the
// subtraction order (8-cycle DSUB chain, loads pipelined).  s is valid in
// lane 0.
JV_INLINE double fold_deps_warp(const SolveArgs& A, int p0, int p1, double s, int lane,
                                double* sp) {
  const unsigned full = 0xffffffffu;
  constexpr int K = kWarpBlock / 32;
  int c[K];
  double v[K], x[K];
  unsigned long long w0[K], w1[K];
  auto issue = [&](int g) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int p = g + 32 * j + lane;
      c[j] = p < p1 ? __ldg(A.col + p) : 0;
      v[j] = p < p1 ? __ldg(A.val + p) : 0.0;
      if (p < p1)
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                     : "=l"(w0[j]), "=l"(w1[j]) : "l"(A.mbox + 2 * (long long)c[j]));
    }
  };
  auto settle = [&](int g) {
    unsigned miss = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int p = g + 32 * j + lane;
      x[j] = 0.0;
      if (p < p1) {
        if ((uint32_t)(w0[j] >> 32) == A.epoch && (uint32_t)(w1[j] >> 32) == A.epoch)
          x[j] = __longlong_as_double((long long)((w0[j] & 0xffffffffull) | (w1[j] << 32)));
        else
          miss |= 1u << j;
      }
    }
    if (__any_sync(full, miss != 0)) gather_conv<K>(A, c, x, miss, full);
  };
  if (p0 >= p1) return s;
  issue(p0);
  for (int g = p0, blk = 0; g < p1; g += kWarpBlock, blk ^= 1) {
    settle(g);
    double* buf = sp + blk * kWarpBlock;
#pragma unroll
    for (int j = 0; j < K; ++j) buf[32 * j + lane] = jv::dmul(v[j], x[j]);
    __syncwarp();
    const int gn = g + kWarpBlock;
    if (gn < p1) issue(gn);     // next block's probes fly during the fold
    if (lane == 0) {
      const int m = min(kWarpBlock, p1 - g);
#pragma unroll 8
      for (int t = 0; t < m; ++t) s = jv::dsub(s, buf[t]);
    }
    __syncwarp();
  }
  return s;
}

template <bool kBackward>
__global__ void __launch_bounds__(256) solve_kernel(SolveArgs A) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  __shared__ double warp_prod[8][2 * kWarpBlock];
  double* sp = warp_prod[threadIdx.x >> 5];
  extern __shared__ __align__(16) unsigned char solve_stage[];
  SolveStage St;
  St.pk = reinterpret_cast<uint64_t*>(solve_stage + (threadIdx.x >> 5) * kSolveStageBytes);
  St.v = reinterpret_cast<double*>(solve_stage + (threadIdx.x >> 5) * kSolveStageBytes +
                                   (size_t)kThreadDeps * 32 * 16);
  St.c = reinterpret_cast<int*>(solve_stage + (threadIdx.x >> 5) * kSolveStageBytes +
                                (size_t)kThreadDeps * 32 * 24);
  const int W = (gridDim.x * blockDim.x) >> 5;
  const jv::Trace T = jv::trace_begin();
  for (;;) {
    const int b = jv::ticket_next(A.ticket, lane, T);
    if (b >= A.nbatch) break;
    const int lo = A.batch_ptr[b], hi = A.batch_ptr[b + 1];
    const bool active = lo + lane < hi;
    const int r = active ? A.order[lo + lane] : 0;
    // dependency range: forward [rs, diag), backward (diag, re)
    int p0 = 0, p1 = 0, dp = 0;
    if (active) {
      dp = __ldg(A.diag + r);
      if (kBackward) { p0 = dp + 1; p1 = __ldg(A.row_start + r + 1); }
      else { p0 = __ldg(A.row_start + r); p1 = dp; }
    }
    // gate: the newest dependency of the batch (forward: the largest column;
    // backward: the smallest column > r)
    int g;
    if (kBackward) {
      g = (active && p1 > p0) ? __ldg(A.col + p0) : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g = min(g, __shfl_xor_sync(full, g, o));
      if (lane == 0 && g != 0x7fffffff && (jv::g_gate & 2)) jv::mbox_gate(A.mbox, g, A.epoch);
    } else {
      g = (active && p1 > p0) ? __ldg(A.col + p1 - 1) : -1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g = max(g, __shfl_xor_sync(full, g, o));
      if (lane == 0 && g >= 0 && (jv::g_gate & 2)) jv::mbox_gate(A.mbox, g, A.epoch);
    }
    __syncwarp();
    const bool small = p1 - p0 <= (kBackward ? kThreadDepsBwd : kThreadDepsFwd);
    const unsigned smask = __ballot_sync(full, active && small);
    if (active && small) {
      double s = jv::g_solve_staged ? fold_deps_staged(A, p0, p1, A.in[r], smask, lane, St)
                                    : fold_deps(A, p0, p1, A.in[r], smask);
      if (kBackward) {
        const double d = __ldg(A.val + dp);
        bool slow;
        const double q = jv::ddiv_fast(s, d, slow);
        s = slow ? __ddiv_rn(s, d) : q;
      }
      A.out[r] = s;
      jv::mbox_put(A.mbox, r, s, A.epoch);
    }
    unsigned pend = __ballot_sync(full, active && !small);
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1;
      const int rr = __shfl_sync(full, r, src);
      const int q0 = __shfl_sync(full, p0, src), q1 = __shfl_sync(full, p1, src);
      double s = fold_deps_warp(A, q0, q1, A.in[rr], lane, sp);
      if (lane == 0) {
        if (kBackward) s = jv::ddiv(s, __ldg(A.val + __ldg(A.diag + rr)));
        A.out[rr] = s;
        jv::mbox_put(A.mbox, rr, s, A.epoch);
      }
      __syncwarp();
    }
  }
  jv::ticket_exit(A.ticket, lane, W);
}

// One level of the paper's CSR-LS baseline (trisolve.py:74-108,
// _kernels.py:369-401): thread per row of the level, the row's chain in the
// reference order; the levels run as consecutive launches (captured into a
// CUDA graph by the host), the launch boundary standing in for the
// reference's barrier.
__global__ void __launch_bounds__(256) level_solve_kernel(int which, const int32_t* rs,
                                                          const int32_t* col, const double* val,
                                                          const int32_t* diag,
                                                          const int32_t* order, int lo, int hi,
                                                          const double* in, double* out) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const int r = order[i];
  double s = in[r];
  if (which == 0) {
    for (int p = rs[r]; p < diag[r]; ++p) s = jv::dsub(s, jv::dmul(val[p], out[col[p]]));
  } else {
    const int d = diag[r];
    for (int p = d + 1; p < rs[r + 1]; ++p) s = jv::dsub(s, jv::dmul(val[p], out[col[p]]));
    s = jv::ddiv(s, val[d]);
  }
  out[r] = s;
}

__global__ void check_zero_diag_kernel(int n, const double* val, const int32_t* diag, int32_t* row) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    if (val[diag[r]] == 0.0) atomicMin(row, r);
}

__global__ void classify_solve_kernel(int n, const int32_t* rs, const int32_t* diag, int backward,
                                      int32_t* cls) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int deps = backward ? rs[r + 1] - diag[r] - 1 : diag[r] - rs[r];
    cls[r] = deps > (backward ? kThreadDepsBwd : kThreadDepsFwd) ? 1 : 0;
  }
}

}  // namespace

extern "C" int jv_solve(int which, int32_t n, const int32_t* row_start, const int32_t* col,
                        const double* val, const int32_t* diag_pos, const int32_t* order,
                        const int32_t* batch_ptr, int32_t nbatch, const double* in, double* out,
                        uint64_t* mbox, uint32_t epoch, int32_t* ticket, void* stream) {
  if (n < 0 || nbatch < 0 || epoch == 0 || (which != 0 && which != 1)) {
    jvh::set_error("jv_solve: bad argument (which=%d n=%d nbatch=%d epoch=%u)", which, n,
                   nbatch, epoch);
    return JV_EINVAL;
  }
  if (n == 0 || nbatch == 0) return JV_OK;
  SolveArgs A{row_start, col, val, diag_pos, order, batch_ptr, nbatch, in, out, mbox, epoch, ticket};
  void* args[] = {&A};
  if (which == 0)
    return jvh::persistent_launch(solve_kernel<false>, 256, args, (cudaStream_t)stream, "jv_solve fwd",
                                  8 * kSolveStageBytes);
  return jvh::persistent_launch(solve_kernel<true>, 256, args, (cudaStream_t)stream, "jv_solve bwd",
                                8 * kSolveStageBytes);
}

extern "C" int jv_solve_level(int which, const int32_t* row_start, const int32_t* col,
                              const double* val, const int32_t* diag_pos, const int32_t* order,
                              int32_t lo, int32_t hi, const double* in, double* out, void* stream) {
  if (hi <= lo) return JV_OK;
  level_solve_kernel<<<(hi - lo + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      which, row_start, col, val, diag_pos, order, lo, hi, in, out);
  JV_CHECK_LAUNCH("jv_solve_level");
  return JV_OK;
}

extern "C" int jv_check_zero_diag(int32_t n, const double* val, const int32_t* diag_pos,
                                  int32_t* row, void* stream) {
  if (n <= 0) return JV_OK;
  int grid = (n + 255) / 256;
  if (grid > 4 * jvh::sm_count()) grid = 4 * jvh::sm_count();
  check_zero_diag_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, val, diag_pos, row);
  JV_CHECK_LAUNCH("jv_check_zero_diag");
  return JV_OK;
}

extern "C" int jv_classify_solve(int which, int32_t n, const int32_t* row_start,
                                 const int32_t* diag_pos, int32_t* cls, void* stream) {
  if (n <= 0) return JV_OK;
  classify_solve_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, row_start, diag_pos,
                                                                         which, cls);
  JV_CHECK_LAUNCH("jv_classify_solve");
  return JV_OK;
}

// ---------------------------------------------------------------------
// Small systems: one triangular sweep in ONE thread block with everything
// in shared memory — the vector, the sweep's dependency entries (column,
// value) of every row compacted by a per-row prefix, the diagonal
// (backward), the level-ordered row list and the level pointers.  Levels
// are separated by __syncthreads (no cross-SM hop, no producer pipeline),
// a thread takes one row of the level and runs the reference chain
// (_kernels.py:348-366: s -= val*x in ascending column order, backward
// divided by the diagonal, every op rounded separately) — bitwise the other
// paths.  Config 1 (4,096 rows, 127 levels): ~0.1 us per level.
namespace {

constexpr int kSmallThreads = 1024;

struct SmallArgs {
  int which, n, nlev, nent, active, width;
  const int32_t* rs;
  const int32_t* col;
  const double* val;
  const int32_t* diag;
  const int32_t* order;
  const int32_t* lptr;
  const int32_t* estart;
  const double* in;
  double* out;
};

__host__ __device__ inline size_t small_bytes(int which, int n, int nlev, long long nent) {
  return 8ull * n + (which ? 8ull * n : 0) + 8ull * nent + 4ull * nent + 4ull * (n + 1) +
         4ull * n + 4ull * (nlev + 1) + 32;
}

__global__ void __launch_bounds__(kSmallThreads, 1) solve_small_kernel(SmallArgs A) {
  extern __shared__ __align__(16) unsigned char ssm[];
  const int n = A.n, tid = threadIdx.x;
  double* x = reinterpret_cast<double*>(ssm);
  double* sd = x + n;                                   // backward only
  double* sv = sd + (A.which ? n : 0);
  int32_t* sc = reinterpret_cast<int32_t*>(sv + A.nent);
  int32_t* se = sc + A.nent + (A.nent & 1);             // [n + 1]
  int32_t* so = se + n + 1;                             // [n] rows in level order
  int32_t* sl = so + n;                                 // [nlev + 1]
  // staging, all 1024 threads: four rows per thread at a time, their bounds
  // loaded together and then their entries, so the dependent global round
  // trips are paid per batch of 4096 rows, not per row
  for (int i = tid; i <= n; i += kSmallThreads) se[i] = A.estart[i];
  for (int i = tid; i < n; i += kSmallThreads) so[i] = A.order[i];
  for (int i = tid; i <= A.nlev; i += kSmallThreads) sl[i] = A.lptr[i];
  constexpr int kB = 4;
  for (int r0 = tid; r0 < n; r0 += kB * kSmallThreads) {
    int a[kB], e0[kB], cnt[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int r = r0 + j * kSmallThreads;
      cnt[j] = 0;
      if (r < n) {
        const int d = A.diag[r];
        a[j] = A.which ? d + 1 : A.rs[r];
        e0[j] = A.estart[r];
        cnt[j] = A.estart[r + 1] - e0[j];
        x[r] = A.in[r];
        if (A.which) sd[r] = A.val[d];
      }
    }
    int most = 0;
#pragma unroll
    for (int j = 0; j < kB; ++j) most = max(most, cnt[j]);
    for (int k = 0; k < most; ++k) {
#pragma unroll
      for (int j = 0; j < kB; ++j)
        if (k < cnt[j]) {
          sc[e0[j] + k] = A.col[a[j] + k];
          sv[e0[j] + k] = A.val[a[j] + k];
        }
    }
  }
  __syncthreads();
  // the sweep: only as many warps as the widest level needs stay (a barrier
  // over 2 warps is much cheaper than over 32; exited threads do not count)
  const int nt = A.active;
  if (tid >= nt) return;
  if (A.width <= nt) {
    // One row per thread and level: everything a row needs except the x
    // values it depends on is independent of the sweep, so it is fetched
    // through a register pipeline three levels deep (level bounds -> row ->
    // entry range and diagonal -> first four entries); each shared-memory
    // load is consumed an iteration after it was issued, and only
    // x[col] -> chain -> store -> barrier stays on the per-level path.
    const int nlev = A.nlev;
    auto bounds_of = [&](int L) { return L < nlev ? make_int2(sl[L] + tid, sl[L + 1]) : make_int2(0, 0); };
    auto row_of = [&](int2 b) { return b.x < b.y ? so[b.x] : -1; };
    struct Row { int r, e0, cnt; double d, xin; };
    auto range_of = [&](int r) {
      Row o{r, 0, 0, 1.0, 0.0};
      if (r >= 0) {
        o.e0 = se[r];
        o.cnt = se[r + 1] - o.e0;
        o.xin = x[r];                       // still the right-hand side: only its owner writes it
        if (A.which) o.d = sd[r];
      }
      return o;
    };
    Row C = range_of(row_of(bounds_of(0)));
    Row B = range_of(row_of(bounds_of(1)));
    int rA = row_of(bounds_of(2));
    int2 bn = bounds_of(3);
    double cv[4];
    int cc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cv[k] = k < C.cnt ? sv[C.e0 + k] : 0.0;
      cc[k] = k < C.cnt ? sc[C.e0 + k] : 0;
    }
    for (int L = 0; L < nlev; ++L) {
      if (C.r >= 0) {
        double s = C.xin;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < C.cnt) s = jv::dsub(s, jv::dmul(cv[k], x[cc[k]]));
        for (int e = C.e0 + 4; e < C.e0 + C.cnt; ++e) s = jv::dsub(s, jv::dmul(sv[e], x[sc[e]]));
        if (A.which) s = jv::ddiv(s, C.d);
        x[C.r] = s;
      }
      // advance the pipeline (none of these loads is used before the next iteration)
      C = B;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cv[k] = k < C.cnt ? sv[C.e0 + k] : 0.0;
        cc[k] = k < C.cnt ? sc[C.e0 + k] : 0;
      }
      B = range_of(rA);
      rA = row_of(bn);
      bn = bounds_of(L + 4);
      __syncthreads();
    }
    for (int r = tid; r < n; r += nt) A.out[r] = x[r];
    return;
  }
  for (int L = 0; L < A.nlev; ++L) {
    const int hi = sl[L + 1];
    for (int i = sl[L] + tid; i < hi; i += nt) {
      const int r = so[i];
      double s = x[r];
      const int e1 = se[r + 1];
      for (int e = se[r]; e < e1; ++e) s = jv::dsub(s, jv::dmul(sv[e], x[sc[e]]));
      if (A.which) s = jv::ddiv(s, sd[r]);
      x[r] = s;
    }
    __syncthreads();
  }
  for (int r = tid; r < n; r += nt) A.out[r] = x[r];
}

}  // namespace

// bytes of shared memory one sweep needs (the host compares with jv_solve_small_max())
extern "C" int64_t jv_solve_small_bytes(int which, int32_t n, int32_t nlev, int64_t nent) {
  return (int64_t)small_bytes(which, n, nlev, nent);
}
extern "C" int64_t jv_solve_small_max(void) { return 220 * 1024; }

/* One sweep of a small system in one thread block (replaces _kernels.py:348-366 for
 * systems that fit shared memory): order = rows sorted by level of the sweep's DAG,
 * lptr[nlev + 1] the level bounds in it, estart[n + 1] the prefix sum of the rows'
 * dependency counts (forward: strict-lower entries, backward: strict-upper); width the
 * largest level (picks the block size).                                           */
extern "C" int jv_solve_small(int which, int32_t n, const int32_t* row_start, const int32_t* col,
                              const double* val, const int32_t* diag_pos, const int32_t* order,
                              const int32_t* lptr, int32_t nlev, const int32_t* estart,
                              int64_t nent, int32_t width, const double* in, double* out,
                              void* stream) {
  if (n < 0 || nlev < 0 || nent < 0 || (which != 0 && which != 1)) {
    jvh::set_error("jv_solve_small: bad argument");
    return JV_EINVAL;
  }
  if (n == 0) return JV_OK;
  const size_t bytes = small_bytes(which, n, nlev, nent);
  if (bytes > (size_t)jv_solve_small_max()) {
    jvh::set_error("jv_solve_small: system does not fit shared memory (%zu bytes)", bytes);
    return JV_EINVAL;
  }
  static bool once = [] {
    cudaFuncSetAttribute(solve_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)jv_solve_small_max());
    return true;
  }();
  (void)once;
  const int active = min(kSmallThreads, max(64, (width + 31) / 32 * 32));
  SmallArgs A{which, n, nlev, (int)nent, active, width, row_start, col, val, diag_pos, order, lptr,
              estart, in, out};
  solve_small_kernel<<<1, kSmallThreads, bytes, (cudaStream_t)stream>>>(A);
  JV_CHECK_LAUNCH("jv_solve_small");
  return JV_OK;
}
