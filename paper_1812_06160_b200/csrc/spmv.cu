// CSR spmv, y = A x (fp64), for sm_100a.
//
// Reference semantics: _kernels.py:28-34 — per row, s = 0; s += val[p]*x[col[p]]
// in ascending p, each product and sum rounded separately (no FMA).
//
// Layout of the work (CSR-stream): CTA t owns the rows whose first nonzero
// lies in [t*kTile, (t+1)*kTile).  Its threads first compute the products
// val[p]*x[col[p]] fully coalesced (val/col streamed once: 12 B/nnz) into
// shared memory, then each row is summed serially from shared memory by one
// thread in the reference order — so every row of up to kTile+1 entries is
// BITWISE equal to the reference while global traffic stays at the
// 12 nnz + 20 n algorithmic bytes.  A row longer than kTile (R-MAT hubs)
// has its products formed by the whole CTA chunk by chunk and summed by one
// thread in order, so it is bitwise too.  The tile -> first-row map is a setup-time plan
// (jv_spmv_plan); without it each CTA binary-searches row_start.
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "../../include/jv.h"

namespace {

#ifndef JV_SPMV_THREADS
#define JV_SPMV_THREADS 128
#endif
#ifndef JV_SPMV_TILE
#define JV_SPMV_TILE 512
#endif
constexpr int kSpmvThreads = JV_SPMV_THREADS;
constexpr int kTile = JV_SPMV_TILE;  // nonzeros per CTA tile
constexpr int kBuf = 2 * kTile;      // shared products: any row <= kTile fits

// first row in [0, n) whose start is >= key (n if none)
JV_INLINE int row_lower_bound(const int32_t* rs, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(rs + mid) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void spmv_plan_kernel(int n, int nnz, int ntiles, const int32_t* rs, int32_t* tile_rows) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles; t += gridDim.x * blockDim.x) {
    int r;
    if (t == 0) r = 0;
    else if (t == ntiles) r = n;
    else r = row_lower_bound(rs, n, t * kTile);
    tile_rows[2 * t] = r;
    tile_rows[2 * t + 1] = rs[r];
  }
}

__global__ void __launch_bounds__(kSpmvThreads) spmv_stream_kernel(
    int n, int nnz, const int32_t* __restrict__ rs, const int32_t* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
    const int32_t* __restrict__ tile_rows, const int32_t* __restrict__ row_map) {
  __shared__ double prod[kBuf];
  const int t = blockIdx.x;
  const int ntiles = gridDim.x;
  int r0, r1, p0, p1;
  if (tile_rows) {
    // (first row, its first nonzero) of this tile and the next: one load
    const int2 a = __ldg(reinterpret_cast<const int2*>(tile_rows) + t);
    const int2 b = __ldg(reinterpret_cast<const int2*>(tile_rows) + t + 1);
    r0 = a.x; p0 = a.y; r1 = b.x; p1 = b.y;
  } else {
    r0 = (t == 0) ? 0 : row_lower_bound(rs, n, t * kTile);
    r1 = (t == ntiles - 1) ? n : row_lower_bound(rs, n, (t + 1) * kTile);
    p0 = __ldg(rs + r0);
    p1 = __ldg(rs + r1);
  }
  if (r0 >= r1) return;
  int rlast = r1;
  if (p1 - p0 > kBuf) {        // the tile's last row is longer than kTile
    rlast = r1 - 1;
    p1 = __ldg(rs + rlast);
  }
  // the first summed row's bounds are loaded now, behind the products'
  // loads, not after the barrier
  const int rfirst = r0 + threadIdx.x;
  int ra = 0, rb = 0;
  if (rfirst < rlast) {
    ra = __ldg(rs + rfirst);
    rb = __ldg(rs + rfirst + 1);
  }
  // products, kU independent load chains per thread in flight (col -> x)
  constexpr int kU = 8;
  for (int b = p0 + threadIdx.x; b < p1; b += kSpmvThreads * kU) {
    int c[kU];
    double v[kU], xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = b + u * kSpmvThreads;
      c[u] = p < p1 ? __ldcs(col + p) : 0;
      v[u] = p < p1 ? __ldcs(val + p) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = b + u * kSpmvThreads;
      if (p < p1) prod[p - p0] = jv::dmul(v[u], xv[u]);
    }
  }
  __syncthreads();
  for (int r = rfirst; r < rlast; r += kSpmvThreads) {
    const int a = (r == rfirst ? ra : __ldg(rs + r)) - p0;
    const int b = (r == rfirst ? rb : __ldg(rs + r + 1)) - p0;
    double s = 0.0;
    for (int q = a; q < b; ++q) s = jv::dadd(s, prod[q]);
    __stcs(y + (row_map ? __ldg(row_map + r) : r), s);
  }
  if (rlast == r1) return;
  // a row longer than a tile (R-MAT hubs): its products chunk by chunk in
  // shared memory (all threads, coalesced), summed serially by one thread in
  // the reference order — bitwise like every other row
  const int a = __ldg(rs + rlast), b = __ldg(rs + rlast + 1);
  double acc = 0.0;
  for (int c0 = a; c0 < b; c0 += kBuf) {
    const int c1 = c0 + kBuf < b ? c0 + kBuf : b;
    __syncthreads();
    for (int q = c0 + threadIdx.x; q < c1; q += kSpmvThreads)
      prod[q - c0] = jv::dmul(__ldcs(val + q), __ldg(x + __ldcs(col + q)));
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < c1 - c0; ++q) acc = jv::dadd(acc, prod[q]);
  }
  if (threadIdx.x == 0) y[row_map ? row_map[rlast] : rlast] = acc;
}


// ---------------------------------------------------------------------
// Persistent bulk-copy variant (large matrices; needs the jv_spmv_plan map).
// The nonzero stream is cut into tiles of T = M*kTile entries; CTA b walks
// the tiles [b*tpc, (b+1)*tpc):
//   * one thread bulk-copies (TMA, cp.async.bulk + mbarrier complete_tx) the
//     col and val tiles S tiles ahead into a shared-memory ring — S*12T
//     bytes per CTA in flight at no register or LSU cost;
//   * the x gathers of tile j+1 are issued (col read from shared memory)
//     before the row sums of tile j, so their L2/DRAM latency runs beside
//     the sums; products go to a double-buffered shared array;
//   * the rows that START in tile k are [F_k, F_{k+1}) with F from the plan
//     (first row whose first nonzero is >= k*T), so every tile's row range —
//     and the row bounds its threads need — is known a tile ahead, without
//     searching; each row that ENDS in the tile is summed serially by one
//     thread in the reference order; the one row that runs on into the next
//     tile hands its partial sum over in shared memory (the sum stays one
//     left-to-right chain: bitwise the reference for rows of any length).
// A CTA whose first tile begins inside a row first folds that row's earlier
// entries (whole CTA forms the products chunk by chunk, one thread adds them
// in order).  Global traffic is the 12 nnz + 20 n algorithmic bytes.
template <int T, int S, int NT>
struct BulkSmem {
  double val[S][T];
  double prod[2][T];
  int32_t col[S][T];
  uint64_t bar[S];
  double carry[2];
};

JV_INLINE uint32_t sp_sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
JV_INLINE void sp_bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SW_%=;\n}" ::"r"(sp_sa(b)), "r"(parity) : "memory");
}
JV_INLINE void sp_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;"
      ::"r"(sp_sa(dst)), "l"(src), "r"(bytes), "r"(sp_sa(b)), "l"(pol) : "memory");
}

template <int T, int S, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) spmv_bulk_kernel(
    int n, int nnz, int ntiles, int tpc, int staged, const int32_t* __restrict__ rs,
    const int32_t* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y, const int2* __restrict__ plan,
    const int32_t* __restrict__ row_map) {
  static_assert(T % kTile == 0 && T % NT == 0, "plan entries are per kTile nonzeros");
  constexpr int kM = T / kTile;
  constexpr int kU = T / NT;
  extern __shared__ __align__(128) unsigned char sp_raw[];
  BulkSmem<T, S, NT>& sm = *reinterpret_cast<BulkSmem<T, S, NT>*>(sp_raw);
  const int tid = threadIdx.x;
  const int kb = blockIdx.x * tpc;
  const int nt = min(kb + tpc, ntiles) - kb;   // > 0 by the grid's construction
  // (first row starting at or behind tile k's first nonzero, that row's start)
  auto first_row = [&](int k) { return k >= ntiles ? make_int2(n, nnz) : __ldg(plan + kM * k); };
  uint64_t pol = 0;
  if (tid == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sp_sa(&sm.bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nfull = staged ? nnz / T - kb : 0;   // the CTA's tiles j < nfull arrive by bulk copy
  auto is_full = [&](int j) { return j < nfull; };
  auto issue = [&](int j) {   // thread 0: fetch the CTA's j-th tile into its ring stage
    if (!is_full(j)) return;
    const long long p = (long long)(kb + j) * T;
    uint64_t* bar = &sm.bar[j % S];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(sp_sa(bar)), "r"((uint32_t)(T * 12)) : "memory");
    sp_bulk(sm.val[j % S], val + p, T * 8, bar, pol);
    sp_bulk(sm.col[j % S], col + p, T * 4, bar, pol);
  };
  if (tid == 0)
    for (int j = 0; j < S && j < nt; ++j) issue(j);

  int2 f0 = first_row(kb), f1 = first_row(kb + 1), f2 = first_row(kb + 2);
  // a row running into the CTA's first tile: fold its earlier entries
  {
    const int ts0 = kb * T;
    double acc = 0.0;
    if (f0.y > ts0) {
      const int a = __ldg(rs + f0.x - 1);
      for (int c0 = a; c0 < ts0; c0 += T) {
        const int c1 = min(c0 + T, ts0);
        __syncthreads();
        for (int q = c0 + tid; q < c1; q += NT)
          sm.prod[1][q - c0] = jv::dmul(__ldg(val + q), __ldg(x + __ldg(col + q)));
        __syncthreads();
        if (tid == 0)
          for (int q = 0; q < c1 - c0; ++q) acc = jv::dadd(acc, sm.prod[1][q]);
      }
    }
    if (tid == 0) sm.carry[0] = acc;   // read behind the first tile's barrier
  }

  // gathers of one tile: x values (and, for an unstaged tile, the matrix values) in registers
  double xv[kU], vv[kU];
  auto gather = [&](int j) {
    const int ts = (kb + j) * T;
    if (is_full(j)) {
      sp_bar_wait(&sm.bar[j % S], (uint32_t)((j / S) & 1));
      const int32_t* sc = sm.col[j % S];
#pragma unroll
      for (int u = 0; u < kU; ++u) xv[u] = __ldg(x + sc[tid + u * NT]);
    } else {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int q = ts + tid + u * NT;
        const bool in = q < nnz;
        vv[u] = in ? __ldcs(val + q) : 0.0;
        xv[u] = in ? __ldg(x + __ldcs(col + q)) : 0.0;
      }
    }
  };
  int rc = f0.x - (f0.y > kb * T ? 1 : 0);   // first row ending in the current tile
  int r0 = rc + tid, ra = 0, rb = 0;          // this thread's first row of the tile, its bounds
  if (r0 < f1.x) { ra = __ldg(rs + r0); rb = __ldg(rs + r0 + 1); }
  gather(0);
  for (int j = 0; j < nt; ++j) {
    const int k = kb + j;
    const int ts = k * T;
    const int te = (int)min((long long)ts + T, (long long)nnz);
    double* prod = sm.prod[j & 1];
    if (is_full(j)) {
      const double* sv = sm.val[j % S];
#pragma unroll
      for (int u = 0; u < kU; ++u) prod[tid + u * NT] = jv::dmul(sv[tid + u * NT], xv[u]);
    } else {
#pragma unroll
      for (int u = 0; u < kU; ++u) prod[tid + u * NT] = jv::dmul(vv[u], xv[u]);
    }
    __syncthreads();
    // the tile's ring stage is free: refill it; then the next tile's gathers and row bounds
    if (tid == 0 && j + S < nt) issue(j + S);
    const int2 f3 = first_row(k + 3);              // used two tiles on: never waited for
    const int rl = f1.x - 1;                       // last row starting in this tile
    const int rcn = f1.x - (f1.y > te ? 1 : 0);    // first row ending in the next tile
    const int rn0 = rcn + tid;
    int rna = 0, rnb = 0;
    if (j + 1 < nt) {
      if (rn0 < f2.x) { rna = __ldg(rs + rn0); rnb = __ldg(rs + rn0 + 1); }
      gather(j + 1);
    }
    const double cin = sm.carry[j & 1];
    for (int r = r0; r <= rl; r += NT) {
      if (r != r0) { ra = __ldg(rs + r); rb = __ldg(rs + r + 1); }
      double s = r == rc ? cin : 0.0;
      const int qb = min(rb, te) - ts;
      int q = max(ra, ts) - ts;
      // eight loads in flight (clamped inside the tile), added in order; the
      // predicated adds keep short rows in one pass without a remainder loop
      for (; q < qb; q += 8) {
        double pv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pv[i] = prod[min(q + i, T - 1)];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (q + i < qb) s = jv::dadd(s, pv[i]);
      }
      if (rb <= te) {
        __stcs(y + (row_map ? __ldg(row_map + r) : r), s);
        if (r == rl) sm.carry[(j + 1) & 1] = 0.0;
      } else {
        sm.carry[(j + 1) & 1] = s;   // r == rl: the row runs on into the next tile
      }
    }
    f1 = f2;
    f2 = f3;
    rc = rcn;
    r0 = rn0;
    ra = rna;
    rb = rnb;
  }
}

int g_spmv_impl = -1;   // -1 auto, 0 stream, 1 bulk

// plan pointer -> "has rows spanning kLongRun whole tiles" (jv_spmv_plan)
std::mutex g_spmv_mu;
std::unordered_map<const void*, bool> g_spmv_long;
constexpr int kLongRun = 2;

// longest run of consecutive tiles in which no row starts (capped at 64)
__global__ void spmv_plan_stat_kernel(int ntiles, const int32_t* tile_rows, int* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles || tile_rows[2 * t] != tile_rows[2 * t + 2]) return;
  if (t > 0 && tile_rows[2 * t - 2] == tile_rows[2 * t]) return;   // not the run's first tile
  int r = 1;
  while (r < 64 && t + r < ntiles && tile_rows[2 * (t + r)] == tile_rows[2 * (t + r) + 2]) ++r;
  atomicMax(out, r);
}

template <int M, int S, int NT, int MINB = 1>
void spmv_bulk_launch(int n, int nnz, const int32_t* rs, const int32_t* col, const double* val,
                      const double* x, double* y, const int32_t* tile_rows,
                      const int32_t* row_map, cudaStream_t st) {
  constexpr int T = M * kTile;
  using Sm = BulkSmem<T, S, NT>;
  static int resident = [] {
    cudaFuncSetAttribute(spmv_bulk_kernel<T, S, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(Sm));
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmv_bulk_kernel<T, S, NT, MINB>, NT,
                                                  sizeof(Sm));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return max(occ, 1) * sms;
  }();
  const int ntiles = (int)(((long long)nnz + T - 1) / T);
  const int tpc = (ntiles + resident - 1) / resident;
  const int grid = (ntiles + tpc - 1) / tpc;
  const int staged =
      ((reinterpret_cast<uintptr_t>(col) | reinterpret_cast<uintptr_t>(val)) & 15) == 0;
  spmv_bulk_kernel<T, S, NT, MINB><<<grid, NT, sizeof(Sm), st>>>(
      n, nnz, ntiles, tpc, staged, rs, col, val, x, y, reinterpret_cast<const int2*>(tile_rows),
      row_map);
}

bool spmv_use_bulk(int nnz, const int32_t* tile_rows) {
  static const int env = [] {
    const char* e = getenv("JV_SPMV_IMPL");
    return e ? atoi(e) : -1;
  }();
  const int impl = g_spmv_impl >= 0 ? g_spmv_impl : env;
  bool bulk = tile_rows != nullptr && nnz > 0 && (impl == 1 || (impl < 0 && nnz >= (1 << 20)));
  if (bulk && impl < 0) {
    std::lock_guard<std::mutex> lock(g_spmv_mu);
    auto it = g_spmv_long.find(tile_rows);
    if (it != g_spmv_long.end() && it->second) bulk = false;
  }
  return bulk;
}

void spmv_launch(int n, int nnz, const int32_t* rs, const int32_t* col, const double* val,
                 const double* x, double* y, const int32_t* tile_rows, const int32_t* row_map,
                 cudaStream_t st) {
  static const int cfg = [] {
    const char* e = getenv("JV_SPMV_CFG");   // tuning: ring depth / threads of the bulk kernel
    return e ? atoi(e) : 0;
  }();
  const bool bulk = spmv_use_bulk(nnz, tile_rows);
  if (!bulk) {
    const int ntiles = nnz > 0 ? (nnz + kTile - 1) / kTile : 1;
    spmv_stream_kernel<<<ntiles, kSpmvThreads, 0, st>>>(n, nnz, rs, col, val, x, y, tile_rows,
                                                       row_map);
    return;
  }
#define JV_SPMV_ARGS n, nnz, rs, col, val, x, y, tile_rows, row_map, st
  // ring shape (tile = M*kTile, S stages, threads, CTAs/SM the registers are bounded for);
  // c2 right after a sweep / back to back: <1,2,128> 47.1 / 42.7 us, <2,2,256> 49.2 / 41.5,
  // <2,3,256> 54.8 / 45.7 — a deeper ring costs L1 (the x gathers' cache) more than its extra
  // bytes in flight gain
  switch (cfg) {
    case 1: spmv_bulk_launch<2, 2, 256, 4>(JV_SPMV_ARGS); break;
    case 2: spmv_bulk_launch<2, 3, 256, 4>(JV_SPMV_ARGS); break;
    default: spmv_bulk_launch<1, 2, 128, 9>(JV_SPMV_ARGS); break;
  }
#undef JV_SPMV_ARGS
}

}  // namespace

extern "C" int jv_spmv_tile(void) { return kTile; }

// -1: by size (bulk from 2^20 nonzeros), 0: CTA-per-tile stream kernel, 1: persistent bulk kernel
extern "C" int jv_set_spmv_impl(int impl) { g_spmv_impl = impl; return JV_OK; }
// 1 when jv_spmv would run the persistent kernel for this matrix and plan, else 0
extern "C" int jv_spmv_impl_for(int32_t nnz, const int32_t* tile_rows) {
  return spmv_use_bulk(nnz, tile_rows) ? 1 : 0;
}

extern "C" int jv_spmv_plan(int32_t n, int32_t nnz, const int32_t* row_start, int32_t* tile_rows,
                            void* stream) {
  if (n < 0 || nnz < 0) { jvh::set_error("jv_spmv_plan: bad size"); return JV_EINVAL; }
  const int ntiles = nnz > 0 ? (nnz + kTile - 1) / kTile : 1;
  cudaStream_t st = (cudaStream_t)stream;
  spmv_plan_kernel<<<(ntiles + 256) / 256, 256, 0, st>>>(n, nnz, ntiles, row_start, tile_rows);
  JV_CHECK_LAUNCH("jv_spmv_plan");
  // Rows spanning whole tiles (power-law hubs): their serial sums stall a
  // persistent CTA's whole tile range, while the CTA-per-tile kernel spreads
  // them over the GPU — remember which kernel this plan's matrix wants.
  // (Setup call: synchronises the stream once.)
  std::lock_guard<std::mutex> lock(g_spmv_mu);
  int run = 0;
  int* drun = nullptr;
  if (cudaMallocAsync(&drun, sizeof(int), st) != cudaSuccess) { cudaGetLastError(); return JV_OK; }
  cudaMemsetAsync(drun, 0, sizeof(int), st);
  spmv_plan_stat_kernel<<<(ntiles + 255) / 256, 256, 0, st>>>(ntiles, tile_rows, drun);
  cudaMemcpyAsync(&run, drun, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(drun, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) { cudaGetLastError(); return JV_OK; }
  g_spmv_long[tile_rows] = run >= kLongRun;
  return JV_OK;
}

extern "C" int jv_spmv(int32_t n, int32_t nnz, const int32_t* row_start, const int32_t* col,
                       const double* val, const double* x, double* y, const int32_t* tile_rows,
                       void* stream) {
  if (n < 0 || nnz < 0) { jvh::set_error("jv_spmv: bad size"); return JV_EINVAL; }
  if (n == 0) return JV_OK;
  spmv_launch(n, nnz, row_start, col, val, x, y, tile_rows, nullptr, (cudaStream_t)stream);
  JV_CHECK_LAUNCH("jv_spmv");
  return JV_OK;
}

extern "C" int jv_spmv_rows(int32_t n, int32_t nnz, const int32_t* row_start, const int32_t* col,
                            const double* val, const double* x, double* y,
                            const int32_t* tile_rows, const int32_t* row_map, void* stream) {
  if (n < 0 || nnz < 0) { jvh::set_error("jv_spmv_rows: bad size"); return JV_EINVAL; }
  if (n == 0) return JV_OK;
  spmv_launch(n, nnz, row_start, col, val, x, y, tile_rows, row_map, (cudaStream_t)stream);
  JV_CHECK_LAUNCH("jv_spmv_rows");
  return JV_OK;
}

namespace {
__global__ void gather_f64_kernel(int n, const int32_t* __restrict__ idx,
                                  const double* __restrict__ src, double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = __ldg(src + __ldg(idx + i));
}
}  // namespace

extern "C" int jv_gather(int32_t n, const int32_t* idx, const double* src, double* dst,
                         void* stream) {
  if (n < 0) { jvh::set_error("jv_gather: bad size"); return JV_EINVAL; }
  if (n == 0) return JV_OK;
  const int grid = min((n + 255) / 256, 148 * 8);
  gather_f64_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  JV_CHECK_LAUNCH("jv_gather");
  return JV_OK;
}
