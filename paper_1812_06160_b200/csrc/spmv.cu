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
#include "common.cuh"
#include "../../include/jv.h"

namespace {

#ifndef JV_SPMV_THREADS
#define JV_SPMV_THREADS 128
#endif
#ifndef JV_SPMV_TILE
#define JV_SPMV_TILE 640
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

}  // namespace

extern "C" int jv_spmv_tile(void) { return kTile; }

extern "C" int jv_spmv_plan(int32_t n, int32_t nnz, const int32_t* row_start, int32_t* tile_rows,
                            void* stream) {
  if (n < 0 || nnz < 0) { jvh::set_error("jv_spmv_plan: bad size"); return JV_EINVAL; }
  const int ntiles = nnz > 0 ? (nnz + kTile - 1) / kTile : 1;
  spmv_plan_kernel<<<(ntiles + 256) / 256, 256, 0, (cudaStream_t)stream>>>(n, nnz, ntiles,
                                                                          row_start, tile_rows);
  JV_CHECK_LAUNCH("jv_spmv_plan");
  return JV_OK;
}

extern "C" int jv_spmv(int32_t n, int32_t nnz, const int32_t* row_start, const int32_t* col,
                       const double* val, const double* x, double* y, const int32_t* tile_rows,
                       void* stream) {
  if (n < 0 || nnz < 0) { jvh::set_error("jv_spmv: bad size"); return JV_EINVAL; }
  if (n == 0) return JV_OK;
  const int ntiles = nnz > 0 ? (nnz + kTile - 1) / kTile : 1;
  spmv_stream_kernel<<<ntiles, kSpmvThreads, 0, (cudaStream_t)stream>>>(n, nnz, row_start, col,
                                                                        val, x, y, tile_rows,
                                                                        nullptr);
  JV_CHECK_LAUNCH("jv_spmv");
  return JV_OK;
}

extern "C" int jv_spmv_rows(int32_t n, int32_t nnz, const int32_t* row_start, const int32_t* col,
                            const double* val, const double* x, double* y,
                            const int32_t* tile_rows, const int32_t* row_map, void* stream) {
  if (n < 0 || nnz < 0) { jvh::set_error("jv_spmv_rows: bad size"); return JV_EINVAL; }
  if (n == 0) return JV_OK;
  const int ntiles = nnz > 0 ? (nnz + kTile - 1) / kTile : 1;
  spmv_stream_kernel<<<ntiles, kSpmvThreads, 0, (cudaStream_t)stream>>>(n, nnz, row_start, col,
                                                                        val, x, y, tile_rows,
                                                                        row_map);
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
