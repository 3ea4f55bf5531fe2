// Device setup: level sets, partition, pattern ops, symbolic ILU(1), assembly.
// All structure outputs are bit-exact with the reference.
//
// Sorting/scans use CUB (header-only, part of the CUDA toolkit): stable
// radix sorts give exactly numpy's kind="stable" argsort and lexsort orders.
#include "common.cuh"
#include "../../include/jv.h"

#include <cub/cub.cuh>
#include <cstdio>

namespace {

constexpr int kSetupThreads = 256;

static inline int grid_for(long long n, int per = kSetupThreads) {
  long long g = (n + per - 1) / per;
  if (g < 1) g = 1;
  if (g > 65535LL * 32) g = 65535LL * 32;
  return (int)g;
}

// stream-ordered temporary buffer
struct Tmp {
  void* p = nullptr;
  cudaStream_t s;
  explicit Tmp(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 1, s); }
  ~Tmp() { if (p) cudaFreeAsync(p, s); }
};

// ---------------------------------------------------------------- levels
// Longest-path depth, sync-free: row r waits on the level words of its
// dependencies (columns < r forward, > r backward) and publishes its own.
// One warp per row (lanes split the row's dependencies, then a max
// reduction), rows in index order (ascending forward, descending backward)
// dealt round-robin to the co-resident warps: a row only waits on rows that
// precede it in that order, so the lowest unfinished row always progresses,
// and no lane ever waits on another lane of its own warp.
struct LevelArgs {
  int n;
  const int32_t* rs;
  const int32_t* col;
  int32_t* level_of;
  uint64_t* box;
  uint32_t epoch;
  int backward;
  int32_t* maxlev;
};

__global__ void __launch_bounds__(256) levels_kernel(LevelArgs A) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int W = (gridDim.x * blockDim.x) >> 5;
  int localmax = -1;
  for (int k = gw; k < A.n; k += W) {
    const int r = A.backward ? A.n - 1 - k : k;
    const int a = A.rs[r], b = A.rs[r + 1];
    int m = -1;
    for (int p = a + lane; p < b; p += 32) {
      const int c = A.col[p];
      const bool dep = A.backward ? (c > r) : (c < r);
      if (dep) {
        const int lc = (int)jv::ibox_wait(A.box, c, A.epoch);
        m = lc > m ? lc : m;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int v = __shfl_xor_sync(0xffffffffu, m, o);
      m = v > m ? v : m;
    }
    const int lev = m + 1;
    if (lane == 0) {
      A.level_of[r] = lev;
      jv::ibox_put(A.box, r, (uint32_t)lev, A.epoch);
    }
    localmax = lev > localmax ? lev : localmax;
  }
  if (lane == 0 && localmax >= 0) atomicMax(A.maxlev, localmax);
}

__global__ void iota_kernel(int n, int32_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = i;
}

// level_ptr from sorted keys (levels are contiguous: every depth 0..max occurs)
__global__ void level_ptr_kernel(int n, int nlev, const int32_t* sorted, int32_t* level_ptr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = sorted[i];
    const int prev = i == 0 ? -1 : sorted[i - 1];
    for (int l = prev + 1; l <= k; ++l) level_ptr[l] = i;
    if (i == n - 1)
      for (int l = k + 1; l <= nlev; ++l) level_ptr[l] = n;
  }
  if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0)
    for (int l = 0; l <= nlev; ++l) level_ptr[l] = 0;
}

// ------------------------------------------------------------- partition
// per-level integer sum of row nnz (exact), then the reference rule
// (ordering.py:119-159) evaluated by one thread with the same float64 ops:
//   ok(l) = count(l) >= min_rows  and  (double)sum(l)/count(l) <= df * ((double)total/n)
__global__ void level_nnz_kernel(int nlev, const int32_t* level_ptr, const int32_t* order,
                                 const int32_t* row_nnz, long long* lev_sum) {
  __shared__ long long part[256 / 32];
  for (int l = blockIdx.x; l < nlev; l += gridDim.x) {
    long long s = 0;
    for (int i = level_ptr[l] + threadIdx.x; i < level_ptr[l + 1]; i += blockDim.x)
      s += row_nnz[order[i]];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += part[w];
      lev_sum[l] = t;
    }
    __syncthreads();
  }
}

__global__ void partition_decide_kernel(int n, int nlev, const int32_t* level_ptr,
                                        const long long* lev_sum, int min_rows, double df,
                                        int suffix_only, int32_t* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  long long total = 0;
  for (int l = 0; l < nlev; ++l) total += lev_sum[l];
  const double mean_nnz = n ? (double)total / (double)n : 0.0;
  const double limit = df * mean_nnz;
  int cut = nlev;
  if (suffix_only) {
    while (cut > 0) {
      const int l = cut - 1;
      const int cnt = level_ptr[l + 1] - level_ptr[l];
      const double mean = cnt ? (double)lev_sum[l] / (double)cnt : 0.0;
      const bool ok = cnt >= min_rows && mean <= limit;
      if (ok) break;
      --cut;
    }
  } else {
    for (int l = 0; l < nlev; ++l) {
      const int cnt = level_ptr[l + 1] - level_ptr[l];
      const double mean = cnt ? (double)lev_sum[l] / (double)cnt : 0.0;
      const bool ok = cnt >= min_rows && mean <= limit;
      if (!ok) { cut = l; break; }
    }
  }
  out[0] = cut;
  out[1] = level_ptr[cut];
}

// --------------------------------------------------------------- batches
__global__ void batch_count_kernel(int nlev, const int32_t* level_ptr, int32_t* cnt) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlev; l += gridDim.x * blockDim.x)
    cnt[l] = (level_ptr[l + 1] - level_ptr[l] + 31) / 32;
}
__global__ void batch_fill_kernel(int nlev, const int32_t* level_ptr, const int32_t* boff,
                                  int32_t* batch_ptr) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlev; l += gridDim.x * blockDim.x) {
    const int a = level_ptr[l], b = level_ptr[l + 1];
    int o = boff[l];
    for (int s = a; s < b; s += 32) batch_ptr[o++] = s;
    if (l == nlev - 1) batch_ptr[o] = b;
  }
}

// class-aware schedule: groups = (level, class) in key order (key = 2*level
// + class); class 0 rows are cut into batches of 32, class 1 rows one each
// batch size per row class: key = nclass * level + class
struct BatchSteps {
  int nclass;
  int step[4];
};
__global__ void group_batch_count_kernel(int ngroups, const int32_t* gptr, BatchSteps bs,
                                         int32_t* cnt) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
    const int c = gptr[g + 1] - gptr[g];
    const int st = bs.step[g % bs.nclass];
    cnt[g] = (c + st - 1) / st;
  }
}
__global__ void group_batch_fill_kernel(int ngroups, const int32_t* gptr, const int32_t* boff,
                                        BatchSteps bs, int32_t* batch_ptr, int m) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
    const int a = gptr[g], b = gptr[g + 1];
    const int step = bs.step[g % bs.nclass];
    int o = boff[g];
    for (int s = a; s < b; s += step) batch_ptr[o++] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) batch_ptr[boff[ngroups]] = m;
}

// ------------------------------------------------------- pattern helpers
__global__ void row_ids_kernel(int n, const int32_t* rs, int32_t* rows) {
  // one warp per row writes its id over the row's nonzeros
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (gridDim.x * blockDim.x) >> 5)
    for (int p = rs[r] + lane; p < rs[r + 1]; p += 32) rows[p] = r;
}

__global__ void count_cols_kernel(int nnz, const int32_t* col, int32_t* cnt) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x)
    atomicAdd(cnt + col[p], 1);
}

// |A row i  ∪  At row i| (optionally restricted to columns < i)
__global__ void union_count_kernel(int n, const int32_t* ars, const int32_t* acol,
                                   const int32_t* brs, const int32_t* bcol, int lower_only,
                                   int32_t* cnt, int32_t* out_col, const int32_t* out_rs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int p = ars[i], pe = ars[i + 1], q = brs[i], qe = brs[i + 1];
    int k = 0;
    int o = out_col ? out_rs[i] : 0;
    while (p < pe || q < qe) {
      int c;
      if (q >= qe || (p < pe && acol[p] < bcol[q])) c = acol[p++];
      else if (p >= pe || bcol[q] < acol[p]) c = bcol[q++];
      else { c = acol[p]; ++p; ++q; }
      if (lower_only && c >= i) break;
      if (out_col) out_col[o + k] = c;
      ++k;
    }
    if (!out_col) cnt[i] = k;
  }
}

__global__ void gather_len_kernel(int n, const int32_t* rs, const int32_t* perm, int32_t* len) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int i = perm[r];
    len[r] = rs[i + 1] - rs[i];
  }
}

__global__ void permute_fill_kernel(int n, const int32_t* rs, const int32_t* col,
                                    const double* val, const int32_t* perm, const int32_t* inv,
                                    const int32_t* ors, int32_t* keys, double* vals) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (gridDim.x * blockDim.x) >> 5) {
    const int i = perm[r];
    const int a = rs[i], len = rs[i + 1] - a, o = ors[r];
    for (int t = lane; t < len; t += 32) {
      keys[o + t] = inv[col[a + t]];
      if (vals) vals[o + t] = val[a + t];
    }
  }
}

__global__ void check_diag_kernel(int n, const int32_t* rs, const int32_t* col, int32_t* row) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int lo = rs[r], hi = rs[r + 1];
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (col[mid] < r) lo = mid + 1; else hi = mid;
    }
    if (!(lo < rs[r + 1] && col[lo] == r)) atomicMin(row, r);
  }
}

// ---------------------------------------------------- ILU(1) symbolic
// candidates of row i: A row i plus strict-upper(A) rows of its strict-lower
// columns m (B.4 of SURVEY: iluk(1) == A ∪ pattern(L_A U_A))
__global__ void iluk1_bound_kernel(int n, const int32_t* rs, const int32_t* col, long long* bound) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    long long b = rs[i + 1] - rs[i];
    for (int p = rs[i]; p < rs[i + 1]; ++p) {
      const int m = col[p];
      if (m >= i) break;
      // strictly-upper part of row m: columns > m
      int lo = rs[m], hi = rs[m + 1];
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (col[mid] <= m) lo = mid + 1; else hi = mid;
      }
      b += rs[m + 1] - lo;
    }
    bound[i] = b;
  }
}

__global__ void iluk1_fill_kernel(int n, const int32_t* rs, const int32_t* col,
                                  const long long* boff, int32_t* cand) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (gridDim.x * blockDim.x) >> 5) {
    long long o = boff[i];
    const int a = rs[i], b = rs[i + 1];
    for (int t = lane; t < b - a; t += 32) cand[o + t] = col[a + t];
    o += b - a;
    for (int p = a; p < b; ++p) {
      const int m = col[p];
      if (m >= i) break;
      int lo = rs[m], hi = rs[m + 1];
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (col[mid] <= m) lo = mid + 1; else hi = mid;
      }
      for (int t = lane; t < rs[m + 1] - lo; t += 32) cand[o + t] = col[lo + t];
      o += rs[m + 1] - lo;
    }
  }
}

__global__ void unique_count_kernel(int n, const long long* boff, const int32_t* cand, int32_t* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int k = 0;
    for (long long p = boff[i]; p < boff[i + 1]; ++p)
      if (p == boff[i] || cand[p] != cand[p - 1]) ++k;
    cnt[i] = k;
  }
}

__global__ void unique_emit_kernel(int n, const long long* boff, const int32_t* cand,
                                   const int32_t* ors, const int32_t* ars, const int32_t* acol,
                                   int32_t* ocol, int32_t* olev) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int o = ors[i];
    int pa = ars[i];
    const int pe = ars[i + 1];
    for (long long p = boff[i]; p < boff[i + 1]; ++p) {
      if (p != boff[i] && cand[p] == cand[p - 1]) continue;
      const int c = cand[p];
      ocol[o] = c;
      if (olev) {
        while (pa < pe && acol[pa] < c) ++pa;
        olev[o] = (pa < pe && acol[pa] == c) ? 0 : 1;
      }
      ++o;
    }
  }
}

// ------------------------------------------------------------ assembly
__global__ void assemble_kernel(int n, const int32_t* ars, const int32_t* acol, const double* aval,
                                const int32_t* frs, const int32_t* fcol, double* fval,
                                int32_t* diag, int32_t* bad_cover, int32_t* bad_diag) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int w = frs[r];
    const int we = frs[r + 1];
    // merge: A row r and factor row r are both sorted
    for (int p = ars[r]; p < ars[r + 1]; ++p) {
      const int c = acol[p];
      while (w < we && fcol[w] < c) ++w;
      if (w < we && fcol[w] == c) fval[w] = aval[p];
      else atomicMin(bad_cover, r);
    }
    int lo = frs[r], hi = we;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (fcol[mid] < r) lo = mid + 1; else hi = mid;
    }
    if (lo < we && fcol[lo] == r) diag[r] = lo;
    else { diag[r] = -1; atomicMin(bad_diag, r); }
  }
}

__global__ void row_norms_kernel(int n, const int32_t* rs, const double* val, double tau,
                                 double* norms) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double m = 0.0;
    if (tau > 0.0)
      for (int p = rs[r]; p < rs[r + 1]; ++p) {
        const double a = fabs(val[p]);
        // np.maximum.at: NaN propagates and sticks
        if (isnan(a) || a > m) m = isnan(m) ? m : a;
      }
    norms[r] = m;
  }
}

__global__ void set_int_kernel(int32_t* p, int32_t v) { *p = v; }

}  // namespace

#define CK_CUDA(expr, what)                                        \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return jvh::cuda_status(_e, what);      \
  } while (0)

extern "C" int jv_reset_row(int32_t* row, void* stream) {
  set_int_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(row, jv::kNoRow);
  JV_CHECK_LAUNCH("jv_reset_row");
  return JV_OK;
}

extern "C" int jv_levels(int backward, int32_t n, const int32_t* row_start, const int32_t* col,
                         int32_t* level_of, uint64_t* ws, uint32_t epoch, int32_t* nlev_h,
                         void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0 || epoch == 0) { jvh::set_error("jv_levels: bad argument"); return JV_EINVAL; }
  if (n == 0) { if (nlev_h) *nlev_h = 0; return JV_OK; }
  Tmp mx(s);
  CK_CUDA(mx.alloc(sizeof(int32_t)), "jv_levels alloc");
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)mx.p, -1);
  LevelArgs A{n, row_start, col, level_of, ws, epoch, backward, (int32_t*)mx.p};
  void* args[] = {&A};
  int rc = jvh::coop_launch(levels_kernel, 256, args, s, "jv_levels");
  if (rc) return rc;
  int32_t m = -1;
  CK_CUDA(cudaMemcpyAsync(&m, mx.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "jv_levels copy");
  CK_CUDA(cudaStreamSynchronize(s), "jv_levels sync");
  if (nlev_h) *nlev_h = m + 1;
  return JV_OK;
}

extern "C" int jv_level_sort(int32_t n, int32_t nlev, const int32_t* level_of, int32_t* order,
                             int32_t* level_ptr, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0 || nlev < 0) { jvh::set_error("jv_level_sort: bad argument"); return JV_EINVAL; }
  if (n == 0) {
    if (level_ptr) level_ptr_kernel<<<1, 1, 0, s>>>(0, nlev, nullptr, level_ptr);
    return JV_OK;
  }
  int bits = 1;
  while ((1LL << bits) < (long long)nlev) ++bits;
  Tmp iota(s), keys(s), tmp(s);
  CK_CUDA(iota.alloc(sizeof(int32_t) * n), "alloc");
  CK_CUDA(keys.alloc(sizeof(int32_t) * n), "alloc");
  iota_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, (int32_t*)iota.p);
  size_t tb = 0;
  CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, level_of, (int32_t*)keys.p,
                                          (const int32_t*)iota.p, order, n, 0, bits, s),
          "sort size");
  CK_CUDA(tmp.alloc(tb), "alloc");
  CK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, level_of, (int32_t*)keys.p,
                                          (const int32_t*)iota.p, order, n, 0, bits, s),
          "sort");
  level_ptr_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, nlev, (const int32_t*)keys.p, level_ptr);
  JV_CHECK_LAUNCH("jv_level_sort");
  return JV_OK;
}

extern "C" int jv_partition(int32_t n, int32_t nlev, const int32_t* level_ptr,
                            const int32_t* order, const int32_t* row_nnz, int32_t min_level_rows,
                            double density_factor, int suffix_only, int32_t* cut_h,
                            int32_t* n_upper_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nlev == 0) { *cut_h = 0; *n_upper_h = 0; return JV_OK; }
  Tmp sums(s), out(s);
  CK_CUDA(sums.alloc(sizeof(long long) * nlev), "alloc");
  CK_CUDA(out.alloc(2 * sizeof(int32_t)), "alloc");
  int g = nlev < 4096 ? nlev : 4096;
  level_nnz_kernel<<<g, 256, 0, s>>>(nlev, level_ptr, order, row_nnz, (long long*)sums.p);
  partition_decide_kernel<<<1, 1, 0, s>>>(n, nlev, level_ptr, (const long long*)sums.p,
                                          min_level_rows, density_factor, suffix_only,
                                          (int32_t*)out.p);
  JV_CHECK_LAUNCH("jv_partition");
  int32_t h[2];
  CK_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  *cut_h = h[0];
  *n_upper_h = h[1];
  return JV_OK;
}

extern "C" int jv_build_batches(int32_t nlev, const int32_t* level_ptr, int32_t* batch_ptr,
                                int32_t* nbatch_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nlev <= 0) {
    set_int_kernel<<<1, 1, 0, s>>>(batch_ptr, 0);
    *nbatch_h = 0;
    return JV_OK;
  }
  Tmp cnt(s), off(s), tmp(s);
  CK_CUDA(cnt.alloc(sizeof(int32_t) * (nlev + 1)), "alloc");
  CK_CUDA(off.alloc(sizeof(int32_t) * (nlev + 1)), "alloc");
  batch_count_kernel<<<grid_for(nlev), kSetupThreads, 0, s>>>(nlev, level_ptr, (int32_t*)cnt.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)cnt.p + nlev, 0);
  size_t tb = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int32_t*)cnt.p, (int32_t*)off.p, nlev + 1, s),
          "scan size");
  CK_CUDA(tmp.alloc(tb), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (int32_t*)cnt.p, (int32_t*)off.p, nlev + 1, s),
          "scan");
  batch_fill_kernel<<<grid_for(nlev), kSetupThreads, 0, s>>>(nlev, level_ptr,
                                                             (const int32_t*)off.p, batch_ptr);
  JV_CHECK_LAUNCH("jv_build_batches");
  int32_t nb = 0;
  CK_CUDA(cudaMemcpyAsync(&nb, (int32_t*)off.p + nlev, sizeof(int32_t), cudaMemcpyDeviceToHost, s),
          "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  *nbatch_h = nb;
  return JV_OK;
}

__global__ void gather_rows_kernel(int nnz, const int32_t* pos, const int32_t* rows, int32_t* t_col) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += gridDim.x * blockDim.x)
    t_col[k] = rows[pos[k]];
}

extern "C" int jv_transpose_pattern(int32_t n, const int32_t* row_start, const int32_t* col,
                                    int32_t* t_row_start, int32_t* t_col, int32_t* t_pos,
                                    void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int32_t nnz = 0;
  CK_CUDA(cudaMemcpyAsync(&nnz, row_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  Tmp rows(s), keys(s), cnt(s), tmp(s), pos(s), spos(s);
  CK_CUDA(cnt.alloc(sizeof(int32_t) * (n + 1)), "alloc");
  CK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (n + 1), s), "memset");
  size_t tb = 0, tb2 = 0;
  if (nnz > 0) {
    CK_CUDA(rows.alloc(sizeof(int32_t) * nnz), "alloc");
    CK_CUDA(keys.alloc(sizeof(int32_t) * nnz), "alloc");
    CK_CUDA(pos.alloc(sizeof(int32_t) * nnz), "alloc");
    CK_CUDA(spos.alloc(sizeof(int32_t) * nnz), "alloc");
    row_ids_kernel<<<grid_for((long long)n * 32), kSetupThreads, 0, s>>>(n, row_start, (int32_t*)rows.p);
    iota_kernel<<<grid_for(nnz), kSetupThreads, 0, s>>>(nnz, (int32_t*)pos.p);
    count_cols_kernel<<<grid_for(nnz), kSetupThreads, 0, s>>>(nnz, col, (int32_t*)cnt.p);
    int bits = 1;
    while ((1LL << bits) < (long long)n) ++bits;
    CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, col, (int32_t*)keys.p,
                                            (const int32_t*)pos.p, (int32_t*)spos.p, nnz, 0, bits, s),
            "sort size");
  }
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, (int32_t*)cnt.p, t_row_start, n + 1, s),
          "scan size");
  CK_CUDA(tmp.alloc(tb > tb2 ? tb : tb2), "alloc");
  if (nnz > 0) {
    int bits = 1;
    while ((1LL << bits) < (long long)n) ++bits;
    CK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, col, (int32_t*)keys.p,
                                            (const int32_t*)pos.p, (int32_t*)spos.p, nnz, 0, bits, s),
            "sort");
    gather_rows_kernel<<<grid_for(nnz), kSetupThreads, 0, s>>>(nnz, (const int32_t*)spos.p,
                                                               (const int32_t*)rows.p, t_col);
    if (t_pos)
      CK_CUDA(cudaMemcpyAsync(t_pos, spos.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s),
              "copy");
  }
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, (int32_t*)cnt.p, t_row_start, n + 1, s), "scan");
  JV_CHECK_LAUNCH("jv_transpose_pattern");
  return JV_OK;
}

extern "C" int jv_sym_lower(int32_t n, const int32_t* row_start, const int32_t* col,
                            const int32_t* t_row_start, const int32_t* t_col, int lower_only,
                            int32_t* out_row_start, int32_t* out_col, int64_t* nnz_h,
                            void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!out_col) {
    Tmp cnt(s), tmp(s);
    CK_CUDA(cnt.alloc(sizeof(int32_t) * (n + 1)), "alloc");
    union_count_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(
        n, row_start, col, t_row_start, t_col, lower_only, (int32_t*)cnt.p, nullptr, nullptr);
    set_int_kernel<<<1, 1, 0, s>>>((int32_t*)cnt.p + n, 0);
    size_t tb = 0;
    CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int32_t*)cnt.p, out_row_start, n + 1, s),
            "scan size");
    CK_CUDA(tmp.alloc(tb), "alloc");
    CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (int32_t*)cnt.p, out_row_start, n + 1, s),
            "scan");
    int32_t nz = 0;
    CK_CUDA(cudaMemcpyAsync(&nz, out_row_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s),
            "copy");
    CK_CUDA(cudaStreamSynchronize(s), "sync");
    *nnz_h = nz;
    return JV_OK;
  }
  union_count_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(
      n, row_start, col, t_row_start, t_col, lower_only, nullptr, out_col, out_row_start);
  JV_CHECK_LAUNCH("jv_sym_lower");
  return JV_OK;
}

extern "C" int jv_permute_symmetric(int32_t n, const int32_t* row_start, const int32_t* col,
                                    const double* val, const int32_t* perm, const int32_t* inv,
                                    int32_t* out_row_start, int32_t* out_col, double* out_val,
                                    void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) { set_int_kernel<<<1, 1, 0, s>>>(out_row_start, 0); return JV_OK; }
  Tmp len(s), tmp(s), keys(s), vals(s);
  CK_CUDA(len.alloc(sizeof(int32_t) * (n + 1)), "alloc");
  gather_len_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, perm, (int32_t*)len.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)len.p + n, 0);
  size_t tb = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int32_t*)len.p, out_row_start, n + 1, s),
          "scan size");
  int32_t nnz = 0;
  CK_CUDA(cudaMemcpyAsync(&nnz, row_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  size_t tb2 = 0;
  if (nnz > 0) {
    if (val)
      CK_CUDA(cub::DeviceSegmentedSort::StableSortPairs(
                  nullptr, tb2, (const int32_t*)nullptr, (int32_t*)nullptr, (const double*)nullptr,
                  (double*)nullptr, nnz, n, out_row_start, out_row_start + 1, s),
              "segsort size");
    else
      CK_CUDA(cub::DeviceSegmentedSort::StableSortKeys(nullptr, tb2, (const int32_t*)nullptr,
                                                      (int32_t*)nullptr, nnz, n, out_row_start,
                                                      out_row_start + 1, s),
              "segsort size");
  }
  CK_CUDA(tmp.alloc(tb > tb2 ? tb : tb2), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (int32_t*)len.p, out_row_start, n + 1, s), "scan");
  if (nnz == 0) return JV_OK;
  CK_CUDA(keys.alloc(sizeof(int32_t) * nnz), "alloc");
  if (val) CK_CUDA(vals.alloc(sizeof(double) * nnz), "alloc");
  permute_fill_kernel<<<grid_for((long long)n * 32), kSetupThreads, 0, s>>>(
      n, row_start, col, val, perm, inv, out_row_start, (int32_t*)keys.p, (double*)vals.p);
  if (val)
    CK_CUDA(cub::DeviceSegmentedSort::StableSortPairs(tmp.p, tb2, (const int32_t*)keys.p, out_col,
                                                      (const double*)vals.p, out_val, nnz, n,
                                                      out_row_start, out_row_start + 1, s),
            "segsort");
  else
    CK_CUDA(cub::DeviceSegmentedSort::StableSortKeys(tmp.p, tb2, (const int32_t*)keys.p, out_col,
                                                     nnz, n, out_row_start, out_row_start + 1, s),
            "segsort");
  JV_CHECK_LAUNCH("jv_permute_symmetric");
  return JV_OK;
}

extern "C" int jv_check_diagonal(int32_t n, const int32_t* row_start, const int32_t* col,
                                 int32_t* row, void* stream) {
  if (n <= 0) return JV_OK;
  check_diag_kernel<<<grid_for(n), kSetupThreads, 0, (cudaStream_t)stream>>>(n, row_start, col, row);
  JV_CHECK_LAUNCH("jv_check_diagonal");
  return JV_OK;
}

extern "C" int jv_iluk1_pattern(int32_t n, const int32_t* row_start, const int32_t* col,
                                int32_t* out_row_start, int32_t* out_col, int32_t* out_lev,
                                int64_t* nnz_h, void* stream) {
  // Single call that recomputes the candidate lists in both phases (setup
  // only; simpler than keeping state between the two calls).
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) { set_int_kernel<<<1, 1, 0, s>>>(out_row_start, 0); *nnz_h = 0; return JV_OK; }
  Tmp bound(s), boff(s), cand(s), sorted(s), cnt(s), tmp(s);
  CK_CUDA(bound.alloc(sizeof(long long) * (n + 1)), "alloc");
  CK_CUDA(boff.alloc(sizeof(long long) * (n + 1)), "alloc");
  iluk1_bound_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, col, (long long*)bound.p);
  CK_CUDA(cudaMemsetAsync((long long*)bound.p + n, 0, sizeof(long long), s), "memset");
  size_t tb = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (long long*)bound.p, (long long*)boff.p, n + 1, s),
          "scan size");
  CK_CUDA(tmp.alloc(tb), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (long long*)bound.p, (long long*)boff.p, n + 1, s),
          "scan");
  long long total = 0;
  CK_CUDA(cudaMemcpyAsync(&total, (long long*)boff.p + n, sizeof(long long), cudaMemcpyDeviceToHost, s),
          "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  if (total >= (1LL << 31)) { jvh::set_error("jv_iluk1_pattern: candidate list too large"); return JV_ENOMEM; }
  CK_CUDA(cand.alloc(sizeof(int32_t) * total), "alloc");
  CK_CUDA(sorted.alloc(sizeof(int32_t) * total), "alloc");
  iluk1_fill_kernel<<<grid_for((long long)n * 32), kSetupThreads, 0, s>>>(
      n, row_start, col, (const long long*)boff.p, (int32_t*)cand.p);
  size_t tb2 = 0;
  CK_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb2, (const int32_t*)cand.p,
                                             (int32_t*)sorted.p, (int)total, n,
                                             (const long long*)boff.p, (const long long*)boff.p + 1, s),
          "segsort size");
  Tmp tmp2(s);
  CK_CUDA(tmp2.alloc(tb2), "alloc");
  CK_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp2.p, tb2, (const int32_t*)cand.p,
                                             (int32_t*)sorted.p, (int)total, n,
                                             (const long long*)boff.p, (const long long*)boff.p + 1, s),
          "segsort");
  CK_CUDA(cnt.alloc(sizeof(int32_t) * (n + 1)), "alloc");
  unique_count_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, (const long long*)boff.p,
                                                            (const int32_t*)sorted.p, (int32_t*)cnt.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)cnt.p + n, 0);
  size_t tb3 = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, (int32_t*)cnt.p, out_row_start, n + 1, s),
          "scan size");
  Tmp tmp3(s);
  CK_CUDA(tmp3.alloc(tb3), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.p, tb3, (int32_t*)cnt.p, out_row_start, n + 1, s), "scan");
  int32_t nz = 0;
  CK_CUDA(cudaMemcpyAsync(&nz, out_row_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  *nnz_h = nz;
  if (out_col)
    unique_emit_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(
        n, (const long long*)boff.p, (const int32_t*)sorted.p, out_row_start, row_start, col,
        out_col, out_lev);
  JV_CHECK_LAUNCH("jv_iluk1_pattern");
  return JV_OK;
}

// ---------------------------------------------------- ILU(k) symbolic, k >= 2
// One round of the level-of-fill closure (symbolic.py:86-138) on a levelled
// pattern: row i keeps its entries and gains (j, a + b + 1) for every strict-
// lower entry (m, a) of row i and strict-upper entry (j, b) of row m with
// a + b + 1 <= K; per column the smallest level wins.  Levels are exact by
// induction on their value — an entry of level l needs a pair of levels
// summing to l - 1, all present after l - 1 rounds — so K rounds from
// (A, level 0) give the reference's ILU(K) pattern and level table.
// Candidates are 64-bit keys (column << 8 | level), segment-sorted per row;
// pairs over the level bound are written as a sentinel that sorts last.
namespace {
constexpr unsigned long long kIlukSent = ~0ull;

__global__ void ilukr_bound_kernel(int n, const int32_t* rs, const int32_t* col,
                                   const int32_t* lev, int K, long long* bound) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    long long b = rs[i + 1] - rs[i];
    for (int p = rs[i]; p < rs[i + 1]; ++p) {
      const int m = col[p];
      if (m >= i) break;
      if (lev[p] >= K) continue;
      int lo = rs[m], hi = rs[m + 1];
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (col[mid] <= m) lo = mid + 1; else hi = mid;
      }
      b += rs[m + 1] - lo;
    }
    bound[i] = b;
  }
}

__global__ void ilukr_fill_kernel(int n, const int32_t* rs, const int32_t* col,
                                  const int32_t* lev, int K, const long long* boff,
                                  unsigned long long* cand) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (gridDim.x * blockDim.x) >> 5) {
    long long o = boff[i];
    const int a = rs[i], b = rs[i + 1];
    for (int t = lane; t < b - a; t += 32)
      cand[o + t] = ((unsigned long long)(unsigned)col[a + t] << 8) | (unsigned)lev[a + t];
    o += b - a;
    for (int p = a; p < b; ++p) {
      const int m = col[p];
      if (m >= i) break;
      const int la = lev[p];
      if (la >= K) continue;
      int lo = rs[m], hi = rs[m + 1];
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (col[mid] <= m) lo = mid + 1; else hi = mid;
      }
      for (int t = lane; t < rs[m + 1] - lo; t += 32) {
        const int l = la + lev[lo + t] + 1;
        cand[o + t] = l <= K ? ((unsigned long long)(unsigned)col[lo + t] << 8) | (unsigned)l
                             : kIlukSent;
      }
      o += rs[m + 1] - lo;
    }
  }
}

__global__ void ilukr_count_kernel(int n, const long long* boff, const unsigned long long* cand,
                                   int32_t* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int k = 0;
    for (long long p = boff[i]; p < boff[i + 1]; ++p) {
      if (cand[p] == kIlukSent) break;
      if (p == boff[i] || (cand[p] >> 8) != (cand[p - 1] >> 8)) ++k;
    }
    cnt[i] = k;
  }
}

__global__ void ilukr_emit_kernel(int n, const long long* boff, const unsigned long long* cand,
                                  const int32_t* ors, int32_t* ocol, int32_t* olev) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int o = ors[i];
    for (long long p = boff[i]; p < boff[i + 1]; ++p) {
      if (cand[p] == kIlukSent) break;
      if (p != boff[i] && (cand[p] >> 8) == (cand[p - 1] >> 8)) continue;
      ocol[o] = (int32_t)(cand[p] >> 8);      // first of its column: the smallest level
      olev[o] = (int32_t)(cand[p] & 0xff);
      ++o;
    }
  }
}
}  // namespace

extern "C" int jv_iluk_round(int32_t n, const int32_t* row_start, const int32_t* col,
                             const int32_t* lev, int32_t K, int32_t* out_row_start,
                             int32_t* out_col, int32_t* out_lev, int64_t* nnz_h, void* stream) {
  // Called twice like jv_iluk1_pattern: out_col == NULL sizes the result.
  cudaStream_t s = (cudaStream_t)stream;
  if (K < 1 || K > 254) { jvh::set_error("jv_iluk_round: fill level out of range"); return JV_EINVAL; }
  if (n == 0) { set_int_kernel<<<1, 1, 0, s>>>(out_row_start, 0); *nnz_h = 0; return JV_OK; }
  Tmp bound(s), boff(s), cand(s), sorted(s), cnt(s), tmp(s);
  CK_CUDA(bound.alloc(sizeof(long long) * (n + 1)), "alloc");
  CK_CUDA(boff.alloc(sizeof(long long) * (n + 1)), "alloc");
  ilukr_bound_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, col, lev, K,
                                                           (long long*)bound.p);
  CK_CUDA(cudaMemsetAsync((long long*)bound.p + n, 0, sizeof(long long), s), "memset");
  size_t tb = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (long long*)bound.p, (long long*)boff.p, n + 1, s),
          "scan size");
  CK_CUDA(tmp.alloc(tb), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (long long*)bound.p, (long long*)boff.p, n + 1, s),
          "scan");
  long long total = 0;
  CK_CUDA(cudaMemcpyAsync(&total, (long long*)boff.p + n, sizeof(long long), cudaMemcpyDeviceToHost, s),
          "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  if (total >= (1LL << 31)) { jvh::set_error("jv_iluk_round: candidate list too large"); return JV_ENOMEM; }
  CK_CUDA(cand.alloc(sizeof(unsigned long long) * total), "alloc");
  CK_CUDA(sorted.alloc(sizeof(unsigned long long) * total), "alloc");
  ilukr_fill_kernel<<<grid_for((long long)n * 32), kSetupThreads, 0, s>>>(
      n, row_start, col, lev, K, (const long long*)boff.p, (unsigned long long*)cand.p);
  size_t tb2 = 0;
  CK_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb2, (const unsigned long long*)cand.p,
                                             (unsigned long long*)sorted.p, (int)total, n,
                                             (const long long*)boff.p, (const long long*)boff.p + 1, s),
          "segsort size");
  Tmp tmp2(s);
  CK_CUDA(tmp2.alloc(tb2), "alloc");
  CK_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp2.p, tb2, (const unsigned long long*)cand.p,
                                             (unsigned long long*)sorted.p, (int)total, n,
                                             (const long long*)boff.p, (const long long*)boff.p + 1, s),
          "segsort");
  CK_CUDA(cnt.alloc(sizeof(int32_t) * (n + 1)), "alloc");
  ilukr_count_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(
      n, (const long long*)boff.p, (const unsigned long long*)sorted.p, (int32_t*)cnt.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)cnt.p + n, 0);
  size_t tb3 = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, (int32_t*)cnt.p, out_row_start, n + 1, s),
          "scan size");
  Tmp tmp3(s);
  CK_CUDA(tmp3.alloc(tb3), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.p, tb3, (int32_t*)cnt.p, out_row_start, n + 1, s), "scan");
  int32_t nz = 0;
  CK_CUDA(cudaMemcpyAsync(&nz, out_row_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  *nnz_h = nz;
  if (out_col)
    ilukr_emit_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(
        n, (const long long*)boff.p, (const unsigned long long*)sorted.p, out_row_start, out_col,
        out_lev);
  JV_CHECK_LAUNCH("jv_iluk_round");
  return JV_OK;
}

extern "C" int jv_assemble(int32_t n, const int32_t* a_row_start, const int32_t* a_col,
                           const double* a_val, const int32_t* f_row_start, const int32_t* f_col,
                           double* f_val, int32_t* diag_pos, int32_t* bad_cover, int32_t* bad_diag,
                           void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return JV_OK;
  int32_t fnnz = 0;
  CK_CUDA(cudaMemcpyAsync(&fnnz, f_row_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  if (fnnz) CK_CUDA(cudaMemsetAsync(f_val, 0, sizeof(double) * fnnz, s), "memset");
  assemble_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, a_row_start, a_col, a_val, f_row_start,
                                                        f_col, f_val, diag_pos, bad_cover, bad_diag);
  JV_CHECK_LAUNCH("jv_assemble");
  return JV_OK;
}

extern "C" int jv_row_norms(int32_t n, const int32_t* row_start, const double* val, double tau,
                            double* norms, void* stream) {
  if (n <= 0) return JV_OK;
  row_norms_kernel<<<grid_for(n), kSetupThreads, 0, (cudaStream_t)stream>>>(n, row_start, val, tau,
                                                                            norms);
  JV_CHECK_LAUNCH("jv_row_norms");
  return JV_OK;
}

extern "C" int jv_build_schedule_n(int32_t m, const int32_t* rows, const int32_t* keys,
                                   int32_t nkeys, int32_t nclass, const int32_t* steps,
                                   int32_t* order, int32_t* batch_ptr, int32_t* nbatch_h,
                                   void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (m < 0 || nkeys < 0 || nclass < 1 || nclass > 4) {
    jvh::set_error("jv_build_schedule: bad argument");
    return JV_EINVAL;
  }
  BatchSteps bs{nclass, {1, 1, 1, 1}};
  for (int c = 0; c < nclass; ++c) {
    if (steps[c] < 1) { jvh::set_error("jv_build_schedule: step < 1"); return JV_EINVAL; }
    bs.step[c] = steps[c];
  }
  if (m == 0) {
    set_int_kernel<<<1, 1, 0, s>>>(batch_ptr, 0);
    *nbatch_h = 0;
    return JV_OK;
  }
  int bits = 1;
  while ((1LL << bits) < (long long)nkeys) ++bits;
  Tmp iota(s), skeys(s), tmp(s), gptr(s), cnt(s), off(s);
  if (!rows) {
    CK_CUDA(iota.alloc(sizeof(int32_t) * m), "alloc");
    iota_kernel<<<grid_for(m), kSetupThreads, 0, s>>>(m, (int32_t*)iota.p);
    rows = (const int32_t*)iota.p;
  }
  CK_CUDA(skeys.alloc(sizeof(int32_t) * m), "alloc");
  size_t tb = 0, tb2 = 0;
  CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, (int32_t*)skeys.p, rows, order, m, 0,
                                          bits, s), "sort size");
  CK_CUDA(cnt.alloc(sizeof(int32_t) * (nkeys + 1)), "alloc");
  CK_CUDA(off.alloc(sizeof(int32_t) * (nkeys + 1)), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, (int32_t*)cnt.p, (int32_t*)off.p, nkeys + 1, s),
          "scan size");
  CK_CUDA(tmp.alloc(tb > tb2 ? tb : tb2), "alloc");
  CK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys, (int32_t*)skeys.p, rows, order, m, 0,
                                          bits, s), "sort");
  CK_CUDA(gptr.alloc(sizeof(int32_t) * (nkeys + 1)), "alloc");
  level_ptr_kernel<<<grid_for(m), kSetupThreads, 0, s>>>(m, nkeys, (const int32_t*)skeys.p,
                                                         (int32_t*)gptr.p);
  group_batch_count_kernel<<<grid_for(nkeys), kSetupThreads, 0, s>>>(nkeys, (const int32_t*)gptr.p,
                                                                     bs, (int32_t*)cnt.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)cnt.p + nkeys, 0);
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, (int32_t*)cnt.p, (int32_t*)off.p, nkeys + 1, s),
          "scan");
  group_batch_fill_kernel<<<grid_for(nkeys), kSetupThreads, 0, s>>>(
      nkeys, (const int32_t*)gptr.p, (const int32_t*)off.p, bs, batch_ptr, m);
  JV_CHECK_LAUNCH("jv_build_schedule");
  int32_t nb = 0;
  CK_CUDA(cudaMemcpyAsync(&nb, (int32_t*)off.p + nkeys, sizeof(int32_t), cudaMemcpyDeviceToHost, s),
          "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  *nbatch_h = nb;
  return JV_OK;
}

extern "C" int jv_build_schedule(int32_t m, const int32_t* rows, const int32_t* keys, int32_t nkeys,
                                 int32_t* order, int32_t* batch_ptr, int32_t* nbatch_h,
                                 void* stream) {
  const int32_t steps[2] = {32, 1};
  return jv_build_schedule_n(m, rows, keys, nkeys, 2, steps, order, batch_ptr, nbatch_h, stream);
}
