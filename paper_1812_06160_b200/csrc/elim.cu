// Elimination lists for heavy rows (setup, once per pattern; see jv.h).
//
// The numeric kernel's warp path finds, per pivot c of row r, the entries of
// U(c) that land in row r by binary search.  For power-law matrices (config
// 5: hub rows with ~5000 pivots whose U rows hold ~15000 entries) that search
// is the whole cost and sits on the critical path, so it moves here: the
// matches of every (row, pivot) pair of a heavy row are found once, by one
// warp per pair over the whole GPU, and stored as (q, w) op pairs in
// ascending column order — the order _factor_row (_kernels.py:165-194)
// applies them in.  Included after setup.cu (shares Tmp / grid_for).

namespace {

constexpr int kElimOut = 1 << 30;   // == factor.cu kOut

// per-row candidate volume -> heavy flag, and the row's count of list pairs
__global__ void elim_heavy_kernel(int n, const int32_t* rs, const int32_t* col,
                                  const int32_t* diag, int milu, long long min_cand,
                                  const int32_t* cls, int8_t* heavy, int32_t* npairs) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int a = rs[r], len = rs[r + 1] - a, nL = diag[r] - a;
    long long cand = 0;
    for (int k = 0; k < nL && cand <= min_cand; ++k) {
      const int c = col[a + k];
      const long long ulen = rs[c + 1] - diag[c] - 1, rem = len - k - 1;
      cand += milu ? ulen : min(ulen, rem);
    }
    // 2: heavy (own path); 1: warp-path row with its list; 0: no list.
    // Tentative: elim_refine_kernel promotes a listed row to 2 once the
    // actual op counts show a 32-pivot chunk over the warp op list.
    int f = 0;
    if (nL > 0 && cand > min_cand) f = min_cand < 256 ? 2 : 1;
    else if (cls != nullptr) f = 1;             // warp-path row (possibly no pivots)
    if (cls != nullptr && cls[r] == 0) f = 0;   // thread-path rows never read a list
    heavy[r] = (int8_t)f;
    npairs[r] = f ? nL : 0;
  }
}

__global__ void elim_pairs_kernel(int n, const int32_t* rs, const int32_t* off, int32_t* prow,
                                  int32_t* ppos) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int b = off[r], m = off[r + 1] - b;
    for (int k = 0; k < m; ++k) {
      prow[b + k] = r;
      ppos[b + k] = rs[r] + k;
    }
  }
}

// final flags of listed rows: 2 (heavy) when a 32-pivot chunk holds more
// than 256 ops (factor.cu kWarpOps); else 1 (pairable: length <= 64 and no
// pivot with more than 160 ops — factor.cu kPairRow / kPairOps) or 3
__global__ void elim_refine_kernel(int n, const int32_t* rs, const int32_t* diag,
                                   const long long* eptr, int8_t* heavy) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (heavy[r] != 1) continue;
    const int a = rs[r], nL = diag[r] - a, len = rs[r + 1] - a;
    int f = len <= 64 ? 1 : 3;
    for (int k0 = 0; k0 < nL; k0 += 32) {
      if (eptr[a + min(k0 + 32, nL)] - eptr[a + k0] > 256) { f = 2; break; }
    }
    if (f == 1)
      for (int k = 0; k < nL; ++k)
        if (eptr[a + k + 1] - eptr[a + k] > 160) { f = 3; break; }
    heavy[r] = (int8_t)f;
  }
}

JV_INLINE int elim_lower_bound(const int32_t* arr, int lo, int hi, int key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (arr[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// one warp per (row, pivot) pair: count (Fill = false) or emit the matches
template <bool Fill>
__global__ void __launch_bounds__(256) elim_match_kernel(
    long long npair, const int32_t* prow, const int32_t* ppos, const int32_t* rs,
    const int32_t* col, const int32_t* diag, int milu, long long* cnt, const long long* ptr,
    int2* ops) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < npair; e += W) {
    const int r = prow[e], p = ppos[e];
    const int a = rs[r], re = rs[r + 1], k = p - a, dloc = diag[r] - a;
    const int c = col[p], dk = diag[c], cek = rs[c + 1];
    const int ulen = cek - dk - 1, rem = re - p - 1;
    long long out = Fill ? ptr[p] : 0;
    long long m = 0;
    if (milu || ulen <= rem) {
      // lanes over U(c), each searched in the rest of row r
      for (int base = dk + 1; base < cek; base += 32) {
        const int q = base + lane;
        int w = -1;
        if (q < cek) {
          const int j = col[q];
          const int t = elim_lower_bound(col, p + 1, re, j);
          if (t < re && col[t] == j) w = t - a;
          else if (milu) w = dloc | kElimOut;
        }
        const unsigned b = __ballot_sync(full, w >= 0);
        if (Fill && w >= 0) ops[out + m + __popc(b & ((1u << lane) - 1))] = make_int2(q, w);
        m += __popc(b);
      }
    } else {
      // lanes over the rest of row r, each searched in U(c)
      for (int base = p + 1; base < re; base += 32) {
        const int t = base + lane;
        int q = -1;
        if (t < re) {
          const int j = col[t];
          const int f = elim_lower_bound(col, dk + 1, cek, j);
          if (f < cek && col[f] == j) q = f;
        }
        const unsigned b = __ballot_sync(full, q >= 0);
        if (Fill && q >= 0) ops[out + m + __popc(b & ((1u << lane) - 1))] = make_int2(q, t - a);
        m += __popc(b);
      }
    }
    if (!Fill && lane == 0) cnt[p] = m;
    (void)k;
  }
}

}  // namespace

extern "C" int jv_elim_lists(int32_t n, const int32_t* row_start, const int32_t* col,
                             const int32_t* diag_pos, int milu, int64_t min_cand,
                             const int32_t* cls, int8_t* heavy,
                             int64_t* elim_ptr, int32_t* elim, int64_t* nops_h, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  *nops_h = 0;
  if (n <= 0) return JV_OK;
  int32_t nnz = 0;
  CK_CUDA(cudaMemcpyAsync(&nnz, row_start + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "copy");
  Tmp npairs(s), off(s), tmp(s), prow(s), ppos(s), cnt(s), tmp2(s);
  CK_CUDA(npairs.alloc(sizeof(int32_t) * (n + 1)), "alloc");
  CK_CUDA(off.alloc(sizeof(int32_t) * (n + 1)), "alloc");
  elim_heavy_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, col, diag_pos, milu,
                                                          (long long)min_cand, cls, heavy,
                                                          (int32_t*)npairs.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)npairs.p + n, 0);
  size_t tb = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int32_t*)npairs.p, (int32_t*)off.p, n + 1, s),
          "scan size");
  CK_CUDA(tmp.alloc(tb), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (int32_t*)npairs.p, (int32_t*)off.p, n + 1, s),
          "scan");
  int32_t np = 0;
  CK_CUDA(cudaMemcpyAsync(&np, (int32_t*)off.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s),
          "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  CK_CUDA(cudaMemsetAsync(elim_ptr, 0, sizeof(int64_t) * ((size_t)nnz + 1), s), "memset");
  if (np == 0) return JV_OK;
  CK_CUDA(prow.alloc(sizeof(int32_t) * np), "alloc");
  CK_CUDA(ppos.alloc(sizeof(int32_t) * np), "alloc");
  elim_pairs_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, (const int32_t*)off.p,
                                                          (int32_t*)prow.p, (int32_t*)ppos.p);
  CK_CUDA(cnt.alloc(sizeof(long long) * ((size_t)nnz + 1)), "alloc");
  CK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(long long) * ((size_t)nnz + 1), s), "memset");
  const int g = grid_for((long long)np * 32);
  elim_match_kernel<false><<<g, 256, 0, s>>>(np, (const int32_t*)prow.p, (const int32_t*)ppos.p,
                                             row_start, col, diag_pos, milu, (long long*)cnt.p,
                                             nullptr, nullptr);
  size_t tb2 = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, (long long*)cnt.p, (long long*)elim_ptr,
                                        nnz + 1, s), "scan size");
  CK_CUDA(tmp2.alloc(tb2), "alloc");
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp2.p, tb2, (long long*)cnt.p, (long long*)elim_ptr,
                                        nnz + 1, s), "scan");
  elim_refine_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, diag_pos,
                                                           (const long long*)elim_ptr, heavy);
  long long total = 0;
  CK_CUDA(cudaMemcpyAsync(&total, elim_ptr + nnz, sizeof(long long), cudaMemcpyDeviceToHost, s),
          "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  *nops_h = total;
  if (elim != nullptr && total > 0)
    elim_match_kernel<true><<<g, 256, 0, s>>>(np, (const int32_t*)prow.p, (const int32_t*)ppos.p,
                                              row_start, col, diag_pos, milu, nullptr,
                                              (const long long*)elim_ptr,
                                              reinterpret_cast<int2*>(elim));
  JV_CHECK_LAUNCH("jv_elim_lists");
  return JV_OK;
}
