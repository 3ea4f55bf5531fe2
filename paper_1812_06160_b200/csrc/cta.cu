// Single-CTA level-synchronous kernels for small systems: the whole
// factorization (or one triangular sweep) of a matrix of at most
// kCtaMaxRows rows in ONE thread block, levels separated by __syncthreads
// instead of cross-SM mailbox hops (t_hop ~0.38 us, SURVEY.md §8d "depth
// bound").  Used for config 1 (4,096 rows, 127 levels) and for the compact
// corner of the two-stage lower tail (config 4: 20,572 rows, 271 levels),
// where the sync-free ticket kernel pays a hop per level.
//
// Factor (_kernels.py:165-204, factor_serial semantics): thread per row of
// the level, the row's pivots in ascending order, each pivot's updates from
// a precomputed list in (pivot, U entry) order — the same (target, pivot,
// q, kind) records the lower-tail plan builds (tail.cu), so tau drops and
// MILU mass follow _factor_row exactly; every op explicitly rounded.  Values
// live in shared memory when they fit (one bulk load, one write back),
// otherwise in L2 (ld/st.cg).  Solves (_kernels.py:348-366): thread per row,
// the reference subtraction order, the vector in shared memory when it fits.
#include "common.cuh"
#include "../../include/jv.h"

namespace {

constexpr int kCtaThreads = 1024;
constexpr int kCtaMaxRows = 1 << 16;
constexpr int kCtaSmemBytes = 200 * 1024;   // dynamic shared memory budget

struct CtaPlan {
  int32_t n;
  int64_t nl, nops;
  int milu;
  int32_t* lstart = nullptr;   // [n+1] first L index of each row
  long long* off = nullptr;    // [nl+1] op range of each L position
  int32_t* otgt = nullptr;
  int32_t* oq = nullptr;
  int8_t* ok = nullptr;
};

void free_cta(CtaPlan* P) {
  if (!P) return;
  void* ptrs[] = {P->lstart, P->off, P->otgt, P->oq, P->ok};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete P;
}

__global__ void cta_lcount_kernel(int n, const int32_t* rs, const int32_t* diag, int32_t* cnt) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    cnt[r] = diag[r] - rs[r];
}

__global__ void cta_lpos_kernel(int n, const int32_t* rs, const int32_t* lstart, int32_t* lpos,
                                int32_t* lrow) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int o = lstart[r], L = lstart[r + 1] - o, a = rs[r];
    for (int k = 0; k < L; ++k) {
      lpos[o + k] = a + k;
      lrow[o + k] = r;
    }
  }
}

// ---- level programs --------------------------------------------------
// Per level a block of int32 [nrows, rowoff[nrows], row programs...]
// (offsets relative to the block start, blocks 16-byte aligned), built on
// the host from the pattern and the update lists (jv_cta_program_host):
//   factor row: [r, a, len, soff, npiv, drel, then per pivot (prel, dc, nops),
//                then per op (wrel | kind << 30, q)]
//               own-row positions relative to a = row_start[r], pivot-row
//               positions (dc, q) absolute; soff = the row's slot in the
//               level's value stage (values in L2 mode)
//   solve row:  [r, a, cnt, soff, d, col[a .. a+cnt)]
// The kernel pipelines three levels: the program block of level L+2 and the
// row data of level L+1 (own-row values / the sweep's values and input
// entry, all final or untouched at that point) are copied with cp.async
// while level L computes; one __syncthreads per level.
constexpr int kHdrF = 6;
constexpr int kHdrS = 5;
constexpr unsigned kKindShift = 30;
constexpr int kPosMask = (1 << 30) - 1;

JV_INLINE uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
JV_INLINE void cpa4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
JV_INLINE void cpa8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
JV_INLINE void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
JV_INLINE void cpa_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct CtaArgs {
  int kind;            // 0 factor, 1 forward, 2 backward
  int n, nlev, nnz;
  const int32_t* prog;
  const int32_t* lbase;   // [nlev+1] block starts (ints)
  int maxblk, maxstage;
  int rb, pb;             // row-data / program ring depths (pb = 2 rb - 1)
  double* val;            // factor: in/out; solves: the factors
  const double* norms;
  double tau;
  int milu;
  const double* in;
  double* out;
  int32_t* err;
};

extern __shared__ __align__(16) double cta_smem[];

JV_INLINE void cpa_wait_n(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
  }
}

// Pipeline: at level L the program block of level L+pb-1 and the row data of
// level L+rb-1 are issued as one cp.async group; after computing L the
// kernel waits for all but the newest rb-2 groups, which leaves the program
// of level L+rb (needed to issue its rows next level) and the rows of L+1
// resident (pb = 2 rb - 1).
template <int Kind, bool Smem>
__global__ void __launch_bounds__(kCtaThreads, 1) cta_kernel(CtaArgs A) {
  const int tid = threadIdx.x;
  const int T = blockDim.x;   // sized to the widest level (jv_cta_run)
  // layout: [resident values (factor: nnz, solve: n) | rb value stages | pb program buffers]
  double* res = cta_smem;
  const int nres = Smem ? (Kind == 0 ? A.nnz : A.n) : 0;
  double* vst0 = res + nres;
  int32_t* pb0 = reinterpret_cast<int32_t*>(vst0 + (size_t)A.rb * A.maxstage);
  int32_t* lb = pb0 + (size_t)A.pb * A.maxblk;   // level block starts, resident
  for (int i = tid; i <= A.nlev; i += T) lb[i] = A.lbase[i];
  __syncthreads();
  // ring slot of level L is L mod depth; the per-level calls below pass
  // levels L, L+rb-1, L+pb-1 whose slots advance by one per level
  auto pbuf = [&](int L) { return pb0 + (size_t)(L % A.pb) * A.maxblk; };
  auto vbuf = [&](int L) { return vst0 + (size_t)(L % A.rb) * A.maxstage; };
  auto fetch_prog = [&](int L) {
    if (L >= A.nlev) return;
    const int b = lb[L], m = lb[L + 1] - b;
    int32_t* dst = pbuf(L);
    for (int i = tid; i < m; i += T) cpa4(dst + i, A.prog + b + i);
  };
  // row data of level L (its program must be resident)
  auto fetch_rows = [&](int L) {
    if (L >= A.nlev) return;
    if (Kind == 0 && Smem) return;
    const int32_t* P = pbuf(L);
    double* st = vbuf(L);
    const int nr = P[0];
    for (int j = tid; j < nr; j += T) {
      const int32_t* R = P + P[1 + j];
      const int r = R[0], a = R[1], len = R[2], soff = R[3];
      for (int k = 0; k < len; ++k) cpa8(st + soff + k, A.val + a + k);
      if (Kind != 0) {
        cpa8(st + soff + len, A.in + r);
        if (Kind == 2) cpa8(st + soff + len + 1, A.val + R[4]);
      }
    }
  };
  if (Smem) {
    if (Kind == 0)
      for (int i = tid; i < A.nnz; i += T) res[i] = A.val[i];
  }
  for (int L = 0; L < A.pb - 1; ++L) fetch_prog(L);
  cpa_commit();
  cpa_wait();
  __syncthreads();
  for (int L = 0; L < A.rb - 1; ++L) fetch_rows(L);
  cpa_commit();
  cpa_wait();
  __syncthreads();
  const bool use_tau = A.tau > 0.0;
  const jv::Trace tr = jv::trace_begin();   // diagnostics: per-level clocks (jv_set_trace)
  for (int L = 0; L < A.nlev; ++L) {
    if (tid == 0) jv::trace_mark(tr, L, 0);
    fetch_prog(L + A.pb - 1);
    fetch_rows(L + A.rb - 1);
    cpa_commit();
    if (tid == 0) jv::trace_mark(tr, L, 1);
    const int32_t* P = pbuf(L);
    double* st = vbuf(L);
    const int nr = P[0];
    for (int j = tid; j < nr; j += T) {
      const int32_t* R = P + P[1 + j];
      const int r = R[0];
      if (Kind == 0) {
        const int a = R[1], len = R[2], soff = R[3], npiv = R[4], drel = R[5];
        double* own = Smem ? res + a : st + soff;
        const double thr = use_tau ? jv::dmul(A.tau, A.norms[r]) : 0.0;
        const int32_t* pv = R + kHdrF;
        const int32_t* op = pv + 3 * npiv;
        for (int k = 0; k < npiv; ++k) {
          const int prel = pv[3 * k], dc = pv[3 * k + 1], no = pv[3 * k + 2];
          const double dv = Smem ? res[dc] : __ldcg(A.val + dc);
          // the pivot's U values do not depend on this row: load them all
          // before the division (one L2 round trip per pivot, not per op)
          constexpr int kB = 8;
          double u[kB];
#pragma unroll
          for (int o = 0; o < kB; ++o)
            if (o < no) u[o] = Smem ? res[op[2 * o + 1]] : __ldcg(A.val + op[2 * o + 1]);
          const double l = jv::ddiv(own[prel], dv);
          const bool drop = use_tau && fabs(l) < thr;
          own[prel] = drop ? 0.0 : l;
          for (int o0 = 0; o0 < no; o0 += kB) {
            if (o0)
#pragma unroll
              for (int o = 0; o < kB; ++o)
                if (o0 + o < no)
                  u[o] = Smem ? res[op[2 * (o0 + o) + 1]] : __ldcg(A.val + op[2 * (o0 + o) + 1]);
#pragma unroll
            for (int o = 0; o < kB; ++o) {
              if (o0 + o >= no) break;
              const int wk = op[2 * (o0 + o)];
              const int kind = (int)((unsigned)wk >> kKindShift);
              const bool apply = kind == 0 ? !drop : (kind == 1 ? true : drop);
              if (apply) {
                const int w = wk & kPosMask;
                own[w] = jv::dsub(own[w], jv::dmul(l, u[o]));
              }
            }
          }
          op += 2 * no;
        }
        if (own[drel] == 0.0) atomicMin(A.err, r);
        if (!Smem)
          for (int k = 0; k < len; ++k) __stcg(A.val + a + k, own[k]);
      } else {
        const int cnt = R[2], soff = R[3];
        const int32_t* cols = R + kHdrS;
        const double* v = st + soff;
        double s = v[cnt];
        double* x = Smem ? res : A.out;
        for (int k = 0; k < cnt; ++k) {
          const double xv = Smem ? x[cols[k]] : __ldcg(x + cols[k]);
          s = jv::dsub(s, jv::dmul(v[k], xv));
        }
        if (Kind == 2) s = jv::ddiv(s, v[cnt + 1]);
        if (Smem) x[r] = s; else __stcg(x + r, s);
      }
    }
    if (tid == 0) jv::trace_mark(tr, L, 2);
    cpa_wait_n(A.rb - 2);
    if (tid == 0) jv::trace_mark(tr, L, 3);
    __syncthreads();
  }
  cpa_wait();
  if (Smem) {
    if (Kind == 0)
      for (int i = tid; i < A.nnz; i += T) A.val[i] = res[i];
    else
      for (int i = tid; i < A.n; i += T) A.out[i] = res[i];
  }
}

template <typename K>
int cta_launch(K kernel, void* args, size_t smem, int threads, cudaStream_t s, const char* what) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return jvh::cuda_status(e, what);
  }
  void* a[] = {args};
  cudaError_t e = cudaLaunchKernel((const void*)kernel, dim3(1), dim3(threads), a, smem, s);
  if (e != cudaSuccess) return jvh::cuda_status(e, what);
  return JV_OK;
}

}  // namespace

extern "C" int jv_cta_max_rows(void) { return kCtaMaxRows; }

extern "C" int64_t jv_cta_plan_build(int32_t n, const int32_t* row_start, const int32_t* col,
                                     const int32_t* diag_pos, int milu, void* stream) {
  if (n < 0 || n > kCtaMaxRows) {
    jvh::set_error("jv_cta_plan_build: n=%d outside [0, %d]", n, kCtaMaxRows);
    return JV_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  CtaPlan* P = new CtaPlan();
  P->n = n;
  P->milu = milu ? 1 : 0;
  auto fail = [&](cudaError_t e, const char* what) -> int64_t {
    free_cta(P);
    return jvh::cuda_status(e, what);
  };
  cudaError_t e;
  Tmp cnt(s), lpos(s), lrow(s), lc(s);
  if ((e = dalloc(P->lstart, n + 1)) != cudaSuccess) return fail(e, "alloc");
  if ((e = cnt.alloc(4 * (size_t)(n + 1))) != cudaSuccess) return fail(e, "alloc");
  cta_lcount_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, diag_pos, (int32_t*)cnt.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)cnt.p + n, 0);
  if ((e = scan_excl((int32_t*)cnt.p, P->lstart, n + 1, s)) != cudaSuccess) return fail(e, "scan");
  int32_t nl = 0;
  cudaMemcpyAsync(&nl, P->lstart + n, 4, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e, "sync");
  P->nl = nl;
  if ((e = lpos.alloc(4 * (size_t)(nl + 1))) != cudaSuccess) return fail(e, "alloc");
  if ((e = lrow.alloc(4 * (size_t)(nl + 1))) != cudaSuccess) return fail(e, "alloc");
  cta_lpos_kernel<<<grid_for(n), kSetupThreads, 0, s>>>(n, row_start, P->lstart, (int32_t*)lpos.p,
                                                        (int32_t*)lrow.p);
  if ((e = lc.alloc(8 * (size_t)(nl + 1))) != cudaSuccess) return fail(e, "alloc");
  if ((e = dalloc(P->off, nl + 1)) != cudaSuccess) return fail(e, "alloc");
  cudaMemsetAsync((long long*)lc.p + nl, 0, 8, s);
  const int gw = grid_for((long long)nl * 32);
  if (nl)
    tail_ops_kernel<false><<<gw, kSetupThreads, 0, s>>>(nl, (const int32_t*)lpos.p,
                                                        (const int32_t*)lrow.p, row_start, col,
                                                        diag_pos, P->milu, (long long*)lc.p,
                                                        nullptr, nullptr, nullptr, nullptr, nullptr);
  if ((e = scan_excl((long long*)lc.p, P->off, (long long)nl + 1, s)) != cudaSuccess)
    return fail(e, "scan");
  long long nops = 0;
  cudaMemcpyAsync(&nops, P->off + nl, 8, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(e, "sync");
  P->nops = nops;
  if ((e = dalloc(P->otgt, nops)) != cudaSuccess) return fail(e, "alloc");
  if ((e = dalloc(P->oq, nops)) != cudaSuccess) return fail(e, "alloc");
  if ((e = dalloc(P->ok, nops)) != cudaSuccess) return fail(e, "alloc");
  int32_t* opiv = nullptr;
  if ((e = dalloc(opiv, nops)) != cudaSuccess) return fail(e, "alloc");
  if (nl && nops)
    tail_ops_kernel<true><<<gw, kSetupThreads, 0, s>>>(nl, (const int32_t*)lpos.p,
                                                       (const int32_t*)lrow.p, row_start, col,
                                                       diag_pos, P->milu, nullptr, P->off, P->otgt,
                                                       opiv, P->oq, P->ok);
  e = cudaStreamSynchronize(s);
  cudaFree(opiv);
  if (e != cudaSuccess) return fail(e, "sync");
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) return fail(le, "jv_cta_plan_build");
  return (int64_t)(intptr_t)P;
}

extern "C" int jv_cta_plan_export(int64_t h, int32_t* lstart_h, int64_t* off_h, int32_t* otgt_h,
                                  int32_t* oq_h, int8_t* ok_h, int64_t* info_h) {
  const CtaPlan* P = (const CtaPlan*)(intptr_t)h;
  if (!P) { jvh::set_error("jv_cta_plan_export: null plan"); return JV_EINVAL; }
  info_h[0] = P->nl;
  info_h[1] = P->nops;
  info_h[2] = P->n;
  info_h[3] = P->milu;
  if (!lstart_h) return JV_OK;
  CK_CUDA(cudaMemcpy(lstart_h, P->lstart, 4 * (size_t)(P->n + 1), cudaMemcpyDeviceToHost), "copy");
  CK_CUDA(cudaMemcpy(off_h, P->off, 8 * (size_t)(P->nl + 1), cudaMemcpyDeviceToHost), "copy");
  if (P->nops) {
    CK_CUDA(cudaMemcpy(otgt_h, P->otgt, 4 * (size_t)P->nops, cudaMemcpyDeviceToHost), "copy");
    CK_CUDA(cudaMemcpy(oq_h, P->oq, 4 * (size_t)P->nops, cudaMemcpyDeviceToHost), "copy");
    if (P->milu)
      CK_CUDA(cudaMemcpy(ok_h, P->ok, (size_t)P->nops, cudaMemcpyDeviceToHost), "copy");
  }
  return JV_OK;
}

extern "C" int jv_cta_plan_free(int64_t h) {
  free_cta((CtaPlan*)(intptr_t)h);
  return JV_OK;
}

// Host: the level programs of one sweep (two calls: sizes, then fill).
// sizes_h = {total ints, max block ints, max stage doubles}.
extern "C" int jv_cta_program_host(int kind, int32_t n, const int32_t* rs, const int32_t* col,
                                   const int32_t* diag, const int32_t* order,
                                   const int32_t* level_ptr, int32_t nlev, const int32_t* lstart,
                                   const int64_t* off, const int32_t* otgt, const int32_t* oq,
                                   const int8_t* ok, int milu, int32_t* prog_h, int32_t* lbase_h,
                                   int64_t* sizes_h) {
  if (n < 0 || nlev < 0 || kind < 0 || kind > 2) {
    jvh::set_error("jv_cta_program_host: bad arguments");
    return JV_EINVAL;
  }
  int64_t pos = 0, maxblk = 0, maxstage = 0;
  for (int L = 0; L < nlev; ++L) {
    const int i0 = level_ptr[L], i1 = level_ptr[L + 1], nr = i1 - i0;
    const int64_t base = pos;
    if (lbase_h) lbase_h[L] = (int32_t)base;
    int64_t cur = 1 + nr;   // header
    int64_t stage = 0;
    for (int j = 0; j < nr; ++j) {
      const int r = order[i0 + j];
      if (prog_h) prog_h[base + 1 + j] = (int32_t)cur;
      int32_t* R = prog_h ? prog_h + base + cur : nullptr;
      const int a = rs[r], d = diag[r];
      if (kind == 0) {
        const int len = rs[r + 1] - a, npiv = d - a;
        int64_t nops = off[lstart[r] + npiv] - off[lstart[r]];
        if (R) {
          R[0] = r; R[1] = a; R[2] = len; R[3] = (int32_t)stage; R[4] = npiv; R[5] = d - a;
          int32_t* pv = R + kHdrF;
          int32_t* op = pv + 3 * npiv;
          for (int k = 0; k < npiv; ++k) {
            const int64_t o0 = off[lstart[r] + k], o1 = off[lstart[r] + k + 1];
            pv[3 * k] = k;
            pv[3 * k + 1] = diag[col[a + k]];
            pv[3 * k + 2] = (int32_t)(o1 - o0);
            for (int64_t o = o0; o < o1; ++o) {
              const int kd = milu ? ok[o] : 0;
              *op++ = (int32_t)(((unsigned)kd << kKindShift) | (unsigned)(otgt[o] - a));
              *op++ = oq[o];
            }
          }
        }
        cur += kHdrF + 3 * npiv + 2 * nops;
        stage += len;
      } else {
        const int lo = kind == 1 ? a : d + 1;
        const int cnt = kind == 1 ? d - a : rs[r + 1] - d - 1;
        if (R) {
          R[0] = r; R[1] = lo; R[2] = cnt; R[3] = (int32_t)stage; R[4] = d;
          for (int k = 0; k < cnt; ++k) R[kHdrS + k] = col[lo + k];
        }
        cur += kHdrS + cnt;
        stage += cnt + 2;
      }
    }
    if (prog_h) prog_h[base] = nr;
    cur = (cur + 3) & ~3LL;   // 16-byte aligned blocks
    pos += cur;
    maxblk = cur > maxblk ? cur : maxblk;
    maxstage = stage > maxstage ? stage : maxstage;
  }
  if (lbase_h) lbase_h[nlev] = (int32_t)pos;
  if (pos >= (1LL << 31)) {
    jvh::set_error("jv_cta_program_host: program too large");
    return JV_EINVAL;
  }
  sizes_h[0] = pos;
  sizes_h[1] = maxblk;
  sizes_h[2] = (maxstage + 1) & ~1LL;
  return JV_OK;
}

// Shared memory a launch needs (bytes) with a row-data ring of depth rb
// (program ring 2 rb - 1), or -1 when it does not fit one CTA.
extern "C" int64_t jv_cta_smem(int kind, int32_t n, int64_t nnz, int32_t nlev, int64_t maxblk,
                               int64_t maxstage, int resident, int rb) {
  if (rb < 2 || rb > 6) return -1;
  const int64_t res = resident ? 8 * (kind == 0 ? nnz : (int64_t)n) : 0;
  const int64_t stage = (kind == 0 && resident) ? 0 : rb * 8 * maxstage;
  const int64_t total = res + stage + (2 * rb - 1) * 4 * maxblk + 4 * ((int64_t)nlev + 1);
  return total <= kCtaSmemBytes ? total : -1;
}

extern "C" int jv_cta_run(int kind, int32_t n, int64_t nnz, int32_t nlev, const int32_t* prog,
                          const int32_t* lbase, int64_t maxblk, int64_t maxstage, int resident,
                          int rb, int32_t maxrows,
                          double* val, const double* norms, double tau, int milu, const double* in,
                          double* out, int32_t* err_row, void* stream) {
  if (n < 0 || n > kCtaMaxRows || kind < 0 || kind > 2) {
    jvh::set_error("jv_cta_run: bad arguments");
    return JV_EINVAL;
  }
  if (n == 0 || nlev == 0) return JV_OK;
  const int64_t smem = jv_cta_smem(kind, n, nnz, nlev, maxblk, maxstage, resident, rb);
  if (smem < 0) {
    jvh::set_error("jv_cta_run: level programs do not fit one CTA's shared memory");
    return JV_EINVAL;
  }
  if (kind == 0 && tau > 0.0 && !norms) {
    jvh::set_error("jv_cta_run: tau > 0 needs row norms");
    return JV_EINVAL;
  }
  CtaArgs A;
  A.kind = kind;
  A.n = n;
  A.nlev = nlev;
  A.nnz = (int)nnz;
  A.prog = prog;
  A.lbase = lbase;
  A.maxblk = (int)maxblk;
  A.maxstage = (kind == 0 && resident) ? 0 : (int)maxstage;   // layout as jv_cta_smem
  A.rb = rb;
  A.pb = 2 * rb - 1;
  // the block is as wide as the widest level (every thread of a level loop
  // costs issue slots, busy or not): 64 .. 1024 threads
  int threads = 64;
  while (threads < maxrows && threads < kCtaThreads) threads *= 2;
  A.val = val;
  A.norms = norms;
  A.tau = tau;
  A.milu = milu;
  A.in = in;
  A.out = out;
  A.err = err_row;
  cudaStream_t s = (cudaStream_t)stream;
  if (kind == 0)
    return resident ? cta_launch(cta_kernel<0, true>, &A, smem, threads, s, "jv_cta_run")
                    : cta_launch(cta_kernel<0, false>, &A, smem, threads, s, "jv_cta_run");
  if (kind == 1)
    return resident ? cta_launch(cta_kernel<1, true>, &A, smem, threads, s, "jv_cta_run")
                    : cta_launch(cta_kernel<1, false>, &A, smem, threads, s, "jv_cta_run");
  return resident ? cta_launch(cta_kernel<2, true>, &A, smem, threads, s, "jv_cta_run")
                  : cta_launch(cta_kernel<2, false>, &A, smem, threads, s, "jv_cta_run");
}
