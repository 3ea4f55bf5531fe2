// Lower-tail ("second stage") factorization: the rows the partition rule
// excluded from level scheduling, rows [n_upper, n) of the level-ordered
// factor storage (reference lower.py:126-318, _kernels.py:221-343).
//
// Stage 1 (the SR / ER stage, jv_tail_upper): every tail row eliminates its
// upper-stage pivots (columns < n_upper).  Those pivots are final when the
// stage starts, so tail rows are independent of each other; within a row the
// reference applies the pivots in ascending column order.  One warp per
// tail row, segmented:
//   * the row's upper-pivot L positions are cut into groups such that no
//     position receives an update from a pivot of its own group (the
//     structural condition the reference's SR needs per level,
//     lower.py:199-211, computed per row here so it also holds for fill
//     patterns); DIVIDE runs over a group's positions in parallel (lanes);
//   * UPDATE is a segmented reduction: the group's updates are sorted by
//     (target position, pivot, U entry) and every segment (one target) is
//     folded by one lane in that order, val[w] -= l*u explicitly rounded,
//     so each stored position sees exactly the reference's subtraction
//     sequence (bitwise, _kernels.py:259-323).  MILU mass and tau drops
//     follow _update_task: a dropped pivot sends all of l*U(c) to the
//     diagonal, a kept one only its out-of-pattern part.
// Stage 2 (the corner, columns >= n_upper, _kernels.py:231-254): exported as
// a compact CSR (jv_tail_corner) that the host factors with the sync-free
// ticket kernel and scatters back.
//
// The plan (ops, groups, segments, corner pattern) depends on the pattern
// only and is built once on the device (jv_tail_plan_build).
#include "common.cuh"
#include "../../include/jv.h"

#include <cub/cub.cuh>

namespace {

struct TailPlan {
  int32_t n, n_upper, nt;
  int32_t tb;          // first storage position of the tail (row_start[n_upper])
  int32_t tnnz;        // storage positions of the tail rows
  int64_t nl;          // upper-pivot L positions of the tail
  int64_t nops, ng, ns;
  int64_t ncorner;
  int milu;
  // device
  int32_t* gbase = nullptr;     // [nt+1] group range per tail row
  int32_t* ga = nullptr;        // [ng+1] first L position of group (ga[G+1] or row end bounds it)
  int32_t* gb = nullptr;        // [ng]   one past the last L position of group
  int32_t* gsp = nullptr;       // [ng+1] segment range per group
  int32_t* seg_tgt = nullptr;   // [ns]
  int32_t* seg_optr = nullptr;  // [ns+1]
  int32_t* op_p = nullptr;      // [nops] sorted (group, target, pivot, q)
  int32_t* op_q = nullptr;
  int8_t* op_k = nullptr;       // kinds (MILU only)
  double* lbuf = nullptr;       // [tnnz] multipliers (tau > 0)
  int8_t* dfl = nullptr;        // [tnnz] drop flags (tau > 0)
  int32_t* crs = nullptr;       // [nt+1] compact corner row_start
  int32_t* ccol = nullptr;      // [ncorner]
  int32_t* cdiag = nullptr;     // [nt]
  int32_t* cpos = nullptr;      // [ncorner] storage position of each corner entry
};

template <typename T>
cudaError_t dalloc(T*& p, size_t count) {
  return cudaMalloc((void**)&p, sizeof(T) * (count ? count : 1));
}

__device__ __forceinline__ int lbound(const int32_t* col, int lo, int hi, int key) {
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (col[m] < key) lo = m + 1; else hi = m;
  }
  return lo;
}

// per tail row: number of upper-pivot L positions and of corner entries
__global__ void tail_count_kernel(int nt, int n_upper, const int32_t* rs, const int32_t* col,
                                  int32_t* lcnt, int32_t* ccnt) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const int r = n_upper + t;
    const int a = rs[r], b = rs[r + 1];
    const int e = lbound(col, a, b, n_upper);
    lcnt[t] = e - a;
    ccnt[t] = b - e;
  }
}

// flat list of the tail's upper-pivot L positions (warp per row)
__global__ void tail_lpos_kernel(int nt, int n_upper, const int32_t* rs, const int32_t* lptr,
                                 int32_t* lpos, int32_t* lrow, const int32_t* crs, const int32_t* col,
                                 const int32_t* diag, int32_t* ccol, int32_t* cdiag, int32_t* cpos) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int W = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < nt; t += W) {
    const int r = n_upper + t;
    const int a = rs[r], b = rs[r + 1];
    const int o = lptr[t], L = lptr[t + 1] - o;
    for (int k = lane; k < L; k += 32) {
      lpos[o + k] = a + k;
      lrow[o + k] = r;
    }
    const int co = crs[t];
    for (int k = a + L + lane; k < b; k += 32) {
      ccol[co + (k - a - L)] = col[k] - n_upper;
      cpos[co + (k - a - L)] = k;
    }
    if (lane == 0) cdiag[t] = co + (diag[r] - a - L);
  }
}

// ops of every (tail row, upper pivot) pair, in (pivot, q) order:
//   non-MILU: in-pattern match w -> (w, kind 0: applied iff the pivot is kept)
//   MILU:     match w != diag -> (w, 0) + (diag, 2: applied iff dropped)
//             match w == diag -> (diag, 1: always)
//             no match        -> (diag, 1: always, out-of-pattern mass)
template <bool Fill>
__global__ void tail_ops_kernel(long long nl, const int32_t* lpos, const int32_t* lrow,
                                const int32_t* rs, const int32_t* col, const int32_t* diag, int milu,
                                long long* cnt, const long long* off, int32_t* otgt, int32_t* op,
                                int32_t* oq, int8_t* ok) {
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = gw; i < nl; i += W) {
    const int p = lpos[i], r = lrow[i];
    const int c = col[p];
    const int re = rs[r + 1], dpos = diag[r];
    const int q0 = diag[c] + 1, q1 = rs[c + 1];
    long long m = 0;
    const long long base = Fill ? off[i] : 0;
    for (int qb = q0; qb < q1; qb += 32) {
      const int q = qb + lane;
      int w = -1, nemit = 0;
      if (q < q1) {
        const int j = col[q];
        const int f = lbound(col, p + 1, re, j);
        if (f < re && col[f] == j) w = f;
        nemit = milu ? ((w >= 0 && w != dpos) ? 2 : 1) : (w >= 0 ? 1 : 0);
      }
      int incl = nemit;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (Fill && nemit) {
        long long at = base + m + incl - nemit;
        if (!milu) {
          otgt[at] = w; op[at] = p; oq[at] = q;
        } else if (w >= 0 && w != dpos) {
          otgt[at] = w; op[at] = p; oq[at] = q; ok[at] = 0;
          otgt[at + 1] = dpos; op[at + 1] = p; oq[at + 1] = q; ok[at + 1] = 2;
        } else {
          otgt[at] = dpos; op[at] = p; oq[at] = q; ok[at] = 1;
        }
      }
      m += tot;
    }
    if (!Fill && lane == 0) cnt[i] = m;
  }
}

__global__ void fill_int_kernel(long long n, int32_t* a, int32_t v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}

// latest pivot position updating each upper-pivot L position
__global__ void tail_maxsrc_kernel(long long nops, int n_upper, int tb, const int32_t* col,
                                   const int32_t* otgt, const int32_t* op, int32_t* maxsrc) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nops;
       i += (long long)gridDim.x * blockDim.x) {
    const int w = otgt[i];
    if (col[w] < n_upper) atomicMax(maxsrc + (w - tb), op[i]);
  }
}

// groups per tail row: a new group starts at position k when k receives an
// update from a pivot of the current group
template <bool Fill>
__global__ void tail_groups_kernel(int nt, int n_upper, int tb, const int32_t* rs,
                                   const int32_t* lptr, const int32_t* maxsrc, int32_t* gcnt,
                                   const int32_t* gbase, int32_t* ga, int32_t* gb, int32_t* gid) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const int r = n_upper + t;
    const int a = rs[r], e = a + (lptr[t + 1] - lptr[t]);
    int g = -1, start = a;
    const int G0 = Fill ? gbase[t] : 0;
    for (int k = a; k < e; ++k) {
      if (k == a || maxsrc[k - tb] >= start) {
        if (Fill && g >= 0) gb[G0 + g] = k;
        start = k;
        ++g;
        if (Fill) ga[G0 + g] = k;
      }
      if (Fill) gid[k - tb] = G0 + g;
    }
    if (Fill && g >= 0) gb[G0 + g] = e;
    if (!Fill) gcnt[t] = g + 1;
  }
}

__global__ void tail_keys_kernel(long long nops, int tb, const int32_t* otgt, const int32_t* op,
                                 const int32_t* gid, unsigned long long* key, int32_t* idx) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nops;
       i += (long long)gridDim.x * blockDim.x) {
    key[i] = ((unsigned long long)(uint32_t)gid[op[i] - tb] << 32) | (uint32_t)otgt[i];
    idx[i] = (int32_t)i;
  }
}

__global__ void tail_heads_kernel(long long nops, const unsigned long long* key, int32_t* head) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nops;
       i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

__global__ void tail_segs_kernel(long long nops, const unsigned long long* key, const int32_t* head,
                                 const int32_t* sid, const int32_t* idx, const int32_t* op,
                                 const int32_t* oq, const int8_t* ok, int32_t* seg_tgt,
                                 int32_t* seg_grp, int32_t* seg_optr, int32_t* sp, int32_t* sq,
                                 int8_t* sk) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nops;
       i += (long long)gridDim.x * blockDim.x) {
    if (head[i]) {
      const int s = sid[i];
      seg_tgt[s] = (int32_t)(key[i] & 0xffffffffull);
      seg_grp[s] = (int32_t)(key[i] >> 32);
      seg_optr[s] = (int32_t)i;
    }
    const int j = idx[i];
    sp[i] = op[j];
    sq[i] = oq[j];
    if (sk) sk[i] = ok[j];
  }
}

__global__ void tail_gsp_kernel(long long ng, long long ns, const int32_t* seg_grp, int32_t* gsp,
                                int32_t* seg_optr, long long nops) {
  for (long long G = (long long)blockIdx.x * blockDim.x + threadIdx.x; G <= ng;
       G += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = ns;
    while (lo < hi) {
      const long long m = (lo + hi) >> 1;
      if (seg_grp[m] < G) lo = m + 1; else hi = m;
    }
    gsp[G] = (int32_t)lo;
    if (G == 0) seg_optr[ns] = (int32_t)nops;
  }
}

// ---------------------------------------------------------------- stage 1
struct TailArgs {
  int nt, n_upper, tb;
  const int32_t* col;
  const int32_t* diag;
  const int32_t* gbase;
  const int32_t* ga;
  const int32_t* gb;
  const int32_t* gsp;
  const int32_t* seg_tgt;
  const int32_t* seg_optr;
  const int32_t* op_p;
  const int32_t* op_q;
  const int8_t* op_k;
  double* val;
  const double* norms;
  double tau;
  int milu;
  double* lbuf;
  int8_t* dfl;
};

__global__ void __launch_bounds__(256) tail_upper_kernel(TailArgs A) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int W = (gridDim.x * blockDim.x) >> 5;
  const bool use_tau = A.tau > 0.0;
  for (int t = gw; t < A.nt; t += W) {
    const int r = A.n_upper + t;
    const double thr = use_tau ? __dmul_rn(A.tau, A.norms[r]) : 0.0;
    const int G0 = A.gbase[t], G1 = A.gbase[t + 1];
    for (int G = G0; G < G1; ++G) {
      // DIVIDE: multipliers of the group's pivots (independent)
      const int a = A.ga[G], b = A.gb[G];
      for (int k = a + lane; k < b; k += 32) {
        const int c = A.col[k];
        const double l = __ddiv_rn(A.val[k], __ldcg(A.val + A.diag[c]));
        if (use_tau) {
          const bool drop = fabs(l) < thr;
          A.lbuf[k - A.tb] = l;
          A.dfl[k - A.tb] = drop ? 1 : 0;
          A.val[k] = drop ? 0.0 : l;
        } else {
          A.val[k] = l;
        }
      }
      __syncwarp();
      // UPDATE: one lane per target, the target's updates in pivot order
      const int s1 = A.gsp[G + 1];
      for (int s = A.gsp[G] + lane; s < s1; s += 32) {
        const int w = A.seg_tgt[s];
        double acc = A.val[w];
        const int o1 = A.seg_optr[s + 1];
        for (int o = A.seg_optr[s]; o < o1; ++o) {
          const int p = A.op_p[o];
          const double u = __ldcg(A.val + A.op_q[o]);
          double l;
          bool apply = true;
          if (use_tau) {
            l = A.lbuf[p - A.tb];
            const bool drop = A.dfl[p - A.tb] != 0;
            const int kind = A.milu ? A.op_k[o] : 0;
            apply = kind == 0 ? !drop : (kind == 1 ? true : drop);
          } else {
            l = A.val[p];
            if (A.milu) apply = A.op_k[o] != 2;
          }
          if (apply) acc = __dsub_rn(acc, __dmul_rn(l, u));
        }
        A.val[w] = acc;
      }
      __syncwarp();
    }
  }
}

__global__ void scatter_f64_kernel(long long n, const int32_t* idx, const double* src, double* dst) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[idx[i]] = src[i];
}

template <typename T>
cudaError_t scan_excl(const T* in, T* out, long long n, cudaStream_t s) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  if (e != cudaSuccess) return e;
  void* tmp = nullptr;
  e = cudaMallocAsync(&tmp, tb ? tb : 1, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n, s);
  cudaFreeAsync(tmp, s);
  return e;
}

void free_plan(TailPlan* P) {
  if (!P) return;
  void* ptrs[] = {P->gbase, P->ga, P->gb, P->gsp, P->seg_tgt, P->seg_optr, P->op_p, P->op_q,
                  P->op_k, P->lbuf, P->dfl, P->crs, P->ccol, P->cdiag, P->cpos};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete P;
}

int build_plan(TailPlan* P, const int32_t* rs, const int32_t* col, const int32_t* diag,
               cudaStream_t s) {
  const int nt = P->nt;
  Tmp lcnt(s), ccnt(s), lptr(s), lpos(s), lrow(s), cnt(s), off(s), otgt(s), op(s), oq(s), ok(s),
      maxsrc(s), gcnt(s), gid(s), key(s), key2(s), idx(s), idx2(s), head(s), sid(s), sgrp(s),
      stmp(s);
  CK_CUDA(lcnt.alloc(4 * (size_t)(nt + 1)), "alloc");
  CK_CUDA(ccnt.alloc(4 * (size_t)(nt + 1)), "alloc");
  CK_CUDA(lptr.alloc(4 * (size_t)(nt + 1)), "alloc");
  CK_CUDA(dalloc(P->crs, nt + 1), "alloc");
  tail_count_kernel<<<grid_for(nt), kSetupThreads, 0, s>>>(nt, P->n_upper, rs, col,
                                                           (int32_t*)lcnt.p, (int32_t*)ccnt.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)lcnt.p + nt, 0);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)ccnt.p + nt, 0);
  CK_CUDA(scan_excl((int32_t*)lcnt.p, (int32_t*)lptr.p, nt + 1, s), "scan");
  CK_CUDA(scan_excl((int32_t*)ccnt.p, P->crs, nt + 1, s), "scan");
  int32_t hv[2] = {0, 0};
  CK_CUDA(cudaMemcpyAsync(&hv[0], (int32_t*)lptr.p + nt, 4, cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaMemcpyAsync(&hv[1], P->crs + nt, 4, cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  P->nl = hv[0];
  P->ncorner = hv[1];
  CK_CUDA(lpos.alloc(4 * (size_t)P->nl), "alloc");
  CK_CUDA(lrow.alloc(4 * (size_t)P->nl), "alloc");
  CK_CUDA(dalloc(P->ccol, P->ncorner), "alloc");
  CK_CUDA(dalloc(P->cpos, P->ncorner), "alloc");
  CK_CUDA(dalloc(P->cdiag, nt), "alloc");
  tail_lpos_kernel<<<grid_for((long long)nt * 32), kSetupThreads, 0, s>>>(
      nt, P->n_upper, rs, (const int32_t*)lptr.p, (int32_t*)lpos.p, (int32_t*)lrow.p, P->crs, col,
      diag, P->ccol, P->cdiag, P->cpos);
  CK_CUDA(dalloc(P->lbuf, P->tnnz), "alloc");
  CK_CUDA(dalloc(P->dfl, P->tnnz), "alloc");
  CK_CUDA(dalloc(P->gbase, nt + 1), "alloc");
  if (P->nl == 0) {
    CK_CUDA(cudaMemsetAsync(P->gbase, 0, 4 * (size_t)(nt + 1), s), "memset");
    P->nops = P->ng = P->ns = 0;
    CK_CUDA(dalloc(P->ga, 1), "alloc");
    CK_CUDA(dalloc(P->gb, 1), "alloc");
    CK_CUDA(dalloc(P->gsp, 1), "alloc");
    CK_CUDA(cudaMemsetAsync(P->gsp, 0, 4, s), "memset");
    CK_CUDA(dalloc(P->seg_tgt, 1), "alloc");
    CK_CUDA(dalloc(P->seg_optr, 1), "alloc");
    CK_CUDA(dalloc(P->op_p, 1), "alloc");
    CK_CUDA(dalloc(P->op_q, 1), "alloc");
    CK_CUDA(cudaStreamSynchronize(s), "sync");
    JV_CHECK_LAUNCH("jv_tail_plan_build");
    return JV_OK;
  }
  // ops
  const long long nl = P->nl;
  CK_CUDA(cnt.alloc(8 * (size_t)(nl + 1)), "alloc");
  CK_CUDA(off.alloc(8 * (size_t)(nl + 1)), "alloc");
  CK_CUDA(cudaMemsetAsync((long long*)cnt.p + nl, 0, 8, s), "memset");
  const int gw = grid_for(nl * 32);
  tail_ops_kernel<false><<<gw, kSetupThreads, 0, s>>>(nl, (const int32_t*)lpos.p,
                                                      (const int32_t*)lrow.p, rs, col, diag,
                                                      P->milu, (long long*)cnt.p, nullptr, nullptr,
                                                      nullptr, nullptr, nullptr);
  CK_CUDA(scan_excl((long long*)cnt.p, (long long*)off.p, nl + 1, s), "scan");
  long long nops = 0;
  CK_CUDA(cudaMemcpyAsync(&nops, (long long*)off.p + nl, 8, cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  if (nops >= (1LL << 31) - 2) {
    jvh::set_error("jv_tail_plan_build: %lld updates exceed int32", nops);
    return JV_EINVAL;
  }
  P->nops = nops;
  const long long no = nops > 0 ? nops : 1;
  CK_CUDA(otgt.alloc(4 * no), "alloc");
  CK_CUDA(op.alloc(4 * no), "alloc");
  CK_CUDA(oq.alloc(4 * no), "alloc");
  CK_CUDA(ok.alloc(no), "alloc");
  tail_ops_kernel<true><<<gw, kSetupThreads, 0, s>>>(
      nl, (const int32_t*)lpos.p, (const int32_t*)lrow.p, rs, col, diag, P->milu, nullptr,
      (const long long*)off.p, (int32_t*)otgt.p, (int32_t*)op.p, (int32_t*)oq.p, (int8_t*)ok.p);
  // groups
  CK_CUDA(maxsrc.alloc(4 * (size_t)P->tnnz), "alloc");
  fill_int_kernel<<<grid_for(P->tnnz), kSetupThreads, 0, s>>>(P->tnnz, (int32_t*)maxsrc.p, -1);
  if (nops)
    tail_maxsrc_kernel<<<grid_for(nops), kSetupThreads, 0, s>>>(
        nops, P->n_upper, P->tb, col, (const int32_t*)otgt.p, (const int32_t*)op.p,
        (int32_t*)maxsrc.p);
  CK_CUDA(gcnt.alloc(4 * (size_t)(nt + 1)), "alloc");
  tail_groups_kernel<false><<<grid_for(nt, 64), 64, 0, s>>>(
      nt, P->n_upper, P->tb, rs, (const int32_t*)lptr.p, (const int32_t*)maxsrc.p,
      (int32_t*)gcnt.p, nullptr, nullptr, nullptr, nullptr);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)gcnt.p + nt, 0);
  CK_CUDA(scan_excl((int32_t*)gcnt.p, P->gbase, nt + 1, s), "scan");
  int32_t ng = 0;
  CK_CUDA(cudaMemcpyAsync(&ng, P->gbase + nt, 4, cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  P->ng = ng;
  CK_CUDA(dalloc(P->ga, ng + 1), "alloc");
  CK_CUDA(dalloc(P->gb, ng + 1), "alloc");
  CK_CUDA(gid.alloc(4 * (size_t)P->tnnz), "alloc");
  tail_groups_kernel<true><<<grid_for(nt, 64), 64, 0, s>>>(
      nt, P->n_upper, P->tb, rs, (const int32_t*)lptr.p, (const int32_t*)maxsrc.p, nullptr,
      P->gbase, P->ga, P->gb, (int32_t*)gid.p);
  // sort ops by (group, target), stable over the (pivot, q) generation order
  CK_CUDA(key.alloc(8 * no), "alloc");
  CK_CUDA(key2.alloc(8 * no), "alloc");
  CK_CUDA(idx.alloc(4 * no), "alloc");
  CK_CUDA(idx2.alloc(4 * no), "alloc");
  if (nops) {
    tail_keys_kernel<<<grid_for(nops), kSetupThreads, 0, s>>>(
        nops, P->tb, (const int32_t*)otgt.p, (const int32_t*)op.p, (const int32_t*)gid.p,
        (unsigned long long*)key.p, (int32_t*)idx.p);
    size_t tb = 0;
    CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, (unsigned long long*)key.p,
                                            (unsigned long long*)key2.p, (int32_t*)idx.p,
                                            (int32_t*)idx2.p, (int)nops, 0, 64, s), "sort size");
    CK_CUDA(stmp.alloc(tb), "alloc");
    CK_CUDA(cub::DeviceRadixSort::SortPairs(stmp.p, tb, (unsigned long long*)key.p,
                                            (unsigned long long*)key2.p, (int32_t*)idx.p,
                                            (int32_t*)idx2.p, (int)nops, 0, 64, s), "sort");
  }
  CK_CUDA(head.alloc(4 * (no + 1)), "alloc");
  CK_CUDA(sid.alloc(4 * (no + 1)), "alloc");
  if (nops)
    tail_heads_kernel<<<grid_for(nops), kSetupThreads, 0, s>>>(nops, (const unsigned long long*)key2.p,
                                                              (int32_t*)head.p);
  set_int_kernel<<<1, 1, 0, s>>>((int32_t*)head.p + nops, 0);
  CK_CUDA(scan_excl((int32_t*)head.p, (int32_t*)sid.p, nops + 1, s), "scan");
  int32_t ns = 0;
  CK_CUDA(cudaMemcpyAsync(&ns, (int32_t*)sid.p + nops, 4, cudaMemcpyDeviceToHost, s), "copy");
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  P->ns = ns;
  CK_CUDA(dalloc(P->seg_tgt, ns), "alloc");
  CK_CUDA(dalloc(P->seg_optr, ns + 1), "alloc");
  CK_CUDA(sgrp.alloc(4 * (size_t)(ns + 1)), "alloc");
  CK_CUDA(dalloc(P->op_p, no), "alloc");
  CK_CUDA(dalloc(P->op_q, no), "alloc");
  if (P->milu) CK_CUDA(dalloc(P->op_k, no), "alloc");
  if (nops)
    tail_segs_kernel<<<grid_for(nops), kSetupThreads, 0, s>>>(
        nops, (const unsigned long long*)key2.p, (const int32_t*)head.p, (const int32_t*)sid.p,
        (const int32_t*)idx2.p, (const int32_t*)op.p, (const int32_t*)oq.p,
        (const int8_t*)ok.p, P->seg_tgt, (int32_t*)sgrp.p, P->seg_optr, P->op_p, P->op_q,
        P->milu ? P->op_k : nullptr);
  CK_CUDA(dalloc(P->gsp, ng + 1), "alloc");
  tail_gsp_kernel<<<grid_for((long long)ng + 1), kSetupThreads, 0, s>>>(
      ng, ns, (const int32_t*)sgrp.p, P->gsp, P->seg_optr, nops);
  CK_CUDA(cudaStreamSynchronize(s), "sync");
  JV_CHECK_LAUNCH("jv_tail_plan_build");
  return JV_OK;
}

}  // namespace

extern "C" int64_t jv_tail_plan_build(int32_t n, int32_t n_upper, const int32_t* row_start,
                                      const int32_t* col, const int32_t* diag_pos, int milu,
                                      void* stream) {
  if (n < 0 || n_upper < 0 || n_upper > n) {
    jvh::set_error("jv_tail_plan_build: bad sizes n=%d n_upper=%d", n, n_upper);
    return JV_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  TailPlan* P = new TailPlan();
  P->n = n;
  P->n_upper = n_upper;
  P->nt = n - n_upper;
  P->milu = milu ? 1 : 0;
  int32_t hv[2] = {0, 0};
  cudaMemcpyAsync(&hv[0], row_start + n_upper, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hv[1], row_start + n, 4, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    free_plan(P);
    return jvh::cuda_status(cudaGetLastError(), "jv_tail_plan_build");
  }
  P->tb = hv[0];
  P->tnnz = hv[1] - hv[0];
  const int rc = build_plan(P, row_start, col, diag_pos, s);
  if (rc != JV_OK) {
    free_plan(P);
    return rc;
  }
  return (int64_t)(intptr_t)P;
}

extern "C" int jv_tail_plan_info(int64_t h, int64_t* info) {
  const TailPlan* P = (const TailPlan*)(intptr_t)h;
  if (!P || !info) { jvh::set_error("jv_tail_plan_info: null"); return JV_EINVAL; }
  info[0] = P->nt;
  info[1] = P->nl;
  info[2] = P->nops;
  info[3] = P->ng;
  info[4] = P->ns;
  info[5] = P->ncorner;
  return JV_OK;
}

extern "C" int jv_tail_corner(int64_t h, int32_t* row_start, int32_t* col, int32_t* diag_pos,
                              int32_t* pos, void* stream) {
  const TailPlan* P = (const TailPlan*)(intptr_t)h;
  if (!P) { jvh::set_error("jv_tail_corner: null plan"); return JV_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  CK_CUDA(cudaMemcpyAsync(row_start, P->crs, 4 * (size_t)(P->nt + 1), cudaMemcpyDeviceToDevice, s),
          "copy");
  if (P->ncorner) {
    CK_CUDA(cudaMemcpyAsync(col, P->ccol, 4 * (size_t)P->ncorner, cudaMemcpyDeviceToDevice, s),
            "copy");
    CK_CUDA(cudaMemcpyAsync(pos, P->cpos, 4 * (size_t)P->ncorner, cudaMemcpyDeviceToDevice, s),
            "copy");
  }
  if (P->nt)
    CK_CUDA(cudaMemcpyAsync(diag_pos, P->cdiag, 4 * (size_t)P->nt, cudaMemcpyDeviceToDevice, s),
            "copy");
  return JV_OK;
}

extern "C" int jv_tail_upper(int64_t h, const int32_t* col, const int32_t* diag_pos, double* val,
                             const double* norms, double tau, void* stream) {
  const TailPlan* P = (const TailPlan*)(intptr_t)h;
  if (!P) { jvh::set_error("jv_tail_upper: null plan"); return JV_EINVAL; }
  if (P->nt == 0 || P->nl == 0) return JV_OK;
  if (tau > 0.0 && norms == nullptr) {
    jvh::set_error("jv_tail_upper: tau > 0 needs row norms");
    return JV_EINVAL;
  }
  TailArgs A;
  A.nt = P->nt;
  A.n_upper = P->n_upper;
  A.tb = P->tb;
  A.col = col;
  A.diag = diag_pos;
  A.gbase = P->gbase;
  A.ga = P->ga;
  A.gb = P->gb;
  A.gsp = P->gsp;
  A.seg_tgt = P->seg_tgt;
  A.seg_optr = P->seg_optr;
  A.op_p = P->op_p;
  A.op_q = P->op_q;
  A.op_k = P->op_k;
  A.val = val;
  A.norms = norms;
  A.tau = tau;
  A.milu = P->milu;
  A.lbuf = P->lbuf;
  A.dfl = P->dfl;
  long long warps = P->nt;
  int grid = (int)((warps * 32 + 255) / 256);
  const int cap = jvh::sm_count() * 8;
  if (grid > cap) grid = cap;
  tail_upper_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A);
  JV_CHECK_LAUNCH("jv_tail_upper");
  return JV_OK;
}

extern "C" int jv_tail_plan_free(int64_t h) {
  free_plan((TailPlan*)(intptr_t)h);
  return JV_OK;
}

extern "C" int jv_scatter(int64_t n, const int32_t* idx, const double* src, double* dst,
                          void* stream) {
  if (n < 0) { jvh::set_error("jv_scatter: bad size"); return JV_EINVAL; }
  if (n == 0) return JV_OK;
  const int grid = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
  scatter_f64_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  JV_CHECK_LAUNCH("jv_scatter");
  return JV_OK;
}
