// Sync-free numeric ILU(k, tau) factorization for sm_100a.
//
// Reference semantics: _kernels.py:165-204 (_factor_row, factor_serial_kernel).
// Row r is eliminated up-looking over its strictly-lower pivots c in
// ascending column order:   l = a_rc / u_cc ; tau drop ; a_rj -= l * u_cj.
// Every operation is an explicitly rounded binary64 op (no FMA), and per
// stored position the updates arrive in ascending pivot order, so the result
// is bitwise equal to factor_serial for ANY schedule that respects the
// dependencies.
//
// Schedule: rows come in level batches (<= 32 rows of one level of the
// factor DAG, so rows of a batch are independent); warp w of a persistent,
// co-resident (cooperative) grid takes batches w, w+W, ...  Because batch b
// only depends on batches < b, the lowest unfinished batch can always make
// progress: no deadlock.  Lane i of the warp owns row order[batch_ptr[b]+i]
// (thread-per-row: the rows of these configs are short, and one thread per
// row gives the memory-level parallelism the latency-bound DAG needs).
//
// Communication: a finished row publishes its U part (diagonal and upper
// entries) as mailbox packets (common.cuh); consumers poll the packets of
// exactly the pivot values they need.  No fences, no flags.
#include "common.cuh"
#include "../../include/jv.h"

namespace {

constexpr int kMaxRow = 32;    // thread path: row length cap
constexpr int kMaxOps = 128;   // thread path: update-op cap
constexpr int kOut = 0x40;     // op target flag: out-of-pattern (MILU -> diagonal)

struct FactorArgs {
  const int32_t* row_start;
  const int32_t* col;
  double* val;
  const int32_t* diag;
  const double* norms;
  double tau;
  int milu;
  const int32_t* order;
  const int32_t* batch_ptr;
  int32_t nbatch;
  int32_t ready_below;
  uint64_t* mbox;
  uint32_t epoch;
  int32_t* err;
};

// value of a pivot row's U entry at position q: final in val[] for rows that
// an earlier call factored, otherwise awaited from the mailbox
JV_INLINE double pivot_value(const FactorArgs& A, int c, int q) {
  if (c < A.ready_below) return __ldcg(A.val + q);
  return jv::mbox_wait(A.mbox, q, A.epoch);
}

// lower_bound of key in col[lo, hi)
JV_INLINE int search_col(const int32_t* col, int lo, int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(col + mid) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Thread path.  Returns false (without side effects) when the row does not
// fit the local buffers; the warp then runs the serial path for it.
__device__ bool factor_row_thread(const FactorArgs& A, int r) {
  const int rs = __ldg(A.row_start + r), re = __ldg(A.row_start + r + 1);
  const int len = re - rs;
  if (len > kMaxRow) return false;
  const int dloc = __ldg(A.diag + r) - rs;
  const int nL = dloc;

  int cj[kMaxRow];
  double a[kMaxRow];
#pragma unroll 4
  for (int i = 0; i < len; ++i) {
    cj[i] = __ldg(A.col + rs + i);
    a[i] = __ldcs(A.val + rs + i);
  }

  // phase 1: structure only (no waiting) — which U entries of which pivot
  // update which position of this row
  int dq[kMaxRow];
  int opend[kMaxRow];
  int opq[kMaxOps];
  unsigned char opw[kMaxOps];
  int nops = 0;
  for (int k = 0; k < nL; ++k) {
    const int c = cj[k];
    const int d = __ldg(A.diag + c);
    const int ce = __ldg(A.row_start + c + 1);
    dq[k] = d;
    const int ulen = ce - d - 1;
    const int rem = len - k - 1;
    if (!A.milu && rem > 0 && ulen > 8 * rem) {
      // long pivot row (hub): search this row's remaining columns in U(c);
      // the update set is the same, and each target is hit once per pivot
      for (int w = k + 1; w < len; ++w) {
        const int q = search_col(A.col, d + 1, ce, cj[w]);
        if (q < ce && __ldg(A.col + q) == cj[w]) {
          if (nops == kMaxOps) return false;
          opq[nops] = q; opw[nops] = (unsigned char)w; ++nops;
        }
      }
    } else {
      int w = k + 1;
      for (int q = d + 1; q < ce; ++q) {
        const int j = __ldg(A.col + q);
        while (w < len && cj[w] < j) ++w;
        if (w < len && cj[w] == j) {
          if (nops == kMaxOps) return false;
          opq[nops] = q; opw[nops] = (unsigned char)w; ++nops;
        } else if (A.milu) {
          if (nops == kMaxOps) return false;
          opq[nops] = q; opw[nops] = (unsigned char)(dloc | kOut); ++nops;
        } else if (w >= len) {
          break;
        }
      }
    }
    opend[k] = nops;
  }

  // phase 2: gather the pivot values (waits on the producers)
  double du[kMaxRow];
  double ov[kMaxOps];
  {
    int o = 0;
    for (int k = 0; k < nL; ++k) {
      const int c = cj[k];
      du[k] = pivot_value(A, c, dq[k]);
      for (; o < opend[k]; ++o) ov[o] = pivot_value(A, c, opq[o]);
    }
  }

  // phase 3: elimination, ascending pivots (reference _kernels.py:172-194)
  const double thresh = jv::dmul(A.tau, A.norms[r]);
  int o = 0;
  for (int k = 0; k < nL; ++k) {
    const double l = jv::ddiv(a[k], du[k]);
    if (A.tau > 0.0 && fabs(l) < thresh) {
      a[k] = 0.0;
      if (A.milu)
        for (; o < opend[k]; ++o) a[dloc] = jv::dsub(a[dloc], jv::dmul(l, ov[o]));
      o = opend[k];
      continue;
    }
    a[k] = l;
    for (; o < opend[k]; ++o) {
      const int t = opw[o];
      const int w = (t & kOut) ? dloc : t;
      a[w] = jv::dsub(a[w], jv::dmul(l, ov[o]));
    }
  }

  // phase 4: publish
  for (int i = 0; i < len; ++i) __stcg(A.val + rs + i, a[i]);
  for (int i = nL; i < len; ++i) jv::mbox_put(A.mbox, rs + i, a[i], A.epoch);
  if (a[dloc] == 0.0) atomicMin(A.err, r);
  return true;
}

// Serial path for long rows: the reference algorithm in place on val[],
// pivot values from the mailbox.  Run by one lane.
__device__ void factor_row_serial(const FactorArgs& A, int r) {
  const int rs = A.row_start[r], re = A.row_start[r + 1];
  const int dpos = A.diag[r];
  double* val = A.val;
  const double thresh = jv::dmul(A.tau, A.norms[r]);
  for (int p = rs; p < re; ++p) {
    const int c = A.col[p];
    if (c >= r) break;
    const int d = A.diag[c], ce = A.row_start[c + 1];
    const double l = jv::ddiv(val[p], pivot_value(A, c, d));
    if (A.tau > 0.0 && fabs(l) < thresh) {
      val[p] = 0.0;
      if (A.milu)
        for (int q = d + 1; q < ce; ++q)
          val[dpos] = jv::dsub(val[dpos], jv::dmul(l, pivot_value(A, c, q)));
      continue;
    }
    val[p] = l;
    const int ulen = ce - d - 1, rem = re - p - 1;
    if (!A.milu && rem > 0 && ulen > 8 * rem) {
      for (int w = p + 1; w < re; ++w) {
        const int q = search_col(A.col, d + 1, ce, A.col[w]);
        if (q < ce && A.col[q] == A.col[w])
          val[w] = jv::dsub(val[w], jv::dmul(l, pivot_value(A, c, q)));
      }
      continue;
    }
    int w = p + 1;
    for (int q = d + 1; q < ce; ++q) {
      const int j = A.col[q];
      while (w < re && A.col[w] < j) ++w;
      if (w < re && A.col[w] == j)
        val[w] = jv::dsub(val[w], jv::dmul(l, pivot_value(A, c, q)));
      else if (A.milu)
        val[dpos] = jv::dsub(val[dpos], jv::dmul(l, pivot_value(A, c, q)));
      else if (w >= re)
        break;
    }
  }
  for (int p = dpos; p < re; ++p) jv::mbox_put(A.mbox, p, val[p], A.epoch);
  if (val[dpos] == 0.0) atomicMin(A.err, r);
}

__global__ void __launch_bounds__(256) factor_kernel(FactorArgs A) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int W = (gridDim.x * blockDim.x) >> 5;
  for (int b = gw; b < A.nbatch; b += W) {
    const int lo = A.batch_ptr[b], hi = A.batch_ptr[b + 1];
    const int idx = lo + lane;
    const bool active = idx < hi;
    const int r = active ? A.order[idx] : -1;
    bool done = true;
    if (active) done = factor_row_thread(A, r);
    unsigned pend = __ballot_sync(0xffffffffu, !done);
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1;
      const int rr = __shfl_sync(0xffffffffu, r, src);
      if (lane == 0) factor_row_serial(A, rr);
      __syncwarp();
    }
  }
}

}  // namespace



extern "C" int jv_factor(int32_t n, const int32_t* row_start, const int32_t* col, double* val,
                         const int32_t* diag_pos, const double* norms, double tau, int milu,
                         const int32_t* order, const int32_t* batch_ptr, int32_t nbatch,
                         int32_t ready_below, uint64_t* mbox, uint32_t epoch, int32_t* err_row,
                         void* stream) {
  if (n < 0 || nbatch < 0 || epoch == 0) {
    jvh::set_error("jv_factor: bad argument (n=%d nbatch=%d epoch=%u)", n, nbatch, epoch);
    return JV_EINVAL;
  }
  if (n == 0 || nbatch == 0) return JV_OK;
  FactorArgs A{row_start, col, val, diag_pos, norms, tau, milu, order, batch_ptr,
               nbatch, ready_below, mbox, epoch, err_row};
  void* args[] = {&A};
  return jvh::coop_launch(factor_kernel, 256, args, (cudaStream_t)stream, "jv_factor");
}
