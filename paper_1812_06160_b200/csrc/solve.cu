// Sync-free sparse triangular solves (stri) over the combined L|U storage.
//
// Reference semantics:
//   forward  (_kernels.py:348-357): y[r] = b[r] - sum_{c<r} l_rc y[c], unit L,
//            subtraction chain in ascending column order;
//   backward (_kernels.py:360-366): x[r] = (y[r] - sum_{c>r} u_rc x[c]) / u_rr.
// Every reference solve path (serial, CSR-LS, p2p, two-stage;
// trisolve.py:60-182) yields the same bits, and so does this kernel: one row
// per thread, the row's chain evaluated in the reference order with
// explicitly rounded ops, dependencies awaited through mailbox packets
// (common.cuh).  Rows come in level batches of the solve's own DAG (forward:
// levels of lower(F); backward: reversed levels of upper(F)); warp w of a
// co-resident grid takes batches w, w+W, ... (deadlock-free: batch b only
// waits on batches < b).
#include "common.cuh"
#include "../../include/jv.h"

namespace {

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
};

constexpr int kProbe = 8;   // dependency values probed together per round

// Wait for the values of columns col[p0..p1) and fold them into s in
// ascending order: s -= val[p] * v[c].  The probes of a group of kProbe
// dependencies are issued back to back so their L2 round trips overlap;
// only not-yet-published ones are re-polled.
JV_INLINE double fold_deps(const SolveArgs& A, int p0, int p1, double s) {
  for (int g = p0; g < p1; g += kProbe) {
    const int m = min(kProbe, p1 - g);
    double v[kProbe];
    int c[kProbe];
    unsigned ready = 0;
#pragma unroll
    for (int t = 0; t < kProbe; ++t) {
      if (t < m) {
        c[t] = __ldg(A.col + g + t);
        if (jv::mbox_try(A.mbox, c[t], A.epoch, v[t])) ready |= 1u << t;
      }
    }
#pragma unroll
    for (int t = 0; t < kProbe; ++t) {
      if (t < m) {
        if (!(ready & (1u << t))) v[t] = jv::mbox_wait(A.mbox, c[t], A.epoch);
        s = jv::dsub(s, jv::dmul(__ldg(A.val + g + t), v[t]));
      }
    }
  }
  return s;
}

__global__ void __launch_bounds__(256) solve_forward_kernel(SolveArgs A) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int W = (gridDim.x * blockDim.x) >> 5;
  for (int b = gw; b < A.nbatch; b += W) {
    const int lo = A.batch_ptr[b], hi = A.batch_ptr[b + 1];
    if (lo + lane >= hi) continue;
    const int r = A.order[lo + lane];
    const int rs = __ldg(A.row_start + r);
    // strictly-lower part = columns < r; diag_pos marks its end
    const int pe = __ldg(A.diag + r);
    double s = A.in[r];
    s = fold_deps(A, rs, pe, s);
    A.out[r] = s;
    jv::mbox_put(A.mbox, r, s, A.epoch);
  }
}

__global__ void __launch_bounds__(256) solve_backward_kernel(SolveArgs A) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int W = (gridDim.x * blockDim.x) >> 5;
  for (int b = gw; b < A.nbatch; b += W) {
    const int lo = A.batch_ptr[b], hi = A.batch_ptr[b + 1];
    if (lo + lane >= hi) continue;
    const int r = A.order[lo + lane];
    const int dp = __ldg(A.diag + r);
    const int re = __ldg(A.row_start + r + 1);
    double s = A.in[r];
    s = fold_deps(A, dp + 1, re, s);
    const double x = jv::ddiv(s, __ldg(A.val + dp));
    A.out[r] = x;
    jv::mbox_put(A.mbox, r, x, A.epoch);
  }
}

__global__ void check_zero_diag_kernel(int n, const double* val, const int32_t* diag, int32_t* row) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    if (val[diag[r]] == 0.0) atomicMin(row, r);
}

}  // namespace

extern "C" int jv_solve(int which, int32_t n, const int32_t* row_start, const int32_t* col,
                        const double* val, const int32_t* diag_pos, const int32_t* order,
                        const int32_t* batch_ptr, int32_t nbatch, const double* in, double* out,
                        uint64_t* mbox, uint32_t epoch, void* stream) {
  if (n < 0 || nbatch < 0 || epoch == 0 || (which != 0 && which != 1)) {
    jvh::set_error("jv_solve: bad argument (which=%d n=%d nbatch=%d epoch=%u)", which, n,
                   nbatch, epoch);
    return JV_EINVAL;
  }
  if (n == 0 || nbatch == 0) return JV_OK;
  SolveArgs A{row_start, col, val, diag_pos, order, batch_ptr, nbatch, in, out, mbox, epoch};
  void* args[] = {&A};
  if (which == 0)
    return jvh::coop_launch(solve_forward_kernel, 256, args, (cudaStream_t)stream, "jv_solve fwd");
  return jvh::coop_launch(solve_backward_kernel, 256, args, (cudaStream_t)stream, "jv_solve bwd");
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
