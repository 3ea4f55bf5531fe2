// Vector kernels of the device Krylov driver (krylov.py: PCG / GMRES over
// jv_spmv and the jv_solve preconditioner).  Reductions are deterministic:
// a fixed grid of partial sums (strided per thread, warp tree, block tree)
// summed in order by one block — the same inputs give the same bits on
// every run (the reference's numpy BLAS dot is not reproducible across
// BLAS builds either; Krylov parity is pinned by iteration counts and
// residuals, tests/test_gpu_krylov.py).  Elementwise updates use explicitly
// rounded products and sums, as numpy's `x += alpha * p`.

namespace {

constexpr int kDotThreads = 256;
constexpr int kDotBlocks = 592;   // 4 per SM

JV_INLINE double block_sum(double s, double* red) {
  for (int o = 16; o > 0; o >>= 1) s = jv::dadd(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kDotThreads / 32; ++w) t = jv::dadd(t, red[w]);
  __syncthreads();
  return t;
}

// partial[b] = sum over this block's grid-stride elements of x[i] * y[i]
__global__ void __launch_bounds__(kDotThreads) dot_partial_kernel(long long n, const double* x,
                                                                  const double* y,
                                                                  double* partial) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kDotThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kDotThreads)
    s = jv::dadd(s, jv::dmul(__ldg(x + i), __ldg(y + i)));
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kDotThreads) sum_partials_kernel(int m, const double* partial,
                                                                   double* out, int sqrt_out) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += kDotThreads) s = jv::dadd(s, partial[i]);
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) *out = sqrt_out ? sqrt(t) : t;
}

// y += a * x, a = sign * coef (host scalar) or sign * (*coef_dev)
__global__ void axpy_kernel(long long n, double a, const double* coef_dev, double sign,
                            const double* x, double* y) {
  const double c = coef_dev ? jv::dmul(sign, *coef_dev) : a;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = jv::dadd(y[i], jv::dmul(c, x[i]));
}

// y = x + b * y
__global__ void xpby_kernel(long long n, const double* x, double b, double* y) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = jv::dadd(x[i], jv::dmul(b, y[i]));
}

// y = a * x
__global__ void scale_kernel(long long n, double a, const double* x, double* y) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = jv::dmul(a, x[i]);
}

// PCG step: x += alpha p ; r -= alpha ap ; partial sums of r.r
__global__ void __launch_bounds__(kDotThreads) pcg_update_kernel(long long n, double alpha,
                                                                 const double* p, const double* ap,
                                                                 double* x, double* r,
                                                                 double* partial) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kDotThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kDotThreads) {
    x[i] = jv::dadd(x[i], jv::dmul(alpha, p[i]));
    const double ri = jv::dsub(r[i], jv::dmul(alpha, ap[i]));
    r[i] = ri;
    s = jv::dadd(s, jv::dmul(ri, ri));
  }
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

inline int ew_grid(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

extern "C" int jv_dot_workspace(void) { return kDotBlocks; }

extern "C" int jv_dot(int64_t n, const double* x, const double* y, double* ws, double* out,
                      int sqrt_out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0) { jvh::set_error("jv_dot: bad size"); return JV_EINVAL; }
  dot_partial_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, x, y, ws);
  sum_partials_kernel<<<1, kDotThreads, 0, s>>>(kDotBlocks, ws, out, sqrt_out);
  JV_CHECK_LAUNCH("jv_dot");
  return JV_OK;
}

extern "C" int jv_axpy(int64_t n, double a, const double* coef_dev, double sign, const double* x,
                       double* y, void* stream) {
  if (n <= 0) return JV_OK;
  axpy_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>(n, a, coef_dev, sign, x, y);
  JV_CHECK_LAUNCH("jv_axpy");
  return JV_OK;
}

extern "C" int jv_xpby(int64_t n, const double* x, double b, double* y, void* stream) {
  if (n <= 0) return JV_OK;
  xpby_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>(n, x, b, y);
  JV_CHECK_LAUNCH("jv_xpby");
  return JV_OK;
}

extern "C" int jv_scale(int64_t n, double a, const double* x, double* y, void* stream) {
  if (n <= 0) return JV_OK;
  scale_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)stream>>>(n, a, x, y);
  JV_CHECK_LAUNCH("jv_scale");
  return JV_OK;
}

extern "C" int jv_pcg_update(int64_t n, double alpha, const double* p, const double* ap, double* x,
                             double* r, double* ws, double* rr, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0) { jvh::set_error("jv_pcg_update: bad size"); return JV_EINVAL; }
  pcg_update_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, alpha, p, ap, x, r, ws);
  sum_partials_kernel<<<1, kDotThreads, 0, s>>>(kDotBlocks, ws, rr, 0);
  JV_CHECK_LAUNCH("jv_pcg_update");
  return JV_OK;
}
