// Per-level cost of a single-CTA level loop (diagnostics for csrc/cta.cu):
// 127 levels, 64 active threads per level, __syncthreads between levels.
//   mode 0: empty levels          mode 1: + 2 dependent smem loads
//   mode 2: + one __ddiv_rn       mode 3: + a 4-byte cp.async + wait_all
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(1024, 1) lv(int mode, int nlev, const int* g, double* out) {
  __shared__ double v[2048];
  __shared__ int idx[2048];
  __shared__ int pf[2048];
  int t = threadIdx.x;
  for (int i = t; i < 2048; i += 1024) { v[i] = 1.0 + i; idx[i] = (i * 7) & 2047; }
  __syncthreads();
  double acc = 0;
  for (int L = 0; L < nlev; ++L) {
    if (mode >= 3) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su(pf + t)), "l"(g + L * 1024 + t) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (t < 64) {
      int r = (L * 64 + t) & 2047;
      double x = 1.0;
      if (mode >= 1) { int j = idx[r]; x = v[idx[j]]; }
      if (mode >= 2) x = __ddiv_rn(v[r], x);
      v[r] = x; acc += x;
    }
    if (mode >= 3) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  if (t == 0) out[0] = acc;
}
int main() {
  int* g; double* o; cudaMalloc(&g, 4 << 20); cudaMemset(g, 0, 4 << 20); cudaMalloc(&o, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    lv<<<1, 1024>>>(mode, 127, g, o);
    cudaEventRecord(a);
    for (int k = 0; k < 10; ++k) lv<<<1, 1024>>>(mode, 127, g, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %d: %.2f us per launch, %.3f us per level\n", mode, ms * 100, ms * 100 / 127);
  }
  return 0;
}
