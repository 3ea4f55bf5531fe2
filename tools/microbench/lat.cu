// Dependent-chain latencies of the ops on the factor's critical path.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1812_06160_b200/csrc lat.cu -o lat
#include <cstdio>
#include "common.cuh"

constexpr int N = 4096;

__global__ void lat_kernel(double* out, long long* cyc, double x0, int sel) {
  __shared__ double sm[1024];
  __shared__ int si[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; si[i] = (i + 1) & 1023; }
  __syncthreads();
  double x = x0, y = 1.0000001;
  int p = threadIdx.x;
  double* gsm = sm;   // generic pointer to smem
  volatile double* vg = gsm;
  long long t0 = clock64();
  switch (sel) {
    case 0: for (int i = 0; i < N; ++i) x = __fma_rn(x, y, 1e-30); break;
    case 1: for (int i = 0; i < N; ++i) x = __dmul_rn(x, y); break;
    case 2: for (int i = 0; i < N; ++i) x = __dsub_rn(x, 1e-30); break;
    case 3: for (int i = 0; i < N; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; } break;
    case 4: for (int i = 0; i < N; ++i) { bool s; x = jv::ddiv_fast(x, y, s); if (s) x = 1.0; } break;
    case 5: for (int i = 0; i < N; ++i) x = __ddiv_rn(x, y); break;
    case 6: for (int i = 0; i < N; ++i) p = si[p]; x = p; break;
    case 7: for (int i = 0; i < N; ++i) { x = vg[((long long)__double_as_longlong(x)) & 1023]; } break;
    case 8: for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, 0) + 1e-30; break;
    case 9: for (int i = 0; i < N; ++i) { __syncwarp(); x = x + 1e-30; } break;
    case 10: for (int i = 0; i < N; ++i) { x = sm[((long long)__double_as_longlong(x)) & 1023]; } break;
    case 11: for (int i = 0; i < N; ++i) x = x * y + 1e-30; break;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x + p; cyc[0] = t1 - t0; }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA", "DMUL", "DADD", "MUFU.RCP64H", "ddiv_fast", "__ddiv_rn", "LDS(int chase)",
                         "generic LD smem (volatile)", "SHFL+DADD", "syncwarp+DADD", "LDS.64 chase", "x*y+c (dfma)"};
  for (int sel = 0; sel < 12; ++sel) {
    for (int rep = 0; rep < 2; ++rep) {
      lat_kernel<<<1, 32>>>(out, cyc, 1.5, sel);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f cycles\n", names[sel], (double)c / N);
  }
  return 0;
}
