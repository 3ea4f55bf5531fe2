// __nanosleep(t) actual duration on this GPU (cycles at the SM clock)
#include <cstdio>
__global__ void k(long long* out, unsigned t, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __nanosleep(t);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  for (unsigned t : {0u, 8u, 16u, 32u, 64u, 128u, 256u, 1000u}) {
    k<<<1, 32>>>(d, t, 1000); cudaDeviceSynchronize();
    k<<<1, 32>>>(d, t, 1000); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("nanosleep(%u ns): %lld cycles per call (%.0f ns at 1.965 GHz)\n", t, c, c / 1.965);
  }
}
