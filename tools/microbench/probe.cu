// Latency of one 16-byte probe of a packet that another SM has just
// published, for several load flavours (cycles, reader side).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__device__ __forceinline__ void ld16(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  if (KIND == 0) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  if (KIND == 1) asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  if (KIND == 2) asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  if (KIND == 3) asm volatile("ld.acquire.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// block 0 (producer) writes slot i with tag i+1 at i*step; block 1 (consumer)
// spins on slot i's tag (gate), then times a probe of the NEXT packet in the
// same 64B group (written just before the gate packet)
template <int KIND>
__global__ void pingpong(unsigned long long* box, int iters, long long* out) {
  if (threadIdx.x != 0) return;
  if (blockIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      unsigned long long* g = box + 8 * i;   // 64 B group
      // data packet first, gate packet second
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" :: "l"(g), "l"(7ull), "l"((unsigned long long)i + 1) : "memory");
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" :: "l"(g + 2), "l"(9ull), "l"((unsigned long long)i + 1) : "memory");
      // wait for the consumer's ack before the next round
      unsigned long long a, b;
      do { ld16<0>(box + 8 * iters + 2 * i, a, b); } while (b != (unsigned long long)i + 1);
    }
  } else {
    long long tot = 0;
    for (int i = 0; i < iters; ++i) {
      unsigned long long* g = box + 8 * i;
      unsigned long long a, b;
      do { ld16<0>(g + 2, a, b); } while (b != (unsigned long long)i + 1);
      long long t0 = clock64();
      ld16<KIND>(g, a, b);
      unsigned long long sum;
      asm volatile("add.u64 %0, %1, %2;" : "=l"(sum) : "l"(a), "l"(b));
      long long t1 = clock64();
      if (sum == 123456789ull) out[7] = 1;
      tot += (t1 - t0) + (long long)(b != (unsigned long long)i + 1) * 1000000;
      asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" :: "l"(box + 8 * iters + 2 * i), "l"(0ull), "l"((unsigned long long)i + 1) : "memory");
    }
    out[KIND] = tot / iters;
  }
}

int main() {
  unsigned long long* box; long long* out; long long h[4];
  const int iters = 2000;
  cudaMalloc(&box, sizeof(unsigned long long) * 10 * iters + 4096);
  cudaMalloc(&out, 64);
  const char* names[] = {"ld.relaxed.gpu", "ld.volatile", "ld.global.cg", "ld.acquire.gpu"};
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(box, 0, sizeof(unsigned long long) * 10 * iters + 4096);
    pingpong<0><<<2, 32>>>(box, iters, out); cudaDeviceSynchronize();
    cudaMemset(box, 0, sizeof(unsigned long long) * 10 * iters + 4096);
    pingpong<1><<<2, 32>>>(box, iters, out); cudaDeviceSynchronize();
    cudaMemset(box, 0, sizeof(unsigned long long) * 10 * iters + 4096);
    pingpong<2><<<2, 32>>>(box, iters, out); cudaDeviceSynchronize();
    cudaMemset(box, 0, sizeof(unsigned long long) * 10 * iters + 4096);
    pingpong<3><<<2, 32>>>(box, iters, out); cudaDeviceSynchronize();
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    for (int k = 0; k < 4; ++k) printf("%-16s probe after gate: %lld cycles (>=1e6 means stale data seen)\n", names[k], h[k]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
