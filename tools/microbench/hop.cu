// Dependency-hop latency microbenchmarks for the sync-free ILU / stri design.
//
// Each test runs a chain of K dependent "rows": step k waits for step k-1,
// reads its value, computes, publishes. Total kernel time / K = hop latency.
//   gflag   : per-step flag in global memory, st.release.gpu / ld.acquire.gpu,
//             data in a separate global array (the classic sync-free scheme)
//   ll16    : {double, u64 tag} published with one 16-byte st.relaxed.gpu,
//             consumer polls the pair (data and flag in one transaction)
//   smem    : chain between warps of one CTA through shared memory
//   gcta    : chain between warps of one CTA through global memory, .cta scope
//   ddiv    : dependent fp64 divisions (latency of one IEEE divide)
//   gridbar : grid-wide barrier (atomic counter + generation) per step
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v; asm volatile("ld.acquire.cta.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void ld_pair(const void* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_pair(void* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" :: "l"(p), "l"(a), "l"(b) : "memory");
}

// chain step k is owned by warp (k % nwarps); warps are spread round-robin
// over CTAs so consecutive steps live on different SMs.
__global__ void chain_gflag(int K, uint32_t* flag, double* data, uint32_t epoch) {
  int nwarps = gridDim.x * (blockDim.x / 32);
  int wid = (threadIdx.x / 32) * gridDim.x + blockIdx.x;
  int lane = threadIdx.x & 31;
  for (int k = wid; k < K; k += nwarps) {
    double v = 0.0;
    if (k > 0) {
      if (lane == 0) while (ld_acquire(flag + k - 1) != epoch) {}
      __syncwarp();
      v = __ldcg(data + k - 1);
    }
    double nv = v + 1.0;
    if (lane == 0) { __stcg(data + k, nv); st_release(flag + k, epoch); }
  }
}

struct __align__(16) Pkt { double v; unsigned long long tag; };
__global__ void chain_ll16(int K, Pkt* box, unsigned long long epoch) {
  int nwarps = gridDim.x * (blockDim.x / 32);
  int wid = (threadIdx.x / 32) * gridDim.x + blockIdx.x;
  int lane = threadIdx.x & 31;
  for (int k = wid; k < K; k += nwarps) {
    double v = 0.0;
    if (k > 0 && lane == 0) {
      unsigned long long a, t;
      do { ld_pair(box + k - 1, a, t); } while (t != epoch);
      v = __longlong_as_double((long long)a);
    }
    double nv = v + 1.0;
    if (lane == 0) st_pair(box + k, (unsigned long long)__double_as_longlong(nv), epoch);
  }
}

__global__ void chain_smem(int K, double* out) {
  __shared__ volatile uint32_t sflag[4096];
  __shared__ volatile double sdata[4096];
  int nw = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sflag[i] = 0;
  __syncthreads();
  for (int k = w; k < K && k < 4096; k += nw) {
    double v = 0.0;
    if (k > 0 && lane == 0) { while (sflag[k - 1] == 0) {} v = sdata[k - 1]; }
    if (lane == 0) { sdata[k] = v + 1.0; __threadfence_block(); sflag[k] = 1; }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[0] = sdata[(K < 4096 ? K : 4096) - 1];
}

__global__ void chain_gcta(int K, uint32_t* flag, double* data, uint32_t epoch) {
  int nw = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int k = w; k < K; k += nw) {
    double v = 0.0;
    if (k > 0 && lane == 0) {
      while (ld_acquire_cta(flag + k - 1) != epoch) {}
      v = data[k - 1];
    }
    if (lane == 0) { data[k] = v + 1.0; st_release_cta(flag + k, epoch); }
  }
}

__global__ void chain_ddiv(int K, double a, double b, double* out) {
  double x = a;
  for (int k = 0; k < K; ++k) x = b / x;   // each divide depends on the last
  if (threadIdx.x == 0) out[0] = x;
}

__global__ void chain_dmulsub(int K, double a, double b, double* out) {
  double x = a;
  for (int k = 0; k < K; ++k) x = __dsub_rn(b, __dmul_rn(x, b));
  if (threadIdx.x == 0) out[0] = x;
}

__global__ void gridbar(int K, unsigned int* bar) {
  // bar[0] arrivals, bar[1] generation
  for (int k = 0; k < K; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int gen = ld_acquire(bar + 1);
      unsigned int arrived = atomicAdd(bar, 1u) + 1;
      if (arrived == gridDim.x) { bar[0] = 0; st_release(bar + 1, gen + 1); }
      else while (ld_acquire(bar + 1) == gen) {}
    }
    __syncthreads();
  }
}

int main1() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  const int K = 20000;
  uint32_t* flag; double* data; Pkt* box; unsigned int* bar; double* out;
  CK(cudaMalloc(&flag, K * 4)); CK(cudaMemset(flag, 0, K * 4));
  CK(cudaMalloc(&data, K * 8)); CK(cudaMalloc(&box, K * sizeof(Pkt)));
  CK(cudaMemset(box, 0, K * sizeof(Pkt)));
  CK(cudaMalloc(&bar, 8)); CK(cudaMemset(bar, 0, 8)); CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int sms = prop.multiProcessorCount;
  for (int rep = 0; rep < 3; ++rep) {
    uint32_t epoch = rep + 1;
    // gflag: 1 warp per CTA, sms CTAs -> every hop crosses SMs
    cudaEventRecord(e0); chain_gflag<<<sms, 32>>>(K, flag, data, epoch); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("gflag  (1 warp/CTA, %d CTAs): %.3f us/hop\n", sms, ms * 1e3 / K);
    cudaEventRecord(e0); chain_gflag<<<sms, 256>>>(K, flag, data, epoch + 100); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("gflag  (8 warp/CTA, %d CTAs): %.3f us/hop\n", sms, ms * 1e3 / K);
    cudaEventRecord(e0); chain_ll16<<<sms, 32>>>(K, box, epoch + 1000); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("ll16   (1 warp/CTA, %d CTAs): %.3f us/hop\n", sms, ms * 1e3 / K);
    cudaEventRecord(e0); chain_smem<<<1, 1024>>>(4096, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("smem   (32 warps, 1 CTA): %.3f us/hop\n", ms * 1e3 / 4096);
    cudaEventRecord(e0); chain_gcta<<<1, 1024>>>(K, flag, data, epoch + 2000); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("gcta   (32 warps, 1 CTA, global .cta): %.3f us/hop\n", ms * 1e3 / K);
    cudaEventRecord(e0); chain_ddiv<<<1, 32>>>(K, 1.5, 2.5, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("ddiv   dependent chain: %.2f ns/div\n", ms * 1e6 / K);
    cudaEventRecord(e0); chain_dmulsub<<<1, 32>>>(K, 1.5, 0.5, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("dmul+dsub dependent chain: %.2f ns/step\n", ms * 1e6 / K);
    int kb = 2000;
    cudaEventRecord(e0); gridbar<<<sms, 128>>>(kb, bar); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("gridbar (%d CTAs): %.3f us/barrier\n", sms, ms * 1e3 / kb);
    cudaEventRecord(e0); gridbar<<<2 * sms, 128>>>(kb, bar); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("gridbar (%d CTAs): %.3f us/barrier\n", 2 * sms, ms * 1e3 / kb);
    // empty-launch cost for reference
    cudaEventRecord(e0); for (int i = 0; i < 100; ++i) chain_ddiv<<<1, 32>>>(0, 1.0, 1.0, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("empty launch back-to-back: %.3f us/launch\n", ms * 1e3 / 100);
  }
  CK(cudaGetLastError());
  return 0;
}

// ---- appended: __nanosleep granularity and a probe round trip
__global__ void sleep_probe(unsigned ns, int reps, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) __nanosleep(ns);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
}
__global__ void ldrelaxed_latency(const unsigned long long* p, int reps, long long* out) {
  unsigned long long a = 0, b = 0;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p + ((a & 1) << 4)) : "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / reps + (long long)(a & 0);
}
int main2() {
  long long* out; cudaMalloc(&out, 8); long long h;
  unsigned long long* buf; cudaMalloc(&buf, 4096); cudaMemset(buf, 0, 4096);
  for (unsigned ns : {0u, 16u, 64u, 256u, 1024u}) {
    sleep_probe<<<1, 32>>>(ns, 1000, out); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("__nanosleep(%u): %lld cycles per call\n", ns, h);
  }
  ldrelaxed_latency<<<1, 32>>>(buf, 1000, out); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("ld.relaxed.gpu.v2 dependent latency: %lld cycles\n", h);
  return 0;
}
int main(int argc, char** argv) {
  if (argc > 1) return main2();
  return main1();
}
