// C-ABI plumbing: error strings, device info, the persistent cooperative
// launch shared by every sync-free kernel, and the hang detector.
#include "common.cuh"
#include "../../include/jv.h"

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>

namespace jvh {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return JV_ECUDA;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 1;
  }
  return cached[dev];
}

// Every warp of a sync-free kernel may spin on rows owned by any other warp,
// so all CTAs must be resident at once: the grid is exactly the occupancy
// limit and the launch is cooperative (the driver refuses rather than
// time-slicing a grid that would not fit).
template <typename K>
int coop_launch(K kernel, int block, void** args, cudaStream_t stream, const char* what,
                size_t smem = 0) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, what);
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
  if (e != cudaSuccess) return cuda_status(e, what);
  if (per_sm < 1) {
    set_error("%s: kernel cannot be resident", what);
    return JV_ECOOP;
  }
  // JV_BLOCKS_PER_SM caps the resident CTAs per SM (tuning experiments)
  static int cap = -1;
  if (cap < 0) {
    const char* env = getenv("JV_BLOCKS_PER_SM");
    cap = env ? atoi(env) : 0;
  }
  if (cap > 0 && per_sm > cap) per_sm = cap;
  const int grid = per_sm * sm_count();
  e = cudaLaunchCooperativeKernel((const void*)kernel, dim3(grid), dim3(block), args, smem, stream);
  if (e != cudaSuccess) return cuda_status(e, what);
  return JV_OK;
}

// Persistent grid sized to the occupancy limit, ordinary launch: kernels that
// take work by ticket never wait on a warp that has not started.
template <typename K>
int persistent_launch(K kernel, int block, void** args, cudaStream_t stream, const char* what,
                      size_t smem = 0) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void*)kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, what);
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
  if (e != cudaSuccess) return cuda_status(e, what);
  if (per_sm < 1) {
    set_error("%s: kernel cannot be resident", what);
    return JV_ECOOP;
  }
  static int cap = -1;
  if (cap < 0) {
    const char* env = getenv("JV_BLOCKS_PER_SM");
    cap = env ? atoi(env) : 0;
  }
  if (cap > 0 && per_sm > cap) per_sm = cap;
  e = cudaLaunchKernel((const void*)kernel, dim3(per_sm * sm_count()), dim3(block), args, smem,
                       stream);
  if (e != cudaSuccess) return cuda_status(e, what);
  return JV_OK;
}

}  // namespace jvh

extern "C" const char* jv_last_error(void) { return jvh::g_err; }

extern "C" int jv_version(void) { return 1; }

// Page-lock a caller's host buffer in place (cudaHostRegister), so the
// drop-in API moves its numpy arrays by DMA with no staging copy.
// (a failure is reported but cleared from the runtime's error state: the
// caller falls back to staged copies)
extern "C" int jv_host_register(void* p, int64_t bytes) {
  const cudaError_t e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault);
  if (e == cudaSuccess) return JV_OK;
  cudaGetLastError();
  return jvh::cuda_status(e, "jv_host_register");
}
extern "C" int jv_host_unregister(void* p) {
  const cudaError_t e = cudaHostUnregister(p);
  if (e == cudaSuccess) return JV_OK;
  cudaGetLastError();
  return jvh::cuda_status(e, "jv_host_unregister");
}
// async copy host <-> device on the caller's stream (kind 0: H2D, 1: D2H)
extern "C" int jv_memcpy_async(void* dst, const void* src, int64_t bytes, int kind, void* stream) {
  const cudaError_t e = cudaMemcpyAsync(
      dst, src, (size_t)bytes, kind == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
      (cudaStream_t)stream);
  return e == cudaSuccess ? JV_OK : jvh::cuda_status(e, "jv_memcpy_async");
}

extern "C" int jv_device_info(int device, int* sms_h, int* coop_h) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_device_info");
  if (sms_h) *sms_h = v;
  e = cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, device);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_device_info");
  if (coop_h) *coop_h = v;
  return JV_OK;
}

extern "C" int jv_set_trace(unsigned long long* buf, long long batches) {
  cudaError_t e = cudaMemcpyToSymbol(jv::g_trace, &buf, sizeof(buf));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(jv::g_trace_cap, &batches, sizeof(batches));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_trace");
  return JV_OK;
}

extern "C" int jv_set_backoff(unsigned cap_ns) {
  cudaError_t e = cudaMemcpyToSymbol(jv::g_backoff_cap, &cap_ns, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_backoff");
  return JV_OK;
}

extern "C" int jv_set_gate(unsigned mask) {
  cudaError_t e = cudaMemcpyToSymbol(jv::g_gate, &mask, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_gate");
  return JV_OK;
}

extern "C" int jv_set_poll(unsigned cap_ns) {
  if (cap_ns < 16) cap_ns = 16;
  cudaError_t e = cudaMemcpyToSymbol(jv::g_poll_cap, &cap_ns, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_poll");
  return JV_OK;
}

extern "C" int jv_set_sfp_group(unsigned g) {
  if (g == 0 || g > 32 || (g & (g - 1))) { jvh::set_error("jv_set_sfp_group: power of 2 <= 32"); return JV_EINVAL; }
  cudaError_t e = cudaMemcpyToSymbol(jv::g_sfp_group, &g, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_sfp_group");
  return JV_OK;
}

extern "C" int jv_set_solve_staged(unsigned on) {
  cudaError_t e = cudaMemcpyToSymbol(jv::g_solve_staged, &on, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_solve_staged");
  return JV_OK;
}

extern "C" int jv_set_spin_limit(unsigned limit) {
  cudaError_t e = cudaMemcpyToSymbol(jv::g_spin_limit, &limit, sizeof(unsigned));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_set_spin_limit");
  return JV_OK;
}

// 1 if any sync-free wait gave up (a producer never published), then
// clears the flag.  Synchronises the device.
extern "C" int jv_status(int* hang_h) {
  int h = 0, z = 0;
  cudaError_t e = cudaMemcpyFromSymbol(&h, jv::g_hang, sizeof(int));
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_status");
  if (h) cudaMemcpyToSymbol(jv::g_hang, &z, sizeof(int));
  if (hang_h) *hang_h = h;
  return JV_OK;
}

// Test hook: out[i] = ddiv_fast(a[i], b[i]) with the __ddiv_rn fallback, so
// the parity tests can compare it with IEEE division bit for bit.
namespace {
__global__ void ddiv_test_kernel(int n, const double* a, const double* b, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    bool slow;
    double q = jv::ddiv_fast(a[i], b[i], slow);
    if (slow) q = __ddiv_rn(a[i], b[i]);
    out[i] = q;
  }
}
}  // namespace

extern "C" int jv_test_ddiv(int32_t n, const double* a, const double* b, double* out, void* stream) {
  if (n <= 0) return JV_OK;
  ddiv_test_kernel<<<(n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096, 256, 0, (cudaStream_t)stream>>>(n, a, b, out);
  JV_CHECK_LAUNCH("jv_test_ddiv");
  return JV_OK;
}

// ---- t_hop: latency of one dependent cross-SM hop through a mailbox packet
// (the primitive every sync-free kernel waits on).  A chain of K steps, step
// k owned by CTA k mod grid (one warp per CTA, consecutive steps on
// different SMs): step k polls step k-1's packet, adds one, publishes.
// Kernel time / K = t_hop, the per-level floor of a DAG sweep whose
// consecutive levels live on different SMs (SURVEY.md §8d "depth bound").
namespace {
__global__ void hop_chain_kernel(int K, uint64_t* box, uint32_t epoch) {
  if (threadIdx.x != 0) return;
  for (int k = blockIdx.x; k < K; k += gridDim.x) {
    double v = 0.0;
    if (k > 0) {
      while (!jv::mbox_try(box, k - 1, epoch, v)) {
      }
    }
    jv::mbox_put(box, k, v + 1.0, epoch);
  }
}
}  // namespace

extern "C" int jv_hop_latency(int32_t hops, double* ns_per_hop_h) {
  if (hops < 2 || !ns_per_hop_h) { jvh::set_error("jv_hop_latency: bad args"); return JV_EINVAL; }
  uint64_t* box = nullptr;
  cudaError_t e = cudaMalloc(&box, 16 * (size_t)hops);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_hop_latency");
  cudaMemset(box, 0, 16 * (size_t)hops);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = jvh::sm_count();
  hop_chain_kernel<<<grid, 32>>>(hops, box, 1u);   // warm-up
  cudaEventRecord(a);
  hop_chain_kernel<<<grid, 32>>>(hops, box, 2u);
  cudaEventRecord(b);
  e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(box);
  if (e != cudaSuccess) return jvh::cuda_status(e, "jv_hop_latency");
  *ns_per_hop_h = (double)ms * 1e6 / hops;
  return JV_OK;
}
