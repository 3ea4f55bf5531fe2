// Reverse Cuthill-McKee on the device, bit-exact with the reference
// rcm_order (ordering.py:199-266) and with jv_rcm_host.
//
// Reference rules: degree = neighbours without self-loops; components are
// taken from candidates in (degree, index) order; a component's root is
// refined George-Liu style (BFS from the candidate, then from the
// minimum-(degree, index) vertex of the last tier while the tier count
// grows); the Cuthill-McKee queue visits each vertex's not-yet-visited
// neighbours in (degree, index) order; the whole order is reversed.
//
// Level-synchronous formulation: the queue is a sequence of BFS levels;
// the children of level l come in the order of their FIRST parent's queue
// position (the parent that dequeues first claims them), then degree, then
// index.  So each level is: discover (atomicMin of the parent position per
// child), then two stable radix sorts (index, then (parent, degree)) —
// exactly the sequential queue.  Tier BFS for the root search uses stamps.
// Degree-0 vertices are components of one vertex each and come first, in
// index order (one stable selection).  Host C++ drives the levels; a graph
// with more than max_components other components returns 1 (the caller then
// uses jv_rcm_host).

namespace {

__global__ void rcm_degree_kernel(int n, const int32_t* rs, const int32_t* col, int32_t* deg) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int d = 0;
    for (int p = rs[v]; p < rs[v + 1]; ++p) d += col[p] != v;
    deg[v] = d;
  }
}

// smallest (degree, index) key among unvisited vertices (or among a list)
__global__ void rcm_min_unvisited(int n, const int32_t* deg, const int8_t* state,
                                  unsigned long long* out) {
  unsigned long long best = ~0ull;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (!state[v]) {
      const unsigned long long k = ((unsigned long long)(uint32_t)deg[v] << 32) | (uint32_t)v;
      best = k < best ? k : best;
    }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
    best = x < best ? x : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(out, best);
}

__global__ void rcm_min_list(int m, const int32_t* list, const int32_t* deg,
                             unsigned long long* out) {
  unsigned long long best = ~0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int v = list[i];
    const unsigned long long k = ((unsigned long long)(uint32_t)deg[v] << 32) | (uint32_t)v;
    best = k < best ? k : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
    best = x < best ? x : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(out, best);
}

// one BFS tier: unseen neighbours of the frontier (stamp != cur) appended
__global__ void rcm_bfs_expand(int m, const int32_t* front, const int32_t* rs,
                               const int32_t* col, int32_t* stamp, int cur, int32_t* next,
                               int32_t* nnext) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int v = front[i];
    for (int p = rs[v]; p < rs[v + 1]; ++p) {
      const int w = col[p];
      if (w != v && stamp[w] != cur && atomicExch(&stamp[w], cur) != cur)
        next[atomicAdd(nnext, 1)] = w;
    }
  }
}

// Cuthill-McKee discovery: unvisited neighbours of the frontier (queue
// positions base + i) get the smallest parent position; first touch lists them
__global__ void rcm_discover(int m, const int32_t* front, int base, const int32_t* rs,
                             const int32_t* col, const int8_t* state, int32_t* parent,
                             int32_t* mark, int32_t* cand, int32_t* ncand) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int v = front[i];
    for (int p = rs[v]; p < rs[v + 1]; ++p) {
      const int w = col[p];
      if (w == v || state[w]) continue;
      atomicMin(&parent[w], base + i);
      if (atomicExch(&mark[w], 1) == 0) cand[atomicAdd(ncand, 1)] = w;
    }
  }
}

__global__ void rcm_key_parent_degree(int m, const int32_t* cand, const int32_t* parent,
                                      const int32_t* deg, int base, unsigned long long* key) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int w = cand[i];
    key[i] = ((unsigned long long)(uint32_t)(parent[w] - base) << 32) | (uint32_t)deg[w];
  }
}

// the sorted children enter the queue: order, state, and scratch reset
__global__ void rcm_enqueue(int m, const int32_t* sorted, int32_t* order, int nord,
                            int8_t* state, int32_t* parent, int32_t* mark) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int w = sorted[i];
    order[nord + i] = w;
    state[w] = 1;
    parent[w] = 0x7fffffff;
    mark[w] = 0;
  }
}

__global__ void rcm_isolated_mark(int n, const int32_t* deg, int8_t* state, int32_t* flag) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    flag[v] = deg[v] == 0;
    if (deg[v] == 0) state[v] = 1;
  }
}

__global__ void rcm_reverse(int n, const int32_t* order, int32_t* perm) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    perm[i] = order[n - 1 - i];
}

__global__ void rcm_fill(int n, int32_t* a, int32_t v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = v;
}

__global__ void rcm_iota(int n, int32_t* a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

}  // namespace

extern "C" int jv_rcm_device(int32_t n, const int32_t* rs, const int32_t* col, int32_t* perm,
                             int32_t max_components, int32_t* ncomp_h, void* stream) {
  if (n < 0) return JV_EINVAL;
  if (ncomp_h) *ncomp_h = 0;
  if (n == 0) return JV_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(n);
  Tmp deg(s), state(s), parent(s), mark(s), stamp(s), order(s), fa(s), fb(s), cnt(s), key(s),
      key2(s), vals2(s), minkey(s), tmp(s);
  CK_CUDA(deg.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(state.alloc((size_t)n), "rcm alloc");
  CK_CUDA(parent.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(mark.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(stamp.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(order.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(fa.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(fb.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(cnt.alloc(8), "rcm alloc");
  CK_CUDA(key.alloc(8 * (size_t)n), "rcm alloc");
  CK_CUDA(key2.alloc(8 * (size_t)n), "rcm alloc");
  CK_CUDA(vals2.alloc(4 * (size_t)n), "rcm alloc");
  CK_CUDA(minkey.alloc(8), "rcm alloc");
  int32_t* D = (int32_t*)deg.p;
  int8_t* ST = (int8_t*)state.p;
  int32_t* PA = (int32_t*)parent.p;
  int32_t* MK = (int32_t*)mark.p;
  int32_t* SP = (int32_t*)stamp.p;
  int32_t* ORD = (int32_t*)order.p;
  int32_t* A = (int32_t*)fa.p;
  int32_t* B = (int32_t*)fb.p;
  int32_t* CN = (int32_t*)cnt.p;
  unsigned long long* K1 = (unsigned long long*)key.p;
  unsigned long long* K2 = (unsigned long long*)key2.p;
  int32_t* V2 = (int32_t*)vals2.p;
  unsigned long long* MN = (unsigned long long*)minkey.p;

  rcm_degree_kernel<<<g, kSetupThreads, 0, s>>>(n, rs, col, D);
  CK_CUDA(cudaMemsetAsync(ST, 0, (size_t)n, s), "rcm memset");
  rcm_fill<<<g, kSetupThreads, 0, s>>>(n, PA, 0x7fffffff);
  CK_CUDA(cudaMemsetAsync(MK, 0, 4 * (size_t)n, s), "rcm memset");
  rcm_fill<<<g, kSetupThreads, 0, s>>>(n, SP, -1);
  // radix-sort temp storage, sized once for n items (keys u64 / u32)
  size_t tb1 = 0, tb2 = 0, tb3 = 0;
  CK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb1, A, B, n, 0, 32, s), "rcm sort size");
  CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, K1, K2, A, V2, n, 0, 64, s),
          "rcm sort size");
  CK_CUDA(cub::DeviceSelect::Flagged(nullptr, tb3, A, MK, B, CN, n, s), "rcm select size");
  CK_CUDA(tmp.alloc(std::max(tb1, std::max(tb2, tb3))), "rcm alloc");
  // degree-0 vertices: one-vertex components, first, in index order
  int32_t nord = 0;
  {
    rcm_iota<<<g, kSetupThreads, 0, s>>>(n, A);
    rcm_isolated_mark<<<g, kSetupThreads, 0, s>>>(n, D, ST, MK);   // MK as flags
    size_t tb = tb3;
    CK_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, A, MK, ORD, CN, n, s), "rcm select");
    CK_CUDA(cudaMemcpyAsync(&nord, CN, 4, cudaMemcpyDeviceToHost, s), "rcm copy");
    CK_CUDA(cudaStreamSynchronize(s), "rcm sync");
    CK_CUDA(cudaMemsetAsync(MK, 0, 4 * (size_t)n, s), "rcm memset");
  }
  int stamp_id = 0;
  int32_t comps = nord;
  int32_t others = 0;
  const unsigned long long none = ~0ull;
  auto read_i32 = [&](int32_t* dev, int32_t& h) -> int {
    CK_CUDA(cudaMemcpyAsync(&h, dev, 4, cudaMemcpyDeviceToHost, s), "rcm copy");
    CK_CUDA(cudaStreamSynchronize(s), "rcm sync");
    return JV_OK;
  };
  // BFS tiers from v: tier count and the (degree, index)-smallest vertex of
  // the last tier
  auto tiers = [&](int32_t v, int32_t& ntiers, int32_t& lastmin) -> int {
    ++stamp_id;
    int32_t* F = A;
    int32_t* X = B;
    CK_CUDA(cudaMemcpyAsync(F, &v, 4, cudaMemcpyHostToDevice, s), "rcm copy");
    CK_CUDA(cudaMemcpyAsync(SP + v, &stamp_id, 4, cudaMemcpyHostToDevice, s), "rcm copy");
    int32_t m = 1;
    ntiers = 0;
    for (;;) {
      ++ntiers;
      CK_CUDA(cudaMemsetAsync(CN, 0, 4, s), "rcm memset");
      rcm_bfs_expand<<<grid_for(m), kSetupThreads, 0, s>>>(m, F, rs, col, SP, stamp_id, X, CN);
      int32_t mn = 0;
      if (read_i32(CN, mn) != JV_OK) return JV_ECUDA;
      if (mn == 0) break;
      std::swap(F, X);
      m = mn;
    }
    CK_CUDA(cudaMemcpyAsync(MN, &none, 8, cudaMemcpyHostToDevice, s), "rcm copy");
    rcm_min_list<<<grid_for(m), kSetupThreads, 0, s>>>(m, F, D, MN);
    unsigned long long k = 0;
    CK_CUDA(cudaMemcpyAsync(&k, MN, 8, cudaMemcpyDeviceToHost, s), "rcm copy");
    CK_CUDA(cudaStreamSynchronize(s), "rcm sync");
    lastmin = (int32_t)(uint32_t)(k & 0xffffffffull);
    return JV_OK;
  };
  while (nord < n) {
    // next component: smallest (degree, index) unvisited vertex
    CK_CUDA(cudaMemcpyAsync(MN, &none, 8, cudaMemcpyHostToDevice, s), "rcm copy");
    rcm_min_unvisited<<<g, kSetupThreads, 0, s>>>(n, D, ST, MN);
    unsigned long long k = 0;
    CK_CUDA(cudaMemcpyAsync(&k, MN, 8, cudaMemcpyDeviceToHost, s), "rcm copy");
    CK_CUDA(cudaStreamSynchronize(s), "rcm sync");
    if (k == none) break;
    if (++others > max_components) return 1;   // caller: jv_rcm_host
    ++comps;
    const int32_t cand = (int32_t)(uint32_t)(k & 0xffffffffull);
    int32_t nt = 0, lm = 0;
    if (tiers(cand, nt, lm) != JV_OK) return JV_ECUDA;
    int32_t root = cand, ecc = nt;
    for (;;) {
      const int32_t pick = lm;
      if (tiers(pick, nt, lm) != JV_OK) return JV_ECUDA;
      if (nt > ecc) {
        root = pick;
        ecc = nt;
      } else {
        break;
      }
    }
    // Cuthill-McKee levels from root
    CK_CUDA(cudaMemcpyAsync(A, &root, 4, cudaMemcpyHostToDevice, s), "rcm copy");
    rcm_enqueue<<<1, 32, 0, s>>>(1, A, ORD, nord, ST, PA, MK);
    int32_t base = nord, m = 1;
    nord += 1;
    for (;;) {
      CK_CUDA(cudaMemsetAsync(CN, 0, 4, s), "rcm memset");
      rcm_discover<<<grid_for(m), kSetupThreads, 0, s>>>(m, ORD + base, base, rs, col, ST, PA, MK,
                                                          B, CN);
      int32_t nc = 0;
      if (read_i32(CN, nc) != JV_OK) return JV_ECUDA;
      if (nc == 0) break;
      // index order, then stable (parent position, degree): the queue order
      size_t t1 = tb1;
      CK_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t1, B, A, nc, 0, 32, s), "rcm sort");
      rcm_key_parent_degree<<<grid_for(nc), kSetupThreads, 0, s>>>(nc, A, PA, D, base, K1);
      size_t t2 = tb2;
      CK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, t2, K1, K2, A, V2, nc, 0, 64, s), "rcm sort");
      rcm_enqueue<<<grid_for(nc), kSetupThreads, 0, s>>>(nc, V2, ORD, nord, ST, PA, MK);
      base = nord;
      nord += nc;
      m = nc;
    }
  }
  if (ncomp_h) *ncomp_h = comps;
  rcm_reverse<<<g, kSetupThreads, 0, s>>>(n, ORD, perm);
  JV_CHECK_LAUNCH("jv_rcm_device");
  CK_CUDA(cudaStreamSynchronize(s), "rcm sync");
  return JV_OK;
}
