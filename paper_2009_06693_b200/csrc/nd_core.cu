// nd_core.cu — level-1 kernel backend, graph residency, roots, results.
//
//   nd_individual_batch      individual_batch      (_ckernels.pyx:136-271)
//   nd_segmented_prefix_sum  segmented_prefix_sum  (_ckernels.pyx:103-116)
//   nd_segment_max           segment_max           (_ckernels.pyx:119-133)
//   nd_graph_create/...      Graph, from_edges     (graph.py:36-129)
//   nd_uniform_roots         _uniform_roots        (apps.py:83-103)
#include <cub/cub.cuh>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "nd_item.cuh"

using namespace nd;

static thread_local std::string g_last_error;

void nd_set_last_error(const char* msg, const char* file, int line) {
  g_last_error = std::string(msg) + " (" + file + ":" + std::to_string(line) + ")";
}

extern "C" const char* nd_last_error(void) { return g_last_error.c_str(); }

#include <chrono>
#include <cstdio>
#include <cstdlib>
void nd_trace(const char* what) {
  static const bool on = getenv("ND_TRACE") && getenv("ND_TRACE")[0] == '1';
  if (!on) return;
  static thread_local auto last = std::chrono::steady_clock::now();
  auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[nd_trace] %-28s +%.3f ms\n", what,
          std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}
extern "C" int nd_version(void) { return 1; }

// Keep stream-ordered allocations cached in the device pool between runs
// (the default release threshold of 0 returns memory to the OS at every
// synchronisation, which costs milliseconds per multi-GB run).
// bytes the sampler keeps mapped in the stream-ordered pool
size_t nd_pool_reserve_bytes(size_t free_bytes) {
  static size_t cached = 0;
  if (cached) return cached;
  double gb = 32.0;
  if (const char* e = getenv("ND_POOL_RESERVE_GB")) gb = atof(e);
  size_t want = (size_t)(gb * (1ull << 30));
  if (free_bytes && want > free_bytes / 3) want = free_bytes / 3;
  cached = want;
  return want;
}

int nd_pool_init() {
  // once per device per process (concurrent runs come from several host threads)
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64 || done[dev]) return ND_OK;
  done[dev] = true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return ND_OK;
  uint64_t thr = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  // Reserve one large chunk up front: multi-GB scratch/result buffers are then
  // carved from mapped memory instead of growing (and page-mapping) the pool
  // mid-run, which costs ~0.5 ms per MB when fragmentation forces a new chunk.
  // ND_POOL_RESERVE_GB overrides (0 disables).
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  size_t want = nd_pool_reserve_bytes(fr);
  if (want >= (1ull << 30)) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, want, 0) == cudaSuccess) {
      cudaFreeAsync(p, 0);
      cudaStreamSynchronize(0);
    }
    cudaGetLastError();
  }
  return ND_OK;
}

// Return the stream-ordered pool's unused memory to the device beyond `keep`
// bytes (after a large job, so the next job's allocations are not carved
// from a pool shaped by the previous one).
extern "C" int nd_pool_trim(int64_t keep) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return ND_ERR_CUDA;
  cudaDeviceSynchronize();
  ND_CUDA_TRY(cudaMemPoolTrimTo(pool, keep > 0 ? (size_t)keep : 0));
  return ND_OK;
}

// one pinned host word-block per thread for small D2H reads (no per-run
// cudaMallocHost/cudaFreeHost, which serialise the device)
__global__ void k_export(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                         int64_t bytes) {
  for (int64_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

int nd_d2h(void* dst, const void* src, int64_t bytes, cudaStream_t s) {
  constexpr int64_t CAP = 1 << 16;
  static thread_local unsigned char* stage = nullptr;  // mapped pinned staging
  static thread_local unsigned char* dstage = nullptr;
  if (bytes <= 0) return ND_OK;
  if (bytes > CAP) {  // large reads: a plain copy (pageable or pinned destination)
    ND_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    return ND_OK;
  }
  if (!stage) {
    ND_CUDA_TRY(cudaHostAlloc((void**)&stage, CAP, cudaHostAllocMapped | cudaHostAllocPortable));
    ND_CUDA_TRY(cudaHostGetDevicePointer((void**)&dstage, stage, 0));
  }
  k_export<<<1, 256, 0, s>>>(static_cast<const unsigned char*>(src), dstage, bytes);
  ND_CUDA_TRY(cudaGetLastError());
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  std::memcpy(dst, stage, bytes);
  return ND_OK;
}

int64_t* nd_pinned_scratch() {
  static thread_local int64_t* p = nullptr;
  if (!p) cudaMallocHost(&p, 64 * sizeof(int64_t));
  return p;
}

extern "C" int nd_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0) return ND_ERR_ARG;
  if (!bytes) return ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  ND_CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, s));
  if (!stream) ND_CUDA_TRY(cudaStreamSynchronize(s));
  return ND_OK;
}

int nd_make_app(int code, const double* params, int64_t n_params, NdApp* a) {
  nd_pool_init();
  *a = NdApp{};
  a->code = code;
  if (code == ND_PPR) {
    if (n_params < 1) return ND_ERR_ARG;
    a->term = params[0];
  } else if (code == ND_NODE2VEC) {
    if (n_params < 3) return ND_ERR_ARG;
    const double p = params[0], q = params[1];
    // factor conventions (apps.py:147-152 / _ckernels.pyx:172-181)
    if (params[2] == 0.0) { a->f_ret = 1.0 / p; a->f_adj = 1.0; a->f_far = 1.0 / q; }
    else { a->f_ret = p; a->f_adj = 1.0 / q; a->f_far = 1.0; }
    a->f_max = a->f_ret;
    if (a->f_adj > a->f_max) a->f_max = a->f_adj;
    if (a->f_far > a->f_max) a->f_max = a->f_far;
  } else if (code != ND_DEEPWALK && code != ND_KHOP && code != ND_MULTIRW) {
    return ND_ERR_APP;
  }
  return ND_OK;
}

// ---- level 1 ------------------------------------------------------------------

// one thread owns one segment: the sequential running sum of the reference
__global__ void k_segmented_prefix(const double* __restrict__ v, const int64_t* __restrict__ off,
                                   int64_t nseg, double* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg;
       s += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int64_t hi = off[s + 1];
    for (int64_t i = off[s]; i < hi; i++) {
      acc = __dadd_rn(acc, v[i]);
      out[i] = acc;
    }
  }
}

__global__ void k_segment_max(const double* __restrict__ v, const int64_t* __restrict__ off,
                              int64_t nseg, double* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg;
       s += (int64_t)gridDim.x * blockDim.x) {
    double m = 0.0;
    const int64_t lo = off[s], hi = off[s + 1];
    for (int64_t i = lo; i < hi; i++) {
      double x = v[i];
      if (i == lo || x > m) m = x;
    }
    out[s] = m;
  }
}

extern "C" int nd_segmented_prefix_sum(const double* values, const int64_t* offsets,
                                       int64_t n_segments, double* out, void* stream) {
  if (n_segments < 0) return ND_ERR_ARG;
  if (n_segments == 0) return ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_segmented_prefix<<<nd_grid(n_segments, 128, 148 * 64), 128, 0, s>>>(values, offsets,
                                                                         n_segments, out);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

extern "C" int nd_segment_max(const double* values, const int64_t* offsets, int64_t n_segments,
                              double* out, void* stream) {
  if (n_segments < 0) return ND_ERR_ARG;
  if (n_segments == 0) return ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_segment_max<<<nd_grid(n_segments, 128, 148 * 64), 128, 0, s>>>(values, offsets, n_segments,
                                                                    out);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

// individual_batch over the reference's own arrays: one thread per item.
__global__ void k_individual_batch_ref(GView<int64_t> g, NdApp a, const int64_t* __restrict__ transits,
                                       const int64_t* __restrict__ t_prev,
                                       const int64_t* __restrict__ sids,
                                       const int64_t* __restrict__ tixs,
                                       const int64_t* __restrict__ slots, int64_t n,
                                       uint64_t base0, int64_t* __restrict__ out, int* stall) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = transits[i];
    const int64_t lo = __ldg(g.row + v);
    const int64_t deg = __ldg(g.row + v + 1) - lo;
    ItemStats st;
    int stl = 0;
    const uint64_t ik = key_item((uint64_t)sids[i], (uint64_t)tixs[i], (uint64_t)slots[i]);
    out[i] = run_item(g, grow(g, lo), a, v, deg, t_prev[i], base0, ik, st, &stl);
    if (stl) atomicExch(stall, 1);
  }
}

extern "C" int nd_individual_batch(int app_code, const double* host_params, int64_t n_params,
                                   const int64_t* row_offsets, const int64_t* col_indices,
                                   const double* weights, const double* weight_prefix,
                                   const double* max_weight, const int64_t* transits,
                                   const int64_t* t_prev, const int64_t* sample_ids,
                                   const int64_t* transit_idxs, const int64_t* slots, int64_t n,
                                   uint64_t seed, int64_t step, int64_t* out, void* stream) {
  NdApp a;
  ND_TRY(nd_make_app(app_code, host_params, n_params, &a));
  if (n < 0) return ND_ERR_ARG;
  if (n == 0) return ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int* stall = nullptr;
  ND_CUDA_TRY(nd_alloc(&stall, 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(stall, 0, sizeof(int), s));
  GView<int64_t> g{row_offsets, col_indices, weights, weight_prefix, max_weight, 0, nullptr, nullptr};
  k_individual_batch_ref<<<nd_grid(n, 256), 256, 0, s>>>(g, a, transits, t_prev, sample_ids,
                                                          transit_idxs, slots, n,
                                                          key_base(seed, (uint64_t)step, 0, 0),
                                                          out, stall);
  ND_CUDA_TRY(cudaGetLastError());
  int h = 0;
  ND_TRY(nd_d2h(&h, stall, sizeof(int), s));
  nd_free(stall, s);
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  return h ? ND_ERR_STALL : ND_OK;
}

__global__ void k_mod(const uint64_t* __restrict__ u, const uint64_t* __restrict__ d, int64_t n,
                      uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mod_u64(u[i], d[i]);
}

extern "C" int nd_mod_u64(const uint64_t* u, const uint64_t* d, int64_t n, uint64_t* out,
                          void* stream) {
  if (n <= 0) return n < 0 ? ND_ERR_ARG : ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_mod<<<nd_grid(n, 256), 256, 0, s>>>(u, d, n, out);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

__global__ void k_keyed_u64(uint64_t base, const int64_t* __restrict__ sids,
                            const int64_t* __restrict__ tixs, const int64_t* __restrict__ slots,
                            int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = draw_u64(base, key_item((uint64_t)sids[i], tixs ? (uint64_t)tixs[i] : 0,
                                     slots ? (uint64_t)slots[i] : 0));
  }
}

extern "C" int nd_keyed_u64(uint64_t seed, const int64_t* sample_ids, int64_t step,
                            const int64_t* transit_idxs, const int64_t* slots, int64_t domain,
                            int64_t draw, int64_t n, uint64_t* out, void* stream) {
  if (n <= 0) return n < 0 ? ND_ERR_ARG : ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_keyed_u64<<<nd_grid(n, 256), 256, 0, s>>>(
      key_base(seed, (uint64_t)step, (uint64_t)domain, (uint64_t)draw), sample_ids, transit_idxs,
      slots, n, out);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

// ---- graph residency --------------------------------------------------------------

__global__ void k_col_narrow(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                             int64_t V, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = in[i];
    if (x < 0 || x >= V) atomicExch(bad, 1);
    out[i] = (int32_t)x;
  }
}

__global__ void k_not_unit(const double* __restrict__ w, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (w[i] != 1.0) { *flag = 1; return; }
  }
}

__global__ void k_unit_max(const int64_t* __restrict__ row, int64_t V, double* __restrict__ mx) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    mx[v] = row[v + 1] > row[v] ? 1.0 : 0.0;
}

static void graph_views(nd_graph* G) {
  G->g.row = G->row;
  G->g.col = G->col;
  G->g.w = G->w;
  G->g.pre = G->pre;
  G->g.mx = G->mx;
}

// finish a graph whose row/col(int32)/weights (or null) are resident
static int graph_finish(nd_graph* G, const double* dev_w, const double* dev_pre,
                        const double* dev_mx, cudaStream_t s) {
  const int64_t V = G->g.V, E = G->g.E;
  int unit = 1;
  if (dev_w && E) {
    int* flag;
    ND_CUDA_TRY(nd_alloc(&flag, 1, s));
    ND_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), s));
    k_not_unit<<<nd_grid(E, 256), 256, 0, s>>>(dev_w, E, flag);
    int h = 0;
    ND_TRY(nd_d2h(&h, flag, sizeof(int), s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    nd_free(flag, s);
    unit = !h;
  }
  G->g.unit = unit;
  ND_CUDA_TRY(cudaMalloc(&G->mx, (V ? V : 1) * sizeof(double)));
  G->bytes += V * sizeof(double);
  if (!unit) {
    ND_CUDA_TRY(cudaMalloc(&G->w, E * sizeof(double)));
    ND_CUDA_TRY(cudaMalloc(&G->pre, E * sizeof(double)));
    G->bytes += 2 * E * sizeof(double);
    ND_CUDA_TRY(cudaMemcpyAsync(G->w, dev_w, E * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (dev_pre)
      ND_CUDA_TRY(cudaMemcpyAsync(G->pre, dev_pre, E * sizeof(double), cudaMemcpyDeviceToDevice, s));
    else
      ND_TRY(nd_segmented_prefix_sum(G->w, G->row, V, G->pre, s));
    if (dev_mx)
      ND_CUDA_TRY(cudaMemcpyAsync(G->mx, dev_mx, V * sizeof(double), cudaMemcpyDeviceToDevice, s));
    else
      ND_TRY(nd_segment_max(G->w, G->row, V, G->mx, s));
  } else if (V) {
    k_unit_max<<<nd_grid(V, 256), 256, 0, s>>>(G->row, V, G->mx);
  }
  graph_views(G);
  G->csr_bytes = G->bytes;
  ND_CUDA_TRY(cudaGetLastError());
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  return ND_OK;
}

extern "C" int nd_graph_destroy(nd_graph* G) {
  if (!G) return ND_OK;
  cudaFree(G->row);
  if (!G->host_mapped) {
    cudaFree(G->col);
    cudaFree(G->w);
    cudaFree(G->pre);
  }
  for (const void* p : G->registered) cudaHostUnregister(const_cast<void*>(p));
  cudaFree(G->mx);
  cudaFree(G->hset);
  cudaFree(G->guide);
  cudaFree(G->vrec);
  cudaFree(G->nbw);
  cudaFree(G->nbp);
  cudaFree(G->nbu);
  cudaFree(G->pl);
  cudaFree(G->vline);
  delete G;
  return ND_OK;
}

int nd_pool_init();
extern "C" int nd_graph_create(const int64_t* row_offsets, const int64_t* col_indices,
                               const double* weights, const double* weight_prefix,
                               const double* max_weight, int64_t n_vertices, int64_t n_edges,
                               int arrays_on_host, void* stream, nd_graph** out) {
  if (n_vertices < 0 || n_edges < 0 || n_vertices >= (1ll << 31)) return ND_ERR_ARG;
  nd_pool_init();
  cudaStream_t s = (cudaStream_t)stream;
  nd_graph* G = new nd_graph();
  cudaGetDevice(&G->device);
  G->g.V = n_vertices;
  G->g.E = n_edges;
  const cudaMemcpyKind kind = arrays_on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  int rc = ND_OK;
  int64_t* col64 = nullptr;
  double *w = nullptr, *pre = nullptr, *mx = nullptr;
  int* bad = nullptr;
  do {
    if (cudaMalloc(&G->row, (n_vertices + 1) * sizeof(int64_t)) != cudaSuccess ||
        cudaMalloc(&G->col, nd_col_alloc(n_edges) * sizeof(int32_t)) != cudaSuccess) {
      rc = ND_ERR_NOMEM;
      break;
    }
    G->bytes = (n_vertices + 1) * 8 + n_edges * 4;
    if (cudaMemcpyAsync(G->row, row_offsets, (n_vertices + 1) * sizeof(int64_t), kind, s) ||
        nd_alloc(&col64, n_edges, s) || nd_alloc(&bad, 1, s) ||
        cudaMemcpyAsync(col64, col_indices, n_edges * sizeof(int64_t), kind, s) ||
        cudaMemsetAsync(bad, 0, sizeof(int), s)) {
      rc = ND_ERR_CUDA;
      break;
    }
    if (n_edges) k_col_narrow<<<nd_grid(n_edges, 256), 256, 0, s>>>(col64, n_edges, G->col, n_vertices, bad);
    int hbad = 0;
    nd_d2h(&hbad, bad, sizeof(int), s);
    auto up = [&](const double* src, int64_t n, double** dst) -> int {
      if (!src) return ND_OK;
      if (nd_alloc(dst, n, s)) return ND_ERR_NOMEM;
      return cudaMemcpyAsync(*dst, src, n * sizeof(double), kind, s) ? ND_ERR_CUDA : ND_OK;
    };
    if ((rc = up(weights, n_edges, &w)) || (rc = up(weight_prefix, n_edges, &pre)) ||
        (rc = up(max_weight, n_vertices, &mx)))
      break;
    if (cudaStreamSynchronize(s) != cudaSuccess) { rc = ND_ERR_CUDA; break; }
    if (hbad) { rc = ND_ERR_ARG; break; }
    rc = graph_finish(G, w, pre, mx, s);
  } while (0);
  nd_free(col64, s);
  nd_free(bad, s);
  nd_free(w, s);
  nd_free(pre, s);
  nd_free(mx, s);
  cudaStreamSynchronize(s);
  if (rc != ND_OK) {
    nd_graph_destroy(G);
    if (rc == ND_ERR_CUDA) nd_set_last_error(cudaGetErrorString(cudaGetLastError()), __FILE__, __LINE__);
    return rc;
  }
  *out = G;
  return ND_OK;
}

// -- device from_edges: stable radix sort of (src, dst) keys carrying the edge id

__global__ void k_pack_keys(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                            int64_t n, int bits, int64_t V, uint64_t* __restrict__ keys,
                            int64_t* __restrict__ ids, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = src[i], b = dst[i];
    if (a < 0 || a >= V || b < 0 || b >= V) atomicExch(bad, 1);
    keys[i] = ((uint64_t)a << bits) | (uint64_t)b;
    ids[i] = i;
  }
}

__global__ void k_unpack_csr(const uint64_t* __restrict__ keys, const int64_t* __restrict__ ids,
                             int64_t n, int bits, const double* __restrict__ w_in,
                             int32_t* __restrict__ col, double* __restrict__ w_out,
                             unsigned long long* __restrict__ counts) {
  const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    col[i] = (int32_t)(k & mask);
    if (w_out) w_out[i] = w_in ? w_in[ids[i]] : 1.0;
    int64_t srcv = (int64_t)(k >> bits);
    // row ends: the last entry of a row records its exclusive end
    if (i + 1 == n || (keys[i + 1] >> bits) != (uint64_t)srcv) counts[srcv + 1] = (unsigned long long)(i + 1);
  }
}

// fill rows without edges: row_off[v] = max over u <= v of recorded ends (inclusive scan max)
struct MaxOp {
  __device__ __forceinline__ unsigned long long operator()(unsigned long long a,
                                                           unsigned long long b) const {
    return a > b ? a : b;
  }
};

static int ceil_log2(int64_t x) {
  int b = 0;
  while ((1ll << b) < x) b++;
  return b < 1 ? 1 : b;
}

static int build_from_edges_dev(const int64_t* src, const int64_t* dst, const double* w,
                                int64_t E, int64_t V, cudaStream_t s, nd_graph** out) {
  if (V <= 0 || V >= (1ll << 31) || E < 0) return ND_ERR_ARG;
  nd_pool_init();
  const int bits = ceil_log2(V);
  if (2 * bits > 64) return ND_ERR_ARG;
  nd_graph* G = new nd_graph();
  cudaGetDevice(&G->device);
  G->g.V = V;
  G->g.E = E;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  int64_t *i0 = nullptr, *i1 = nullptr;
  double* wtmp = nullptr;
  int* bad = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc = ND_OK;
  do {
    if (cudaMalloc(&G->row, (V + 1) * sizeof(int64_t)) || cudaMalloc(&G->col, nd_col_alloc(E) * 4)) {
      rc = ND_ERR_NOMEM;
      break;
    }
    G->bytes = (V + 1) * 8 + E * 4;
    if (nd_alloc(&k0, E, s) || nd_alloc(&k1, E, s) || nd_alloc(&i0, E, s) ||
        nd_alloc(&i1, E, s) || nd_alloc(&bad, 1, s) || nd_alloc(&wtmp, w ? E : 1, s)) {
      rc = ND_ERR_NOMEM;
      break;
    }
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    if (E) k_pack_keys<<<nd_grid(E, 256), 256, 0, s>>>(src, dst, E, bits, V, k0, i0, bad);
    cub::DoubleBuffer<uint64_t> dk(k0, k1);
    cub::DoubleBuffer<int64_t> dv(i0, i1);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, E, 0, 2 * bits, s);
    if (nd_alloc((char**)&tmp, tmp_bytes, s)) { rc = ND_ERR_NOMEM; break; }
    if (E) cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dk, dv, E, 0, 2 * bits, s);
    unsigned long long* ends = reinterpret_cast<unsigned long long*>(G->row);
    cudaMemsetAsync(G->row, 0, (V + 1) * sizeof(int64_t), s);
    if (E)
      k_unpack_csr<<<nd_grid(E, 256), 256, 0, s>>>(dk.Current(), dv.Current(), E, bits, w,
                                                   G->col, w ? wtmp : nullptr, ends);
    // rows without edges inherit the previous end: inclusive max-scan
    size_t tb2 = 0;
    cub::DeviceScan::InclusiveScan(nullptr, tb2, ends, ends, MaxOp(), V + 1, s);
    void* tmp2 = nullptr;
    if (nd_alloc((char**)&tmp2, tb2, s)) { rc = ND_ERR_NOMEM; break; }
    cub::DeviceScan::InclusiveScan(tmp2, tb2, ends, ends, MaxOp(), V + 1, s);
    nd_free(tmp2, s);
    int hbad = 0;
    nd_d2h(&hbad, bad, sizeof(int), s);
    if (cudaStreamSynchronize(s)) { rc = ND_ERR_CUDA; break; }
    if (hbad) { rc = ND_ERR_ARG; break; }
    rc = graph_finish(G, w ? wtmp : nullptr, nullptr, nullptr, s);
  } while (0);
  nd_free(k0, s); nd_free(k1, s); nd_free(i0, s); nd_free(i1, s);
  nd_free(bad, s); nd_free(wtmp, s); nd_free(tmp, s);
  cudaStreamSynchronize(s);
  // the build's sort buffers (~32 B/edge) go back to the OS down to the
  // sampler's reserve, which stays mapped for the runs that follow
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolTrimTo(pool, nd_pool_reserve_bytes(0));
  }
  if (rc != ND_OK) {
    nd_graph_destroy(G);
    return rc;
  }
  *out = G;
  return ND_OK;
}

int nd_build_from_edges_dev(const int64_t* src, const int64_t* dst, const double* w, int64_t E,
                            int64_t V, cudaStream_t s, nd_graph** out) {
  return build_from_edges_dev(src, dst, w, E, V, s, out);
}

extern "C" int nd_graph_from_edges(const int64_t* src, const int64_t* dst, const double* weights,
                                   int64_t n_edges, int64_t n_vertices, void* stream,
                                   nd_graph** out) {
  return build_from_edges_dev(src, dst, weights, n_edges, n_vertices, (cudaStream_t)stream, out);
}

// -- keyed RMAT: 16-bit quadrant draws, 4 levels
// per keyed u64 (domain 16), endpoints through a keyed bijection (domain 17),
// weight 1 + 4u keyed on the edge index (domain 3, graph.py:168-169 formula).
__device__ __forceinline__ uint64_t rmat_bij(uint64_t x, int scale, uint64_t k1, uint64_t k2) {
  const uint64_t mask = scale >= 64 ? ~0ull : ((1ull << scale) - 1);
  const int sh = scale / 2 + 1;
  x = (x * (k1 | 1ull)) & mask;
  x ^= x >> sh;
  x = (x * (k2 | 1ull)) & mask;
  x ^= x >> sh;
  return x;
}

__global__ void k_rmat(int scale, int64_t n_edges, uint32_t ta, uint32_t tab, uint32_t tabc,
                       uint64_t seed, uint64_t k1, uint64_t k2, int undirected, int weighted,
                       int64_t* __restrict__ src, int64_t* __restrict__ dst,
                       double* __restrict__ w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_edges;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = 0, d = 0, u = 0;
    const uint64_t ik = key_item((uint64_t)e, 0, 0);
    for (int l = 0; l < scale; l++) {
      if ((l & 3) == 0) u = draw_u64(key_base(seed, (uint64_t)(l >> 2), 16, 0), ik);
      uint32_t r = (uint32_t)((u >> (16 * (l & 3))) & 0xFFFFu);
      s = (s << 1) | (uint64_t)(r >= tab);
      d = (d << 1) | (uint64_t)((r >= ta && r < tab) || r >= tabc);
    }
    s = rmat_bij(s, scale, k1, k2);
    d = rmat_bij(d, scale, k1, k2);
    double we = 1.0;
    if (weighted) we = __dadd_rn(1.0, __dmul_rn(4.0, to_unit(draw_u64(key_base(seed, 0, 3, 0), ik))));
    if (undirected) {
      src[2 * e] = (int64_t)s; dst[2 * e] = (int64_t)d;
      src[2 * e + 1] = (int64_t)d; dst[2 * e + 1] = (int64_t)s;
      if (w) { w[2 * e] = we; w[2 * e + 1] = we; }
    } else {
      src[e] = (int64_t)s; dst[e] = (int64_t)d;
      if (w) w[e] = we;
    }
  }
}

extern "C" int nd_graph_rmat(int scale, int64_t n_edges, uint32_t ta, uint32_t tab, uint32_t tabc,
                             uint64_t seed, int undirected, int weighted, void* stream,
                             nd_graph** out) {
  if (scale < 1 || scale > 30 || n_edges < 0) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t m = n_edges * (undirected ? 2 : 1);
  int64_t *src = nullptr, *dst = nullptr;
  double* w = nullptr;
  ND_CUDA_TRY(nd_alloc(&src, m, s));
  ND_CUDA_TRY(nd_alloc(&dst, m, s));
  if (weighted) ND_CUDA_TRY(nd_alloc(&w, m, s));
  const uint64_t k1 = fin64(fin64(key_base(seed, 0, 17, 0) + key_item(0, 0, 0)));
  const uint64_t k2 = fin64(fin64(key_base(seed, 0, 17, 1) + key_item(0, 0, 0)));
  if (n_edges)
    k_rmat<<<nd_grid(n_edges, 256, 148 * 64), 256, 0, s>>>(scale, n_edges, ta, tab, tabc, seed, k1,
                                                          k2, undirected, weighted, src, dst, w);
  ND_CUDA_TRY(cudaGetLastError());
  int rc = build_from_edges_dev(src, dst, w, m, 1ll << scale, s, out);
  nd_free(src, s);
  nd_free(dst, s);
  nd_free(w, s);
  cudaStreamSynchronize(s);
  return rc;
}

extern "C" int nd_graph_info(const nd_graph* g, int64_t* n_vertices, int64_t* n_edges,
                             int* unit_weights, int64_t* bytes) {
  if (!g) return ND_ERR_ARG;
  if (n_vertices) *n_vertices = g->g.V;
  if (n_edges) *n_edges = g->g.E;
  if (unit_weights) *unit_weights = g->g.unit;
  if (bytes) *bytes = g->bytes;
  return ND_OK;
}

// A graph whose column / weight / prefix arrays stay in host memory and are
// read by the kernels in place over the host link (zero copy): the
// out-of-core fallback for apps the partition shuttle does not run
// (node2vec's second row, collective apps).  Row offsets and per-row maxima
// are device-resident; no index or record structure is ever built (the
// kernels take their plain-CSR paths).  Host arrays: int64 row offsets
// [V+1], int32 columns [E], f64 weights and inclusive prefix [E] (both NULL
// for unit weights); caller-owned, alive until destroy.
static const void* map_host(const void* p, size_t bytes, nd_graph* G, cudaError_t* err) {
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess || at.type != cudaMemoryTypeHost) {  // not page-locked yet: register it
    cudaGetLastError();
    e = cudaHostRegister(const_cast<void*>(p), bytes,
                         cudaHostRegisterMapped | cudaHostRegisterReadOnly);
    if (e != cudaSuccess) { *err = e; return nullptr; }
    G->registered.push_back(p);
  }
  void* d = nullptr;
  e = cudaHostGetDevicePointer(&d, const_cast<void*>(p), 0);
  if (e != cudaSuccess) { *err = e; return nullptr; }
  return d;
}

extern "C" int nd_graph_create_mapped(const int64_t* row_offsets, const int32_t* col,
                                      const double* weights, const double* prefix,
                                      int64_t n_vertices, int64_t n_edges, void* stream,
                                      nd_graph** out) {
  if (!row_offsets || !out || n_vertices <= 0 || n_edges <= 0 || !col || n_vertices >= (1ll << 31) ||
      (!weights) != (!prefix))
    return ND_ERR_ARG;
  if (row_offsets[0] != 0 || row_offsets[n_vertices] != n_edges) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  auto* G = new nd_graph();
  G->host_mapped = true;
  G->device = 0;
  cudaGetDevice(&G->device);
  G->g.V = n_vertices;
  G->g.E = n_edges;
  G->skipped = ND_IDX_VREC | ND_IDX_NBW | ND_IDX_NBP | ND_IDX_NBU | ND_IDX_GUIDE | ND_IDX_HSET |
               ND_IDX_LINES;
  cudaError_t err = cudaSuccess;
  G->col = const_cast<int32_t*>(static_cast<const int32_t*>(map_host(col, n_edges * 4, G, &err)));
  if (weights && G->col) {
    G->w = const_cast<double*>(static_cast<const double*>(map_host(weights, n_edges * 8, G, &err)));
    G->pre = const_cast<double*>(static_cast<const double*>(map_host(prefix, n_edges * 8, G, &err)));
  }
  if (err == cudaSuccess) err = cudaMalloc(&G->row, (n_vertices + 1) * sizeof(int64_t));
  if (err == cudaSuccess) err = cudaMalloc(&G->mx, n_vertices * sizeof(double));
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(G->row, row_offsets, (n_vertices + 1) * 8, cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) {
    nd_set_last_error(cudaGetErrorString(err), __FILE__, __LINE__);
    nd_graph_destroy(G);
    return ND_ERR_CUDA;
  }
  G->bytes = (n_vertices + 1) * 8 + n_vertices * 8;
  G->g.unit = weights ? 0 : 1;
  if (weights) {
    int rc = nd_segment_max(G->w, G->row, n_vertices, G->mx, s);  // streams the weights once
    if (rc != ND_OK) { nd_graph_destroy(G); return rc; }
  } else {
    k_unit_max<<<nd_grid(n_vertices, 256), 256, 0, s>>>(G->row, n_vertices, G->mx);
  }
  graph_views(G);
  G->csr_bytes = G->bytes;
  if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    nd_graph_destroy(G);
    return ND_ERR_CUDA;
  }
  *out = G;
  return ND_OK;
}

extern "C" int nd_graph_footprint(const nd_graph* g, int64_t* csr_bytes, int64_t* index_bytes,
                                  double* prep_ms, int* built, int* skipped) {
  if (!g) return ND_ERR_ARG;
  if (csr_bytes) *csr_bytes = g->csr_bytes;
  if (index_bytes) *index_bytes = g->bytes - g->csr_bytes;
  if (prep_ms) *prep_ms = g->prep_ms;
  if (built) *built = g->built;
  if (skipped) *skipped = g->skipped;
  return ND_OK;
}

extern "C" int nd_graph_arrays(const nd_graph* g, const int64_t** row_offsets, const int32_t** col,
                               const double** weights, const double** prefix,
                               const double** max_w) {
  if (!g) return ND_ERR_ARG;
  if (row_offsets) *row_offsets = g->row;
  if (col) *col = g->col;
  if (weights) *weights = g->w;
  if (prefix) *prefix = g->pre;
  if (max_w) *max_w = g->mx;
  return ND_OK;
}

// ---- roots (apps.py:83-103) ---------------------------------------------------------

template <typename OutT>
__global__ void k_uniform_roots(int64_t V, int64_t count, uint64_t base, int64_t sample_lo,
                                int64_t n, OutT* __restrict__ roots) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    OutT* r = roots + i * count;
    const uint64_t ik = key_item((uint64_t)(sample_lo + i), 0, 0);
    const bool distinct = V >= count;
    int64_t have = 0;
    uint64_t b = base;  // draw d: base + C_DRAW*d
    while (have < count) {
      int64_t v = (int64_t)mod_u64(draw_u64(b, ik), (uint64_t)V);
      b += C_DRAW;
      if (distinct) {
        bool dup = false;
        for (int64_t k = 0; k < have; k++)
          if ((int64_t)r[k] == v) { dup = true; break; }
        if (dup) continue;
      }
      r[have++] = (OutT)v;
    }
  }
}

// count > 1 (batch roots): one warp per sample.  The lanes draw the first
// `count` keyed candidates at once; when they hold no repeat -- nearly always
// for V >> count -- they are the roots (apps.py:92-101 keeps every draw that
// is new).  Otherwise lane 0 replays the sequential rejection loop.
constexpr int ROOTS_WARP_MAX = 256;

template <typename OutT>
__global__ void k_uniform_roots_warp(int64_t V, int64_t count, uint64_t base, int64_t sample_lo,
                                     int64_t n, OutT* __restrict__ roots) {
  __shared__ int64_t cand[8][ROOTS_WARP_MAX];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool distinct = V >= count;
  for (int64_t i = warp; i < n; i += nw) {
    const uint64_t ik = key_item((uint64_t)(sample_lo + i), 0, 0);
    for (int64_t d = lane; d < count; d += 32)
      cand[wib][d] = (int64_t)mod_u64(draw_u64(base + C_DRAW * (uint64_t)d, ik), (uint64_t)V);
    __syncwarp();
    bool dup = false;
    if (distinct)
      for (int64_t d = lane; d < count && !dup; d += 32)
        for (int64_t e = 0; e < d; e++)
          if (cand[wib][e] == cand[wib][d]) { dup = true; break; }
    dup = __any_sync(0xffffffffu, dup);
    OutT* r = roots + i * count;
    if (!dup) {
      for (int64_t d = lane; d < count; d += 32) r[d] = (OutT)cand[wib][d];
    } else if (lane == 0) {
      int64_t have = 0;
      uint64_t b = base;
      while (have < count) {
        const int64_t v = (int64_t)mod_u64(draw_u64(b, ik), (uint64_t)V);
        b += C_DRAW;
        bool rep = false;
        for (int64_t k = 0; k < have; k++)
          if ((int64_t)r[k] == v) { rep = true; break; }
        if (rep) continue;
        r[have++] = (OutT)v;
      }
    }
    __syncwarp();
  }
}

template <typename OutT>
static void launch_uniform_roots(int64_t V, int64_t count, uint64_t base, int64_t sample_lo,
                                 int64_t n, OutT* roots, cudaStream_t s) {
  if (count > 1 && count <= ROOTS_WARP_MAX)
    k_uniform_roots_warp<OutT><<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(V, count, base,
                                                                             sample_lo, n, roots);
  else
    k_uniform_roots<OutT><<<nd_grid(n, 128), 128, 0, s>>>(V, count, base, sample_lo, n, roots);
}

extern "C" int nd_uniform_roots(const nd_graph* g, int64_t count, uint64_t seed, int64_t sample_lo,
                                int64_t n_samples, int64_t* roots, void* stream) {
  if (!g || count < 0 || n_samples < 0) return ND_ERR_ARG;
  if (!n_samples || !count) return ND_OK;
  if (g->g.V <= 0) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  launch_uniform_roots<int64_t>(g->g.V, count, key_base(seed, 0, 2, 0), sample_lo, n_samples,
                                roots, s);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

int nd_uniform_roots_i32(const DevGraph& g, int64_t count, uint64_t seed, int64_t sample_lo,
                         int64_t n, int32_t* roots, cudaStream_t s) {
  if (!n || !count) return ND_OK;
  if (g.V <= 0) return ND_ERR_ARG;
  launch_uniform_roots<int32_t>(g.V, count, key_base(seed, 0, 2, 0), sample_lo, n, roots, s);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

// ---- results ------------------------------------------------------------------------

extern "C" int nd_result_info(const nd_result* r, int64_t* n_samples, int64_t* n_steps,
                              int64_t* total_sampled, int64_t* total_recorded) {
  if (!r) return ND_ERR_ARG;
  if (n_samples) *n_samples = r->n;
  if (n_steps) *n_steps = r->n_steps;
  if (total_sampled) *total_sampled = r->total_sampled;
  if (total_recorded) *total_recorded = r->total_recorded;
  return ND_OK;
}

// Runs write the final ids once, as int32 (ND_F_FINAL_IDS32: half the bytes of
// every read and gather).  The reference-width int64 field is derived on the
// first request, on the result's stream, and kept.
__global__ void k_widen_ids(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  const int64_t half = n >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < half; i += stride) {
    const int2 x = reinterpret_cast<const int2*>(in)[i];
    reinterpret_cast<longlong2*>(out)[i] = make_longlong2(x.x, x.y);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[n - 1] = in[n - 1];
}

static std::mutex g_result_mu;

// int64 field `f64` derived from its int32 source `f32` on first request
static int ensure_wide(const nd_result* rc, int f64, int f32) {
  nd_result* r = const_cast<nd_result*>(rc);
  std::lock_guard<std::mutex> lock(g_result_mu);
  if (r->ptr[f64] || !r->ptr[f32]) return ND_OK;
  const int64_t n = r->cnt[f32];
  int64_t* out = nullptr;
  ND_CUDA_TRY(nd_alloc(&out, n > 0 ? n : 1, r->stream));
  if (n)
    k_widen_ids<<<nd_grid((n + 1) / 2, 256, 148 * 16), 256, 0, r->stream>>>(
        static_cast<const int32_t*>(r->ptr[f32]), n, out);
  ND_CUDA_TRY(cudaGetLastError());
  ND_CUDA_TRY(cudaStreamSynchronize(r->stream));
  r->set(f64, out, n);
  return ND_OK;
}

// a field the run deferred (nd_result::lazy_build), built once on request
static int ensure_lazy(const nd_result* rc, int field) {
  nd_result* r = const_cast<nd_result*>(rc);
  std::lock_guard<std::mutex> lock(g_result_mu);
  if (r->lazy_field != field || r->ptr[field] || !r->lazy_build) return ND_OK;
  const int rc2 = r->lazy_build(r);
  if (r->lazy_free) r->lazy_free();
  r->lazy_build = nullptr;
  r->lazy_free = nullptr;
  if (rc2 == ND_OK) ND_CUDA_TRY(cudaStreamSynchronize(r->stream));
  return rc2;
}

static int ensure_derived(const nd_result* r, int field) {
  if (field == ND_F_FINAL_IDS) return ensure_wide(r, ND_F_FINAL_IDS, ND_F_FINAL_IDS32);
  if (field == ND_F_STEP_VALS) {
    ND_TRY(ensure_lazy(r, ND_F_STEP_VALS32));
    return ensure_wide(r, ND_F_STEP_VALS, ND_F_STEP_VALS32);
  }
  return ensure_lazy(r, field);
}

extern "C" int nd_result_field(const nd_result* r, int field, const void** ptr, int64_t* count) {
  if (!r || field < 0 || field >= ND_N_FIELDS) return ND_ERR_ARG;
  ND_TRY(ensure_derived(r, field));
  *ptr = r->ptr[field];
  *count = r->cnt[field];
  return ND_OK;
}

extern "C" int nd_result_counters(const nd_result* r, int64_t* host_counters, int64_t n) {
  if (!r) return ND_ERR_ARG;
  for (int64_t i = 0; i < n && i < ND_N_COUNTERS; i++) host_counters[i] = r->counters[i];
  return ND_OK;
}

extern "C" int nd_result_copy(const nd_result* r, int field, void* dst, void* stream) {
  if (!r || field < 0 || field >= ND_N_FIELDS) return ND_ERR_ARG;
  ND_TRY(ensure_derived(r, field));
  if (!r->ptr[field] || !r->cnt[field]) return ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  ND_CUDA_TRY(cudaMemcpyAsync(dst, r->ptr[field], r->cnt[field] * r->esz[field], cudaMemcpyDefault, s));
  if (!stream) ND_CUDA_TRY(cudaStreamSynchronize(s));
  return ND_OK;
}

// int64 -> int32 ids: 16-byte loads, 8-byte stores, grid-stride over pairs
__global__ void k_narrow_ids(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  const int64_t half = n >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < half; i += stride) {
    const longlong2 x = __ldcs(reinterpret_cast<const longlong2*>(in) + i);
    __stcs(reinterpret_cast<int2*>(out) + i, make_int2((int32_t)x.x, (int32_t)x.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[n - 1] = (int32_t)in[n - 1];
}

extern "C" int nd_result_narrow_ids(nd_result* r, void* stream) {
  if (!r) return ND_ERR_ARG;
  if (r->ptr[ND_F_FINAL_IDS32] || !r->ptr[ND_F_FINAL_IDS]) return ND_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = r->cnt[ND_F_FINAL_IDS];
  int32_t* out = nullptr;
  ND_CUDA_TRY(nd_alloc(&out, n > 0 ? n : 1, s));
  if (n) k_narrow_ids<<<nd_grid((n + 1) / 2, 256, 148 * 16), 256, 0, s>>>(
      static_cast<const int64_t*>(r->ptr[ND_F_FINAL_IDS]), n, out);
  ND_CUDA_TRY(cudaGetLastError());
  r->set(ND_F_FINAL_IDS32, out, n);
  return ND_OK;
}

// dense final rows (the frontend's getFinalSamples, frontend/src/index.ts:
// 160-171): row i = sample i's roots then sampled vertices, padded with NULL
__global__ void k_dense_rows(const int64_t* __restrict__ off, const int32_t* __restrict__ ids,
                             int64_t n, int64_t width, int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const int64_t a = off[i], len = off[i + 1] - a;
    for (int64_t k = lane; k < width; k += 32) out[i * width + k] = k < len ? ids[a + k] : -1;
  }
}

__global__ void k_max_row(const int64_t* __restrict__ off, int64_t n, unsigned long long* __restrict__ mx) {
  unsigned long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long len = (unsigned long long)(off[i + 1] - off[i]);
    m = len > m ? len : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_down_sync(0xffffffffu, m, o);
    m = x > m ? x : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

extern "C" int nd_result_max_row(const nd_result* r, int64_t* host_width) {
  if (!r || !host_width) return ND_ERR_ARG;
  *host_width = 0;
  if (!r->ptr[ND_F_FINAL_OFF] || r->n <= 0) return ND_OK;
  unsigned long long* mx = nullptr;
  ND_CUDA_TRY(nd_alloc(&mx, 1, r->stream));
  ND_CUDA_TRY(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), r->stream));
  k_max_row<<<nd_grid(r->n, 256), 256, 0, r->stream>>>(
      static_cast<const int64_t*>(r->ptr[ND_F_FINAL_OFF]), r->n, mx);
  unsigned long long h = 0;
  ND_TRY(nd_d2h(&h, mx, sizeof(h), r->stream));
  ND_CUDA_TRY(cudaStreamSynchronize(r->stream));
  nd_free(mx, r->stream);
  *host_width = (int64_t)h;
  return ND_OK;
}

extern "C" int nd_result_dense(const nd_result* r, int64_t width, int32_t* out, void* stream) {
  if (!r || width < 0 || (!out && r->n * width > 0)) return ND_ERR_ARG;
  if (!r->ptr[ND_F_FINAL_OFF] || !r->ptr[ND_F_FINAL_IDS32] || r->n * width == 0) return ND_OK;
  cudaStream_t s = stream ? (cudaStream_t)stream : r->stream;
  k_dense_rows<<<nd_grid(r->n * 32, 256, 148 * 32), 256, 0, s>>>(
      static_cast<const int64_t*>(r->ptr[ND_F_FINAL_OFF]),
      static_cast<const int32_t*>(r->ptr[ND_F_FINAL_IDS32]), r->n, width, out);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

extern "C" int nd_result_destroy(nd_result* r) {
  if (!r) return ND_OK;
  if (r->lazy_free) r->lazy_free();
  for (int f = 0; f < ND_N_FIELDS; f++)
    if (r->ptr[f]) cudaFreeAsync(r->ptr[f], r->stream);
  delete r;
  return ND_OK;
}
