// nd_index.cu — exact per-row indexes that shorten the sampler's dependent
// search chains (DESIGN.md §3/§8):
//   * guide tables for the inverse-CDF weighted pick (DeepWalk, PPR, node2vec
//     step 0): guide[lo+j] = upper_bound(prefix[lo:hi], j*(total/deg));
//   * hash sets for node2vec's has_edge(t, u) (graph.py:78-81,
//     _ckernels.pyx:77-87): open addressing, linear probing, load <= 1/2.
// Built once per graph on first use; answers are identical to the binary
// searches they replace (tests/test_gpu_kernels.py::test_index_equivalence).
#include <cub/cub.cuh>

#include <chrono>
#include <cstdlib>
#include <mutex>

#include "nd_internal.h"

using namespace nd;

namespace {

__global__ void k_build_guide(const int64_t* __restrict__ row, const double* __restrict__ pre,
                              int64_t V, int32_t* __restrict__ guide) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < V; v += nw) {
    const int64_t lo = row[v], deg = row[v + 1] - lo;
    if (deg <= GUIDE_MIN_DEG) continue;
    const double total = pre[lo + deg - 1];
    const double width = __ddiv_rn(total, (double)deg);
    for (int64_t j = lane; j < deg; j += 32) {
      const double y = __dmul_rn(width, (double)j);
      int64_t a = 0, b = deg;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (pre[lo + mid] <= y) a = mid + 1; else b = mid;
      }
      guide[lo + j] = (int32_t)a;
    }
  }
}

__global__ void k_build_hset(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                             int64_t V, int32_t* __restrict__ hset) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < V; v += nw) {
    const int64_t lo = row[v], deg = row[v + 1] - lo;
    if (deg <= HASH_MIN_DEG) continue;
    int32_t* tab = hset + 4 * lo;
    const int64_t size = hset_size(deg);
    const uint32_t mask = (uint32_t)size - 1;
    const int sh = 32 - (63 - __clzll(size));
    for (int64_t e = lane; e < deg; e += 32) {
      const int32_t u = col[lo + e];
      uint32_t p = hset_hash((uint32_t)u) >> sh;
      while (true) {
        const int32_t old = atomicCAS(tab + p, -1, u);
        if (old == -1 || old == u) break;
        p = (p + 1) & mask;
      }
    }
  }
}

__global__ void k_build_vrec(const int64_t* __restrict__ row, const double* __restrict__ mx,
                             const double* __restrict__ pre, int64_t V, VRec* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    VRec r;
    r.lo = row[v];
    r.deg = row[v + 1] - r.lo;
    r.mx = mx[v];
    r.total = pre ? (r.deg > 0 ? pre[r.lo + r.deg - 1] : 0.0) : (double)r.deg;
    out[v] = r;
  }
}

__global__ void k_build_nbr(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                            const double* __restrict__ w, const double* __restrict__ pre,
                            const double* __restrict__ mx, int64_t E, NbrW* __restrict__ nw,
                            NbrP* __restrict__ np_, NbrU* __restrict__ nu) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = col[e];
    const int64_t lo = row[u], deg = row[u + 1] - lo;
    if (nu) {
      NbrU r;
      r.col = u;
      r.deg = (int32_t)deg;
      r.lo = lo;
      nu[e] = r;
      continue;
    }
    if (nw) {
      NbrW r;
      r.col = u;
      r.deg = (int32_t)deg;
      r.lo = lo;
      r.w = w[e];
      r.mx = mx[u];
      nw[e] = r;
    }
    if (np_) {
      NbrP r;
      r.pre = pre[e];
      r.col = u;
      r.deg = (int32_t)deg;
      r.lo = lo;
      r.total = deg > 0 ? pre[lo + deg - 1] : 0.0;
      np_[e] = r;
    }
  }
}

// lines per row: ceil(deg / 3)
__global__ void k_line_counts(const int64_t* __restrict__ row, int64_t V, int64_t* __restrict__ cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= V;
       v += (int64_t)gridDim.x * blockDim.x)
    cnt[v] = v < V ? (row[v + 1] - row[v] + 2) / 3 : 0;
}

__global__ void k_vline32(const int64_t* __restrict__ first, int64_t V, int32_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = (int32_t)first[v];
}

// one warp per row, a lane per line: the line's three records and
// guide[j] = upper_bound(prefix row, rn(rn(total/deg) * j)) for its four
// buckets, exactly as k_build_guide
__global__ void k_build_lines(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                              const double* __restrict__ pre, const int32_t* __restrict__ vline,
                              int64_t V, PickLine* __restrict__ pl) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < V; v += nw) {
    const int64_t lo = row[v], deg = row[v + 1] - lo;
    if (deg <= 0) continue;
    const double total = pre[lo + deg - 1];
    const double width = __ddiv_rn(total, (double)deg);
    const int64_t n_lines = (deg + 2) / 3;
    for (int64_t L = lane; L < n_lines; L += 32) {
      PickLine ln;
      for (int q = 0; q < 4; q++) {
        const int64_t j = 3 * L + q;
        int64_t a = deg;
        if (j < deg && width > 0.0) {
          const double y = __dmul_rn(width, (double)j);
          int64_t b = deg;
          a = 0;
          while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (pre[lo + mid] <= y) a = mid + 1; else b = mid;
          }
        }
        ln.g[q] = (int32_t)a;
      }
      for (int q = 0; q < 3; q++) {
        const int64_t k = 3 * L + q;
        PickRec r{__longlong_as_double(0x7FF0000000000000ll), 0.0, -1, 0, 0, 0};
        if (k < deg) {
          const int32_t u = col[lo + k];
          const int64_t ulo = row[u], udeg = row[u + 1] - ulo;
          r.pre = pre[lo + k];
          r.total = udeg > 0 ? pre[ulo + udeg - 1] : 0.0;
          r.col = u;
          r.deg = (int32_t)udeg;
          r.llo = vline[u];
        }
        ln.r[q] = r;
      }
      ln.spare[0] = ln.spare[1] = ln.spare[2] = ln.spare[3] = 0;
      pl[vline[v] + L] = ln;
    }
  }
}

}  // namespace

// lazy index builds may be requested by concurrent runs on one graph
static std::mutex g_index_mu;

// Every structure below is an accelerator, not a requirement: the kernels
// fall back to the plain CSR (row/col/weights/prefix, same answers) when a
// pointer is null.  A structure is built only when it fits beside a margin
// kept free for the runs' own buffers (walk windows, final rows, sort
// scratch): ND_INDEX_MARGIN_MB, default 8 GiB.
static bool room_for(double need) {
  static const double margin = [] {
    const char* e = getenv("ND_INDEX_MARGIN_MB");
    return (e && e[0] ? atof(e) : 8192.0) * (1 << 20);
  }();
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
  return need + margin <= (double)fr;
}

namespace {
struct PrepTimer {  // host wall time of a build (each build ends in a stream sync)
  nd_graph* G;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  NvtxRange nvtx{"nd_graph index build"};
  explicit PrepTimer(nd_graph* g) : G(g) {}
  ~PrepTimer() {
    G->prep_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                      .count();
  }
};
}  // namespace

int nd_graph_ensure_records(nd_graph* G, int want_tries, cudaStream_t s) {
  static const bool disabled = getenv("ND_NO_PACK") && getenv("ND_NO_PACK")[0] == '1';
  if (disabled) return ND_OK;
  std::lock_guard<std::mutex> lock(g_index_mu);
  const int64_t V = G->g.V, E = G->g.E;
  const bool need_vrec = !G->vrec && V > 0 && !(G->skipped & ND_IDX_VREC);
  const bool need_nbu = E > 0 && G->g.unit && !G->nbu && !(G->skipped & ND_IDX_NBU);
  const bool need_nbp = E > 0 && !G->g.unit && !G->nbp && !(G->skipped & ND_IDX_NBP);
  const bool need_nbw = E > 0 && !G->g.unit && want_tries && !G->nbw && !(G->skipped & ND_IDX_NBW);
  if (!need_vrec && !need_nbu && !need_nbp && !need_nbw) return ND_OK;
  PrepTimer timer(G);
  bool built = false;
  if (need_vrec) {
    if (room_for((double)V * sizeof(VRec))) {
      built = true;
      ND_CUDA_TRY(cudaMalloc(&G->vrec, V * sizeof(VRec)));
      G->bytes += V * sizeof(VRec);
      G->built |= ND_IDX_VREC;
      k_build_vrec<<<nd_grid(V, 256), 256, 0, s>>>(G->row, G->mx, G->g.unit ? nullptr : G->pre, V,
                                                    G->vrec);
      ND_CUDA_TRY(cudaGetLastError());
      G->g.vrec = G->vrec;
    } else {
      G->skipped |= ND_IDX_VREC;
    }
  }
  NbrW* nw = nullptr;
  NbrP* np_ = nullptr;
  NbrU* nu = nullptr;
  if (need_nbu) {
    if (room_for((double)E * sizeof(NbrU))) ND_CUDA_TRY(cudaMalloc(&nu, E * sizeof(NbrU)));
    else G->skipped |= ND_IDX_NBU;
  }
  if (need_nbp) {
    if (room_for((double)E * sizeof(NbrP))) ND_CUDA_TRY(cudaMalloc(&np_, E * sizeof(NbrP)));
    else G->skipped |= ND_IDX_NBP;
  }
  if (need_nbw) {  // tries read nbw only beside nbp: without nbp it would sit idle
    if ((np_ || G->nbp) && room_for((double)E * sizeof(NbrW)))
      ND_CUDA_TRY(cudaMalloc(&nw, E * sizeof(NbrW)));
    else
      G->skipped |= ND_IDX_NBW;
  }
  if (nw || np_ || nu) {
    built = true;
    k_build_nbr<<<nd_grid(E, 256, 148 * 64), 256, 0, s>>>(G->row, G->col, G->w, G->pre, G->mx, E,
                                                           nw, np_, nu);
    ND_CUDA_TRY(cudaGetLastError());
    if (nw) { G->nbw = nw; G->g.nbw = nw; G->bytes += E * sizeof(NbrW); G->built |= ND_IDX_NBW; }
    if (np_) { G->nbp = np_; G->g.nbp = np_; G->bytes += E * sizeof(NbrP); G->built |= ND_IDX_NBP; }
    if (nu) { G->nbu = nu; G->g.nbu = nu; G->bytes += E * sizeof(NbrU); G->built |= ND_IDX_NBU; }
  }
  // other streams may use the records as soon as this call returns
  if (built) ND_CUDA_TRY(cudaStreamSynchronize(s));
  return ND_OK;
}

int nd_graph_ensure_index(nd_graph* G, int want_hset, int want_guide, cudaStream_t s) {
  static const bool disabled = getenv("ND_NO_INDEX") && getenv("ND_NO_INDEX")[0] == '1';
  if (disabled) return ND_OK;
  std::lock_guard<std::mutex> lock(g_index_mu);
  const int64_t V = G->g.V, E = G->g.E;
  const bool need_guide = want_guide && !G->guide && !G->g.unit && E > 0 &&
                          !(G->skipped & ND_IDX_GUIDE);
  const bool need_hset = want_hset && !G->hset && E > 0 && !(G->skipped & ND_IDX_HSET);
  if (!need_guide && !need_hset) return ND_OK;
  PrepTimer timer(G);
  if (need_guide) {
    // +8 entries: the walker kernels read guide entries as aligned 32-byte chunks
    if (room_for((double)(E + 8) * sizeof(int32_t))) {
      ND_CUDA_TRY(cudaMalloc(&G->guide, (E + 8) * sizeof(int32_t)));
      G->bytes += E * 4;
      G->built |= ND_IDX_GUIDE;
      k_build_guide<<<148 * 16, 256, 0, s>>>(G->row, G->pre, V, G->guide);
      ND_CUDA_TRY(cudaGetLastError());
      ND_CUDA_TRY(cudaStreamSynchronize(s));
      G->g.guide = G->guide;
    } else {
      G->skipped |= ND_IDX_GUIDE;
    }
  }
  if (need_hset) {
    // +8 slots: the walker kernels read the tables as aligned 32-byte chunks
    if (room_for((double)(4 * E + 8) * sizeof(int32_t))) {
      ND_CUDA_TRY(cudaMalloc(&G->hset, (4 * E + 8) * sizeof(int32_t)));
      G->bytes += 16 * E;
      G->built |= ND_IDX_HSET;
      ND_CUDA_TRY(cudaMemsetAsync(G->hset, 0xFF, (4 * E + 8) * sizeof(int32_t), s));
      k_build_hset<<<148 * 16, 256, 0, s>>>(G->row, G->col, V, G->hset);
      ND_CUDA_TRY(cudaGetLastError());
      ND_CUDA_TRY(cudaStreamSynchronize(s));
      G->g.hset = G->hset;
    } else {
      G->skipped |= ND_IDX_HSET;
    }
  }
  return ND_OK;
}

int nd_graph_ensure_lines(nd_graph* G, cudaStream_t s) {
  static const bool disabled = getenv("ND_NO_LINES") && getenv("ND_NO_LINES")[0] == '1';
  if (disabled || G->g.unit || G->g.E <= 0) return ND_OK;
  std::lock_guard<std::mutex> lock(g_index_mu);
  if (G->pl || (G->skipped & ND_IDX_LINES)) return ND_OK;
  PrepTimer timer(G);
  const int64_t V = G->g.V;
  int64_t *cnt = nullptr, *first = nullptr;
  ND_CUDA_TRY(nd_alloc(&cnt, V + 1, s));
  ND_CUDA_TRY(nd_alloc(&first, V + 1, s));
  k_line_counts<<<nd_grid(V + 1, 256), 256, 0, s>>>(G->row, V, cnt);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, first, V + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, first, V + 1, s));
    nd_free(tmp, s);
  }
  int64_t n_lines = 0;
  ND_TRY(nd_d2h(&n_lines, first + V, sizeof(int64_t), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  // int32 line offsets; without room the picks use the nbp records
  const double need = (double)n_lines * sizeof(PickLine) + (double)V * 4;
  if (n_lines >= (1ll << 31) || !room_for(need)) {
    G->skipped |= ND_IDX_LINES;
    nd_free(cnt, s); nd_free(first, s);
    return ND_OK;
  }
  ND_CUDA_TRY(cudaMalloc(&G->vline, V * sizeof(int32_t)));
  ND_CUDA_TRY(cudaMalloc(&G->pl, (n_lines > 0 ? n_lines : 1) * sizeof(PickLine)));
  G->bytes += V * 4 + n_lines * (int64_t)sizeof(PickLine);
  G->built |= ND_IDX_LINES;
  k_vline32<<<nd_grid(V, 256), 256, 0, s>>>(first, V, G->vline);
  k_build_lines<<<148 * 16, 256, 0, s>>>(G->row, G->col, G->pre, G->vline, V, G->pl);
  ND_CUDA_TRY(cudaGetLastError());
  nd_free(cnt, s);
  nd_free(first, s);
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  G->g.pl = G->pl;
  G->g.vline = G->vline;
  return ND_OK;
}

extern "C" int nd_graph_build_index(nd_graph* g, int flags, void* stream) {
  if (!g) return ND_ERR_ARG;
  ND_TRY(nd_graph_ensure_index(g, flags & 1, flags & 2, (cudaStream_t)stream));
  if (flags & 4) ND_TRY(nd_graph_ensure_records(g, flags & 1, (cudaStream_t)stream));
  return ND_OK;
}
