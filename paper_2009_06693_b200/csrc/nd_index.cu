// nd_index.cu — exact per-row indexes that shorten the sampler's dependent
// search chains (DESIGN.md §3/§8):
//   * guide tables for the inverse-CDF weighted pick (DeepWalk, PPR, node2vec
//     step 0): guide[lo+j] = upper_bound(prefix[lo:hi], j*(total/deg));
//   * hash sets for node2vec's has_edge(t, u) (graph.py:78-81,
//     _ckernels.pyx:77-87): open addressing, linear probing, load <= 1/2.
// Built once per graph on first use; answers are identical to the binary
// searches they replace (tests/test_gpu_kernels.py::test_index_equivalence).
#include <cub/cub.cuh>

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

int nd_graph_ensure_records(nd_graph* G, int want_tries, cudaStream_t s) {
  static const bool disabled = getenv("ND_NO_PACK") && getenv("ND_NO_PACK")[0] == '1';
  if (disabled) return ND_OK;
  std::lock_guard<std::mutex> lock(g_index_mu);
  const int64_t V = G->g.V, E = G->g.E;
  bool built = false;
  if (!G->vrec && V > 0) {
    built = true;
    ND_CUDA_TRY(cudaMalloc(&G->vrec, V * sizeof(VRec)));
    G->bytes += V * sizeof(VRec);
    k_build_vrec<<<nd_grid(V, 256), 256, 0, s>>>(G->row, G->mx, G->g.unit ? nullptr : G->pre, V,
                                                  G->vrec);
    ND_CUDA_TRY(cudaGetLastError());
    G->g.vrec = G->vrec;
  }
  if (E > 0) {
    NbrW* nw = nullptr;
    NbrP* np_ = nullptr;
    NbrU* nu = nullptr;
    if (G->g.unit) {
      if (!G->nbu) ND_CUDA_TRY(cudaMalloc(&nu, E * sizeof(NbrU)));
    } else {
      if (!G->nbp) ND_CUDA_TRY(cudaMalloc(&np_, E * sizeof(NbrP)));
      if (want_tries && !G->nbw) ND_CUDA_TRY(cudaMalloc(&nw, E * sizeof(NbrW)));
    }
    if (nw || np_ || nu) {
      built = true;
      k_build_nbr<<<nd_grid(E, 256, 148 * 64), 256, 0, s>>>(G->row, G->col, G->w, G->pre, G->mx,
                                                             E, nw, np_, nu);
      ND_CUDA_TRY(cudaGetLastError());
      if (nw) { G->nbw = nw; G->g.nbw = nw; G->bytes += E * sizeof(NbrW); }
      if (np_) { G->nbp = np_; G->g.nbp = np_; G->bytes += E * sizeof(NbrP); }
      if (nu) { G->nbu = nu; G->g.nbu = nu; G->bytes += E * sizeof(NbrU); }
    }
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
  if (want_guide && !G->guide && !G->g.unit && E > 0) {
    // +8 entries: the walker kernels read guide entries as aligned 32-byte chunks
    ND_CUDA_TRY(cudaMalloc(&G->guide, (E + 8) * sizeof(int32_t)));
    G->bytes += E * 4;
    k_build_guide<<<148 * 16, 256, 0, s>>>(G->row, G->pre, V, G->guide);
    ND_CUDA_TRY(cudaGetLastError());
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    G->g.guide = G->guide;
  }
  if (want_hset && !G->hset && E > 0) {
    // +8 slots: the walker kernels read the tables as aligned 32-byte chunks
    ND_CUDA_TRY(cudaMalloc(&G->hset, (4 * E + 8) * sizeof(int32_t)));
    G->bytes += 16 * E;
    ND_CUDA_TRY(cudaMemsetAsync(G->hset, 0xFF, (4 * E + 8) * sizeof(int32_t), s));
    k_build_hset<<<148 * 16, 256, 0, s>>>(G->row, G->col, V, G->hset);
    ND_CUDA_TRY(cudaGetLastError());
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    G->g.hset = G->hset;
  }
  return ND_OK;
}

int nd_graph_ensure_lines(nd_graph* G, cudaStream_t s) {
  static const bool disabled = getenv("ND_NO_LINES") && getenv("ND_NO_LINES")[0] == '1';
  if (disabled || G->g.unit || G->g.E <= 0) return ND_OK;
  std::lock_guard<std::mutex> lock(g_index_mu);
  if (G->pl) return ND_OK;
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
  // int32 line offsets; and the layout is an accelerator, not a requirement:
  // without room for it (plus a margin) the picks use the nbp records
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const double need = (double)n_lines * sizeof(PickLine) + (double)V * 4 + (double)(2ull << 30);
  if (n_lines >= (1ll << 31) || need > (double)fr) {
    nd_free(cnt, s); nd_free(first, s);
    return ND_OK;
  }
  ND_CUDA_TRY(cudaMalloc(&G->vline, V * sizeof(int32_t)));
  ND_CUDA_TRY(cudaMalloc(&G->pl, (n_lines > 0 ? n_lines : 1) * sizeof(PickLine)));
  G->bytes += V * 4 + n_lines * (int64_t)sizeof(PickLine);
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
