// nd_ooc.cu — out-of-core sub-graph shuttling.
//
// A graph larger than the device budget stays in (page-locked) host memory.
// Its vertices are cut into contiguous partitions whose edge slices (int32
// columns, plus the f64 inclusive prefix for weighted graphs) fit half of the
// budget; only the int64 row offsets stay resident.  A run shuttles the
// partitions through two device slice buffers on a copy stream, one ahead of
// the compute stream, and a partition's kernel advances every sample whose
// current transit lies in it:
//   * DeepWalk (chain.py:64-179): a walker keeps stepping while its next
//     vertex stays in the resident partition, then waits for its partition's
//     turn in the next round.  Rounds repeat until every walker is done; each
//     round uploads only partitions that hold a waiting walker.
//   * k-hop (driver.py:203-235, fixed fanouts): per step, every partition
//     holding a parent transit is uploaded once and samples its parents'
//     slots.
// Every draw is keyed on (seed, sample, step, transit_idx, slot) exactly as
// in-core, so the rows equal nd_run_walk / nd_run_individual byte for byte
// whatever the partition schedule (tests/test_gpu_ooc.py).
//   * PPR (unbounded walks, step cap): as DeepWalk, with each step's value
//     appended to a (walker, vertex) log that a stable sort by walker turns
//     into the final rows.
// node2vec's next() reads a second row (has_edge on the previous transit),
// which a single resident partition cannot answer: ND_ERR_APP.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "nd_internal.h"
#include "nd_item.cuh"

using namespace nd;

extern "C" int nd_ooc_graph_destroy(nd_ooc_graph* G);

struct nd_ooc_graph {
  int64_t V = 0, E = 0;
  int unit = 0;
  int64_t* row_d = nullptr;          // resident row offsets [V+1]
  const int64_t* row_h = nullptr;    // host copies (caller-owned)
  const int32_t* col_h = nullptr;
  const double* pre_h = nullptr;     // null for unit-weight graphs
  bool reg_col = false, reg_pre = false;
  const int32_t* col_map = nullptr;  // device views of the registered host arrays (zero copy)
  const double* pre_map = nullptr;
  std::vector<int64_t> vcut;         // partition p = vertices [vcut[p], vcut[p+1])
  int64_t* vcut_d = nullptr;
  int64_t slice_cap = 0;             // edges per slice buffer
  int32_t* col_d[2] = {};
  double* pre_d[2] = {};
  int64_t bytes_shuttled = 0;        // host->device slice bytes over the graph's life
  int64_t uploads = 0;
  int64_t parts() const { return (int64_t)vcut.size() - 1; }
  int64_t e0(int64_t p) const { return row_h[vcut[p]]; }
  int64_t e1(int64_t p) const { return row_h[vcut[p + 1]]; }
};

namespace {

__device__ __forceinline__ int part_of(const int64_t* __restrict__ vcut, int P, int64_t v) {
  int lo = 0, hi = P;  // vcut[lo] <= v < vcut[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(vcut + mid) <= v) lo = mid; else hi = mid;
  }
  return lo;
}

// walkers waiting per partition (live walkers: step < L)
__global__ void k_ooc_walk_hist(const int32_t* __restrict__ cur, const int32_t* __restrict__ stp,
                                int64_t n, int L, const int64_t* __restrict__ vcut, int P,
                                unsigned long long* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (stp[i] < L) atomicAdd(cnt + part_of(vcut, P, cur[i]), 1ull);
}

// DeepWalk steps of the walkers whose current vertex is in [v0, v1), the
// partition's columns / prefix at colp / prep (edge ebase = index 0)
__global__ void k_ooc_walk(const int64_t* __restrict__ row, const int32_t* __restrict__ colp,
                           const double* __restrict__ prep, int64_t ebase, int64_t v0, int64_t v1,
                           int unit, int32_t* __restrict__ cur, int32_t* __restrict__ stp,
                           int64_t* __restrict__ clen, int32_t* __restrict__ out, int L, int64_t n,
                           uint64_t seed, int64_t sample_lo, unsigned long long* __restrict__ ctr) {
  unsigned long long bytes = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int s = stp[i];
    if (s >= L) continue;
    int64_t v = cur[i];
    if (v < v0 || v >= v1) continue;
    const uint64_t ik = key_item((uint64_t)(sample_lo + i), 0, 0);  // chain.py:52-54
    while (true) {
      const int64_t lo = __ldg(row + v), deg = __ldg(row + v + 1) - lo;
      if (deg <= 0) {  // dead end: NULL at this step ends the walk (core.py:192)
        clen[i] = s + 1;
        s = L;
        break;
      }
      const SRow r{colp + (lo - ebase), unit ? nullptr : prep + (lo - ebase), nullptr};
      const double u01 = to_unit(draw_u64(key_base(seed, (uint64_t)s, 0, 0), ik));
      const int64_t nb = r.c(pick_rel(r, unit, deg, u01));
      bytes += 2 * SECTOR + 8 + (unit ? 0 : SECTOR * search_sectors(deg));
      out[i * (int64_t)L + s] = (int32_t)nb;
      if (++s == L) {
        clen[i] = L;
        break;
      }
      v = nb;
      if (v < v0 || v >= v1) break;  // waits for its partition's turn
    }
    stp[i] = s;
    cur[i] = (int32_t)v;
  }
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_down_sync(0xffffffffu, bytes, o);
  if ((threadIdx.x & 31) == 0 && bytes) atomicAdd(ctr, bytes);
}

// final rows of the walk window: roots, then the walk's non-NULL prefix
__global__ void k_ooc_walk_lens(const int64_t* __restrict__ clen, const int32_t* __restrict__ out,
                                int L, int64_t n, int64_t* __restrict__ flen) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { flen[n] = 0; continue; }
    const int64_t c = clen[i];
    const int64_t nnz = c > 0 && out[i * (int64_t)L + c - 1] < 0 ? c - 1 : c;
    flen[i] = 1 + nnz;
  }
}

__global__ void k_ooc_walk_emit(const int32_t* __restrict__ roots, const int32_t* __restrict__ out,
                                int L, int64_t n, const int64_t* __restrict__ off,
                                int32_t* __restrict__ ids, int64_t* __restrict__ roots_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const int64_t o = off[i], len = off[i + 1] - o;
    if (lane == 0) {
      ids[o] = roots[i];
      roots_out[i] = roots[i];
    }
    for (int64_t s = lane; s + 1 < len; s += 32) ids[o + 1 + s] = out[i * (int64_t)L + s];
  }
}

// PPR steps (apps.py:47-49: draw 0 < term ends the walk with NULL, else
// draw 1 picks) of the walkers in [v0, v1).  Walks have no length bound, so
// each step's value is appended to a log of (walker << 32 | vertex) words; a
// walker stops where the log is full (it resumes there next round).  nnz[i]
// counts its logged values; clen[i] is set when it ends (NULL included).
__global__ void k_ooc_ppr(const int64_t* __restrict__ row, const int32_t* __restrict__ colp,
                          const double* __restrict__ prep, int64_t ebase, int64_t v0, int64_t v1,
                          int unit, double term, int32_t* __restrict__ cur,
                          int32_t* __restrict__ stp, int64_t* __restrict__ clen,
                          int32_t* __restrict__ nnz, uint64_t* __restrict__ log,
                          unsigned long long* __restrict__ log_n, int64_t log_cap, int cap,
                          int64_t n, uint64_t seed, int64_t sample_lo,
                          unsigned long long* __restrict__ ctr) {
  unsigned long long bytes = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int s = stp[i];
    if (s >= cap) continue;
    int64_t v = cur[i];
    if (v < v0 || v >= v1) continue;
    const uint64_t ik = key_item((uint64_t)(sample_lo + i), 0, 0);  // chain.py:52-54
    int k = nnz[i];
    while (true) {
      const uint64_t base0 = key_base(seed, (uint64_t)s, 0, 0);
      const int64_t lo = __ldg(row + v), deg = __ldg(row + v + 1) - lo;
      if (deg <= 0 || to_unit(draw_u64(base0, ik)) < term) {  // NULL: the walk ends
        clen[i] = s + 1;
        s = cap;
        break;
      }
      const unsigned long long slot = atomicAdd(log_n, 1ull);
      if ((int64_t)slot >= log_cap) break;  // log full: resume here next round
      const SRow r{colp + (lo - ebase), unit ? nullptr : prep + (lo - ebase), nullptr};
      const int64_t nb = r.c(pick_rel(r, unit, deg, to_unit(draw_u64(base0 + C_DRAW, ik))));
      bytes += 2 * SECTOR + 8 + (unit ? 0 : SECTOR * search_sectors(deg));
      log[slot] = ((uint64_t)i << 32) | (uint32_t)nb;
      k++;
      if (++s == cap) {  // the step cap (core.py:37): no NULL
        clen[i] = cap;
        v = nb;
        break;
      }
      v = nb;
      if (v < v0 || v >= v1) break;
    }
    nnz[i] = k;
    stp[i] = s;
    cur[i] = (int32_t)v;
  }
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_down_sync(0xffffffffu, bytes, o);
  if ((threadIdx.x & 31) == 0 && bytes) atomicAdd(ctr, bytes);
}

__global__ void k_ooc_flen(const int32_t* __restrict__ nnz, int64_t n, int64_t* __restrict__ flen) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    flen[i] = i < n ? 1 + nnz[i] : 0;
}

// the walker-sorted log into the final rows: entry k of walker w (its
// (k - logoff[w])-th step) after w's root
__global__ void k_ooc_log_emit(const uint64_t* __restrict__ sorted, int64_t m,
                               const int64_t* __restrict__ off, int32_t* __restrict__ ids) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = sorted[k];
    const int64_t w = (int64_t)(e >> 32);
    // off[w] - w = values logged by walkers before w (each row holds 1 root)
    const int64_t j = k - (off[w] - w);
    ids[off[w] + 1 + j] = (int32_t)(uint32_t)e;
  }
}

__global__ void k_ooc_roots_emit(const int32_t* __restrict__ roots, int64_t n,
                                 const int64_t* __restrict__ off, int32_t* __restrict__ ids,
                                 int64_t* __restrict__ roots_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ids[off[i]] = roots[i];
    roots_out[i] = roots[i];
  }
}

// transit_idx of every parent slot: rank among the sample block's non-NULL
// entries (core.py:97,180-181); nn[i] = non-NULL parents of sample i
__global__ void k_ooc_rank(const int32_t* __restrict__ blk, int64_t n, int64_t B,
                           int32_t* __restrict__ rank, int64_t* __restrict__ nn) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    int32_t base = 0;
    for (int64_t p0 = 0; p0 < B; p0 += 32) {
      const int64_t p = p0 + lane;
      const bool ok = p < B && blk[i * B + p] >= 0;
      const unsigned mk = __ballot_sync(0xffffffffu, ok);
      if (p < B) rank[i * B + p] = ok ? base + __popc(mk & ((1u << lane) - 1)) : -1;
      base += __popc(mk);
    }
    if (lane == 0) nn[i] = base;
  }
}

__global__ void k_ooc_parent_hist(const int32_t* __restrict__ blk, int64_t N,
                                  const int64_t* __restrict__ vcut, int P,
                                  unsigned long long* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    if (blk[i] >= 0) atomicAdd(cnt + part_of(vcut, P, blk[i]), 1ull);
}

// one k-hop step over the parents in [v0, v1): slot `slot` of parent ip,
// u % deg over the resident partition's columns (_ckernels.pyx:212-223)
__global__ void k_ooc_khop(const int64_t* __restrict__ row, const int32_t* __restrict__ colp,
                           int64_t ebase, int64_t v0, int64_t v1, const int32_t* __restrict__ prev,
                           const int32_t* __restrict__ rank, int64_t N, FastDiv Bp, FastDiv m,
                           uint64_t base0, int64_t sample_lo, int32_t* __restrict__ next,
                           unsigned long long* __restrict__ ctr) {
  unsigned long long bytes = 0;
  const int64_t items = N * m.d;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < items;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t ip = m.div((uint32_t)q), slot = (uint32_t)q - ip * m.d;
    const int64_t v = prev[ip];
    if (v < v0 || v >= v1) continue;  // NULL parents (-1) and other partitions
    if (slot == 0) bytes += SECTOR + 8;
    const int64_t lo = __ldg(row + v), deg = __ldg(row + v + 1) - lo;
    if (deg <= 0) continue;           // NULL slots (prefilled)
    const uint32_t i = Bp.div(ip);
    const uint64_t ik = key_item((uint64_t)(sample_lo + i), (uint64_t)rank[ip], slot);
    const uint64_t k = mod_u64(draw_u64(base0, ik), (uint64_t)deg);
    next[q] = colp[lo - ebase + (int64_t)k];
    bytes += SECTOR + 8;
  }
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_down_sync(0xffffffffu, bytes, o);
  if ((threadIdx.x & 31) == 0 && bytes) atomicAdd(ctr, bytes);
}

struct OocSteps {
  const int32_t* blk[8];
  int64_t B[8];
  int n_steps;
};

// per-sample non-NULL slots over every step block
__global__ void k_ooc_khop_lens(OocSteps S, int64_t n, int64_t R, int64_t* __restrict__ flen) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i <= n; i += nw) {
    if (i == n) { if (lane == 0) flen[n] = 0; continue; }
    int64_t c = 0;
    for (int s = 0; s < S.n_steps; s++)
      for (int64_t p = lane; p < S.B[s]; p += 32) c += S.blk[s][i * S.B[s] + p] >= 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if (lane == 0) flen[i] = R + c;
  }
}

// final rows: roots, then each step's non-NULL slots in block order
__global__ void k_ooc_khop_emit(OocSteps S, const int32_t* __restrict__ roots, int64_t n, int64_t R,
                                const int64_t* __restrict__ off, int32_t* __restrict__ ids,
                                int64_t* __restrict__ roots_out, int64_t* __restrict__ roots_off) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    int32_t* dst = ids + off[i];
    for (int64_t r = lane; r < R; r += 32) {
      dst[r] = roots[i * R + r];
      roots_out[i * R + r] = roots[i * R + r];
    }
    if (lane == 0) {
      roots_off[i] = i * R;
      if (i == n - 1) roots_off[n] = n * R;
    }
    int64_t pos = R;
    for (int s = 0; s < S.n_steps; s++) {
      const int64_t B = S.B[s];
      for (int64_t p0 = 0; p0 < B; p0 += 32) {
        const int64_t p = p0 + lane;
        const int32_t v = p < B ? S.blk[s][i * B + p] : -1;
        const unsigned mk = __ballot_sync(0xffffffffu, v >= 0);
        if (v >= 0) dst[pos + __popc(mk & ((1u << lane) - 1))] = v;
        pos += __popc(mk);
      }
    }
  }
}

// step rows (F_STEP_VALS32): the slots of real pairs of step s, sample-major
__global__ void k_ooc_step_vals(const int32_t* __restrict__ next, const int32_t* __restrict__ rank,
                                int64_t n, int64_t Bp, int64_t m, const int64_t* __restrict__ soff,
                                int32_t* __restrict__ vals) {
  const int64_t total = n * Bp * m;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ip = q / m, slot = q - ip * m;
    const int32_t r = rank[ip];
    if (r < 0) continue;
    vals[soff[ip / Bp] + (int64_t)r * m + slot] = next[q];
  }
}

__global__ void k_ooc_step_counts(const int64_t* __restrict__ nn, int64_t n, int64_t m,
                                  int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = nn[i] * m;
}

__global__ void k_iota_off(int64_t* __restrict__ off, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    off[i] = i;
}

__global__ void k_ooc_narrow(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

// Shuttle: partition p's slice into buffer b on the copy stream, ordered
// after the compute work that last read buffer b; the compute stream waits
// for the copy before the partition's kernel.
struct Shuttle {
  nd_ooc_graph* G;
  cudaStream_t s = nullptr, cs = nullptr;
  cudaEvent_t copied[2] = {}, freed[2] = {};
  int next_buf = 0;
  int init() {
    ND_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int b = 0; b < 2; b++) {
      ND_CUDA_TRY(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
      ND_CUDA_TRY(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
      ND_CUDA_TRY(cudaEventRecord(freed[b], s));
    }
    return ND_OK;
  }
  // issue the upload of partition p; returns its buffer
  int upload(int64_t p, int& b) {
    b = next_buf;
    next_buf ^= 1;
    const int64_t a = G->e0(p), e = G->e1(p) - a;
    ND_CUDA_TRY(cudaStreamWaitEvent(cs, freed[b], 0));
    if (e > 0) {
      ND_CUDA_TRY(cudaMemcpyAsync(G->col_d[b], G->col_h + a, e * 4, cudaMemcpyHostToDevice, cs));
      if (!G->unit)
        ND_CUDA_TRY(cudaMemcpyAsync(G->pre_d[b], G->pre_h + a, e * 8, cudaMemcpyHostToDevice, cs));
    }
    G->bytes_shuttled += e * (G->unit ? 4 : 12);
    G->uploads++;
    ND_CUDA_TRY(cudaEventRecord(copied[b], cs));
    return ND_OK;
  }
  int use(int b) { ND_CUDA_TRY(cudaStreamWaitEvent(s, copied[b], 0)); return ND_OK; }
  int release(int b) { ND_CUDA_TRY(cudaEventRecord(freed[b], s)); return ND_OK; }
  void destroy() {  // idempotent; also run by the destructor on early returns
    if (cs) cudaStreamSynchronize(cs);
    for (int b = 0; b < 2; b++) {
      if (copied[b]) cudaEventDestroy(copied[b]);
      if (freed[b]) cudaEventDestroy(freed[b]);
      copied[b] = freed[b] = nullptr;
    }
    if (cs) cudaStreamDestroy(cs);
    cs = nullptr;
  }
  ~Shuttle() { destroy(); }
};

// Few walkers left (the geometric tail of PPR, the last DeepWalk stragglers):
// uploading whole partitions for them costs more than reading their rows
// straight from the page-locked host arrays over the link (zero copy), so
// below this many waiting walkers one launch over the whole vertex range
// finishes them (ND_OOC_ZC: the threshold; 0 disables).
static int64_t zero_copy_threshold(int64_t n) {
  static const int64_t env = getenv("ND_OOC_ZC") ? atoll(getenv("ND_OOC_ZC")) : -1;
  if (env >= 0) return env;
  return std::max<int64_t>(4096, n / 32);
}

// partitions with work, in order, from a device histogram
static int busy_parts(const unsigned long long* cnt_d, int64_t P, cudaStream_t s,
                      std::vector<int64_t>& busy, int64_t* total) {
  std::vector<unsigned long long> h(P);
  ND_CUDA_TRY(cudaMemcpyAsync(h.data(), cnt_d, P * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  busy.clear();
  *total = 0;
  for (int64_t p = 0; p < P; p++)
    if (h[p]) { busy.push_back(p); *total += (int64_t)h[p]; }
  return ND_OK;
}

}  // namespace

extern "C" int nd_ooc_graph_create(const int64_t* row_offsets, const int32_t* col,
                                   const double* prefix, int64_t n_vertices, int64_t n_edges,
                                   int64_t device_budget_bytes, int register_host, void* stream,
                                   nd_ooc_graph** out) {
  NvtxRange nvtx("nd_ooc_graph_create");
  if (!row_offsets || !out || n_vertices <= 0 || n_edges < 0 || n_vertices >= (1ll << 31) ||
      (n_edges > 0 && !col))
    return ND_ERR_ARG;
  if (row_offsets[0] != 0 || row_offsets[n_vertices] != n_edges) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  auto* G = new nd_ooc_graph();
  G->V = n_vertices;
  G->E = n_edges;
  G->unit = prefix == nullptr;
  G->row_h = row_offsets;
  G->col_h = col;
  G->pre_h = prefix;
  const int64_t bpe = G->unit ? 4 : 12;
  const int64_t resident = (n_vertices + 1) * 8;
  // two slice buffers share what the resident offsets leave of the budget
  G->slice_cap = (device_budget_bytes - resident) / (2 * bpe);
  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n_vertices; v++)
    maxdeg = std::max(maxdeg, row_offsets[v + 1] - row_offsets[v]);
  if (G->slice_cap < std::max<int64_t>(maxdeg, 1)) {
    delete G;
    nd_set_last_error("device budget below two slices of the largest row", __FILE__, __LINE__);
    return ND_ERR_NOMEM;
  }
  // contiguous vertex ranges, each slice <= slice_cap edges
  G->vcut.push_back(0);
  int64_t start_e = 0;
  for (int64_t v = 0; v < n_vertices; v++)
    if (row_offsets[v + 1] - start_e > G->slice_cap) {
      G->vcut.push_back(v);
      start_e = row_offsets[v];
    }
  G->vcut.push_back(n_vertices);
  const int64_t cap = std::min<int64_t>(G->slice_cap, std::max<int64_t>(n_edges, 1));
  int rc = ND_OK;
  auto fail = [&](cudaError_t e) {
    nd_set_last_error(cudaGetErrorString(e), __FILE__, __LINE__);
    rc = e == cudaErrorMemoryAllocation ? ND_ERR_NOMEM : ND_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&G->row_d, (n_vertices + 1) * 8)) != cudaSuccess) fail(e);
  if (rc == ND_OK && (e = cudaMalloc(&G->vcut_d, G->vcut.size() * 8)) != cudaSuccess) fail(e);
  for (int b = 0; b < 2 && rc == ND_OK; b++) {
    if ((e = cudaMalloc(&G->col_d[b], cap * 4)) != cudaSuccess) fail(e);
    if (rc == ND_OK && !G->unit && (e = cudaMalloc(&G->pre_d[b], cap * 8)) != cudaSuccess) fail(e);
  }
  if (rc == ND_OK && register_host && n_edges > 0) {
    // page-lock the host slices so uploads run at full link speed, async
    // (memory the caller already page-locked is used as is)
    auto pinned = [](const void* p) {
      cudaPointerAttributes at{};
      const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
      cudaGetLastError();
      return ok;
    };
    if (!pinned(col) &&
        cudaHostRegister((void*)col, n_edges * 4, cudaHostRegisterMapped | cudaHostRegisterReadOnly) ==
            cudaSuccess)
      G->reg_col = true;
    cudaGetLastError();  // not registrable: pageable copies still work
    if (!G->unit && !pinned(prefix) &&
        cudaHostRegister((void*)prefix, n_edges * 8,
                         cudaHostRegisterMapped | cudaHostRegisterReadOnly) == cudaSuccess)
      G->reg_pre = true;
    cudaGetLastError();
  }
  if (register_host && n_edges > 0) {  // zero-copy views for sparse late rounds
    void* dc = nullptr;
    void* dp = nullptr;
    cudaPointerAttributes ac{}, ap{};
    const bool cm = cudaPointerGetAttributes(&ac, col) == cudaSuccess && ac.type == cudaMemoryTypeHost;
    const bool pm = G->unit || (cudaPointerGetAttributes(&ap, prefix) == cudaSuccess &&
                                ap.type == cudaMemoryTypeHost);
    cudaGetLastError();
    if (cm && pm && cudaHostGetDevicePointer(&dc, (void*)col, 0) == cudaSuccess &&
        (G->unit || cudaHostGetDevicePointer(&dp, (void*)prefix, 0) == cudaSuccess)) {
      G->col_map = static_cast<const int32_t*>(dc);
      G->pre_map = static_cast<const double*>(dp);
    }
    cudaGetLastError();
  }
  if (rc == ND_OK &&
      (e = cudaMemcpyAsync(G->row_d, row_offsets, (n_vertices + 1) * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    fail(e);
  if (rc == ND_OK && (e = cudaMemcpyAsync(G->vcut_d, G->vcut.data(), G->vcut.size() * 8,
                                          cudaMemcpyHostToDevice, s)) != cudaSuccess)
    fail(e);
  if (rc == ND_OK && (e = cudaStreamSynchronize(s)) != cudaSuccess) fail(e);
  if (rc != ND_OK) {
    nd_ooc_graph_destroy(G);
    return rc;
  }
  *out = G;
  return ND_OK;
}

extern "C" int nd_ooc_graph_destroy(nd_ooc_graph* G) {
  if (!G) return ND_OK;
  if (G->reg_col) cudaHostUnregister((void*)G->col_h);
  if (G->reg_pre) cudaHostUnregister((void*)G->pre_h);
  cudaFree(G->row_d);
  cudaFree(G->vcut_d);
  for (int b = 0; b < 2; b++) {
    cudaFree(G->col_d[b]);
    cudaFree(G->pre_d[b]);
  }
  delete G;
  return ND_OK;
}

extern "C" int nd_ooc_graph_info(const nd_ooc_graph* G, int64_t* n_parts, int64_t* slice_edges,
                                 int64_t* device_bytes, int64_t* bytes_shuttled, int64_t* uploads) {
  if (!G) return ND_ERR_ARG;
  if (n_parts) *n_parts = G->parts();
  if (slice_edges) *slice_edges = G->slice_cap;
  if (device_bytes)
    *device_bytes = (G->V + 1) * 8 + 2 * std::min<int64_t>(G->slice_cap, std::max<int64_t>(G->E, 1)) *
                                         (G->unit ? 4 : 12);
  if (bytes_shuttled) *bytes_shuttled = G->bytes_shuttled;
  if (uploads) *uploads = G->uploads;
  return ND_OK;
}

extern "C" int nd_ooc_graph_parts(const nd_ooc_graph* G, int64_t* vcut, int64_t n_max) {
  if (!G || !vcut) return ND_ERR_ARG;
  for (int64_t p = 0; p < (int64_t)G->vcut.size() && p < n_max; p++) vcut[p] = G->vcut[p];
  return ND_OK;
}

// PPR over a shuttled graph: rounds over the partitions holding live walkers
// until every walk has ended (NULL) or reached `cap` steps (the run loop's
// step cap, core.py:37); values go to a growing log, sorted by walker
// (stable: each walker's values stay in step order) into the final rows.
static int run_ppr_ooc(nd_ooc_graph* G, double term, int64_t sample_lo, int64_t n,
                       const int64_t* roots, uint64_t seed, int64_t cap_steps, cudaStream_t s,
                       nd_result** out) {
  if (cap_steps < 1 || cap_steps >= (1ll << 30)) return ND_ERR_ARG;
  const int cap = (int)cap_steps;
  const int P = (int)G->parts();
  DevGraph gv;
  gv.V = G->V;
  int32_t *roots32 = nullptr, *cur = nullptr, *stp = nullptr, *nnz = nullptr;
  int64_t* clen = nullptr;
  uint64_t* log = nullptr;
  unsigned long long *hist = nullptr, *ctr = nullptr, *log_n = nullptr;
  int64_t log_cap = std::max<int64_t>(n * 32, 1 << 20);
  ND_CUDA_TRY(nd_alloc(&roots32, std::max<int64_t>(n, 1), s));
  ND_CUDA_TRY(nd_alloc(&cur, std::max<int64_t>(n, 1), s));
  ND_CUDA_TRY(nd_alloc(&stp, std::max<int64_t>(n, 1), s));
  ND_CUDA_TRY(nd_alloc(&nnz, std::max<int64_t>(n, 1), s));
  ND_CUDA_TRY(nd_alloc(&clen, std::max<int64_t>(n, 1), s));
  ND_CUDA_TRY(nd_alloc(&log, log_cap, s));
  ND_CUDA_TRY(nd_alloc(&hist, P, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 1, s));
  ND_CUDA_TRY(nd_alloc(&log_n, 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, s));
  ND_CUDA_TRY(cudaMemsetAsync(log_n, 0, 8, s));
  if (roots) {
    if (n) k_ooc_narrow<<<nd_grid(n, 256), 256, 0, s>>>(roots, n, roots32);
  } else {
    ND_TRY(nd_uniform_roots_i32(gv, 1, seed, sample_lo, n, roots32, s));
  }
  if (n) ND_CUDA_TRY(cudaMemcpyAsync(cur, roots32, n * 4, cudaMemcpyDeviceToDevice, s));
  ND_CUDA_TRY(cudaMemsetAsync(stp, 0, std::max<int64_t>(n, 1) * 4, s));
  ND_CUDA_TRY(cudaMemsetAsync(nnz, 0, std::max<int64_t>(n, 1) * 4, s));
  ND_CUDA_TRY(cudaMemsetAsync(clen, 0, std::max<int64_t>(n, 1) * 8, s));
  Shuttle sh{G, s, nullptr};
  ND_TRY(sh.init());
  std::vector<int64_t> busy;
  int64_t waiting = 0, rounds = 0;
  unsigned long long* h = reinterpret_cast<unsigned long long*>(nd_pinned_scratch());
  while (n > 0) {
    ND_CUDA_TRY(cudaMemsetAsync(hist, 0, P * 8, s));
    k_ooc_walk_hist<<<nd_grid(n, 256), 256, 0, s>>>(cur, stp, n, cap, G->vcut_d, P, hist);
    ND_TRY(busy_parts(hist, P, s, busy, &waiting));
    if (waiting == 0) break;
    rounds++;
    if (G->col_map && waiting <= zero_copy_threshold(n)) {  // the geometric tail, zero copy
      k_ooc_ppr<<<nd_grid(n, 256, 148 * 16), 256, 0, s>>>(
          G->row_d, G->col_map, G->pre_map, 0, 0, G->V, G->unit, term, cur, stp, clen, nnz, log,
          log_n, log_cap, cap, n, seed, sample_lo, ctr);
      ND_CUDA_TRY(cudaGetLastError());
    } else {
      int b = 0, nb = 0;
      ND_TRY(sh.upload(busy[0], b));
      for (size_t k = 0; k < busy.size(); k++) {
        const int64_t p = busy[k];
        if (k + 1 < busy.size()) ND_TRY(sh.upload(busy[k + 1], nb));
        ND_TRY(sh.use(b));
        k_ooc_ppr<<<nd_grid(n, 256, 148 * 16), 256, 0, s>>>(
            G->row_d, G->col_d[b], G->pre_d[b], G->e0(p), G->vcut[p], G->vcut[p + 1], G->unit,
            term, cur, stp, clen, nnz, log, log_n, log_cap, cap, n, seed, sample_lo, ctr);
        ND_CUDA_TRY(cudaGetLastError());
        ND_TRY(sh.release(b));
        b = nb;
      }
    }
    // a full log: grow it (the walkers that found no slot resume next round)
    ND_TRY(nd_d2h(h, log_n, 8, s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    if ((int64_t)h[0] >= log_cap) {
      const int64_t valid = log_cap;
      const int64_t ncap = log_cap * 2;
      uint64_t* nl = nullptr;
      ND_CUDA_TRY(nd_alloc(&nl, ncap, s));
      ND_CUDA_TRY(cudaMemcpyAsync(nl, log, valid * 8, cudaMemcpyDeviceToDevice, s));
      nd_free(log, s);
      log = nl;
      log_cap = ncap;
      const unsigned long long v = (unsigned long long)valid;
      ND_CUDA_TRY(cudaMemcpyAsync(log_n, &v, 8, cudaMemcpyHostToDevice, s));
      ND_CUDA_TRY(cudaStreamSynchronize(s));
    }
  }
  sh.destroy();
  // the log sorted by walker (stable), the final rows
  ND_TRY(nd_d2h(h, log_n, 8, s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t m = std::min<int64_t>((int64_t)h[0], log_cap);
  int wbits = 1;
  while ((1ll << wbits) < std::max<int64_t>(n, 2)) wbits++;
  uint64_t* sorted = nullptr;
  int64_t *flen = nullptr, *final_off = nullptr, *roots_out = nullptr, *roots_off = nullptr;
  ND_CUDA_TRY(nd_alloc(&sorted, std::max<int64_t>(m, 1), s));
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, std::max<int64_t>(n, 1), s));
  ND_CUDA_TRY(nd_alloc(&roots_off, n + 1, s));
  {
    size_t t1 = 0, t2 = 0;
    if (m) cub::DeviceRadixSort::SortKeys(nullptr, t1, log, sorted, m, 32, 32 + wbits, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, flen, final_off, n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, std::max(t1, t2), s));
    if (m) ND_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, t1, log, sorted, m, 32, 32 + wbits, s));
    k_ooc_flen<<<nd_grid(n + 1, 256), 256, 0, s>>>(nnz, n, flen);
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, t2, flen, final_off, n + 1, s));
    nd_free(tmp, s);
  }
  int64_t* mx = nullptr;
  ND_CUDA_TRY(nd_alloc(&mx, 1, s));
  {
    size_t tb = 0;
    cub::DeviceReduce::Max(nullptr, tb, clen, mx, std::max<int64_t>(n, 1), s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    if (n) ND_CUDA_TRY(cub::DeviceReduce::Max(tmp, tb, clen, mx, n, s));
    else ND_CUDA_TRY(cudaMemsetAsync(mx, 0, 8, s));
    nd_free(tmp, s);
  }
  int64_t* hh = nd_pinned_scratch();
  ND_TRY(nd_d2h(hh, final_off + n, 8, s));
  ND_TRY(nd_d2h(hh + 1, mx, 8, s));
  ND_TRY(nd_d2h(hh + 2, ctr, 8, s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t total = hh[0], n_steps = hh[1], slot_bytes = hh[2];
  int32_t* final_ids = nullptr;
  ND_CUDA_TRY(nd_alloc(&final_ids, std::max<int64_t>(total, 1), s));
  if (n) k_ooc_roots_emit<<<nd_grid(n, 256), 256, 0, s>>>(roots32, n, final_off, final_ids, roots_out);
  if (m) k_ooc_log_emit<<<nd_grid(m, 256, 148 * 64), 256, 0, s>>>(sorted, m, final_off, final_ids);
  k_iota_off<<<nd_grid(n + 1, 256), 256, 0, s>>>(roots_off, n + 1);
  ND_CUDA_TRY(cudaGetLastError());
  nd_result* res = new nd_result();
  res->stream = s;
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n);
  res->set(ND_F_ROOTS_OFF, roots_off, n + 1);
  res->set(ND_F_CHAIN_LEN, clen, n);
  res->counters[NDC_SLOT_BYTES] = slot_bytes;
  res->counters[NDC_STEPS] = rounds;
  *out = res;
  nd_free(roots32, s); nd_free(cur, s); nd_free(stp, s); nd_free(nnz, s); nd_free(log, s);
  nd_free(sorted, s); nd_free(hist, s); nd_free(ctr, s); nd_free(log_n, s); nd_free(flen, s);
  nd_free(mx, s);
  return ND_OK;
}

extern "C" int nd_run_walk_ooc(nd_ooc_graph* G, int app_code, const double* host_params,
                               int64_t n_params, int64_t sample_lo, int64_t n, const int64_t* roots,
                               uint64_t seed, int64_t steps, void* stream, nd_result** out) {
  NvtxRange nvtx("nd_run_walk_ooc");
  if (!G || !out || n < 0 || sample_lo < 0 || n >= (1ll << 31) || steps < 0 || steps >= (1 << 20))
    return ND_ERR_ARG;
  if (app_code == ND_PPR) {
    if (!host_params || n_params < 1) return ND_ERR_ARG;
    return run_ppr_ooc(G, host_params[0], sample_lo, n, roots, seed, steps, (cudaStream_t)stream, out);
  }
  if (app_code != ND_DEEPWALK) return ND_ERR_APP;  // see the file comment
  (void)host_params;
  (void)n_params;
  cudaStream_t s = (cudaStream_t)stream;
  const int L = (int)steps;
  const int P = (int)G->parts();
  DevGraph gv;
  gv.V = G->V;
  int32_t *roots32 = nullptr, *cur = nullptr, *stp = nullptr, *win = nullptr;
  int64_t* clen = nullptr;
  unsigned long long *hist = nullptr, *ctr = nullptr;
  ND_CUDA_TRY(nd_alloc(&roots32, n, s));
  ND_CUDA_TRY(nd_alloc(&cur, n, s));
  ND_CUDA_TRY(nd_alloc(&stp, n, s));
  ND_CUDA_TRY(nd_alloc(&clen, n, s));
  ND_CUDA_TRY(nd_alloc(&win, (int64_t)n * std::max(L, 1), s));
  ND_CUDA_TRY(nd_alloc(&hist, P, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, s));
  if (roots) {
    if (n) k_ooc_narrow<<<nd_grid(n, 256), 256, 0, s>>>(roots, n, roots32);
  } else {
    ND_TRY(nd_uniform_roots_i32(gv, 1, seed, sample_lo, n, roots32, s));
  }
  if (n) ND_CUDA_TRY(cudaMemcpyAsync(cur, roots32, n * 4, cudaMemcpyDeviceToDevice, s));
  ND_CUDA_TRY(cudaMemsetAsync(stp, 0, n * 4, s));
  ND_CUDA_TRY(cudaMemsetAsync(clen, 0, n * 8, s));
  ND_CUDA_TRY(cudaMemsetAsync(win, 0xFF, (int64_t)n * std::max(L, 1) * 4, s));
  if (L == 0) ND_CUDA_TRY(cudaMemsetAsync(stp, 0x7F, n * 4, s));  // nothing to walk
  Shuttle sh{G, s, nullptr};
  ND_TRY(sh.init());
  std::vector<int64_t> busy;
  int64_t waiting = 0, rounds = 0;
  while (n > 0 && L > 0) {
    ND_CUDA_TRY(cudaMemsetAsync(hist, 0, P * 8, s));
    k_ooc_walk_hist<<<nd_grid(n, 256), 256, 0, s>>>(cur, stp, n, L, G->vcut_d, P, hist);
    ND_TRY(busy_parts(hist, P, s, busy, &waiting));
    if (waiting == 0) break;
    rounds++;
    if (G->col_map && waiting <= zero_copy_threshold(n)) {  // the stragglers, zero copy
      k_ooc_walk<<<nd_grid(n, 256, 148 * 16), 256, 0, s>>>(
          G->row_d, G->col_map, G->pre_map, 0, 0, G->V, G->unit, cur, stp, clen, win, L, n, seed,
          sample_lo, ctr);
      ND_CUDA_TRY(cudaGetLastError());
      continue;
    }
    int b = 0, nb = 0;
    ND_TRY(sh.upload(busy[0], b));
    for (size_t k = 0; k < busy.size(); k++) {
      const int64_t p = busy[k];
      if (k + 1 < busy.size()) ND_TRY(sh.upload(busy[k + 1], nb));  // next slice in flight
      ND_TRY(sh.use(b));
      k_ooc_walk<<<nd_grid(n, 256, 148 * 16), 256, 0, s>>>(
          G->row_d, G->col_d[b], G->pre_d[b], G->e0(p), G->vcut[p], G->vcut[p + 1], G->unit, cur,
          stp, clen, win, L, n, seed, sample_lo, ctr);
      ND_CUDA_TRY(cudaGetLastError());
      ND_TRY(sh.release(b));
      b = nb;
    }
  }
  sh.destroy();
  // final rows
  int64_t *flen = nullptr, *final_off = nullptr, *roots_out = nullptr, *roots_off = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, n, s));
  ND_CUDA_TRY(nd_alloc(&roots_off, n + 1, s));
  k_ooc_walk_lens<<<nd_grid(n + 1, 256), 256, 0, s>>>(clen, win, std::max(L, 1), n, flen);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flen, final_off, n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flen, final_off, n + 1, s));
    int64_t* mx = nullptr;
    size_t tb2 = 0;
    ND_CUDA_TRY(nd_alloc(&mx, 1, s));
    cub::DeviceReduce::Max(nullptr, tb2, clen, mx, n, s);
    void* tmp2 = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp2, tb2, s));
    if (n) ND_CUDA_TRY(cub::DeviceReduce::Max(tmp2, tb2, clen, mx, n, s));
    else ND_CUDA_TRY(cudaMemsetAsync(mx, 0, 8, s));
    int64_t* h = nd_pinned_scratch();
    ND_TRY(nd_d2h(h, final_off + n, 8, s));
    ND_TRY(nd_d2h(h + 1, mx, 8, s));
    ND_TRY(nd_d2h(h + 2, ctr, 8, s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    nd_free(tmp, s); nd_free(tmp2, s); nd_free(mx, s);
    const int64_t total = h[0], n_steps = h[1], slot_bytes = h[2];
    int32_t* final_ids = nullptr;
    ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
    k_ooc_walk_emit<<<nd_grid(n * 32, 256), 256, 0, s>>>(roots32, win, std::max(L, 1), n, final_off,
                                                         final_ids, roots_out);
    k_iota_off<<<nd_grid(n + 1, 256), 256, 0, s>>>(roots_off, n + 1);
    ND_CUDA_TRY(cudaGetLastError());
    nd_result* res = new nd_result();
    res->stream = s;
    res->n = n;
    res->n_steps = n_steps;
    res->total_sampled = total - n;
    res->set(ND_F_FINAL_OFF, final_off, n + 1);
    res->set(ND_F_FINAL_IDS32, final_ids, total);
    res->set(ND_F_ROOTS, roots_out, n);
    res->set(ND_F_ROOTS_OFF, roots_off, n + 1);
    res->set(ND_F_CHAIN_LEN, clen, n);
    res->counters[NDC_SLOT_BYTES] = slot_bytes;
    res->counters[NDC_STEPS] = rounds;  // shuttle rounds
    *out = res;
  }
  nd_free(flen, s); nd_free(roots32, s); nd_free(cur, s); nd_free(stp, s); nd_free(win, s);
  nd_free(hist, s); nd_free(ctr, s);
  return ND_OK;
}

extern "C" int nd_run_individual_ooc(nd_ooc_graph* G, int app_code, const int64_t* host_fanouts,
                                     int64_t n_fanouts, int64_t sample_lo, int64_t n,
                                     const int64_t* roots, uint64_t seed, void* stream,
                                     nd_result** out) {
  NvtxRange nvtx("nd_run_individual_ooc");
  if (!G || !out || n <= 0 || sample_lo < 0 || n >= (1ll << 31) || n_fanouts < 1 || n_fanouts > 8)
    return ND_ERR_ARG;
  if (app_code != ND_KHOP) return ND_ERR_APP;
  for (int64_t k = 0; k < n_fanouts; k++)
    if (host_fanouts[k] < 1) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t S = n_fanouts, R = 1;
  const int P = (int)G->parts();
  int64_t B[9];
  B[0] = R;
  for (int64_t k = 0; k < S; k++) {
    B[k + 1] = B[k] * host_fanouts[k];
    if ((double)n * (double)B[k + 1] >= 4.0e9) return ND_ERR_ARG;  // 32-bit item indices
  }
  DevGraph gv;
  gv.V = G->V;
  int32_t* blk[9] = {};
  int32_t* rank[8] = {};
  int64_t* nn[8] = {};
  unsigned long long *hist = nullptr, *ctr = nullptr;
  ND_CUDA_TRY(nd_alloc(&blk[0], n, s));
  ND_CUDA_TRY(nd_alloc(&hist, P, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, s));
  if (roots) k_ooc_narrow<<<nd_grid(n, 256), 256, 0, s>>>(roots, n, blk[0]);
  else ND_TRY(nd_uniform_roots_i32(gv, 1, seed, sample_lo, n, blk[0], s));
  Shuttle sh{G, s, nullptr};
  ND_TRY(sh.init());
  std::vector<int64_t> busy;
  std::vector<int64_t> parents(S, 0);
  int64_t n_steps = S;
  for (int64_t k = 0; k < S; k++) {
    const int64_t N = n * B[k];
    ND_CUDA_TRY(nd_alloc(&rank[k], N, s));
    ND_CUDA_TRY(nd_alloc(&nn[k], n, s));
    ND_CUDA_TRY(nd_alloc(&blk[k + 1], n * B[k + 1], s));
    ND_CUDA_TRY(cudaMemsetAsync(blk[k + 1], 0xFF, n * B[k + 1] * 4, s));
    k_ooc_rank<<<nd_grid(n * 32, 256), 256, 0, s>>>(blk[k], n, B[k], rank[k], nn[k]);
    ND_CUDA_TRY(cudaMemsetAsync(hist, 0, P * 8, s));
    k_ooc_parent_hist<<<nd_grid(N, 256), 256, 0, s>>>(blk[k], N, G->vcut_d, P, hist);
    ND_TRY(busy_parts(hist, P, s, busy, &parents[k]));
    if (parents[k] == 0 && n_steps == S) n_steps = k;  // no sample has a transit (core.py:187-203)
    const uint64_t base0 = key_base(seed, (uint64_t)k, 0, 0);
    int b = 0, nb = 0;
    if (!busy.empty()) ND_TRY(sh.upload(busy[0], b));
    for (size_t j = 0; j < busy.size(); j++) {
      const int64_t p = busy[j];
      if (j + 1 < busy.size()) ND_TRY(sh.upload(busy[j + 1], nb));
      ND_TRY(sh.use(b));
      k_ooc_khop<<<nd_grid(N * host_fanouts[k], 256, 148 * 32), 256, 0, s>>>(
          G->row_d, G->col_d[b], G->e0(p), G->vcut[p], G->vcut[p + 1], blk[k], rank[k], N,
          FastDiv((uint32_t)B[k]), FastDiv((uint32_t)host_fanouts[k]), base0, sample_lo,
          blk[k + 1], ctr);
      ND_CUDA_TRY(cudaGetLastError());
      ND_TRY(sh.release(b));
      b = nb;
    }
  }
  sh.destroy();
  // final rows, step counts and step rows
  OocSteps FS;
  FS.n_steps = (int)S;
  for (int64_t k = 0; k < S; k++) { FS.blk[k] = blk[k + 1]; FS.B[k] = B[k + 1]; }
  int64_t *flen = nullptr, *final_off = nullptr, *step_counts = nullptr, *soff = nullptr,
          *roots_out = nullptr, *roots_off = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&step_counts, S * n + 1, s));
  ND_CUDA_TRY(nd_alloc(&soff, S * n + 1, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, n, s));
  ND_CUDA_TRY(nd_alloc(&roots_off, n + 1, s));
  k_ooc_khop_lens<<<nd_grid((n + 1) * 32, 256), 256, 0, s>>>(FS, n, R, flen);
  for (int64_t k = 0; k < S; k++)
    k_ooc_step_counts<<<nd_grid(n, 256), 256, 0, s>>>(nn[k], n, host_fanouts[k], step_counts + k * n);
  ND_CUDA_TRY(cudaMemsetAsync(step_counts + S * n, 0, 8, s));
  {
    size_t t1 = 0, t2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t1, flen, final_off, n + 1, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, step_counts, soff, S * n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, std::max(t1, t2), s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, t1, flen, final_off, n + 1, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, t2, step_counts, soff, S * n + 1, s));
    nd_free(tmp, s);
  }
  int64_t* h = nd_pinned_scratch();
  ND_TRY(nd_d2h(h, final_off + n, 8, s));
  ND_TRY(nd_d2h(h + 1, soff + S * n, 8, s));
  ND_TRY(nd_d2h(h + 2, ctr, 8, s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t total = h[0], total_items = h[1], slot_bytes = h[2];
  int32_t *final_ids = nullptr, *vals = nullptr;
  ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
  ND_CUDA_TRY(nd_alloc(&vals, std::max<int64_t>(total_items, 1), s));
  k_ooc_khop_emit<<<nd_grid(n * 32, 256), 256, 0, s>>>(FS, blk[0], n, R, final_off, final_ids,
                                                       roots_out, roots_off);
  for (int64_t k = 0; k < S; k++)
    k_ooc_step_vals<<<nd_grid(n * B[k + 1], 256, 148 * 64), 256, 0, s>>>(
        blk[k + 1], rank[k], n, B[k], host_fanouts[k], soff + k * n, vals);
  ND_CUDA_TRY(cudaGetLastError());
  nd_result* res = new nd_result();
  res->stream = s;
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n * R;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n * R);
  res->set(ND_F_ROOTS_OFF, roots_off, n + 1);
  // the run loop's steps: step rows and counts of the steps that ran
  int64_t items_run = 0;
  {
    // step k's slot count = soff[(k+1)*n] - soff[k*n]; keep the first n_steps steps
    if (n_steps > 0) ND_TRY(nd_d2h(h + 3, soff + n_steps * n, 8, s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    items_run = n_steps > 0 ? h[3] : 0;
  }
  res->set(ND_F_STEP_COUNTS, step_counts, n_steps * n);
  res->set(ND_F_STEP_VALS32, vals, items_run);
  res->counters[NDC_ITEMS] = items_run;
  res->counters[NDC_SLOT_BYTES] = slot_bytes;
  res->counters[NDC_STEPS] = n_steps;
  *out = res;
  for (int64_t k = 0; k <= S; k++) nd_free(blk[k], s);
  for (int64_t k = 0; k < S; k++) { nd_free(rank[k], s); nd_free(nn[k], s); }
  nd_free(flen, s); nd_free(soff, s); nd_free(hist, s); nd_free(ctr, s);
  return ND_OK;
}
