// nd_collective.cu — collective apps on device (layer, FastGCN/LADIES, MVS,
// ClusterGCN).
//
// Reference path: tp_step's collective branch (transit_parallel.py:187-198)
// -> build_combined (collective.py:39-120) -> collective_select
// (collective.py:123-141) -> the apps' next functions (apps.py:247-386).
// Per step every alive sample's transits are its previous step's non-NULL
// vertices (roots at step 0, duplicates kept, core.py:168-184); the combined
// neighbourhood is the concatenation of the transits' adjacency lists in
// transit order.  The device never materialises it: a combined entry e of
// sample i is located by a binary search over the per-sample exclusive scan
// of transit degrees (entry e -> transit k, offset e - cdeg[k]).
//   layer       take = min(m, max(0, cap - size)); slot < take -> combined[u % n]
//   importance  v = u % V (or the deg^2 inverse CDF); record (t, v) for every
//               transit t with an edge t->v (slot-major, transit order)
//   mvs         i = u % n; record (src_transit[i], nbr[i])
//   clustergcn  record every combined entry whose neighbour is a root
//               (per-sample root bitmap; one warp per (sample, transit) pair
//               walks the adjacency twice: count, then ordered write)
// The transit-parallel build statistics (groups of equal transits classed
// by members * degree, collective.py:107-114) are computed on device from a
// radix sort of the step's transit occurrences.
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <vector>

#include "nd_tp.cuh"

using namespace nd;

namespace {

template <typename T>
int scan_excl(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  void* tmp = nullptr;
  ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
  ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n, s));
  nd_free(tmp, s);
  return ND_OK;
}

template <typename T>
int dcopy_to_host(T* h, const T* d, int64_t n, cudaStream_t s) {
  ND_TRY(nd_d2h(h, d, n * sizeof(T), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  return ND_OK;
}

struct WidenFlag {
  __host__ __device__ int64_t operator()(uint8_t x) const { return (int64_t)x; }
};

// degrees of the flattened transits (+1 trailing 0 for the exclusive scan)
__global__ void k_tdeg(const int32_t* __restrict__ tv, int64_t T, const int64_t* __restrict__ row,
                       int64_t* __restrict__ d) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= T;
       j += (int64_t)gridDim.x * blockDim.x)
    d[j] = j < T ? row[tv[j] + 1] - row[tv[j]] : 0;
}

// locate combined entry e of sample i: transit index k in [a, b) with
// cdeg[k] - cdeg[a] <= e < cdeg[k+1] - cdeg[a]
__device__ __forceinline__ int64_t locate(const int64_t* __restrict__ cdeg, int64_t a, int64_t b,
                                          int64_t e) {
  const int64_t base = cdeg[a];
  int64_t lo = a, hi = b;  // last k with cdeg[k] - base <= e
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (cdeg[mid] - base <= e) lo = mid; else hi = mid;
  }
  return lo;
}

struct SelCtx {
  DevGraph g;
  int kind;
  int64_t m, max_size, V;
  uint64_t base0;
  int64_t sample_lo;
  const int64_t* toff;     // [n+1] transit offsets per sample (this step)
  const int32_t* tv;       // transits
  const int64_t* cdeg;     // [T+1] exclusive scan of transit degrees
  const int64_t* size;     // per sample size before this step
  const uint8_t* alive;
  const double* cum;       // deg^2 CDF (importance, degree_sq)
  int distribution;
  int32_t* out;            // [n*m]
  int32_t* rec_t1;         // mvs: one record per slot ([n*m], -1 = none)
};

// layer / importance / mvs slot selection: one thread per (sample, slot)
__global__ void k_select(SelCtx c, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n * c.m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = j / c.m, slot = j - i * c.m;
    int32_t o = -1, rt = -1;
    if (c.alive[i]) {
      const int64_t a = c.toff[i], b = c.toff[i + 1];
      const int64_t total = c.cdeg[b] - c.cdeg[a];
      const uint64_t u = draw_u64(c.base0, key_item((uint64_t)(c.sample_lo + i), 0, (uint64_t)slot));
      if (c.kind == ND_LAYER) {
        int64_t take = c.max_size - c.size[i];
        if (take < 0) take = 0;
        if (take > c.m) take = c.m;
        if (total > 0 && slot < take) {
          const int64_t e = (int64_t)mod_u64(u, (uint64_t)total);
          const int64_t k = locate(c.cdeg, a, b, e);
          const int64_t t = c.tv[k];
          o = __ldg(c.g.col + __ldg(c.g.row + t) + (e - (c.cdeg[k] - c.cdeg[a])));
        }
      } else if (c.kind == ND_MVS) {
        if (total > 0) {
          const int64_t e = (int64_t)mod_u64(u, (uint64_t)total);
          const int64_t k = locate(c.cdeg, a, b, e);
          const int64_t t = c.tv[k];
          o = __ldg(c.g.col + __ldg(c.g.row + t) + (e - (c.cdeg[k] - c.cdeg[a])));
          rt = (int32_t)t;
        }
      } else {  // importance
        if (c.distribution == 0) {
          o = (int32_t)mod_u64(u, (uint64_t)c.V);
        } else {
          const double x = __dmul_rn(to_unit(u), c.cum[c.V - 1]);
          int64_t lo = 0, hi = c.V;
          while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (c.cum[mid] <= x) lo = mid + 1; else hi = mid;
          }
          o = (int32_t)(lo < c.V - 1 ? lo : c.V - 1);
        }
      }
    }
    c.out[j] = o;
    if (c.rec_t1) c.rec_t1[j] = rt;
  }
}

// importance hits: one warp per (sample, slot), lanes over the sample's
// transits (flag index tri_off[i] + slot * T + k, the triple order of
// apps.py:286-312)
__global__ void k_imp_hits(const DevGraph g, const int64_t* __restrict__ toff,
                           const int32_t* __restrict__ tv, const int32_t* __restrict__ out,
                           const uint8_t* __restrict__ alive, const int64_t* __restrict__ tri_off,
                           int64_t n, int64_t m, int64_t total_tri, uint8_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ps = warp; ps < n * m; ps += nw) {
    const int64_t i = ps / m, slot = ps - i * m;
    if (!alive[i]) continue;
    const int64_t T = toff[i + 1] - toff[i];
    const int64_t v = out[i * m + slot];
    for (int64_t k = lane; k < T; k += 32) {
      const int64_t j = tri_off[i] + slot * T + k;
      const int64_t t = tv[toff[i] + k];
      const int64_t rlo = __ldg(g.row + t), rhi = __ldg(g.row + t + 1);
    // has_edge(t, v) (graph.py:78-81): the exact hash set when built, else the
    // sorted-row binary search; same answer
      const bool hit = (g.hset != nullptr && rhi - rlo > HASH_MIN_DEG)
                           ? (v >= 0 && hset_contains(g.hset + 4 * rlo, hset_size(rhi - rlo), (int32_t)v))
                           : has_edge(g.col, rlo, rhi, v);
      flag[j] = hit ? 1 : 0;
    }
  }
}

__global__ void k_imp_write(const int64_t* __restrict__ toff, const int32_t* __restrict__ tv,
                            const int32_t* __restrict__ out, const int64_t* __restrict__ tri_off,
                            int64_t n, int64_t m, int64_t total_tri, const uint8_t* __restrict__ flag,
                            const int64_t* __restrict__ pos, int64_t* __restrict__ rt,
                            int64_t* __restrict__ rv) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total_tri;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[j]) continue;
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (tri_off[mid] <= j) lo = mid; else hi = mid;
    }
    const int64_t i = lo;
    const int64_t T = toff[i + 1] - toff[i];
    const int64_t r = j - tri_off[i];
    const int64_t slot = r / T, k = r - slot * T;
    rt[pos[j]] = tv[toff[i] + k];
    rv[pos[j]] = out[i * m + slot];
  }
}

// per-sample triple offsets (importance): m * transits, 0 when dead
__global__ void k_tri_len(const int64_t* __restrict__ toff, const uint8_t* __restrict__ alive,
                          int64_t n, int64_t m, int64_t* __restrict__ len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    len[i] = (i < n && alive[i]) ? m * (toff[i + 1] - toff[i]) : 0;
}

// per-sample counts between offsets of a scanned flag array
__global__ void k_seg_counts(const int64_t* __restrict__ seg, const int64_t* __restrict__ pos,
                             int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = pos[seg[i + 1]] - pos[seg[i]];
}

// ---- clustergcn -------------------------------------------------------------------
__global__ void k_bitmap_set(const int64_t* __restrict__ roff, const int32_t* __restrict__ roots,
                             int64_t n, int64_t words, uint32_t* __restrict__ bm) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
    for (int64_t k = roff[i] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < roff[i + 1];
         k += (int64_t)gridDim.x * blockDim.x) {
      const uint32_t v = (uint32_t)roots[k];
      atomicOr(bm + i * words + (v >> 5), 1u << (v & 31));
    }
}

// ClusterGCN record scan (apps.py:372-379: every combined entry whose
// neighbour is one of the sample's roots).  The combined neighbourhoods of
// all samples are one flattened edge range (cdeg = exclusive scan of the
// pairs' row lengths), cut into units of CG_UNIT edges, one warp per unit and
// 32 edges per iteration, so a hub's row spreads over many warps instead of
// serialising one.  Each lane finds its edge's pair by a binary search of
// cdeg inside the unit's pair range (cached while the pair repeats).  Pass 0
// counts hits per unit (and per sample); pass 1 writes them at the unit's
// scanned base in flattened order = pair order, then adjacency order.
constexpr int64_t CG_UNIT = 1024;

struct CgArgs {
  DevGraph g;
  const int64_t* toff;  // per-sample pair offsets [n+1]
  const int32_t* tv;    // pair transits [T]
  const int64_t* cdeg;  // flattened edge offset of each pair [T+1]
  int64_t n, T;
  const uint32_t* bm;   // per-sample root bitmaps
  int64_t words;
};

// last pair starting at or before flattened edge k, searched in [a, b]
__device__ __forceinline__ int64_t cg_pair_of(const int64_t* __restrict__ cdeg, int64_t k,
                                              int64_t a, int64_t b) {
  while (a < b) {
    const int64_t mid = (a + b + 1) >> 1;
    if (__ldg(cdeg + mid) <= k) a = mid; else b = mid - 1;
  }
  return a;
}

// One warp scans flattened edges [e0, e1) 32 at a time; returns the hits and,
// with rt/rv, writes them from position acc0 in edge order.  (Four chunks in
// flight per iteration measured slower: 5.3 vs 4.8 ms on C4 ClusterGCN.)
__device__ __forceinline__ int64_t cg_scan(const CgArgs& A, int64_t e0, int64_t e1, int64_t acc0,
                                           int64_t* __restrict__ rt, int64_t* __restrict__ rv) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  if (e1 <= e0) return acc0;
  const int64_t plo = cg_pair_of(A.cdeg, e0, 0, A.T - 1);
  const int64_t phi = cg_pair_of(A.cdeg, e1 - 1, plo, A.T - 1);
  int64_t q = -1, t = 0, base = 0, smp = 0, qend = -1;  // this lane's cached pair
  int64_t acc = acc0;
  for (int64_t c = e0; c < e1; c += 32) {
    const int64_t k = c + lane;
    bool hit = false;
    uint32_t v = 0;
    if (k < e1) {
      if (k >= qend) {
        q = cg_pair_of(A.cdeg, k, q < 0 ? plo : q, phi);
        t = A.tv[q];
        base = __ldg(A.g.row + t) - __ldg(A.cdeg + q);
        qend = __ldg(A.cdeg + q + 1);
        int64_t a = 0, b = A.n - 1;  // owner sample: last i with toff[i] <= q
        while (a < b) {
          const int64_t mid = (a + b + 1) >> 1;
          if (__ldg(A.toff + mid) <= q) a = mid; else b = mid - 1;
        }
        smp = a;
      }
      v = (uint32_t)__ldg(A.g.col + base + k);
      hit = (__ldg(A.bm + smp * A.words + (v >> 5)) >> (v & 31)) & 1u;
    }
    const unsigned hm = __ballot_sync(0xffffffffu, hit);
    if (rt != nullptr && hit) {
      const int64_t pos = acc + __popc(hm & lt);
      rt[pos] = t;
      rv[pos] = v;
    }
    acc += __popc(hm);
  }
  return acc;
}

// pass 0: hits per unit; pass 1: write the unit's hits at its scanned base
template <int PASS>
__global__ void __launch_bounds__(256) k_cgcn(const CgArgs A, int64_t* __restrict__ ucnt,
                                              const int64_t* __restrict__ ubase,
                                              int64_t* __restrict__ rt, int64_t* __restrict__ rv) {
  const int64_t ET = A.cdeg[A.T];
  const int64_t units = (ET + CG_UNIT - 1) / CG_UNIT;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < units; u += nw) {
    const int64_t e0 = u * CG_UNIT, e1 = e0 + CG_UNIT < ET ? e0 + CG_UNIT : ET;
    if (PASS == 0) {
      const int64_t h = cg_scan(A, e0, e1, 0, nullptr, nullptr);
      if ((threadIdx.x & 31) == 0) ucnt[u] = h;
    } else {
      cg_scan(A, e0, e1, ubase[u], rt, rv);
    }
  }
}

// hits before each sample's first edge (the unit's base + a partial rescan),
// then per-sample record counts
__global__ void k_cgcn_bounds(const CgArgs A, const int64_t* __restrict__ ubase,
                              int64_t* __restrict__ hb) {
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i <= A.n; i += nw) {
    const int64_t eb = A.cdeg[i < A.n ? A.toff[i] : A.T];
    const int64_t u = eb / CG_UNIT;
    const int64_t h = cg_scan(A, u * CG_UNIT, eb, ubase[u], nullptr, nullptr);
    if ((threadIdx.x & 31) == 0) hb[i] = h;
  }
}

__global__ void k_diff(const int64_t* __restrict__ hb, int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = hb[i + 1] - hb[i];
}

// ---- step plumbing ----------------------------------------------------------------------
__global__ void k_alive_from_toff(const int64_t* __restrict__ toff, int64_t n,
                                  uint8_t* __restrict__ alive) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    alive[i] = toff[i + 1] > toff[i];
}

__global__ void k_step_counts(const uint8_t* __restrict__ alive, int64_t n, int64_t m,
                              int64_t* __restrict__ cnt, int64_t* __restrict__ nn_flags_len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = alive[i] ? m : 0;
}

// non-NULL slots of alive samples -> next transits; per-sample next counts
__global__ void k_nonnull(const int32_t* __restrict__ out, const uint8_t* __restrict__ alive,
                          int64_t n, int64_t m, int64_t* __restrict__ flag) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= n * m;
       j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = (j < n * m && alive[j / m] && out[j] >= 0) ? 1 : 0;
}

__global__ void k_next_transits(const int32_t* __restrict__ out, const int64_t* __restrict__ flag,
                                const int64_t* __restrict__ pos, int64_t nm, int32_t* __restrict__ ntv) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nm;
       j += (int64_t)gridDim.x * blockDim.x)
    if (flag[j]) ntv[pos[j]] = out[j];
}

__global__ void k_next_transits_sid(const int32_t* __restrict__ out, const int64_t* __restrict__ flag,
                                    const int64_t* __restrict__ pos, int64_t nm, int64_t m,
                                    int32_t* __restrict__ ntv, int32_t* __restrict__ nsid) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nm;
       j += (int64_t)gridDim.x * blockDim.x)
    if (flag[j]) {
      ntv[pos[j]] = out[j];
      nsid[pos[j]] = (int32_t)(j / m);
    }
}

__global__ void k_size_add(int64_t* __restrict__ size, const int64_t* __restrict__ c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    size[i] += c[i];
}

__global__ void k_next_toff(const int64_t* __restrict__ pos, int64_t n, int64_t m,
                            int64_t* __restrict__ ntoff, int64_t* __restrict__ size) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ntoff[i] = pos[i * m];
    if (i < n) size[i] += pos[(i + 1) * m] - pos[i * m];
  }
}

// out slots of alive samples, compacted in step-major sample order
__global__ void k_emit_slots(const int32_t* __restrict__ out, const uint8_t* __restrict__ alive,
                             const int64_t* __restrict__ base, int64_t n, int64_t m,
                             int64_t* __restrict__ vals) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n * m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = j / m;
    if (alive[i]) vals[base[i] * m + (j - i * m)] = out[j];
  }
}

__global__ void k_alive_idx(const uint8_t* __restrict__ alive, int64_t n, int64_t* __restrict__ a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = i < n ? alive[i] : 0;
}

// mvs: records from one-per-slot (t, v) where v non-NULL
__global__ void k_mvs_flags(const int32_t* __restrict__ rec_t1, int64_t nm, int64_t* __restrict__ f) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= nm;
       j += (int64_t)gridDim.x * blockDim.x)
    f[j] = (j < nm && rec_t1[j] >= 0) ? 1 : 0;
}

__global__ void k_mvs_write(const int32_t* __restrict__ rec_t1, const int32_t* __restrict__ out,
                            const int64_t* __restrict__ f, const int64_t* __restrict__ pos, int64_t nm,
                            int64_t* __restrict__ rt, int64_t* __restrict__ rv) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nm;
       j += (int64_t)gridDim.x * blockDim.x)
    if (f[j]) {
      rt[pos[j]] = rec_t1[j];
      rv[pos[j]] = out[j];
    }
}

__global__ void k_mvs_counts(const int64_t* __restrict__ pos, int64_t n, int64_t m,
                             int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = pos[(i + 1) * m] - pos[i * m];
}

// TP build stats: group classes with work = members * degree(transit)
__global__ void k_classify_deg(const uint32_t* __restrict__ keys, const int* __restrict__ gstart,
                               const int* __restrict__ n_groups, const int64_t* __restrict__ row,
                               unsigned long long* __restrict__ stats) {
  const int G = *n_groups;
  int cnt[3] = {0, 0, 0};
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    const uint32_t t = keys[gstart[g]];
    const int64_t work = (int64_t)(gstart[g + 1] - gstart[g]) * (row[t + 1] - row[t]);
    cnt[work < SMALL_MAX_WORK ? 0 : (work <= LARGE_MIN_WORK ? 1 : 2)]++;
  }
  for (int c = 0; c < 3; c++) {
    int v = cnt[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(stats + c, (unsigned long long)v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats + 3, (unsigned long long)G);
}

__global__ void k_u32(const int32_t* __restrict__ a, int64_t n, uint32_t* __restrict__ k,
                      uint64_t* __restrict__ v) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    k[j] = (uint32_t)a[j];
    v[j] = (uint64_t)j;
  }
}

__global__ void k_deg2(const int64_t* __restrict__ row, int64_t V, int64_t* __restrict__ d2) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = row[v + 1] - row[v];
    d2[v] = d * d;
  }
}

__global__ void k_i64_to_f64(const int64_t* __restrict__ a, int64_t n, double* __restrict__ b) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    b[v] = (double)a[v];
}

// clustergcn roots: cluster of each vertex keyed on (seed, vertex) domain 4
__global__ void k_cluster_flags(int64_t V, uint64_t base4, int64_t nc, const uint8_t* __restrict__ chosen,
                                int64_t* __restrict__ flag) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= V;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (v == V) { flag[V] = 0; continue; }
    const uint64_t u = draw_u64(base4, key_item((uint64_t)v, 0, 0));
    flag[v] = chosen[mod_u64(u, (uint64_t)nc)] ? 1 : 0;
  }
}

__global__ void k_cluster_write(const int64_t* __restrict__ flag, const int64_t* __restrict__ pos,
                                int64_t V, int32_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    if (flag[v]) out[pos[v]] = (int32_t)v;
}

__global__ void k_widen32(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    b[j] = a[j];
}

__global__ void k_narrow64(const int64_t* __restrict__ a, int64_t n, int32_t* __restrict__ b) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    b[j] = (int32_t)a[j];
}

// final rows: roots then every step's non-NULL slots.  Block rows stride over
// samples (blockIdx.y) and threads over a sample's entries, so one huge
// sample (ClusterGCN: ~20% of V roots) is copied by many blocks, coalesced.
__global__ void k_coll_final(const int64_t* __restrict__ roff, const int32_t* __restrict__ roots,
                             int64_t n, const int64_t* __restrict__ off, int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    const int64_t a = roff[i], len = roff[i + 1] - a, o = off[i];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * blockDim.x)
      ids[o + k] = roots[a + k];
  }
}

__global__ void k_coll_final_step(const int32_t* __restrict__ ntv, const int64_t* __restrict__ ntoff,
                                  int64_t n, const int64_t* __restrict__ off,
                                  const int64_t* __restrict__ fill, int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    const int64_t a = ntoff[i], len = ntoff[i + 1] - a, o = off[i] + fill[i];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len;
         k += (int64_t)gridDim.x * blockDim.x)
      ids[o + k] = ntv[a + k];
  }
}

// 2-D grid for a segmented copy of `total` entries over n segments
static dim3 seg_grid(int64_t total, int64_t n) {
  const int64_t avg = n > 0 ? (total + n - 1) / n : 0;
  int64_t gx = (avg + 255) / 256;
  gx = gx < 1 ? 1 : (gx > 512 ? 512 : gx);
  int64_t gy = n < 1 ? 1 : (n > 65535 ? 65535 : n);
  return dim3((unsigned)gx, (unsigned)gy);
}

__global__ void k_fill_add(int64_t* __restrict__ fill, const int64_t* __restrict__ ntoff, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    fill[i] += ntoff[i + 1] - ntoff[i];
}

struct CStep {
  int64_t* counts = nullptr;     // [n]
  int64_t* vals = nullptr;       // alive*m
  int64_t nvals = 0;
  int64_t* rec_cnt = nullptr;    // [n]
  int64_t* rec_t = nullptr;
  int64_t* rec_v = nullptr;
  int64_t nrec = 0;
  int32_t* ntv = nullptr;        // next transits (non-NULL of this step)
  int64_t* ntoff = nullptr;      // [n+1]
};

}  // namespace

extern "C" int nd_run_collective(const nd_graph* G, int kind, int64_t step_size, int64_t max_size,
                                 int distribution, int64_t steps, int64_t batch_size,
                                 int64_t clusters_per_sample, int64_t num_clusters,
                                 int64_t sample_lo, int64_t n, const int64_t* roots_off_in,
                                 const int64_t* roots_in, uint64_t seed, int64_t step_cap,
                                 const uint8_t* host_unique, int64_t n_unique, void* stream,
                                 nd_result** out_res) {
  NvtxRange nvtx_run("nd_run_collective");
  nd_pool_init();
  if (!G || n < 0 || sample_lo < 0 || step_size < 1 || kind < 0 || kind > 3) return kind < 0 || kind > 3 ? ND_ERR_APP : ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  // FastGCN/LADIES test has_edge(t, v) for every (draw, transit) pair: build
  // the exact per-row hash sets once per graph (nd_index.cu)
  if (kind == ND_IMPORTANCE) ND_TRY(nd_graph_ensure_index(const_cast<nd_graph*>(G), 1, 0, s));
  const DevGraph& g = G->g;
  const int64_t V = g.V;
  const int64_t m = step_size;
  const int64_t S_max = steps >= 0 ? std::min(steps, step_cap) : step_cap;
  std::vector<int64_t> h_roff(n + 1, 0);

  // ---- roots (CSR, int32) ---------------------------------------------------------
  int64_t* roff = nullptr;
  int32_t* roots = nullptr;
  ND_CUDA_TRY(nd_alloc(&roff, n + 1, s));
  if (roots_in) {
    ND_CUDA_TRY(cudaMemcpyAsync(roff, roots_off_in, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    ND_TRY(dcopy_to_host(h_roff.data(), roff, n + 1, s));
    ND_CUDA_TRY(nd_alloc(&roots, h_roff[n], s));
    if (h_roff[n]) k_narrow64<<<nd_grid(h_roff[n], 256), 256, 0, s>>>(roots_in, h_roff[n], roots);
  } else if (kind == ND_CLUSTERGCN) {
    if (num_clusters < 1 || clusters_per_sample < 0) return ND_ERR_ARG;
    // chosen clusters per sample (apps.py:357-366): keyed draws until distinct
    const int64_t want = std::min(clusters_per_sample, num_clusters);
    std::vector<std::vector<int32_t>> parts(n);
    int64_t* flag = nullptr;
    int64_t* pos = nullptr;
    uint8_t* chosen = nullptr;
    ND_CUDA_TRY(nd_alloc(&flag, V + 1, s));
    ND_CUDA_TRY(nd_alloc(&pos, V + 1, s));
    ND_CUDA_TRY(nd_alloc(&chosen, num_clusters, s));
    std::vector<int32_t*> rparts(n, nullptr);
    for (int64_t i = 0; i < n; i++) {
      std::vector<uint8_t> ch(num_clusters, 0);
      int64_t have = 0;
      uint64_t b = key_base(seed, 0, 5, 0);
      const uint64_t ik = key_item((uint64_t)(sample_lo + i), 0, 0);
      while (have < want) {
        const uint64_t c = fin64(fin64(b + ik)) % (uint64_t)num_clusters;
        b += C_DRAW;
        if (!ch[c]) { ch[c] = 1; have++; }
      }
      ND_CUDA_TRY(cudaMemcpyAsync(chosen, ch.data(), num_clusters, cudaMemcpyHostToDevice, s));
      k_cluster_flags<<<nd_grid(V + 1, 256), 256, 0, s>>>(V, key_base(seed, 0, 4, 0), num_clusters,
                                                           chosen, flag);
      ND_TRY(scan_excl(flag, pos, V + 1, s));
      int64_t cnt = 0;
      ND_TRY(dcopy_to_host(&cnt, pos + V, 1, s));
      ND_CUDA_TRY(nd_alloc(&rparts[i], cnt, s));
      if (V) k_cluster_write<<<nd_grid(V, 256), 256, 0, s>>>(flag, pos, V, rparts[i]);
      h_roff[i + 1] = h_roff[i] + cnt;
    }
    ND_CUDA_TRY(nd_alloc(&roots, h_roff[n], s));
    for (int64_t i = 0; i < n; i++) {
      const int64_t c = h_roff[i + 1] - h_roff[i];
      if (c) ND_CUDA_TRY(cudaMemcpyAsync(roots + h_roff[i], rparts[i], c * 4, cudaMemcpyDeviceToDevice, s));
      nd_free(rparts[i], s);
    }
    ND_CUDA_TRY(cudaMemcpyAsync(roff, h_roff.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    nd_free(flag, s); nd_free(pos, s); nd_free(chosen, s);
  } else {
    const int64_t R = kind == ND_LAYER ? 1 : batch_size;
    if (R < 1) return ND_ERR_ARG;
    for (int64_t i = 0; i <= n; i++) h_roff[i] = i * R;
    ND_CUDA_TRY(cudaMemcpyAsync(roff, h_roff.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    ND_CUDA_TRY(nd_alloc(&roots, n * R, s));
    ND_TRY(nd_uniform_roots_i32(g, R, seed, sample_lo, n, roots, s));
  }
  const int64_t n_roots = h_roff[n];

  // deg^2 CDF (apps.py:291-296): exact integer prefix converted to f64
  double* cum = nullptr;
  if (kind == ND_IMPORTANCE && distribution == 1 && V > 0) {
    int64_t *d2 = nullptr, *c2 = nullptr;
    ND_CUDA_TRY(nd_alloc(&d2, V, s));
    ND_CUDA_TRY(nd_alloc(&c2, V, s));
    ND_CUDA_TRY(nd_alloc(&cum, V, s));
    k_deg2<<<nd_grid(V, 256), 256, 0, s>>>(g.row, V, d2);
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, d2, c2, V, s);
    void* tmp;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp, tb, d2, c2, V, s));
    k_i64_to_f64<<<nd_grid(V, 256), 256, 0, s>>>(c2, V, cum);
    nd_free(tmp, s); nd_free(d2, s); nd_free(c2, s);
  }

  // ---- step loop -----------------------------------------------------------------------
  int64_t *size = nullptr, *toff = nullptr;
  uint8_t* alive = nullptr;
  int32_t* tv = roots;
  unsigned long long* stats = nullptr;
  ND_CUDA_TRY(nd_alloc(&size, n, s));
  ND_CUDA_TRY(nd_alloc(&alive, n, s));
  ND_CUDA_TRY(nd_alloc(&toff, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&stats, 4 * (S_max + 1), s));
  ND_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * (S_max + 1) * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemcpyAsync(toff, roff, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  {
    std::vector<int64_t> hs(n);
    for (int64_t i = 0; i < n; i++) hs[i] = h_roff[i + 1] - h_roff[i];
    if (n) ND_CUDA_TRY(cudaMemcpyAsync(size, hs.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
  }
  int64_t T = n_roots;
  std::vector<CStep> steps_v;
  const int key_bits = key_bits_for(V);
  int64_t step = 0;
  int64_t total_rec = 0;
  Profiler prof(s);
  while (step < S_max) {
    if (n) k_alive_from_toff<<<nd_grid(n, 256), 256, 0, s>>>(toff, n, alive);
    if (T == 0) break;  // no sample has transits (is_alive, core.py:195-203)
    prof.step_begin();
    CStep cs;
    // TP build statistics over the step's transit occurrences
    {
      TPScratch S;
      ND_TRY(S.alloc(T, key_bits, s));
      uint32_t *k0, *k1;
      uint64_t *v0, *v1;
      ND_CUDA_TRY(nd_alloc(&k0, T, s)); ND_CUDA_TRY(nd_alloc(&k1, T, s));
      ND_CUDA_TRY(nd_alloc(&v0, T, s)); ND_CUDA_TRY(nd_alloc(&v1, T, s));
      k_u32<<<nd_grid(T, 256), 256, 0, s>>>(tv, T, k0, v0);
      cub::DoubleBuffer<uint32_t> dk(k0, k1);
      cub::DoubleBuffer<uint64_t> dv(v0, v1);
      ND_TRY(tp_sort(dk, dv, T, key_bits, S, s));
      k_mark<<<nd_grid(T, 256), 256, 0, s>>>(dk.Current(), T, S.flags);
      size_t tb = S.cub_bytes;
      ND_CUDA_TRY(cub::DeviceScan::InclusiveSum(S.cub_tmp, tb, S.flags, S.gid, (int)T, s));
      ND_CUDA_TRY(cudaMemsetAsync(S.counters, 0, 4 * sizeof(int), s));
      k_gstart<<<nd_grid(T, 256), 256, 0, s>>>(S.flags, S.gid, T, S.gstart, S.counters);
      k_classify_deg<<<nd_grid(T, 256), 256, 0, s>>>(dk.Current(), S.gstart, S.counters, g.row,
                                                      stats + 4 * step);
      nd_free(k0, s); nd_free(k1, s); nd_free(v0, s); nd_free(v1, s);
      S.release(s);
    }
    // combined-neighbourhood index: exclusive scan of transit degrees
    int64_t *dg = nullptr, *cdeg = nullptr;
    ND_CUDA_TRY(nd_alloc(&dg, T + 1, s));
    ND_CUDA_TRY(nd_alloc(&cdeg, T + 1, s));
    k_tdeg<<<nd_grid(T + 1, 256), 256, 0, s>>>(tv, T, g.row, dg);
    ND_TRY(scan_excl(dg, cdeg, T + 1, s));
    prof.step_built();
    int32_t* out = nullptr;
    int32_t* rec1 = nullptr;
    ND_CUDA_TRY(nd_alloc(&out, n * m, s));
    ND_CUDA_TRY(nd_alloc(&cs.counts, n, s));
    ND_CUDA_TRY(nd_alloc(&cs.rec_cnt, n, s));
    ND_CUDA_TRY(cudaMemsetAsync(cs.rec_cnt, 0, n * sizeof(int64_t), s));
    if (kind == ND_MVS) ND_CUDA_TRY(nd_alloc(&rec1, n * m, s));
    if (kind != ND_CLUSTERGCN) {
      SelCtx c{g, kind, m, max_size, V, key_base(seed, (uint64_t)step, 0, 0), sample_lo, toff, tv,
               cdeg, size, alive, cum, distribution, out, rec1};
      if (n * m) k_select<<<nd_grid(n * m, 256, 148 * 64), 256, 0, s>>>(c, n);
    } else {
      ND_CUDA_TRY(cudaMemsetAsync(out, 0xFF, n * m * sizeof(int32_t), s));  // all NULL
    }
    // recorded edges
    if (kind == ND_IMPORTANCE) {
      int64_t *tl = nullptr, *tri_off = nullptr;
      ND_CUDA_TRY(nd_alloc(&tl, n + 1, s));
      ND_CUDA_TRY(nd_alloc(&tri_off, n + 1, s));
      k_tri_len<<<nd_grid(n + 1, 256), 256, 0, s>>>(toff, alive, n, m, tl);
      ND_TRY(scan_excl(tl, tri_off, n + 1, s));
      int64_t tot_tri = 0;
      ND_TRY(dcopy_to_host(&tot_tri, tri_off + n, 1, s));
      uint8_t* fl = nullptr;
      int64_t* pos = nullptr;
      ND_CUDA_TRY(nd_alloc(&fl, tot_tri + 1, s));
      ND_CUDA_TRY(nd_alloc(&pos, tot_tri + 1, s));
      ND_CUDA_TRY(cudaMemsetAsync(fl, 0, tot_tri + 1, s));
      if (tot_tri)
        k_imp_hits<<<nd_grid(n * m * 32, 256, 148 * 64), 256, 0, s>>>(g, toff, tv, out, alive,
                                                                      tri_off, n, m, tot_tri, fl);
      // exclusive scan of the byte flags, widened on the fly
      {
        auto it = thrust::make_transform_iterator(fl, WidenFlag{});
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, it, pos, tot_tri + 1, s);
        void* tmp = nullptr;
        ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
        ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, it, pos, tot_tri + 1, s));
        nd_free(tmp, s);
      }
      ND_TRY(dcopy_to_host(&cs.nrec, pos + tot_tri, 1, s));
      ND_CUDA_TRY(nd_alloc(&cs.rec_t, cs.nrec, s));
      ND_CUDA_TRY(nd_alloc(&cs.rec_v, cs.nrec, s));
      if (tot_tri)
        k_imp_write<<<nd_grid(tot_tri, 256, 148 * 64), 256, 0, s>>>(toff, tv, out, tri_off, n, m,
                                                                    tot_tri, fl, pos, cs.rec_t,
                                                                    cs.rec_v);
      if (n) k_seg_counts<<<nd_grid(n, 256), 256, 0, s>>>(tri_off, pos, n, cs.rec_cnt);
      nd_free(tl, s); nd_free(tri_off, s); nd_free(fl, s); nd_free(pos, s);
    } else if (kind == ND_MVS) {
      int64_t *f = nullptr, *pos = nullptr;
      ND_CUDA_TRY(nd_alloc(&f, n * m + 1, s));
      ND_CUDA_TRY(nd_alloc(&pos, n * m + 1, s));
      k_mvs_flags<<<nd_grid(n * m + 1, 256), 256, 0, s>>>(rec1, n * m, f);
      ND_TRY(scan_excl(f, pos, n * m + 1, s));
      ND_TRY(dcopy_to_host(&cs.nrec, pos + n * m, 1, s));
      ND_CUDA_TRY(nd_alloc(&cs.rec_t, cs.nrec, s));
      ND_CUDA_TRY(nd_alloc(&cs.rec_v, cs.nrec, s));
      if (n * m) k_mvs_write<<<nd_grid(n * m, 256), 256, 0, s>>>(rec1, out, f, pos, n * m, cs.rec_t, cs.rec_v);
      if (n) k_mvs_counts<<<nd_grid(n, 256), 256, 0, s>>>(pos, n, m, cs.rec_cnt);
      nd_free(f, s); nd_free(pos, s);
    } else if (kind == ND_CLUSTERGCN) {
      // the sample's own roots as a bitmap (np.isin against sample.roots)
      const int64_t words = (V + 31) / 32;
      uint32_t* bm = nullptr;
      ND_CUDA_TRY(nd_alloc(&bm, n * words, s));
      ND_CUDA_TRY(cudaMemsetAsync(bm, 0, n * words * sizeof(uint32_t), s));
      if (n_roots) {
        dim3 gr((unsigned)std::min<int64_t>(1024, (n_roots / std::max<int64_t>(n, 1) + 255) / 256 + 1),
                (unsigned)std::min<int64_t>(n, 65535));
        k_bitmap_set<<<gr, 256, 0, s>>>(roff, roots, n, words, bm);
      }
      // m slots each record the same set (apps.py:372-379 runs per slot):
      // count once (per unit, then per sample), write once per slot
      int64_t ET = 0;
      ND_TRY(dcopy_to_host(&ET, cdeg + T, 1, s));
      const int64_t units = (ET + CG_UNIT - 1) / CG_UNIT;
      const CgArgs A{g, toff, tv, cdeg, n, T, bm, words};
      int64_t *ucnt = nullptr, *ubase = nullptr, *hb = nullptr;
      ND_CUDA_TRY(nd_alloc(&ucnt, units + 1, s));
      ND_CUDA_TRY(nd_alloc(&ubase, units + 1, s));
      ND_CUDA_TRY(nd_alloc(&hb, n + 1, s));
      ND_CUDA_TRY(cudaMemsetAsync(ucnt, 0, (units + 1) * sizeof(int64_t), s));
      if (units) k_cgcn<0><<<148 * 16, 256, 0, s>>>(A, ucnt, nullptr, nullptr, nullptr);
      ND_TRY(scan_excl(ucnt, ubase, units + 1, s));
      if (n && T) {
        k_cgcn_bounds<<<nd_grid((n + 1) * 32, 256), 256, 0, s>>>(A, ubase, hb);
        k_diff<<<nd_grid(n, 256), 256, 0, s>>>(hb, n, cs.rec_cnt);
      }
      int64_t nr = 0;
      ND_TRY(dcopy_to_host(&nr, ubase + units, 1, s));
      for (int64_t sl = 0; sl < m; sl++) {
        int64_t *rt = nullptr, *rv = nullptr;
        ND_CUDA_TRY(nd_alloc(&rt, cs.nrec + nr, s));
        ND_CUDA_TRY(nd_alloc(&rv, cs.nrec + nr, s));
        if (cs.nrec) {
          ND_CUDA_TRY(cudaMemcpyAsync(rt, cs.rec_t, cs.nrec * 8, cudaMemcpyDeviceToDevice, s));
          ND_CUDA_TRY(cudaMemcpyAsync(rv, cs.rec_v, cs.nrec * 8, cudaMemcpyDeviceToDevice, s));
        }
        if (units)
          k_cgcn<1><<<148 * 16, 256, 0, s>>>(A, nullptr, ubase, rt + cs.nrec, rv + cs.nrec);
        nd_free(cs.rec_t, s);
        nd_free(cs.rec_v, s);
        cs.rec_t = rt;
        cs.rec_v = rv;
        cs.nrec += nr;
      }
      nd_free(bm, s); nd_free(ucnt, s); nd_free(ubase, s); nd_free(hb, s);
    }
    total_rec += cs.nrec;
    prof.step_sampled();
    const bool uniq = nd_unique_at(host_unique, n_unique, step);
    // next transits = non-NULL slots (stable); with unique() the sorted distinct
    // values per sample (finish_step, driver.py:165-172)
    int32_t* nsid = nullptr;
    {
      int64_t *f = nullptr, *pos = nullptr;
      ND_CUDA_TRY(nd_alloc(&f, n * m + 1, s));
      ND_CUDA_TRY(nd_alloc(&pos, n * m + 1, s));
      k_nonnull<<<nd_grid(n * m + 1, 256), 256, 0, s>>>(out, alive, n, m, f);
      ND_TRY(scan_excl(f, pos, n * m + 1, s));
      int64_t nt = 0;
      ND_TRY(dcopy_to_host(&nt, pos + n * m, 1, s));
      ND_CUDA_TRY(nd_alloc(&cs.ntv, nt, s));
      ND_CUDA_TRY(nd_alloc(&cs.ntoff, n + 1, s));
      if (uniq) {
        ND_CUDA_TRY(nd_alloc(&nsid, nt, s));
        if (n * m) k_next_transits_sid<<<nd_grid(n * m, 256), 256, 0, s>>>(out, f, pos, n * m, m, cs.ntv, nsid);
        int32_t *usid = nullptr, *uval = nullptr;
        int64_t um = 0;
        int64_t* cnt_u = nullptr;
        ND_CUDA_TRY(nd_alloc(&cnt_u, n + 1, s));
        ND_TRY(nd_dedup_segments(nsid, cs.ntv, nt, n, V, &usid, &uval, &um, cnt_u, s));
        ND_CUDA_TRY(cudaMemsetAsync(cnt_u + n, 0, sizeof(int64_t), s));
        ND_TRY(scan_excl(cnt_u, cs.ntoff, n + 1, s));
        if (n) k_size_add<<<nd_grid(n, 256), 256, 0, s>>>(size, cnt_u, n);
        if (n) ND_CUDA_TRY(cudaMemcpyAsync(cs.counts, cnt_u, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        nd_free(cs.ntv, s);
        nd_free(nsid, s);
        nd_free(usid, s);
        nd_free(cnt_u, s);
        cs.ntv = uval;
        nt = um;
        cs.nvals = um;
        ND_CUDA_TRY(nd_alloc(&cs.vals, um, s));
        if (um) k_widen32<<<nd_grid(um, 256), 256, 0, s>>>(uval, um, cs.vals);
      } else {
        if (n * m) k_next_transits<<<nd_grid(n * m, 256), 256, 0, s>>>(out, f, pos, n * m, cs.ntv);
        k_next_toff<<<nd_grid(n + 1, 256), 256, 0, s>>>(pos, n, m, cs.ntoff, size);
        // per-step slots of alive samples (NULLs kept)
        if (n) k_step_counts<<<nd_grid(n, 256), 256, 0, s>>>(alive, n, m, cs.counts, nullptr);
        int64_t *ai = nullptr, *abase = nullptr;
        ND_CUDA_TRY(nd_alloc(&ai, n + 1, s));
        ND_CUDA_TRY(nd_alloc(&abase, n + 1, s));
        k_alive_idx<<<nd_grid(n + 1, 256), 256, 0, s>>>(alive, n, ai);
        ND_TRY(scan_excl(ai, abase, n + 1, s));
        int64_t na = 0;
        ND_TRY(dcopy_to_host(&na, abase + n, 1, s));
        cs.nvals = na * m;
        ND_CUDA_TRY(nd_alloc(&cs.vals, cs.nvals, s));
        if (n * m) k_emit_slots<<<nd_grid(n * m, 256), 256, 0, s>>>(out, alive, abase, n, m, cs.vals);
        nd_free(ai, s);
        nd_free(abase, s);
      }
      ND_CUDA_TRY(cudaMemcpyAsync(toff, cs.ntoff, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
      T = nt;
      tv = cs.ntv;
      nd_free(f, s);
      nd_free(pos, s);
    }
    nd_free(out, s); nd_free(rec1, s); nd_free(dg, s); nd_free(cdeg, s);
    ND_CUDA_TRY(cudaGetLastError());
    steps_v.push_back(cs);
    step++;
  }
  const int64_t n_steps = step;
  ND_CUDA_TRY(cudaStreamSynchronize(s));

  // ---- outputs ------------------------------------------------------------------------
  int32_t* final_ids = nullptr;  // int32 vertex ids (F_FINAL_IDS32; int64 derived on request)
  int64_t *final_off = nullptr, *flen = nullptr, *fill = nullptr,
          *roots_out = nullptr, *roots_off = nullptr, *step_counts = nullptr, *step_vals = nullptr,
          *rec_counts = nullptr, *rec_t = nullptr, *rec_v = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&fill, n, s));
  // size[] = roots + all non-NULL slots = final row lengths
  ND_CUDA_TRY(cudaMemsetAsync(flen + n, 0, sizeof(int64_t), s));
  if (n) ND_CUDA_TRY(cudaMemcpyAsync(flen, size, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  ND_TRY(scan_excl(flen, final_off, n + 1, s));
  int64_t total = 0;
  ND_TRY(dcopy_to_host(&total, final_off + n, 1, s));
  ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
  if (n) k_coll_final<<<seg_grid(n_roots, n), 256, 0, s>>>(roff, roots, n, final_off, final_ids);
  {
    // fill = root counts
    std::vector<int64_t> hr(n);
    for (int64_t i = 0; i < n; i++) hr[i] = h_roff[i + 1] - h_roff[i];
    if (n) ND_CUDA_TRY(cudaMemcpyAsync(fill, hr.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
  }
  for (auto& cs : steps_v) {
    if (n) {
      k_coll_final_step<<<seg_grid(cs.nvals, n), 256, 0, s>>>(cs.ntv, cs.ntoff, n, final_off, fill,
                                                             final_ids);
      k_fill_add<<<nd_grid(n, 256), 256, 0, s>>>(fill, cs.ntoff, n);
    }
  }
  ND_CUDA_TRY(nd_alloc(&roots_out, n_roots, s));
  ND_CUDA_TRY(nd_alloc(&roots_off, n + 1, s));
  if (n_roots) k_widen32<<<nd_grid(n_roots, 256), 256, 0, s>>>(roots, n_roots, roots_out);
  ND_CUDA_TRY(cudaMemcpyAsync(roots_off, roff, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  int64_t tot_vals = 0;
  for (auto& cs : steps_v) tot_vals += cs.nvals;
  ND_CUDA_TRY(nd_alloc(&step_counts, n_steps * n, s));
  ND_CUDA_TRY(nd_alloc(&step_vals, tot_vals, s));
  ND_CUDA_TRY(nd_alloc(&rec_counts, n_steps * n, s));
  ND_CUDA_TRY(nd_alloc(&rec_t, total_rec, s));
  ND_CUDA_TRY(nd_alloc(&rec_v, total_rec, s));
  int64_t pv = 0, pr = 0;
  for (int64_t st = 0; st < n_steps; st++) {
    CStep& cs = steps_v[st];
    if (n) {
      ND_CUDA_TRY(cudaMemcpyAsync(step_counts + st * n, cs.counts, n * 8, cudaMemcpyDeviceToDevice, s));
      ND_CUDA_TRY(cudaMemcpyAsync(rec_counts + st * n, cs.rec_cnt, n * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (cs.nvals) ND_CUDA_TRY(cudaMemcpyAsync(step_vals + pv, cs.vals, cs.nvals * 8, cudaMemcpyDeviceToDevice, s));
    if (cs.nrec) {
      ND_CUDA_TRY(cudaMemcpyAsync(rec_t + pr, cs.rec_t, cs.nrec * 8, cudaMemcpyDeviceToDevice, s));
      ND_CUDA_TRY(cudaMemcpyAsync(rec_v + pr, cs.rec_v, cs.nrec * 8, cudaMemcpyDeviceToDevice, s));
    }
    pv += cs.nvals;
    pr += cs.nrec;
  }
  ND_CUDA_TRY(cudaGetLastError());
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  for (auto& cs : steps_v) {
    nd_free(cs.counts, s); nd_free(cs.vals, s); nd_free(cs.rec_cnt, s); nd_free(cs.rec_t, s);
    nd_free(cs.rec_v, s); nd_free(cs.ntv, s); nd_free(cs.ntoff, s);
  }
  nd_free(size, s); nd_free(alive, s); nd_free(toff, s); nd_free(cum, s); nd_free(flen, s);
  nd_free(fill, s); nd_free(roff, s); nd_free(roots, s);
  nd_result* res = new nd_result();
  res->stream = s;
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n_roots;
  res->total_recorded = total_rec;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n_roots);
  res->set(ND_F_ROOTS_OFF, roots_off, n + 1);
  res->set(ND_F_STEP_COUNTS, step_counts, n_steps * n);
  res->set(ND_F_STEP_VALS, step_vals, tot_vals);
  res->set(ND_F_REC_COUNTS, rec_counts, n_steps * n);
  res->set(ND_F_REC_T, rec_t, total_rec);
  res->set(ND_F_REC_V, rec_v, total_rec);
  res->set(ND_F_STATS, stats, 4 * n_steps);
  res->counters[NDC_STEPS] = n_steps;
  if (prof.on) {  // the stream was synchronised above
    const auto st = prof.to_result(res);
    res->prof_ms[0] = st[0];
    res->prof_ms[1] = st[1];
  }
  prof.destroy();
  *out_res = res;
  return ND_OK;
}
