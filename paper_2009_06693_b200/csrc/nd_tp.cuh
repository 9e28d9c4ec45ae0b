// nd_tp.cuh — the transit-parallel step machinery shared by the engines.
//
// Per step (transit_parallel.py:185-230, paper §6 / PAPER.md:793-840):
//   1. transit -> sample inversion: CUB stable radix sort of (transit key,
//      payload) over ceil(log2 V) bits (build_transit_map, :71-83);
//   2. run-length boundaries -> dense group ids (inclusive scan of flags) and
//      group starts;
//   3. work classes by members*m: small < 32, medium 32..1024, large > 1024
//      (partition_work_classes, :86-101);
//   4. class kernels:
//        small  — one thread per item; lanes of a warp that share a transit
//                 form a sub-warp (__match_any_sync) and broadcast the row
//                 header with shuffles (paper's sub-warp kernel);
//        medium — one CTA per group; the transit's adjacency (col, prefix,
//                 weights as the app needs) is staged in shared memory with
//                 cp.async and every member samples from it;
//        large  — the group's members are split into 1024-item chunks, one
//                 CTA each, each staging the adjacency (global fallback when
//                 the row exceeds the staging budget).
// Outputs are order independent (keyed RNG), so group member order and the
// order of the next-step state do not affect results.
#pragma once

#include <cub/cub.cuh>

#include "nd_item.cuh"

namespace nd {

constexpr int TP_BLOCK = 256;
constexpr int LARGE_CHUNK = 1024;
constexpr int STAGE_BYTES = 48 * 1024;

struct StageSpec {
  int need_pre = 0;
  int need_w = 0;
  int64_t cap = 0;  // entries that fit
};

inline StageSpec stage_spec(int need_pre, int need_w) {
  StageSpec s;
  s.need_pre = need_pre;
  s.need_w = need_w;
  const int per = 4 + 8 * need_pre + 8 * need_w;
  s.cap = STAGE_BYTES / per;
  return s;
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Stage v's row [lo, lo+deg) into shared memory; returns the shared row view.
__device__ __forceinline__ SRow stage_row(const DevGraph& g, int64_t lo, int64_t deg,
                                          const StageSpec& sp, unsigned char* smem) {
  double* s_pre = reinterpret_cast<double*>(smem);
  double* s_w = s_pre + (sp.need_pre ? sp.cap : 0);
  int32_t* s_col = reinterpret_cast<int32_t*>(s_w + (sp.need_w ? sp.cap : 0));
  for (int64_t k = threadIdx.x; k < deg; k += blockDim.x) {
    cp_async4(s_col + k, g.col + lo + k);
    if (sp.need_pre) cp_async8(s_pre + k, g.pre + lo + k);
    if (sp.need_w) cp_async8(s_w + k, g.w + lo + k);
  }
  cp_async_wait_all();
  __syncthreads();
  return SRow{s_col, s_pre, s_w};
}

// warp-aggregated append of one element per alive lane; returns slot or -1
__device__ __forceinline__ int64_t warp_append(bool alive, int* counter) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, alive);
  const int lane = threadIdx.x & 31;
  int base = 0;
  const int leader = __ffs(m) - 1;
  if (m && lane == leader) base = atomicAdd(counter, __popc(m));
  const int src = m ? leader : (__ffs(act) - 1);
  base = __shfl_sync(act, base, src);
  if (!alive) return -1;
  return base + __popc(m & ((1u << lane) - 1));
}

// per-block reduction of the byte/try counters into global counters
__device__ __forceinline__ void flush_stats(const ItemStats& st, unsigned long long* ctr) {
  unsigned long long b = (unsigned long long)st.bytes, t = (unsigned long long)st.tries,
                     q = (unsigned long long)st.sect;
  for (int o = 16; o > 0; o >>= 1) {
    b += __shfl_down_sync(0xffffffffu, b, o);
    t += __shfl_down_sync(0xffffffffu, t, o);
    q += __shfl_down_sync(0xffffffffu, q, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (b) atomicAdd(ctr + 0, b);
    if (t) atomicAdd(ctr + 1, t);
    if (q) atomicAdd(ctr + 2, q);
  }
}

// ---- grouping kernels ------------------------------------------------------------

static __global__ void k_mark(const uint32_t* __restrict__ keys, int64_t n, int* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

static __global__ void k_gstart(const int* __restrict__ flags, const int* __restrict__ gid, int64_t n,
                         int* __restrict__ gstart, int* __restrict__ n_groups) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flags[i]) gstart[gid[i] - 1] = (int)i;
    if (i == n - 1) {
      gstart[gid[i]] = (int)n;
      *n_groups = gid[i];
    }
  }
}

// classes by work = members*m; per-step class counts into stats[0..3];
// medium groups and large-group chunks appended to work lists
static __global__ void k_classify(const int* __restrict__ gstart, const int* __restrict__ n_groups,
                           int64_t m, signed char* __restrict__ gclass, int* __restrict__ med_list,
                           int* __restrict__ n_med, int2* __restrict__ large_units,
                           int* __restrict__ n_large, unsigned long long* __restrict__ stats) {
  const int G = *n_groups;
  int cnt[3] = {0, 0, 0};
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    const int size = gstart[g + 1] - gstart[g];
    const int64_t work = (int64_t)size * m;
    int c = work < SMALL_MAX_WORK ? 0 : (work <= LARGE_MIN_WORK ? 1 : 2);
    gclass[g] = (signed char)c;
    cnt[c]++;
    if (c == 1) {
      med_list[atomicAdd(n_med, 1)] = g;
    } else if (c == 2) {
      const int chunks = (size + LARGE_CHUNK - 1) / LARGE_CHUNK;
      const int b = atomicAdd(n_large, chunks);
      for (int k = 0; k < chunks; k++) large_units[b + k] = make_int2(g, k);
    }
  }
  for (int c = 0; c < 3; c++) {
    int v = cnt[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(stats + c, (unsigned long long)v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats + 3, (unsigned long long)G);
}

// ---- class kernels, generic over the per-item action ------------------------------
// Act provides:  template <class RowT> __device__ void operator()(int64_t i,
//                  int64_t v, uint64_t val, const RowT& row, int64_t deg,
//                  ItemStats& st) const;   (must be reached by every active lane)

template <class Act>
__global__ void __launch_bounds__(TP_BLOCK) k_flat(const uint32_t* __restrict__ keys,
                                                   const uint64_t* __restrict__ vals, int64_t n,
                                                   DevGraph g, Act act,
                                                   unsigned long long* __restrict__ ctr) {
  ItemStats st;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const int64_t v = keys[i];
    const int64_t lo = __ldg(g.row + v), deg = __ldg(g.row + v + 1) - lo;
    st.bytes += SECTOR + 8;
    act(i, v, vals[i], grow(view(g), lo), deg, st);
  }
  flush_stats(st, ctr);
}

template <class Act>
__global__ void __launch_bounds__(TP_BLOCK) k_small(const uint32_t* __restrict__ keys,
                                                    const uint64_t* __restrict__ vals, int64_t n,
                                                    const int* __restrict__ gid,
                                                    const signed char* __restrict__ gclass,
                                                    DevGraph g, Act act,
                                                    unsigned long long* __restrict__ ctr) {
  ItemStats st;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && gclass[gid[i] - 1] == 0) {
    const uint32_t v = keys[i];
    // sub-warp: lanes sharing the transit read its row header once
    const unsigned act_m = __activemask();
    const unsigned peers = __match_any_sync(act_m, v);
    const int leader = __ffs(peers) - 1;
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = 0;
    if (lane == leader) {
      lo = __ldg(g.row + v);
      hi = __ldg(g.row + v + 1);
    }
    lo = __shfl_sync(act_m, lo, leader);
    hi = __shfl_sync(act_m, hi, leader);
    st.bytes += SECTOR + 8;
    act(i, (int64_t)v, vals[i], grow(view(g), lo), hi - lo, st);
  }
  flush_stats(st, ctr);
}

// one CTA per medium group; persistent over the list
template <class Act>
__global__ void __launch_bounds__(TP_BLOCK) k_medium(const uint32_t* __restrict__ keys,
                                                     const uint64_t* __restrict__ vals,
                                                     const int* __restrict__ gstart,
                                                     const int* __restrict__ med_list,
                                                     const int* __restrict__ n_med, DevGraph g,
                                                     StageSpec sp, Act act,
                                                     unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  ItemStats st;
  const int U = *n_med;
  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    const int gi = med_list[u];
    const int start = gstart[gi], size = gstart[gi + 1] - start;
    const int64_t v = keys[start];
    const int64_t lo = __ldg(g.row + v), deg = __ldg(g.row + v + 1) - lo;
    // stage only when the members re-read a fair share of the row (each
    // member touches ~1-2 entries); otherwise the copy costs more than it saves
    if (deg <= sp.cap && deg > 0 && 4 * (int64_t)size >= deg) {
      SRow r = stage_row(g, lo, deg, sp, smem);
      for (int k = threadIdx.x; k < size; k += blockDim.x) {
        st.bytes += SECTOR + 8;
        act(start + k, v, vals[start + k], r, deg, st);
      }
    } else {
      auto r = grow(view(g), lo);
      for (int k = threadIdx.x; k < size; k += blockDim.x) {
        st.bytes += SECTOR + 8;
        act(start + k, v, vals[start + k], r, deg, st);
      }
    }
    __syncthreads();
  }
  flush_stats(st, ctr);
}

template <class Act>
__global__ void __launch_bounds__(TP_BLOCK) k_large(const uint32_t* __restrict__ keys,
                                                    const uint64_t* __restrict__ vals,
                                                    const int* __restrict__ gstart,
                                                    const int2* __restrict__ units,
                                                    const int* __restrict__ n_units, DevGraph g,
                                                    StageSpec sp, Act act,
                                                    unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  ItemStats st;
  const int U = *n_units;
  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    const int2 un = units[u];
    const int gs = gstart[un.x], ge = gstart[un.x + 1];
    const int start = gs + un.y * LARGE_CHUNK;
    const int end = min(ge, start + LARGE_CHUNK);
    const int64_t v = keys[gs];
    const int64_t lo = __ldg(g.row + v), deg = __ldg(g.row + v + 1) - lo;
    if (deg <= sp.cap && deg > 0 && 4 * (int64_t)(end - start) >= deg) {
      SRow r = stage_row(g, lo, deg, sp, smem);
      for (int k = start + threadIdx.x; k < end; k += blockDim.x) {
        st.bytes += SECTOR + 8;
        act(k, v, vals[k], r, deg, st);
      }
    } else {
      auto r = grow(view(g), lo);
      for (int k = start + threadIdx.x; k < end; k += blockDim.x) {
        st.bytes += SECTOR + 8;
        act(k, v, vals[k], r, deg, st);
      }
    }
    __syncthreads();
  }
  flush_stats(st, ctr);
}

// ---- host-side driver of one TP step ------------------------------------------------

struct TPScratch {
  int64_t cap = 0;
  int* flags = nullptr;
  int* gid = nullptr;
  int* gstart = nullptr;
  signed char* gclass = nullptr;
  int* med_list = nullptr;
  int2* large_units = nullptr;
  int* counters = nullptr;  // [0]=n_groups [1]=n_med [2]=n_large
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;

  int alloc(int64_t n, int key_bits, cudaStream_t s) {
    cap = n;
    ND_CUDA_TRY(nd_alloc(&flags, n, s));
    ND_CUDA_TRY(nd_alloc(&gid, n, s));
    ND_CUDA_TRY(nd_alloc(&gstart, n + 1, s));
    ND_CUDA_TRY(nd_alloc(&gclass, n, s));
    ND_CUDA_TRY(nd_alloc(&med_list, n, s));
    ND_CUDA_TRY(nd_alloc(&large_units, n, s));
    ND_CUDA_TRY(nd_alloc(&counters, 4, s));
    size_t b1 = 0, b2 = 0;
    cub::DoubleBuffer<uint32_t> dk(nullptr, nullptr);
    cub::DoubleBuffer<uint64_t> dv(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, b1, dk, dv, (int)n, 0, key_bits, s);
    cub::DeviceScan::InclusiveSum(nullptr, b2, flags, gid, (int)n, s);
    cub_bytes = b1 > b2 ? b1 : b2;
    ND_CUDA_TRY(nd_alloc((char**)&cub_tmp, cub_bytes, s));
    return ND_OK;
  }
  void release(cudaStream_t s) {
    nd_free(flags, s); nd_free(gid, s); nd_free(gstart, s); nd_free(gclass, s);
    nd_free(med_list, s); nd_free(large_units, s); nd_free(counters, s); nd_free(cub_tmp, s);
  }
};

inline int key_bits_for(int64_t V) {
  int b = 1;
  while ((1ll << b) < V) b++;
  return b;
}

// Group + classify one step's sorted (keys, vals) and run the three class
// kernels with `act`.  m = slots per pair (work = members*m).  stats[0..3]
// receive the step's {small, medium, large, groups} counts.
template <class Act>
int tp_run_sorted(const uint32_t* keys, const uint64_t* vals, int64_t n, int64_t m,
                  const DevGraph& g, const StageSpec& sp, const Act& act, TPScratch& S,
                  unsigned long long* ctr, unsigned long long* stats, cudaStream_t s) {
  if (n == 0) return ND_OK;
  k_mark<<<nd_grid(n, 256), 256, 0, s>>>(keys, n, S.flags);
  size_t tb = S.cub_bytes;
  ND_CUDA_TRY(cub::DeviceScan::InclusiveSum(S.cub_tmp, tb, S.flags, S.gid, (int)n, s));
  ND_CUDA_TRY(cudaMemsetAsync(S.counters, 0, 4 * sizeof(int), s));
  k_gstart<<<nd_grid(n, 256), 256, 0, s>>>(S.flags, S.gid, n, S.gstart, S.counters);
  k_classify<<<nd_grid(n, 256), 256, 0, s>>>(S.gstart, S.counters, m, S.gclass, S.med_list,
                                              S.counters + 1, S.large_units, S.counters + 2,
                                              stats);
  k_small<Act><<<(unsigned)((n + TP_BLOCK - 1) / TP_BLOCK), TP_BLOCK, 0, s>>>(
      keys, vals, n, S.gid, S.gclass, g, act, ctr);
  const int pgrid = 148 * 4;
  k_medium<Act><<<pgrid, TP_BLOCK, STAGE_BYTES, s>>>(keys, vals, S.gstart, S.med_list,
                                                     S.counters + 1, g, sp, act, ctr);
  k_large<Act><<<pgrid, TP_BLOCK, STAGE_BYTES, s>>>(keys, vals, S.gstart, S.large_units,
                                                    S.counters + 2, g, sp, act, ctr);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

// stable radix sort of the step's (transit, payload) pairs (build_transit_map)
inline int tp_sort(cub::DoubleBuffer<uint32_t>& dk, cub::DoubleBuffer<uint64_t>& dv, int64_t n,
                   int key_bits, TPScratch& S, cudaStream_t s) {
  if (n == 0) return ND_OK;
  size_t tb = S.cub_bytes;
  ND_CUDA_TRY(cub::DeviceRadixSort::SortPairs(S.cub_tmp, tb, dk, dv, (int)n, 0, key_bits, s));
  return ND_OK;
}

template <class Act>
int sp_step(const uint32_t* keys, const uint64_t* vals, int64_t n, const DevGraph& g,
            const Act& act, unsigned long long* ctr, unsigned long long* stats, cudaStream_t s) {
  if (n == 0) return ND_OK;
  k_flat<Act><<<(unsigned)((n + TP_BLOCK - 1) / TP_BLOCK), TP_BLOCK, 0, s>>>(keys, vals, n, g, act,
                                                                            ctr);
  ND_CUDA_TRY(cudaGetLastError());
  return ND_OK;
}

}  // namespace nd
