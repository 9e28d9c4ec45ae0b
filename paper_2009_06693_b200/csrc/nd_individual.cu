// nd_individual.cu — multi-slot individual apps (GraphSAGE k-hop) on device.
//
// The reference's generic run loop (driver.py:203-235) with StepPlan
// semantics (driver.py:80-144): at step s every alive sample contributes one
// pair per transit (sample-major; transit_idx = rank among the previous
// step's non-NULL slots, core.py:84-97,168-184) and each pair expands into
// m = fanout[s] slots at out[pair*m + slot].  A sample stays alive while it
// has transits (core.py:195-203).
//
// Transit-parallel step (transit_parallel.py:185-230): the pairs are radix
// sorted by transit, grouped, classed by work = members*m and run by
//   small  — one warp per group, lanes = the group's (member, slot) items
//            (the paper's sub-warp kernel: one row header, m lanes per sample);
//   medium — one CTA per group, adjacency staged in shared memory (cp.async);
//   large  — groups split into chunks of ~1024 items, one CTA per chunk.
// The next step's pairs come from a stable compaction of the non-NULL slots
// (exclusive scan), which also yields transit_idx and per-sample counts.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include <string>
#include <vector>

#include "nd_bulk.cuh"
#include "nd_tp.cuh"

using namespace nd;

namespace {

constexpr int IND_BLOCK = 256;

struct IndCtx {
  GView<int32_t> gv;
  NdApp a;
  uint64_t base0;
  int64_t sample_lo;
  int64_t m;
  const uint32_t* pt;    // pair transit
  const int32_t* psid;   // pair sample (local)
  const int32_t* ptix;   // pair transit index
  int32_t* out;          // [P*m]
  int* stall;
};

template <class RowT>
__device__ __forceinline__ void ind_item(const IndCtx& c, int64_t p, int64_t slot, int64_t v,
                                         const RowT& row, int64_t deg, ItemStats& st) {
  int stl = 0;
  const uint64_t ik = key_item((uint64_t)(c.sample_lo + c.psid[p]), (uint64_t)c.ptix[p],
                               (uint64_t)slot);
  const int64_t o = run_item(c.gv, row, c.a, v, deg, -1, c.base0, ik, st, &stl);
  if (stl) atomicExch(c.stall, 1);
  c.out[p * c.m + slot] = (int32_t)o;
}

// sample-parallel: one thread per (pair, slot) item in plan order
__global__ void __launch_bounds__(IND_BLOCK) k_ind_flat(IndCtx c, int64_t P,
                                                        unsigned long long* ctr) {
  ItemStats st;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < P * c.m) {
    const int64_t p = j / c.m, slot = j - p * c.m;
    const int64_t v = c.pt[p];
    const int64_t lo = __ldg(c.gv.row + v), deg = __ldg(c.gv.row + v + 1) - lo;
    if (slot == 0) st.bytes += SECTOR + 8;
    ind_item(c, p, slot, v, grow(c.gv, lo), deg, st);
  }
  flush_stats(st, ctr);
}

// classes for the multi-slot engine: every class gets a work list
__global__ void k_ind_classify(const int* __restrict__ gstart, const int* __restrict__ n_groups,
                               int64_t m, int* __restrict__ small_list, int* __restrict__ n_small,
                               int2* __restrict__ units, int* __restrict__ n_units,
                               unsigned long long* __restrict__ stats) {
  const int G = *n_groups;
  int cnt[3] = {0, 0, 0};
  const int per_chunk = (int)(LARGE_CHUNK / m > 0 ? LARGE_CHUNK / m : 1);
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    const int size = gstart[g + 1] - gstart[g];
    const int64_t work = (int64_t)size * m;
    const int c = work < SMALL_MAX_WORK ? 0 : (work <= LARGE_MIN_WORK ? 1 : 2);
    cnt[c]++;
    if (c == 0) {
      small_list[atomicAdd(n_small, 1)] = g;
    } else if (c == 1) {
      units[atomicAdd(n_units, 1)] = make_int2(g, -1);
    } else {
      const int chunks = (size + per_chunk - 1) / per_chunk;
      const int b = atomicAdd(n_units, chunks);
      for (int k = 0; k < chunks; k++) units[b + k] = make_int2(g, k);
    }
  }
  for (int c = 0; c < 3; c++) {
    int v = cnt[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(stats + c, (unsigned long long)v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats + 3, (unsigned long long)G);
}

// small class: one warp per group; lanes walk the group's (member, slot) items
__global__ void __launch_bounds__(IND_BLOCK) k_ind_small(IndCtx c, const uint32_t* __restrict__ keys,
                                                         const uint64_t* __restrict__ vals,
                                                         const int* __restrict__ gstart,
                                                         const int* __restrict__ list,
                                                         const int* __restrict__ n_list,
                                                         unsigned long long* ctr) {
  ItemStats st;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int U = *n_list;
  for (int u = warp; u < U; u += nwarps) {
    const int g = list[u];
    const int gs = gstart[g], size = gstart[g + 1] - gs;
    const int64_t v = keys[gs];
    int64_t lo = 0, hi = 0;
    if (lane == 0) {
      lo = __ldg(c.gv.row + v);
      hi = __ldg(c.gv.row + v + 1);
    }
    lo = __shfl_sync(0xffffffffu, lo, 0);
    hi = __shfl_sync(0xffffffffu, hi, 0);
    const auto row = grow(c.gv, lo);
    const int64_t items = (int64_t)size * c.m;
    for (int64_t j = lane; j < items; j += 32) {
      const int64_t q = gs + j / c.m, slot = j - (j / c.m) * c.m;
      if (slot == 0) st.bytes += SECTOR + 8;
      ind_item(c, (int64_t)vals[q], slot, v, row, hi - lo, st);
    }
  }
  flush_stats(st, ctr);
}

// medium groups (chunk -1) and large-group chunks: one CTA each, row staged
__global__ void __launch_bounds__(IND_BLOCK) k_ind_group(IndCtx c, const uint32_t* __restrict__ keys,
                                                         const uint64_t* __restrict__ vals,
                                                         const int* __restrict__ gstart,
                                                         const int2* __restrict__ units,
                                                         const int* __restrict__ n_units,
                                                         DevGraph g, StageSpec sp,
                                                         unsigned long long* ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  ItemStats st;
  const int U = *n_units;
  const int per_chunk = (int)(LARGE_CHUNK / c.m > 0 ? LARGE_CHUNK / c.m : 1);
  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    const int2 un = units[u];
    const int gs = gstart[un.x], ge = gstart[un.x + 1];
    const int ms = un.y < 0 ? gs : gs + un.y * per_chunk;
    const int me = un.y < 0 ? ge : min(ge, ms + per_chunk);
    const int64_t v = keys[gs];
    const int64_t lo = __ldg(g.row + v), deg = __ldg(g.row + v + 1) - lo;
    const int64_t items = (int64_t)(me - ms) * c.m;
    if (deg > 0 && deg <= sp.cap && 4 * items >= deg) {
      const SRow r = stage_row(g, lo, deg, sp, smem);
      for (int64_t j = threadIdx.x; j < items; j += blockDim.x) {
        const int64_t q = ms + j / c.m, slot = j - (j / c.m) * c.m;
        if (slot == 0) st.bytes += SECTOR + 8;
        ind_item(c, (int64_t)vals[q], slot, v, r, deg, st);
      }
    } else {
      const auto r = grow(c.gv, lo);
      for (int64_t j = threadIdx.x; j < items; j += blockDim.x) {
        const int64_t q = ms + j / c.m, slot = j - (j / c.m) * c.m;
        if (slot == 0) st.bytes += SECTOR + 8;
        ind_item(c, (int64_t)vals[q], slot, v, r, deg, st);
      }
    }
    __syncthreads();
  }
  flush_stats(st, ctr);
}

__global__ void k_ind_init(const int64_t* __restrict__ roots64, const int32_t* __restrict__ roots32,
                           int64_t n, int64_t R, uint32_t* __restrict__ pt, int32_t* __restrict__ psid,
                           int32_t* __restrict__ ptix, int64_t* __restrict__ spo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / R;
    pt[i] = roots64 ? (uint32_t)roots64[i] : (uint32_t)roots32[i];
    psid[i] = (int32_t)s;
    ptix[i] = (int32_t)(i - s * R);
    if (i - s * R == 0) spo[s] = s * R;
    if (i == n * R - 1) spo[n] = n * R;
  }
}

__global__ void k_iota_pairs(const uint32_t* __restrict__ pt, int64_t P, uint32_t* __restrict__ keys,
                             uint64_t* __restrict__ vals) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    keys[p] = pt[p];
    vals[p] = (uint64_t)p;
  }
}

__global__ void k_add_fetch(unsigned long long* st, unsigned long long n) { st[3] += n; }

__global__ void k_flags_nonnull(const int32_t* __restrict__ out, int64_t n, int32_t* __restrict__ f) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    f[j] = out[j] >= 0;
}

// per-sample slot counts and non-NULL counts of this step
__global__ void k_ind_counts(const int64_t* __restrict__ spo, int64_t n, int64_t m,
                             const int64_t* __restrict__ sc, int64_t* __restrict__ cnt_row,
                             int64_t* __restrict__ nnz, int64_t* __restrict__ tot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { nnz[n] = 0; continue; }
    const int64_t a = spo[i] * m, b = spo[i + 1] * m;
    cnt_row[i] = b - a;
    const int64_t k = sc[b] - sc[a];
    nnz[i] = k;
  }
}

// next pairs from the non-NULL slots (stable), with transit_idx = rank in sample
__global__ void k_ind_compact(const int32_t* __restrict__ out, int64_t items, int64_t m,
                              const int64_t* __restrict__ sc, const int32_t* __restrict__ psid,
                              const int64_t* __restrict__ spo_next, uint32_t* __restrict__ npt,
                              int32_t* __restrict__ npsid, int32_t* __restrict__ nptix) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < items;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = out[j];
    if (v < 0) continue;
    const int64_t pos = sc[j];
    const int32_t s = psid[j / m];
    npt[pos] = (uint32_t)v;
    npsid[pos] = s;
    nptix[pos] = (int32_t)(pos - spo_next[s]);
  }
}

__global__ void k_tot_add(int64_t* __restrict__ tot, const int64_t* __restrict__ c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    tot[i] += c[i];
}

// transit_idx of a deduped list = rank within its sample; fallback flags
// (output.py:34-40: 0 < distinct < m)
__global__ void k_dedup_tix(const int32_t* __restrict__ sid, int64_t cnt,
                            const int64_t* __restrict__ spo_next, int32_t* __restrict__ tix) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt;
       j += (int64_t)gridDim.x * blockDim.x)
    tix[j] = (int32_t)(j - spo_next[sid[j]]);
}

__global__ void k_fallback(const int64_t* __restrict__ cnt, int64_t n, int64_t m,
                           uint8_t* __restrict__ fb, int* __restrict__ nfb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool f = cnt[i] > 0 && cnt[i] < m;
    fb[i] = f;
    if (f) atomicAdd(nfb, 1);
  }
}

// pairs of samples not flagged for the SP fallback (their transits form the
// TP groups, transit_parallel.py:200-209); flagged pairs count as fetches
__global__ void k_keep_unflagged(const uint32_t* __restrict__ pt, const int32_t* __restrict__ psid,
                                 const uint8_t* __restrict__ fb, int64_t P,
                                 int64_t* __restrict__ flag) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= P;
       p += (int64_t)gridDim.x * blockDim.x)
    flag[p] = (p < P && !fb[psid[p]]) ? 1 : 0;
}

__global__ void k_keep_write(const uint32_t* __restrict__ pt, const int64_t* __restrict__ flag,
                             const int64_t* __restrict__ pos, int64_t P, uint32_t* __restrict__ keys,
                             uint64_t* __restrict__ vals) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x)
    if (flag[p]) {
      keys[pos[p]] = pt[p];
      vals[pos[p]] = (uint64_t)p;
    }
}

// final rows: roots, then each step's compacted values at R + cum + tix
template <typename RootT>
__global__ void k_ind_roots(const RootT* __restrict__ roots, int64_t n, int64_t R,
                            const int64_t* __restrict__ off, int32_t* __restrict__ ids,
                            int64_t* __restrict__ roots_out, int64_t* __restrict__ roots_off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / R;
    ids[off[s] + (i - s * R)] = (int32_t)roots[i];
    roots_out[i] = (int64_t)roots[i];
    if (i - s * R == 0) roots_off[s] = s * R;
    if (i == n * R - 1) roots_off[n] = n * R;
  }
}

__global__ void k_ind_final(const uint32_t* __restrict__ npt, const int32_t* __restrict__ npsid,
                            const int32_t* __restrict__ nptix, int64_t cnt,
                            const int64_t* __restrict__ off, const int64_t* __restrict__ cum,
                            int64_t R, int32_t* __restrict__ ids) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = npsid[j];
    ids[off[s] + R + cum[s] + nptix[j]] = (int32_t)npt[j];
  }
}


__global__ void k_plus_r(int64_t* __restrict__ a, int64_t n, int64_t R) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] += R;
}


struct StepData {
  int32_t* out = nullptr;   // [P*m]
  int64_t items = 0;
  bool dedup = false;       // unique() step: the step's slots are npt (distinct, sorted)
  uint32_t* npt = nullptr;  // compacted next pairs
  int32_t* npsid = nullptr;
  int32_t* nptix = nullptr;
  int64_t nnext = 0;
  int64_t* cum = nullptr;   // per-sample nnz before this step (for the final rows)
};

// ---- fixed-layout sample-parallel run (k-hop without unique steps) -------------
// Every step's slots live in per-sample blocks with NULL holes where a parent
// slot was NULL: block of sample i at step s has B_s = R * m_0 * ... * m_s
// slots, item (i, p, slot) = parent p of the previous block (the roots at
// s = 0) and slot < m_s.  A non-NULL parent's transit_idx is its rank among
// the non-NULL entries of its block (core.py:97, driver.py:80-144), so the
// draws are exactly the run loop's.  Nothing between steps needs the host:
// one count pass, one scan and emit kernels build the reference's final rows,
// step rows and statistics, with a single host synchronisation at the end.

// per sample (one warp): rank of each non-NULL entry of `blk` (block size B),
// the sample's non-NULL count, and the step's pair total for the statistics
__global__ void k_fx_rank(const int32_t* __restrict__ blk, int64_t n, int64_t B,
                          int32_t* __restrict__ rank, int64_t* __restrict__ nn,
                          unsigned long long* __restrict__ fetch) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long tot = 0;
  for (int64_t i = warp; i < n; i += nw) {
    int32_t base = 0;
    for (int64_t p0 = 0; p0 < B; p0 += 32) {
      const int64_t p = p0 + lane;
      const bool ok = p < B && blk[i * B + p] >= 0;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (p < B) rank[i * B + p] = ok ? base + __popc(m & ((1u << lane) - 1)) : -1;
      base += __popc(m);
    }
    if (lane == 0) nn[i] = base;
    tot += base;
  }
  if (lane == 0 && tot) atomicAdd(fetch, tot);
}

// one thread per (sample, parent, slot) item of step s
// (also counts each sample's non-NULL slots into cnt[i]: warp-aggregated atomics)
__global__ void __launch_bounds__(IND_BLOCK) k_fx_sample(GView<int32_t> gv, NdApp a, uint64_t base0,
                                                        int64_t sample_lo, int64_t n, FastDiv Bp,
                                                        FastDiv m, const int32_t* __restrict__ prev,
                                                        const int32_t* __restrict__ rank,
                                                        int32_t* __restrict__ out,
                                                        unsigned long long* __restrict__ cnt,
                                                        int* stall, unsigned long long* ctr) {
  ItemStats st;
  const int64_t total = n * (int64_t)Bp.d * m.d;  // < 2^32 (checked by the host)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x; q0 < total; q0 += stride) {
    const int64_t q = q0 + threadIdx.x;
    int64_t i = -1;
    int32_t o = -1;
    if (q < total) {
      const uint32_t ip = m.div((uint32_t)q), slot = (uint32_t)q - ip * m.d;  // ip = i * Bp + p
      const int32_t v = prev[ip];
      i = Bp.div(ip);
      if (v >= 0) {
        const int64_t lo = __ldg(gv.row + v), deg = __ldg(gv.row + v + 1) - lo;
        if (slot == 0) st.bytes += SECTOR + 8;
        int stl = 0;
        const uint64_t ik = key_item((uint64_t)(sample_lo + i), (uint64_t)rank[ip], (uint64_t)slot);
        o = (int32_t)run_item(gv, grow(gv, lo), a, v, deg, -1, base0, ik, st, &stl);
        if (stl) atomicExch(stall, 1);
      }
      out[q] = o;
    }
    // per-sample non-NULL counts: lanes of one sample add once
    const unsigned act = __ballot_sync(0xffffffffu, o >= 0);
    const unsigned same = __match_any_sync(0xffffffffu, i);
    const unsigned grp = act & same;
    if (o >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(cnt + i, (unsigned long long)__popc(grp));
  }
  flush_stats(st, ctr);
}

__global__ void k_fx_flen(const unsigned long long* __restrict__ cnt, int64_t n, int64_t R,
                          int64_t* __restrict__ flen) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    flen[i] = i < n ? R + (int64_t)cnt[i] : 0;
}

// per sample (one warp): final row length R + non-NULL slots of every step
struct FxSteps {
  const int32_t* blk[8];
  int64_t B[8];
  int n_steps;
};

// ---- transit-parallel order for the fixed layout ------------------------------------
// The parent slots of a step are radix-sorted by transit (NULL parents keyed
// past every vertex), so the items of one transit -- all samples' pairs at a
// hub -- run in consecutive threads and share its row in L1/L2
// (transit_parallel.py:71-83's inversion); outputs land at the same fixed
// positions, so the rows are identical to the sample-parallel order.
__global__ void k_fx_keys(const int32_t* __restrict__ prev, const int32_t* __restrict__ rank,
                          int64_t N, uint32_t sentinel, uint32_t* __restrict__ keys,
                          uint64_t* __restrict__ vals) {
  for (int64_t ip = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ip < N;
       ip += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = prev[ip];
    keys[ip] = v >= 0 ? (uint32_t)v : sentinel;
    vals[ip] = (uint64_t)(uint32_t)ip | ((uint64_t)(uint32_t)rank[ip] << 32);
  }
}

// work classes of the step's transit groups (transit_parallel.py:86-101):
// work = members * m; small < 32, medium 32..1024, large > 1024; [3] = groups
__global__ void k_fx_classes(const uint32_t* __restrict__ keys, int64_t N, uint32_t sentinel,
                             int64_t m, unsigned long long* __restrict__ stats) {
  unsigned long long c0 = 0, c1 = 0, c2 = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[r];
    if (k == sentinel || (r > 0 && keys[r - 1] == k)) continue;
    int64_t lo = r + 1, hi = N;  // end of the group: first key > k
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] <= k) lo = mid + 1; else hi = mid;
    }
    const int64_t work = (lo - r) * m;
    if (work < SMALL_MAX_WORK) c0++; else if (work <= LARGE_MIN_WORK) c1++; else c2++;
  }
  for (int o = 16; o > 0; o >>= 1) {
    c0 += __shfl_down_sync(0xffffffffu, c0, o);
    c1 += __shfl_down_sync(0xffffffffu, c1, o);
    c2 += __shfl_down_sync(0xffffffffu, c2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (c0) atomicAdd(stats + 0, c0);
    if (c1) atomicAdd(stats + 1, c1);
    if (c2) atomicAdd(stats + 2, c2);
    if (c0 + c1 + c2) atomicAdd(stats + 3, c0 + c1 + c2);
  }
}

// one thread per (sorted parent, slot)
// payload = parent slot ip (low 32 bits) | its transit_idx (high 32 bits)
__global__ void __launch_bounds__(IND_BLOCK) k_fx_sample_tp(GView<int32_t> gv, NdApp a, uint64_t base0,
                                                           int64_t sample_lo, int64_t N, FastDiv Bp,
                                                           FastDiv m, uint32_t sentinel,
                                                           const uint32_t* __restrict__ keys,
                                                           const uint64_t* __restrict__ vals,
                                                           int32_t* __restrict__ out, int* stall,
                                                           unsigned long long* ctr) {
  ItemStats st;
  const int64_t total = N * (int64_t)m.d;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = m.div((uint32_t)q), slot = (uint32_t)q - r * m.d;
    const uint64_t pv = vals[r];
    const uint32_t ip = (uint32_t)pv;
    const uint32_t v = keys[r];
    int32_t o = -1;
    if (v != sentinel) {
      const int64_t lo = __ldg(gv.row + v), deg = __ldg(gv.row + v + 1) - lo;
      if (slot == 0) st.bytes += SECTOR + 8;
      int stl = 0;
      const uint64_t ik = key_item((uint64_t)(sample_lo + Bp.div(ip)), pv >> 32, (uint64_t)slot);
      o = (int32_t)run_item(gv, grow(gv, lo), a, (int64_t)v, deg, -1, base0, ik, st, &stl);
      if (stl) atomicExch(stall, 1);
    }
    out[(int64_t)ip * m.d + slot] = o;
  }
  flush_stats(st, ctr);
}

// ---- transit-parallel order for the fixed layout: hub-bucket inversion ----------
// The transit -> sample inversion (transit_parallel.py:71-83) without a sort:
// one pass counts each transit's members with warp-aggregated atomics (the
// returned old count is the member's position in its group), and a transit is
// appended to the hub list when its count crosses the medium threshold
// (work = members*m >= 32, transit_parallel.py:86-101).  The per-step class
// counts fall out of the same pass: groups = transits reaching 1 member,
// medium+large = crossings of the medium threshold, large = crossings of the
// large one (work > 1024).  A placement pass then writes every hub member's
// record at its group position and collects the small-class parents.  Class
// kernels:
//   sub-warp     small class: the m lanes of one parent cache the transit's
//                row in registers when it fits and read it with shuffles;
//   warp         hubs with work <= HUB_WARP_MAX: one warp per hub;
//   thread block hubs up to HUB_UNIT items: one CTA;
//   grid         larger hubs: HUB_UNIT-item units over several CTAs.
// The warp and CTA tiers stage the row (and the CTA tier the unit's member
// records) in shared memory by bulk copies (nd_bulk.cuh), the next hub's
// copy in flight while the current one is sampled.  Output positions are
// fixed per (parent, slot), so any member order gives the same rows.
constexpr int HUB_WARP_MAX = 256;   // work of a warp-tier hub
constexpr int HUB_UNIT = 8192;      // items per CTA unit (larger hubs span several CTAs)
constexpr int HUB_SLICE_W = 512;    // staged row entries per warp stage
constexpr int HUB_SLICE_C = 2048;   // staged row entries per CTA stage
constexpr int HUB_MEM_SLICE = 1024; // staged member records per CTA stage
constexpr int REG_K = 4;            // row entries cached per sub-warp lane
constexpr int FX_ILP = 4;           // independent items (or parents) in flight per thread

struct HubThr {
  int32_t tm, tl;  // member counts at which a group becomes medium / large
};
inline HubThr hub_thresholds(int64_t m) {
  HubThr t;
  if (m <= 0) { t.tm = t.tl = 0x7fffffff; return t; }
  t.tm = (int32_t)((SMALL_MAX_WORK + m - 1) / m);  // members*m >= 32
  t.tl = (int32_t)(LARGE_MIN_WORK / m + 1);        // members*m > 1024
  return t;
}

// A parent slot as the class kernels see it: its index (output position
// ip*m + slot) and the sample/transit part of its RNG key,
// C_SAMPLE*(sid+1) + C_TRANSIT*(tix+1) (rng.py:52-71), computed once per
// parent instead of once per slot.
struct __align__(16) MemRec {
  uint32_t ip, pad;
  uint64_t key;
};

// Per-warp staging of list appends: a warp collects up to 32 entries in
// shared memory and reserves their global slots with one atomic.  Every lane
// calls push/flush with warp-uniform control flow.
template <typename T>
struct WarpBuf {
  T* sbuf;      // this warp's 32 entries in shared memory
  int n = 0;    // buffered entries (warp-uniform)
  __device__ __forceinline__ int64_t flush(T* glist, int32_t* gcount) {
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (n) {
      if (lane == 0) base = atomicAdd(gcount, n);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (lane < n) glist[base + lane] = sbuf[lane];
      __syncwarp();
    }
    n = 0;
    return base;
  }
  __device__ __forceinline__ void push(bool f, const T& x, T* glist, int32_t* gcount) {
    const unsigned bm = __ballot_sync(0xffffffffu, f);
    if (!bm) return;
    if (n + __popc(bm) > 32) flush(glist, gcount);
    if (f) sbuf[n + __popc(bm & ((1u << (threadIdx.x & 31)) - 1))] = x;
    n += __popc(bm);
    __syncwarp();
  }
};

__device__ __forceinline__ void hub_flush(WarpBuf<int32_t>& wb, int32_t* hubs, int32_t* nhub,
                                          int2* vinfo) {
  const int lane = threadIdx.x & 31;
  const int cnt = wb.n;
  const int32_t v = lane < cnt ? wb.sbuf[lane] : 0;
  const int64_t base = wb.flush(hubs, nhub);
  if (lane < cnt) vinfo[v].y = (int32_t)(base + lane);
}

// Member counting of Q tiles of 32 parent slots (every lane calls it; lane
// entries with v >= 0 are non-NULL parents ip with transit v): the Q tiles'
// warp-aggregated atomics on the per-vertex count are in flight together; the
// returned old count is each member's position in its group, and threshold
// crossings go to the hub list through the warp buffer.
template <int Q>
__device__ __forceinline__ void count_tiles(const int32_t (&v)[Q], const int64_t (&ip)[Q],
                                            int2* vinfo, int32_t* gpos, WarpBuf<int32_t>& wb,
                                            int32_t* hubs, int32_t* nhub, const HubThr& th,
                                            unsigned long long& ng, unsigned long long& nm,
                                            unsigned long long& nl) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  int old[Q], c[Q];
  unsigned peers[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const bool ok = v[q] >= 0;
    const unsigned mk = __ballot_sync(0xffffffffu, ok);
    old[q] = 0;
    c[q] = 0;
    peers[q] = 0;
    if (ok) {
      peers[q] = __match_any_sync(mk, v[q]);
      c[q] = __popc(peers[q]);
      if (lane == __ffs(peers[q]) - 1) old[q] = atomicAdd(&vinfo[v[q]].x, c[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < Q; q++) {
    bool cross = false;
    if (v[q] >= 0) {
      const int leader = __ffs(peers[q]) - 1;
      const int o = __shfl_sync(peers[q], old[q], leader);
      gpos[ip[q]] = o + __popc(peers[q] & lt);
      if (lane == leader) {
        ng += o == 0;
        cross = o < th.tm && o + c[q] >= th.tm;
        nm += cross;
        nl += o < th.tl && o + c[q] >= th.tl;
      }
    }
    const unsigned cm = __ballot_sync(0xffffffffu, cross);
    if (cm) {
      if (wb.n + __popc(cm) > 32) hub_flush(wb, hubs, nhub, vinfo);
      if (cross) wb.sbuf[wb.n + __popc(cm & lt)] = v[q];
      wb.n += __popc(cm);
      __syncwarp();
    }
  }
}

// transit_idx ranks as k_fx_rank (rank among the sample block's non-NULL
// entries), per-sample non-NULL counts, and member counting.  Blocks of B < 32
// slots: several samples per 32-lane tile (one lane segment each), FX_ILP
// tiles per warp iteration; larger blocks: one sample per warp, its 32-slot
// chunks in order.  vinfo[v] = {member count, hub index}.
template <int Q>
__global__ void __launch_bounds__(256) k_fx_rank_count(const int32_t* __restrict__ blk, int64_t n,
                                                       int64_t B, int32_t* __restrict__ rank,
                                                       int64_t* __restrict__ nn,
                                                       int2* __restrict__ vinfo,
                                                       int32_t* __restrict__ gpos,
                                                       int32_t* __restrict__ hubs,
                                                       int32_t* __restrict__ nhub, HubThr th,
                                                       unsigned long long* __restrict__ stats) {
  __shared__ int32_t s_hub[256];
  WarpBuf<int32_t> wb;
  wb.sbuf = s_hub + (threadIdx.x & ~31);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long ng = 0, nm = 0, nl = 0;
  if (B < 32) {
    const int spw = 32 / (int)B, seg = lane / (int)B, pos = lane % (int)B;
    const unsigned segm = (unsigned)(((1ull << B) - 1) << (seg * B));
    const int64_t tiles = (n + spw - 1) / spw;
    for (int64_t t0 = warp * Q; t0 < tiles; t0 += nw * Q) {
      int32_t v[Q];
      int64_t ip[Q];
#pragma unroll
      for (int q = 0; q < Q; q++) {
        const int64_t i = (t0 + q) * spw + seg;
        const bool valid = seg < spw && i < n;
        ip[q] = valid ? i * B + pos : -1;
        v[q] = valid ? blk[ip[q]] : -2;
      }
#pragma unroll
      for (int q = 0; q < Q; q++) {
        const unsigned mk = __ballot_sync(0xffffffffu, v[q] >= 0);
        if (ip[q] >= 0) {
          rank[ip[q]] = v[q] >= 0 ? __popc(mk & segm & lt) : -1;
          if (pos == 0) nn[ip[q] / B] = __popc(mk & segm);
        }
      }
      count_tiles<Q>(v, ip, vinfo, gpos, wb, hubs, nhub, th, ng, nm, nl);
    }
  } else {
    for (int64_t i = warp; i < n; i += nw) {
      int32_t base = 0;
      for (int64_t p0 = 0; p0 < B; p0 += 32) {
        const int64_t p = p0 + lane;
        int32_t v[1] = {p < B ? blk[i * B + p] : -2};
        int64_t ip[1] = {p < B ? i * B + p : -1};
        const unsigned mk = __ballot_sync(0xffffffffu, v[0] >= 0);
        if (p < B) rank[ip[0]] = v[0] >= 0 ? base + __popc(mk & lt) : -1;
        base += __popc(mk);
        count_tiles<1>(v, ip, vinfo, gpos, wb, hubs, nhub, th, ng, nm, nl);
      }
      if (lane == 0) nn[i] = base;
    }
  }
  hub_flush(wb, hubs, nhub, vinfo);
  for (int o = 16; o > 0; o >>= 1) {
    ng += __shfl_down_sync(0xffffffffu, ng, o);
    nm += __shfl_down_sync(0xffffffffu, nm, o);
    nl += __shfl_down_sync(0xffffffffu, nl, o);
  }
  // a warp can cross a threshold of a group another warp opened: the class
  // deltas are signed per warp and sum to the exact counts over the grid
  if (lane == 0 && (ng | nm | nl)) {
    if (ng != nm) atomicAdd(stats + 0, ng - nm);
    if (nm != nl) atomicAdd(stats + 1, nm - nl);
    if (nl) atomicAdd(stats + 2, nl);
    if (ng) atomicAdd(stats + 3, ng);
  }
}

// hub sizes (members) and CTA-unit counts, zero past the hub count
__global__ void k_hub_sizes(const int32_t* __restrict__ hubs, const int32_t* __restrict__ nhub,
                            int64_t cap, const int2* __restrict__ vinfo, int64_t m,
                            int32_t* __restrict__ hsz, int32_t* __restrict__ hun) {
  const int64_t H = *nhub;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= cap;
       j += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = 0, u = 0;
    if (j < H) {
      c = vinfo[hubs[j]].x;
      const int64_t w = (int64_t)c * m;
      u = w > HUB_WARP_MAX ? (int32_t)((w + HUB_UNIT - 1) / HUB_UNIT) : 0;
    }
    hsz[j] = c;
    hun[j] = u;
  }
}

// the CTA units of the hubs above the warp tier: one 32-byte descriptor per
// unit (row, group start, item range) for the producer warp of k_fx_hub_cta
struct __align__(32) HubUnit {
  int64_t lo;
  int32_t deg, start, t0, t1, pad0, pad1;
};

__global__ void k_hub_units(const int32_t* __restrict__ nhub, const int32_t* __restrict__ hubs,
                            const int32_t* __restrict__ hoff, const int32_t* __restrict__ uoff,
                            const int32_t* __restrict__ hun, const int64_t* __restrict__ row,
                            int64_t m, HubUnit* __restrict__ units, int2* __restrict__ vinfo) {
  const int64_t H = *nhub;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < H;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = hubs[j];
    // the hub's first member slot replaces its hub index: placement reads it
    // with the member count, one dependent lookup fewer per member
    vinfo[v].y = hoff[j];
    const int32_t nu = hun[j];
    if (nu == 0) continue;
    HubUnit d;
    d.lo = row[v];
    d.deg = (int32_t)(row[v + 1] - d.lo);
    d.start = hoff[j];
    const int64_t work = (int64_t)(hoff[j + 1] - d.start) * m;
    d.pad0 = d.pad1 = 0;
    const int32_t u0 = uoff[j];
    for (int32_t c = 0; c < nu; c++) {
      d.t0 = c * HUB_UNIT;
      d.t1 = (int32_t)min(work, (int64_t)d.t0 + HUB_UNIT);
      units[u0 + c] = d;
    }
  }
}

// Placement, FX_ILP tiles of 32 consecutive parent slots per warp: NULL
// parents give m NULL slots; hub members' records go to their group
// position, small-class parents' records to the small list.  The final-row
// lengths come from here too: a k-hop pick from a non-empty row is never
// NULL, so a sample gains m values per parent whose transit has edges.
template <int Q>
__global__ void __launch_bounds__(256) k_fx_place(const int32_t* __restrict__ prev,
                                                  const int32_t* __restrict__ rank, int64_t N,
                                                  FastDiv Bp, int64_t m, int64_t sample_lo,
                                                  const int64_t* __restrict__ row,
                                                  const int2* __restrict__ vinfo, int32_t tm,
                                                  const int32_t* __restrict__ gpos,
                                                  const int32_t* __restrict__ hoff,
                                                  MemRec* __restrict__ perm,
                                                  MemRec* __restrict__ small,
                                                  int32_t* __restrict__ nsmall,
                                                  int32_t* __restrict__ out,
                                                  unsigned long long* __restrict__ scnt) {
  __shared__ MemRec s_small[256];
  const int lane = threadIdx.x & 31;
  WarpBuf<MemRec> wb;
  wb.sbuf = s_small + (threadIdx.x & ~31);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b0 = warp * 32 * Q; b0 < N; b0 += nw * 32 * Q) {
    int32_t v[Q], rk[Q], gp[Q], ho[Q];
    int2 vi[Q];
    int64_t dg[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int64_t ip = b0 + q * 32 + lane;
      v[q] = ip < N ? prev[ip] : -2;
      rk[q] = ip < N ? rank[ip] : -1;
      gp[q] = ip < N ? gpos[ip] : 0;
    }
#pragma unroll
    for (int q = 0; q < Q; q++) {
      vi[q] = v[q] >= 0 ? vinfo[v[q]] : make_int2(0, 0);
      dg[q] = v[q] >= 0 ? __ldg(row + v[q] + 1) - __ldg(row + v[q]) : 0;
    }
#pragma unroll
    for (int q = 0; q < Q; q++) ho[q] = vi[q].x >= tm ? vi[q].y : 0;  // hub's first slot (k_hub_units)
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int64_t ip = b0 + q * 32 + lane;
      bool sm = false;
      MemRec r;
      const int64_t i = v[q] >= 0 ? (int64_t)Bp.div((uint32_t)ip) : -1;
      if (v[q] == -1) {
        for (int64_t j = 0; j < m; j++) out[ip * m + j] = -1;
      } else if (v[q] >= 0) {
        r.ip = (uint32_t)ip;
        r.pad = 0;
        r.key = C_SAMPLE * (uint64_t)(sample_lo + i + 1) + C_TRANSIT * (uint64_t)(rk[q] + 1);
        if (vi[q].x >= tm) perm[ho[q] + gp[q]] = r;
        else sm = true;
      }
      wb.push(sm, r, small, nsmall);
      // per-sample non-NULL slots: lanes of one sample add once
      const bool gain = dg[q] > 0;
      const unsigned gb = __ballot_sync(0xffffffffu, gain);
      const unsigned same = __match_any_sync(0xffffffffu, i);
      const unsigned grp = gb & same;
      if (gain && lane == __ffs(grp) - 1) atomicAdd(scnt + i, (unsigned long long)(__popc(grp) * m));
    }
  }
  wb.flush(small, nsmall);
}

struct FxHub {
  GView<int32_t> gv;
  uint64_t base0;   // key_base(seed, step, 0, 0)
  FastDiv m;
  const int32_t* hubs;
  const int32_t* nhub;
  const int32_t* hoff;  // [cap+1] member offsets into perm
  const int32_t* uoff;  // [cap+1] CTA-unit offsets (uoff[cap] = unit count)
  int64_t cap;
  const HubUnit* units; // CTA-unit descriptors
  const MemRec* perm;   // member records in group order
  int32_t* out;
  unsigned long long* ctr;
};

// one item: slot `slot` of member record `r`, the transit's row at `srow`
// (shared memory) or `col + lo`; returns the vertex (NULL for an empty row)
__device__ __forceinline__ int32_t fx_pick(uint64_t base0, const MemRec& r, uint32_t slot,
                                           const ModU64& md, int64_t deg, const int32_t* srow,
                                           const int32_t* col, int64_t lo) {
  if (deg <= 0) return -1;  // a transit without out-edges gives NULL slots (_ckernels.pyx:212-223)
  const uint64_t k = md.mod(draw_u64(base0, r.key + C_SLOT * (uint64_t)(slot + 1)));
  return srow ? srow[k] : __ldg(col + lo + (int64_t)k);
}

// Algorithmic bytes of a range [t0, t1) of a hub's items:
// S+8 per pair (slot 0 items) plus S+8 per slot when the row is non-empty.
__device__ __forceinline__ int64_t fx_range_bytes(int32_t t0, int32_t t1, uint32_t m, int64_t deg) {
  const int64_t pairs = (int64_t)((t1 + m - 1) / m) - (int64_t)((t0 + m - 1) / m);
  return pairs * (SECTOR + 8) + (deg > 0 ? (int64_t)(t1 - t0) * (SECTOR + 8) : 0);
}

// small class: one thread per (small parent, slot); the lanes of one parent
// form a sub-warp that holds the transit's row in registers when it fits
// (REG_K entries per lane) and reads it with warp shuffles
__global__ void __launch_bounds__(IND_BLOCK) k_fx_small(GView<int32_t> gv, uint64_t base0,
                                                       FastDiv m, const int32_t* __restrict__ prev,
                                                       const MemRec* __restrict__ small,
                                                       const int32_t* __restrict__ nsmall,
                                                       int32_t* __restrict__ out,
                                                       unsigned long long* __restrict__ ctr) {
  ItemStats st;
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)(*nsmall) * m.d;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x; q0 < total; q0 += stride) {
    const int64_t q = q0 + threadIdx.x;
    const bool act = q < total;
    const unsigned am = __ballot_sync(0xffffffffu, act);
    if (!act) continue;
    const uint32_t e = m.div((uint32_t)q), slot = (uint32_t)q - e * m.d;
    const unsigned peers = __match_any_sync(am, e);
    const int leader = __ffs(peers) - 1;
    const int sw = __popc(peers);
    const int r = lane - leader;
    MemRec rec;
    int64_t lo = 0, hi = 0;
    if (lane == leader) {
      rec = small[e];
      const int32_t v = prev[rec.ip];
      lo = __ldg(gv.row + v);
      hi = __ldg(gv.row + v + 1);
    }
    rec.ip = __shfl_sync(peers, rec.ip, leader);
    rec.key = __shfl_sync(peers, rec.key, leader);
    lo = __shfl_sync(peers, lo, leader);
    hi = __shfl_sync(peers, hi, leader);
    const int64_t deg = hi - lo;
    int32_t o = -1;
    if (slot == 0) st.bytes += SECTOR + 8;
    if (deg > 0) {
      st.bytes += SECTOR + 8;
      const uint64_t k = mod_u64(draw_u64(base0, rec.key + C_SLOT * (uint64_t)(slot + 1)),
                                 (uint64_t)deg);
      if (deg <= (int64_t)REG_K * sw) {
        // the row in the sub-warp's registers: lane r holds entries r, r+sw, ...
        int32_t c[REG_K];
#pragma unroll
        for (int j = 0; j < REG_K; j++) {
          const int64_t x = r + (int64_t)j * sw;
          c[j] = x < deg ? __ldg(gv.col + lo + x) : -1;
        }
        const int src = leader + (int)(k % (uint64_t)sw);
        const int kj = (int)(k / (uint64_t)sw);
#pragma unroll
        for (int j = 0; j < REG_K; j++) {
          const int32_t x = __shfl_sync(peers, c[j], src);
          if (j == kj) o = x;
        }
      } else {
        o = __ldg(gv.col + lo + (int64_t)k);
      }
    }
    out[(uint64_t)rec.ip * m.d + slot] = o;
  }
  flush_stats(st, ctr);
}

__device__ __forceinline__ bool hub_stage(int64_t deg, int64_t items, int64_t slice) {
  // stage when the copy costs less than the picks' random sectors (8 entries each)
  return deg > 0 && deg + 8 <= slice && deg <= 8 * items;
}

// warp tier: one warp per hub with work <= HUB_WARP_MAX, two bulk-copy stages
// per warp (the next hub's row lands while this one is sampled)
__global__ void __launch_bounds__(IND_BLOCK) k_fx_hub_warp(FxHub h) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm) + 2 * wib;
  int32_t* buf0 = reinterpret_cast<int32_t*>(dsm + 16 * (IND_BLOCK / 32)) +
                  (size_t)wib * 2 * (HUB_SLICE_W + 8);
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  __syncwarp();
  ItemStats st;
  const int64_t H = *h.nhub;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t m = h.m.d;
  uint32_t ph = 0;  // bit b: parity of stage b's next phase
  // hub j's descriptor (warp-uniform); staged when in the warp tier and worth it
  auto desc = [&](int64_t j, int64_t& lo, int64_t& deg, int32_t& start, int32_t& work,
                  bool& staged, int b) {
    const int32_t v = h.hubs[j];
    lo = __ldg(h.gv.row + v);
    deg = __ldg(h.gv.row + v + 1) - lo;
    start = h.hoff[j];
    const int64_t w = (int64_t)(h.hoff[j + 1] - start) * m;
    work = w <= HUB_WARP_MAX ? (int32_t)w : 0;  // larger hubs: the CTA tiers
    staged = work > 0 && hub_stage(deg, work, HUB_SLICE_W);
    if (staged && lane == 0)
      stage_row_bulk(buf0 + b * (HUB_SLICE_W + 8), h.gv.col, row_span(lo, deg), bar + b);
  };
  int64_t lo = 0, deg = 0;
  int32_t start = 0, work = 0;
  bool staged = false;
  if (w0 < H) desc(w0, lo, deg, start, work, staged, 0);
  int it = 0;
  for (int64_t j = w0; j < H; j += nw, it++) {
    const int b = it & 1;
    int64_t nlo = 0, ndeg = 0;
    int32_t nstart = 0, nwork = 0;
    bool nstaged = false;
    if (j + nw < H) desc(j + nw, nlo, ndeg, nstart, nwork, nstaged, b ^ 1);  // prefetch
    if (work > 0) {
      const int32_t* srow = nullptr;
      if (staged) {
        mbar_wait(bar + b, (ph >> b) & 1u);
        ph ^= 1u << b;
        srow = buf0 + b * (HUB_SLICE_W + 8) + row_span(lo, deg).skew;
      }
      const ModU64 md((uint64_t)(deg > 0 ? deg : 1));
      if (lane == 0) st.bytes += fx_range_bytes(0, work, m, deg);
      for (int32_t tb = 0; tb < work; tb += 32 * FX_ILP) {
        MemRec r[FX_ILP];
        uint32_t slot[FX_ILP];
#pragma unroll
        for (int q = 0; q < FX_ILP; q++) {
          const int32_t t = min(tb + q * 32 + lane, work - 1);
          const uint32_t mem = h.m.div((uint32_t)t);
          slot[q] = (uint32_t)t - mem * m;
          r[q] = h.perm[start + mem];
        }
        int32_t o[FX_ILP];
#pragma unroll
        for (int q = 0; q < FX_ILP; q++) o[q] = fx_pick(h.base0, r[q], slot[q], md, deg, srow, h.gv.col, lo);
#pragma unroll
        for (int q = 0; q < FX_ILP; q++)
          if (tb + q * 32 + lane < work) h.out[r[q].ip * m + slot[q]] = o[q];
      }
    }
    __syncwarp();
    lo = nlo; deg = ndeg; start = nstart; work = nwork; staged = nstaged;
  }
  flush_stats(st, h.ctr);
}

// thread-block tier (a hub's items in one CTA) and grid tier (a hub above
// HUB_UNIT items split over several CTAs), one CTA per unit of the unit
// list, warp-specialised: the producer warp walks the CTA's units ahead of the
// consumers and stages, by bulk copies into a ring of HUB_STAGES shared-memory
// stages, the unit's row (when it fits and pays) and its slice of the member
// records (full barrier: the bytes landed; empty barrier: every consumer warp
// is done with the stage).  The eight consumer warps sample, FX_ILP items per
// thread in flight.
constexpr int HUB_STAGES = 4;
constexpr int HUB_STAGE_MEMS = 0;  // stage the unit's member records too (1) or read them through L1 (0)
constexpr int HUB_CONSUMERS = IND_BLOCK / 32;
constexpr size_t HUB_STAGE_BYTES = (size_t)(HUB_SLICE_C + 8) * 4 + (size_t)HUB_MEM_SLICE * 16 * HUB_STAGE_MEMS;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct HubStage {
  HubUnit d;
  int32_t rskew;  // row entry 0 in the row buffer, or -1 (not staged)
  int32_t mstg;   // member records staged (from member t0/m)
  int32_t m0;     // first member of the unit
};

// the consumer loop of one unit: Q items per thread in flight
template <int Q, bool SREC, bool SROW>
__device__ __forceinline__ void hub_items(const FxHub& h, const MemRec* __restrict__ recs,
                                          const int32_t* __restrict__ srow, int32_t t0, int32_t t1,
                                          int warp, int lane, const ModU64& md, int64_t deg,
                                          int64_t lo) {
  const uint32_t m = h.m.d;
  for (int32_t tb = t0 + warp * 32 * Q; tb < t1; tb += IND_BLOCK * Q) {
    MemRec r[Q];
    uint32_t slot[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int32_t t = min(tb + q * 32 + lane, t1 - 1);
      const uint32_t mem = h.m.div((uint32_t)t);
      slot[q] = (uint32_t)t - mem * m;
      if (SREC) {
        r[q] = recs[mem];
      } else {
        const int4 x = __ldg(reinterpret_cast<const int4*>(recs + mem));
        r[q].ip = (uint32_t)x.x;
        r[q].key = (uint64_t)(uint32_t)x.z | ((uint64_t)(uint32_t)x.w << 32);
      }
    }
    int32_t o[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) {
      if (deg <= 0) { o[q] = -1; continue; }
      const uint64_t k = md.mod(draw_u64(h.base0, r[q].key + C_SLOT * (uint64_t)(slot[q] + 1)));
      o[q] = SROW ? srow[k] : __ldg(h.gv.col + lo + (int64_t)k);
    }
#pragma unroll
    for (int q = 0; q < Q; q++)
      if (tb + q * 32 + lane < t1) h.out[r[q].ip * m + slot[q]] = o[q];
  }
}

template <int Q>
__global__ void __launch_bounds__(IND_BLOCK + 32, 4) k_fx_hub_cta(FxHub h) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ HubStage sd[HUB_STAGES];
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
  uint64_t* empty = full + HUB_STAGES;
  unsigned char* stage0 = dsm + 16 * HUB_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int k = 0; k < HUB_STAGES; k++) {
      mbar_init(full + k, 1);
      mbar_init(empty + k, HUB_CONSUMERS);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t U = h.uoff[h.cap];
  const uint32_t m = h.m.d;
  if (warp == HUB_CONSUMERS) {  // producer
    if (lane == 0) {
      int it = 0;
      for (int64_t u = blockIdx.x; u < U; u += gridDim.x, it++) {
        const int sg = it % HUB_STAGES, use = it / HUB_STAGES;
        if (use > 0) mbar_wait(empty + sg, (use - 1) & 1);
        HubStage g;
        g.d = h.units[u];
        int32_t* rbuf = reinterpret_cast<int32_t*>(stage0 + sg * HUB_STAGE_BYTES);
        MemRec* mbuf = reinterpret_cast<MemRec*>(rbuf + HUB_SLICE_C + 8);
        const bool stg = hub_stage(g.d.deg, g.d.t1 - g.d.t0, HUB_SLICE_C);
        g.m0 = g.d.t0 / (int32_t)m;
        const int32_t nm = (g.d.t1 - 1) / (int32_t)m + 1 - g.m0;
        g.mstg = HUB_STAGE_MEMS && nm <= HUB_MEM_SLICE;
        const RowSpan rs = row_span(g.d.lo, g.d.deg);
        g.rskew = stg ? (int32_t)rs.skew : -1;
        sd[sg] = g;
        const uint32_t bytes = (stg ? rs.n * 4u : 0u) + (g.mstg ? (uint32_t)nm * 16u : 0u);
        if (bytes) {
          mbar_arrive_expect_tx(full + sg, bytes);
          if (stg) bulk_g2s(rbuf, h.gv.col + rs.a, rs.n * 4u, full + sg);
          if (g.mstg) bulk_g2s(mbuf, h.perm + g.d.start + g.m0, (uint32_t)nm * 16u, full + sg);
        } else {
          mbar_arrive(full + sg);
        }
      }
    }
    return;
  }
  ItemStats st;
  int it = 0;
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x, it++) {
    const int sg = it % HUB_STAGES, use = it / HUB_STAGES;
    mbar_wait(full + sg, use & 1);
    const HubStage g = sd[sg];
    const int32_t* rbuf = reinterpret_cast<const int32_t*>(stage0 + sg * HUB_STAGE_BYTES);
    const MemRec* mbuf = reinterpret_cast<const MemRec*>(rbuf + HUB_SLICE_C + 8);
    const int32_t* srow = g.rskew >= 0 ? rbuf + g.rskew : nullptr;
    const int64_t lo = g.d.lo, deg = g.d.deg;
    const ModU64 md((uint64_t)(deg > 0 ? deg : 1));
    if (threadIdx.x == 0) st.bytes += fx_range_bytes(g.d.t0, g.d.t1, m, deg);
    // member records from the stage (shared) or from global memory; the row
    // from the stage or global: four specialised loops keep every load typed
    if (g.mstg) {
      const MemRec* recs = mbuf - g.m0;
      if (srow) hub_items<Q, true, true>(h, recs, srow, g.d.t0, g.d.t1, warp, lane, md, deg, lo);
      else hub_items<Q, true, false>(h, recs, srow, g.d.t0, g.d.t1, warp, lane, md, deg, lo);
    } else {
      const MemRec* recs = h.perm + g.d.start;
      if (srow) hub_items<Q, false, true>(h, recs, srow, g.d.t0, g.d.t1, warp, lane, md, deg, lo);
      else hub_items<Q, false, false>(h, recs, srow, g.d.t0, g.d.t1, warp, lane, md, deg, lo);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + sg);
  }
  flush_stats(st, h.ctr);
}

constexpr size_t HUB_WARP_SMEM = 16 * (IND_BLOCK / 32) + (size_t)(IND_BLOCK / 32) * 2 * (HUB_SLICE_W + 8) * 4;
constexpr size_t HUB_CTA_SMEM = 16 * HUB_STAGES + HUB_STAGES * HUB_STAGE_BYTES;

// per sample (one warp): non-NULL slots of one step block, added to cnt[i]
__global__ void k_fx_block_counts(const int32_t* __restrict__ blk, int64_t n, int64_t B,
                                  unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    unsigned long long c = 0;
    for (int64_t p0 = 0; p0 < B; p0 += 32) {
      const int64_t p = p0 + lane;
      c += __popc(__ballot_sync(0xffffffffu, p < B && blk[i * B + p] >= 0));
    }
    if (lane == 0) cnt[i] += c;
  }
}

// final rows: roots, then each step's non-NULL slots in block order
template <typename RootT>
__global__ void k_fx_final(FxSteps S, const RootT* __restrict__ roots, int64_t n, int64_t R,
                           const int64_t* __restrict__ off, int32_t* __restrict__ ids,
                           int64_t* __restrict__ roots_out, int64_t* __restrict__ roots_off) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    int32_t* dst = ids + off[i];
    for (int64_t r = lane; r < R; r += 32) {
      const int64_t x = (int64_t)roots[i * R + r];
      dst[r] = (int32_t)x;
      roots_out[i * R + r] = x;
    }
    if (lane == 0) {
      roots_off[i] = i * R;
      if (i == n - 1) roots_off[n] = n * R;
    }
    int64_t pos = R;
    for (int s = 0; s < S.n_steps; s++) {
      const int64_t B = S.B[s];
      const int32_t* src = S.blk[s] + i * B;
      // eight 32-slot chunks loaded back to back, then compacted in order
      for (int64_t p0 = 0; p0 < B; p0 += 32 * 8) {
        int32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int64_t p = p0 + 32 * u + lane;
          v[u] = p < B ? src[p] : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const unsigned mk = __ballot_sync(0xffffffffu, v[u] >= 0);
          if (v[u] >= 0) dst[pos + __popc(mk & ((1u << lane) - 1))] = v[u];
          pos += __popc(mk);
        }
      }
    }
  }
}

// step rows (F_STEP_VALS): the slots of real pairs (non-NULL parents) of step s,
// sample-major, at off_s[i] + rank(parent) * m + slot
__global__ void k_fx_step_vals(const int32_t* __restrict__ out, const int32_t* __restrict__ prev_rank,
                               int64_t n, int64_t Bp, int64_t m, const int64_t* __restrict__ soff,
                               int32_t* __restrict__ vals) {
  const int64_t total = n * Bp * m;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ip = q / m, slot = q - ip * m;
    const int32_t r = prev_rank[ip];
    if (r < 0) continue;
    vals[soff[ip / Bp] + (int64_t)r * m + slot] = out[q];
  }
}

__global__ void k_fx_step_counts(const int64_t* __restrict__ nn, int64_t n, int64_t m,
                                 int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = nn[i] * m;
}

}  // namespace

__global__ void k_fx_narrow_roots(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

// launch knobs of the TP fixed-layout kernels (ND_FX_KNOBS="rc,pl,hc,rc_grid,pl_grid,hc_grid,
// hw_grid": ILP of the rank/count, placement and CTA-tier kernels and grid sizes; for
// ablations only, the defaults are the measured best)
struct FxKnobs {
  int rc = 4, pl = 4, hc = 4;
  int rc_grid = 148 * 32, pl_grid = 148 * 16, hc_grid = 148 * 4, hw_grid = 148 * 6;
};
static FxKnobs fx_knobs() {
  static FxKnobs k = [] {
    FxKnobs x;
    if (const char* e = getenv("ND_FX_KNOBS"))
      sscanf(e, "%d,%d,%d,%d,%d,%d,%d", &x.rc, &x.pl, &x.hc, &x.rc_grid, &x.pl_grid, &x.hc_grid,
             &x.hw_grid);
    return x;
  }();
  return k;
}

// dynamic shared memory above 48 KB for the hub kernels (once per process)
static int fx_hub_attrs() {
  static int rc = -1;
  if (rc < 0) {
    rc = ND_OK;
    if (cudaFuncSetAttribute(k_fx_hub_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)HUB_WARP_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k_fx_hub_cta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)HUB_CTA_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k_fx_hub_cta<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)HUB_CTA_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k_fx_hub_cta<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)HUB_CTA_SMEM) != cudaSuccess)
      rc = ND_ERR_CUDA;
  }
  return rc;
}

// fixed-layout SP run (see k_fx_*); returns ND_ERR_ARG when the layout does not apply
static int run_individual_fixed(const nd_graph* G, const NdApp& a, const int64_t* fan, int64_t S,
                                int64_t sample_lo, int64_t n, const int64_t* roots, int64_t R,
                                uint64_t seed, bool tp, cudaStream_t s, nd_result** out_res) {
  const DevGraph& g = G->g;
  if (S < 1 || S > 8 || n <= 0) return ND_ERR_ARG;
  int64_t B[9];
  B[0] = R;
  double cells = 0;
  for (int64_t k = 0; k < S; k++) {
    B[k + 1] = B[k] * fan[k];
    cells += (double)n * (double)B[k + 1];
    if (B[k + 1] >= (1ll << 31)) return ND_ERR_ARG;
  }
  if (cells > 1.5e9) return ND_ERR_ARG;
  nd_trace("fx:start");
  int32_t* blk[9] = {};
  int32_t* rank[8] = {};
  int64_t* nn[8] = {};
  ND_CUDA_TRY(nd_alloc(&blk[0], n * R, s));
  if (roots) k_fx_narrow_roots<<<nd_grid(n * R, 256), 256, 0, s>>>(roots, n * R, blk[0]);
  else ND_TRY(nd_uniform_roots_i32(g, R, seed, sample_lo, n, blk[0], s));
  unsigned long long *stats = nullptr, *ctr = nullptr;
  int* stall = nullptr;
  ND_CUDA_TRY(nd_alloc(&stats, 4 * S, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 4, s));
  ND_CUDA_TRY(nd_alloc(&stall, 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * S * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stall, 0, sizeof(int), s));
  const int kbits = key_bits_for(g.V);
  const uint32_t sentinel = 1u << kbits;  // past every vertex id
  unsigned long long* tp_scratch = nullptr;  // TP mode: pair counts are not the fetches
  ND_CUDA_TRY(nd_alloc(&tp_scratch, 1, s));
  unsigned long long* scnt = nullptr;  // per-sample non-NULL slots over all steps
  ND_CUDA_TRY(nd_alloc(&scnt, n, s));
  ND_CUDA_TRY(cudaMemsetAsync(scnt, 0, n * sizeof(unsigned long long), s));
  const GView<int32_t> gv = view(g);
  static const bool sort_tp = getenv("ND_FX_TP") && std::string(getenv("ND_FX_TP")) == "sort";
  const FxKnobs knob = fx_knobs();
  int2* vinfo = nullptr;  // TP: per-vertex {member count, hub index}
  int32_t* nhub = nullptr;
  if (tp && !sort_tp) {
    ND_TRY(fx_hub_attrs());
    ND_CUDA_TRY(nd_alloc(&vinfo, g.V, s));
    ND_CUDA_TRY(nd_alloc(&nhub, 2, s));  // [0] hubs, [1] small parents
  }
  Profiler prof(s);
  for (int64_t k = 0; k < S; k++) {
    ND_CUDA_TRY(nd_alloc(&rank[k], n * B[k], s));
    ND_CUDA_TRY(nd_alloc(&nn[k], n, s));
    ND_CUDA_TRY(nd_alloc(&blk[k + 1], n * B[k + 1], s));
    const int64_t items = n * B[k + 1];
    prof.step_begin();
    if (!tp) {
      k_fx_rank<<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(blk[k], n, B[k], rank[k], nn[k],
                                                              stats + 4 * k + 3);
      prof.step_built();
      k_fx_sample<<<nd_grid(items, IND_BLOCK, 148 * 64), IND_BLOCK, 0, s>>>(
          gv, a, key_base(seed, (uint64_t)k, 0, 0), sample_lo, n, FastDiv((uint32_t)B[k]),
          FastDiv((uint32_t)fan[k]), blk[k], rank[k], blk[k + 1], scnt, stall, ctr);
      prof.step_sampled();
      continue;
    }
    if (sort_tp) {  // ND_FX_TP=sort: the round-1 radix-sorted order (A/B only)
      k_fx_rank<<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(blk[k], n, B[k], rank[k], nn[k],
                                                              tp_scratch);
      const int64_t N = n * B[k];
      uint32_t *k0 = nullptr, *k1 = nullptr;
      uint64_t *v0 = nullptr, *v1 = nullptr;
      ND_CUDA_TRY(nd_alloc(&k0, N, s)); ND_CUDA_TRY(nd_alloc(&k1, N, s));
      ND_CUDA_TRY(nd_alloc(&v0, N, s)); ND_CUDA_TRY(nd_alloc(&v1, N, s));
      k_fx_keys<<<nd_grid(N, 256), 256, 0, s>>>(blk[k], rank[k], N, sentinel, k0, v0);
      {
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, N, 0, kbits + 1, s);
        void* tmp = nullptr;
        ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
        ND_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, N, 0, kbits + 1, s));
        nd_free(tmp, s);
      }
      k_fx_classes<<<nd_grid(N, 256, 148 * 16), 256, 0, s>>>(k1, N, sentinel, fan[k], stats + 4 * k);
      prof.step_built();
      k_fx_sample_tp<<<nd_grid(items, IND_BLOCK, 148 * 64), IND_BLOCK, 0, s>>>(
          gv, a, key_base(seed, (uint64_t)k, 0, 0), sample_lo, N, FastDiv((uint32_t)B[k]),
          FastDiv((uint32_t)fan[k]), sentinel, k1, v1, blk[k + 1], stall, ctr);
      k_fx_block_counts<<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(blk[k + 1], n, B[k + 1], scnt);
      prof.step_sampled();
      nd_free(k0, s); nd_free(k1, s); nd_free(v0, s); nd_free(v1, s);
      continue;
    }
    // transit-parallel order: hub-bucket inversion, small class by sub-warps,
    // hubs in the warp / thread-block / grid tiers
    {
      const int64_t N = n * B[k];
      const HubThr th = hub_thresholds(fan[k]);
      const int64_t cap = th.tm >= 0x7fffffff ? 1 : N / th.tm + 1;
      const int64_t ucap = cap + N * fan[k] / HUB_UNIT + 1;
      // the step's scratch in one pool allocation (nine arrays carved from it):
      // fewer stream-ordered allocations per step keep the step's cost
      // independent of how earlier jobs left the pool
      int32_t *gpos = nullptr, *hubs = nullptr, *hsz = nullptr, *hun = nullptr, *hoff = nullptr,
              *uoff = nullptr;
      MemRec *perm = nullptr, *small = nullptr;
      HubUnit* units = nullptr;
      char* arena = nullptr;
      size_t scan_bytes = 0, o_scan = 0;
      {
        size_t off = 0;
        auto carve = [&](size_t bytes) {
          const size_t at = off;
          off += (bytes + 255) & ~(size_t)255;
          return at;
        };
        const size_t o_gpos = carve(N * 4), o_hubs = carve(cap * 4), o_hsz = carve((cap + 1) * 4),
                     o_hun = carve((cap + 1) * 4), o_hoff = carve((cap + 1) * 4),
                     o_uoff = carve((cap + 1) * 4), o_units = carve(ucap * sizeof(HubUnit)),
                     o_perm = carve(N * sizeof(MemRec)), o_small = carve(N * sizeof(MemRec));
        cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, hsz, hoff, cap + 1, s);
        o_scan = carve(scan_bytes);
        ND_CUDA_TRY(nd_alloc(&arena, off, s));
        gpos = reinterpret_cast<int32_t*>(arena + o_gpos);
        hubs = reinterpret_cast<int32_t*>(arena + o_hubs);
        hsz = reinterpret_cast<int32_t*>(arena + o_hsz);
        hun = reinterpret_cast<int32_t*>(arena + o_hun);
        hoff = reinterpret_cast<int32_t*>(arena + o_hoff);
        uoff = reinterpret_cast<int32_t*>(arena + o_uoff);
        units = reinterpret_cast<HubUnit*>(arena + o_units);
        perm = reinterpret_cast<MemRec*>(arena + o_perm);
        small = reinterpret_cast<MemRec*>(arena + o_small);
      }
      ND_CUDA_TRY(cudaMemsetAsync(vinfo, 0, g.V * sizeof(int2), s));
      ND_CUDA_TRY(cudaMemsetAsync(nhub, 0, 2 * sizeof(int32_t), s));
      {
        auto krc = knob.rc == 1 ? k_fx_rank_count<1> : knob.rc == 2 ? k_fx_rank_count<2>
                                                                    : k_fx_rank_count<4>;
        krc<<<nd_grid(n * 32, 256, knob.rc_grid), 256, 0, s>>>(blk[k], n, B[k], rank[k], nn[k], vinfo,
                                                              gpos, hubs, nhub, th, stats + 4 * k);
      }
      k_hub_sizes<<<nd_grid(cap + 1, 256), 256, 0, s>>>(hubs, nhub, cap, vinfo, fan[k], hsz, hun);
      {
        size_t tb = scan_bytes;
        void* tmp = arena + o_scan;
        ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, hsz, hoff, cap + 1, s));
        ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, hun, uoff, cap + 1, s));
      }
      k_hub_units<<<nd_grid(cap, 256), 256, 0, s>>>(nhub, hubs, hoff, uoff, hun, g.row, fan[k],
                                                   units, vinfo);
      const FastDiv fB((uint32_t)B[k]), fm((uint32_t)fan[k]);
      auto kpl = knob.pl == 1 ? k_fx_place<1> : knob.pl == 2 ? k_fx_place<2> : k_fx_place<4>;
      kpl<<<nd_grid(N, 256 * knob.pl, knob.pl_grid), 256, 0, s>>>(
          blk[k], rank[k], N, fB, fan[k], sample_lo, g.row, vinfo, th.tm, gpos, hoff, perm, small,
          nhub + 1, blk[k + 1], scnt);
      prof.step_built();
      const uint64_t b0 = key_base(seed, (uint64_t)k, 0, 0);
      k_fx_small<<<nd_grid(items, IND_BLOCK, 148 * 16), IND_BLOCK, 0, s>>>(
          gv, b0, fm, blk[k], small, nhub + 1, blk[k + 1], ctr);
      FxHub hb{gv, b0, fm, hubs, nhub, hoff, uoff, cap, units, perm, blk[k + 1], ctr};
      k_fx_hub_warp<<<knob.hw_grid, IND_BLOCK, HUB_WARP_SMEM, s>>>(hb);
      auto kh = knob.hc == 1 ? k_fx_hub_cta<1> : knob.hc == 2 ? k_fx_hub_cta<2> : k_fx_hub_cta<4>;
      kh<<<knob.hc_grid, IND_BLOCK + 32, HUB_CTA_SMEM, s>>>(hb);
      prof.step_sampled();
      ND_CUDA_TRY(cudaGetLastError());
      nd_free(arena, s);
    }
  }
  // final rows and step rows: counts, scans, one synchronisation for the totals
  FxSteps FS;
  FS.n_steps = (int)S;
  for (int64_t k = 0; k < S; k++) { FS.blk[k] = blk[k + 1]; FS.B[k] = B[k + 1]; }
  int64_t *flen = nullptr, *final_off = nullptr, *step_counts = nullptr, *soff = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&step_counts, S * n + 1, s));
  ND_CUDA_TRY(nd_alloc(&soff, S * n + 1, s));
  const size_t e_fin0 = prof.mark();
  k_fx_flen<<<nd_grid(n + 1, 256), 256, 0, s>>>(scnt, n, R, flen);
  for (int64_t k = 0; k < S; k++)
    k_fx_step_counts<<<nd_grid(n, 256), 256, 0, s>>>(nn[k], n, fan[k], step_counts + k * n);
  ND_CUDA_TRY(cudaMemsetAsync(step_counts + S * n, 0, sizeof(int64_t), s));
  {
    size_t t1 = 0, t2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t1, flen, final_off, n + 1, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, step_counts, soff, S * n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, t1 > t2 ? t1 : t2, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, t1, flen, final_off, n + 1, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, t2, step_counts, soff, S * n + 1, s));
    nd_free(tmp, s);
  }
  int64_t* h = nd_pinned_scratch();  // [0] total, [1] step values, [2] stall, [3..6] ctr, [8..] stats
  ND_TRY(nd_d2h(h, final_off + n, 8, s));
  ND_TRY(nd_d2h(h + 1, soff + S * n, 8, s));
  ND_TRY(nd_d2h(h + 2, stall, sizeof(int), s));
  ND_TRY(nd_d2h(h + 3, ctr, 4 * 8, s));
  ND_TRY(nd_d2h(h + 8, stats, 4 * S * 8, s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  nd_trace("fx:totals(synced)");
  const int64_t total = h[0], total_items = h[1];
  const int h_stall = (int)(h[2] & 0xFFFFFFFF);
  const int64_t slot_bytes = h[3];
  // the run loop stops once no sample has a transit left (core.py:187-203)
  int64_t n_steps = S;
  for (int64_t k = 0; k < S; k++)
    if (h[8 + 4 * k + 3] == 0) { n_steps = k; break; }
  int32_t* final_ids = nullptr;
  int64_t *roots_out = nullptr, *roots_off = nullptr;
  ND_CUDA_TRY(nd_alloc(&final_ids, total > 0 ? total : 1, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, n * R, s));
  ND_CUDA_TRY(nd_alloc(&roots_off, n + 1, s));
  k_fx_final<int32_t><<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(FS, blk[0], n, R, final_off,
                                                                   final_ids, roots_out, roots_off);
  const size_t e_fin1 = prof.mark();
  ND_CUDA_TRY(cudaGetLastError());
  for (int64_t k = 0; k < S; k++) nd_free(nn[k], s);
  nd_free(flen, s); nd_free(scnt, s); nd_free(ctr, s); nd_free(stall, s); nd_free(tp_scratch, s);
  nd_free(vinfo, s); nd_free(nhub, s);
  // step rows (F_STEP_VALS32) are built on first request from the blocks and
  // ranks, which the result keeps until then
  std::vector<int32_t*> kb(blk, blk + S + 1), kr(rank, rank + S);
  std::vector<int64_t> kB(B, B + S + 1), kf(fan, fan + S);
  auto release = [kb, kr, soff, s]() {
    for (auto p : kb) nd_free(p, s);
    for (auto p : kr) nd_free(p, s);
    nd_free(soff, s);
  };
  if (h_stall) {
    release();
    nd_free(final_off, s); nd_free(final_ids, s); nd_free(roots_out, s);
    nd_free(roots_off, s); nd_free(step_counts, s); nd_free(stats, s);
    prof.destroy();
    return ND_ERR_STALL;
  }
  nd_result* res = new nd_result();
  res->stream = s;
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n * R;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n * R);
  res->set(ND_F_ROOTS_OFF, roots_off, n + 1);
  res->set(ND_F_STEP_COUNTS, step_counts, n_steps * n);
  res->set(ND_F_STEP_VALS32, nullptr, total_items);
  res->lazy_field = ND_F_STEP_VALS32;
  res->lazy_build = [kb, kr, kB, kf, soff, n, n_steps, total_items](nd_result* r) {
    int32_t* vals = nullptr;
    ND_CUDA_TRY(nd_alloc(&vals, total_items > 0 ? total_items : 1, r->stream));
    for (int64_t k = 0; k < n_steps; k++) {
      const int64_t items = n * kB[k + 1];
      k_fx_step_vals<<<nd_grid(items, 256, 148 * 64), 256, 0, r->stream>>>(
          kb[k + 1], kr[k], n, kB[k], kf[k], soff + k * n, vals);
    }
    ND_CUDA_TRY(cudaGetLastError());
    r->set(ND_F_STEP_VALS32, vals, total_items);
    return ND_OK;
  };
  res->lazy_free = release;
  res->set(ND_F_STATS, stats, 4 * n_steps);
  res->counters[NDC_ITEMS] = total_items;
  res->counters[NDC_SLOT_BYTES] = slot_bytes;
  res->counters[NDC_STEPS] = n_steps;
  res->counters[NDC_LAUNCHES] = 2 * S + 6;
  if (prof.on) {
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    const auto st = prof.to_result(res);
    res->prof_ms[0] = st[0];
    res->prof_ms[1] = st[1];
    res->prof_ms[2] = prof.between(e_fin0, e_fin1);
  }
  prof.destroy();
  *out_res = res;
  nd_trace("fx:done");
  return ND_OK;
}

extern "C" int nd_run_individual(const nd_graph* G, int app_code, const double* host_params,
                                 int64_t n_params, const int64_t* host_fanouts, int64_t n_fanouts,
                                 int64_t sample_lo, int64_t n, const int64_t* roots, int64_t R,
                                 uint64_t seed, int64_t step_cap, int paradigm,
                                 const uint8_t* host_unique, int64_t n_unique, void* stream,
                                 nd_result** out_res) {
  NvtxRange nvtx_run("nd_run_individual");
  NdApp a;
  ND_TRY(nd_make_app(app_code, host_params, n_params, &a));
  if (!G || n < 0 || R < 1 || n_fanouts < 0 || sample_lo < 0 || n >= (1ll << 31)) return ND_ERR_ARG;
  if (app_code == ND_NODE2VEC || app_code == ND_MULTIRW) return ND_ERR_ARG;  // walk engine
  for (int64_t k = 0; k < n_fanouts; k++)
    if (host_fanouts[k] < 1) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const DevGraph& g = G->g;
  const int key_bits = key_bits_for(g.V);
  const int64_t S_max = n_fanouts < step_cap ? n_fanouts : step_cap;
  // k-hop without unique steps: the fixed-layout run (sample-parallel, or
  // transit-sorted for TP; one host synchronisation; identical outputs and
  // TP class statistics).  ND_IND_FIXED=0 disables it.
  static const bool fixed_off = getenv("ND_IND_FIXED") && getenv("ND_IND_FIXED")[0] == '0';
  bool any_unique = false;
  for (int64_t k = 0; k < S_max; k++) any_unique |= nd_unique_at(host_unique, n_unique, k);
  if (!fixed_off && app_code == ND_KHOP && !any_unique) {
    const int rc = run_individual_fixed(G, a, host_fanouts, S_max, sample_lo, n, roots, R, seed,
                                        paradigm == ND_TP, s, out_res);
    if (rc != ND_ERR_ARG) return rc;  // ND_ERR_ARG: the layout does not fit, run the loop
  }

  int32_t* roots32 = nullptr;
  if (!roots) {
    ND_CUDA_TRY(nd_alloc(&roots32, n * R, s));
    ND_TRY(nd_uniform_roots_i32(g, R, seed, sample_lo, n, roots32, s));
  }
  int64_t P = n * R;
  uint32_t* pt = nullptr;
  int32_t *psid = nullptr, *ptix = nullptr;
  int64_t *spo = nullptr, *tot = nullptr, *nnz = nullptr, *stats = nullptr;
  unsigned long long* ctr = nullptr;
  int* stall = nullptr;
  ND_CUDA_TRY(nd_alloc(&pt, P, s));
  ND_CUDA_TRY(nd_alloc(&psid, P, s));
  ND_CUDA_TRY(nd_alloc(&ptix, P, s));
  ND_CUDA_TRY(nd_alloc(&spo, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&tot, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&nnz, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 4, s));
  ND_CUDA_TRY(nd_alloc(&stall, 1, s));
  ND_CUDA_TRY(nd_alloc(&stats, 4 * (S_max + 1), s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stall, 0, sizeof(int), s));
  ND_CUDA_TRY(cudaMemsetAsync(tot, 0, (n + 1) * sizeof(int64_t), s));
  ND_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * (S_max + 1) * sizeof(int64_t), s));
  ND_CUDA_TRY(cudaMemsetAsync(spo, 0, (n + 1) * sizeof(int64_t), s));
  if (P) k_ind_init<<<nd_grid(P, 256), 256, 0, s>>>(roots, roots32, n, R, pt, psid, ptix, spo);
  uint32_t* const pt0 = pt;  // step-0 pairs (the roots); later steps' pairs live in `steps`
  int32_t* const psid0 = psid;
  int32_t* const ptix0 = ptix;

  // step-count matrix [S_max, n] and scratch
  int64_t* step_counts = nullptr;
  ND_CUDA_TRY(nd_alloc(&step_counts, S_max * n, s));
  std::vector<StepData> steps;
  TPScratch TS;
  int64_t tp_cap = 0;
  int64_t* h_tmp = nd_pinned_scratch();
  uint8_t* fb = nullptr;      // per-sample SP-fallback flags after a unique step
  int* nfb = nullptr;
  unsigned long long* scratch_stats = nullptr;
  ND_CUDA_TRY(nd_alloc(&fb, n, s));
  ND_CUDA_TRY(nd_alloc(&nfb, 1, s));
  ND_CUDA_TRY(nd_alloc(&scratch_stats, 4, s));
  int64_t n_flagged = 0;      // host copy for the current step
  int64_t step = 0;
  Profiler prof(s);
  nd_trace("ind:start");
  while (step < S_max && P > 0) {
    nd_trace("ind:step-begin");
    const int64_t m = host_fanouts[step];
    const int64_t items = P * m;
    StepData sd;
    sd.items = items;
    ND_CUDA_TRY(nd_alloc(&sd.out, items, s));
    ND_CUDA_TRY(nd_alloc(&sd.cum, n, s));
    ND_CUDA_TRY(cudaMemcpyAsync(sd.cum, tot, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    IndCtx c{view(g), a, key_base(seed, (uint64_t)step, 0, 0), sample_lo, m, pt, psid, ptix,
             sd.out, stall};
    unsigned long long* st_step = reinterpret_cast<unsigned long long*>(stats + 4 * step);
    prof.step_begin();
    if (paradigm == ND_TP && n_flagged > 0) {
      // statistics over the unflagged pairs only; flagged pairs are single fetches
      int64_t *kf = nullptr, *kp = nullptr;
      ND_CUDA_TRY(nd_alloc(&kf, P + 1, s));
      ND_CUDA_TRY(nd_alloc(&kp, P + 1, s));
      k_keep_unflagged<<<nd_grid(P + 1, 256), 256, 0, s>>>(pt, psid, fb, P, kf);
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, kf, kp, P + 1, s);
      void* tmp;
      ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
      ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, kf, kp, P + 1, s));
      ND_TRY(nd_d2h(h_tmp, kp + P, sizeof(int64_t), s));
      ND_CUDA_TRY(cudaStreamSynchronize(s));
      const int64_t K = h_tmp[0];
      if (K > tp_cap) {
        if (tp_cap) TS.release(s);
        ND_TRY(TS.alloc(K, key_bits, s));
        tp_cap = K;
      }
      if (K) {
        uint32_t *k0, *k1;
        uint64_t *v0, *v1;
        ND_CUDA_TRY(nd_alloc(&k0, K, s)); ND_CUDA_TRY(nd_alloc(&k1, K, s));
        ND_CUDA_TRY(nd_alloc(&v0, K, s)); ND_CUDA_TRY(nd_alloc(&v1, K, s));
        k_keep_write<<<nd_grid(P, 256), 256, 0, s>>>(pt, kf, kp, P, k0, v0);
        cub::DoubleBuffer<uint32_t> dk(k0, k1);
        cub::DoubleBuffer<uint64_t> dv(v0, v1);
        ND_TRY(tp_sort(dk, dv, K, key_bits, TS, s));
        k_mark<<<nd_grid(K, 256), 256, 0, s>>>(dk.Current(), K, TS.flags);
        size_t t2 = TS.cub_bytes;
        ND_CUDA_TRY(cub::DeviceScan::InclusiveSum(TS.cub_tmp, t2, TS.flags, TS.gid, (int)K, s));
        ND_CUDA_TRY(cudaMemsetAsync(TS.counters, 0, 4 * sizeof(int), s));
        k_gstart<<<nd_grid(K, 256), 256, 0, s>>>(TS.flags, TS.gid, K, TS.gstart, TS.counters);
        k_ind_classify<<<nd_grid(K, 256), 256, 0, s>>>(TS.gstart, TS.counters, m, TS.med_list,
                                                        TS.counters + 1, TS.large_units,
                                                        TS.counters + 2, st_step);
        nd_free(k0, s); nd_free(k1, s); nd_free(v0, s); nd_free(v1, s);
      }
      k_add_fetch<<<1, 1, 0, s>>>(st_step, (unsigned long long)(P - K));
      nd_free(kf, s); nd_free(kp, s); nd_free(tmp, s);
      st_step = scratch_stats;  // the execution below still runs TP; its stats are discarded
      ND_CUDA_TRY(cudaMemsetAsync(scratch_stats, 0, 4 * sizeof(unsigned long long), s));
    }
    if (paradigm == ND_TP) {
      if (P > tp_cap) {
        if (tp_cap) TS.release(s);
        ND_TRY(TS.alloc(P, key_bits, s));
        tp_cap = P;
      }
      uint32_t *k0, *k1;
      uint64_t *v0, *v1;
      ND_CUDA_TRY(nd_alloc(&k0, P, s));
      ND_CUDA_TRY(nd_alloc(&k1, P, s));
      ND_CUDA_TRY(nd_alloc(&v0, P, s));
      ND_CUDA_TRY(nd_alloc(&v1, P, s));
      k_iota_pairs<<<nd_grid(P, 256), 256, 0, s>>>(pt, P, k0, v0);
      cub::DoubleBuffer<uint32_t> dk(k0, k1);
      cub::DoubleBuffer<uint64_t> dv(v0, v1);
      ND_TRY(tp_sort(dk, dv, P, key_bits, TS, s));
      const uint32_t* keys = dk.Current();
      const uint64_t* vals = dv.Current();
      k_mark<<<nd_grid(P, 256), 256, 0, s>>>(keys, P, TS.flags);
      size_t tb = TS.cub_bytes;
      ND_CUDA_TRY(cub::DeviceScan::InclusiveSum(TS.cub_tmp, tb, TS.flags, TS.gid, (int)P, s));
      ND_CUDA_TRY(cudaMemsetAsync(TS.counters, 0, 4 * sizeof(int), s));
      k_gstart<<<nd_grid(P, 256), 256, 0, s>>>(TS.flags, TS.gid, P, TS.gstart, TS.counters);
      // lists: small groups -> med_list, medium/large units -> large_units
      k_ind_classify<<<nd_grid(P, 256), 256, 0, s>>>(TS.gstart, TS.counters, m, TS.med_list,
                                                      TS.counters + 1, TS.large_units,
                                                      TS.counters + 2, st_step);
      const StageSpec sp = stage_spec(!g.unit && (app_code == ND_DEEPWALK || app_code == ND_PPR), 0);
      prof.step_built();
      k_ind_small<<<148 * 8, IND_BLOCK, 0, s>>>(c, keys, vals, TS.gstart, TS.med_list,
                                                TS.counters + 1, ctr);
      k_ind_group<<<148 * 4, IND_BLOCK, STAGE_BYTES, s>>>(c, keys, vals, TS.gstart,
                                                          TS.large_units, TS.counters + 2, g, sp,
                                                          ctr);
      prof.step_sampled();
      ND_CUDA_TRY(cudaGetLastError());
      nd_free(k0, s); nd_free(k1, s); nd_free(v0, s); nd_free(v1, s);
    } else {
      prof.step_built();
      k_ind_flat<<<(unsigned)((items + IND_BLOCK - 1) / IND_BLOCK), IND_BLOCK, 0, s>>>(c, P, ctr);
      prof.step_sampled();
      // SP fetches: one adjacency read per (sample, transit) pair
      k_add_fetch<<<1, 1, 0, s>>>(st_step, (unsigned long long)P);
    }
    nd_trace("ind:sampled(issued)");
    // stable compaction of the non-NULL slots -> next pairs
    int32_t* flags = nullptr;
    int64_t *sc = nullptr, *spo_next = nullptr;
    ND_CUDA_TRY(nd_alloc(&flags, items + 1, s));
    ND_CUDA_TRY(nd_alloc(&sc, items + 1, s));
    ND_CUDA_TRY(nd_alloc(&spo_next, n + 1, s));
    ND_CUDA_TRY(cudaMemsetAsync(flags + items, 0, sizeof(int32_t), s));
    k_flags_nonnull<<<nd_grid(items, 256), 256, 0, s>>>(sd.out, items, flags);
    {
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, sc, items + 1, s);
      void* tmp;
      ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
      ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flags, sc, items + 1, s));
      k_ind_counts<<<nd_grid(n + 1, 256), 256, 0, s>>>(spo, n, m, sc, step_counts + step * n, nnz,
                                                       tot);
      size_t tb2 = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb2, nnz, spo_next, n + 1, s);
      void* tmp2;
      ND_CUDA_TRY(nd_alloc((char**)&tmp2, tb2, s));
      ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp2, tb2, nnz, spo_next, n + 1, s));
      nd_free(tmp, s);
      nd_free(tmp2, s);
    }
    ND_TRY(nd_d2h(h_tmp, sc + items, sizeof(int64_t), s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    const int64_t Pn = h_tmp[0];
    nd_trace("ind:compacted(synced)");
    sd.nnext = Pn;
    ND_CUDA_TRY(nd_alloc(&sd.npt, Pn, s));
    ND_CUDA_TRY(nd_alloc(&sd.npsid, Pn, s));
    ND_CUDA_TRY(nd_alloc(&sd.nptix, Pn, s));
    if (items)
      k_ind_compact<<<nd_grid(items, 256), 256, 0, s>>>(sd.out, items, m, sc, psid, spo_next,
                                                         sd.npt, sd.npsid, sd.nptix);
    ND_CUDA_TRY(cudaGetLastError());
    n_flagged = 0;
    if (nd_unique_at(host_unique, n_unique, step)) {
      // finish_step (driver.py:165-172): each sample's step becomes its sorted
      // distinct non-NULL vertices; the next transits are that list
      int32_t *usid = nullptr, *uval = nullptr;
      int64_t um = 0;
      ND_TRY(nd_dedup_segments(sd.npsid, reinterpret_cast<const int32_t*>(sd.npt), Pn, n, g.V,
                               &usid, &uval, &um, nnz, s));
      ND_CUDA_TRY(cudaMemsetAsync(nnz + n, 0, sizeof(int64_t), s));
      {
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, nnz, spo_next, n + 1, s);
        void* tmp;
        ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
        ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, nnz, spo_next, n + 1, s));
        nd_free(tmp, s);
      }
      int32_t* utix = nullptr;
      ND_CUDA_TRY(nd_alloc(&utix, um, s));
      if (um) k_dedup_tix<<<nd_grid(um, 256), 256, 0, s>>>(usid, um, spo_next, utix);
      if (n) ND_CUDA_TRY(cudaMemcpyAsync(step_counts + step * n, nnz, n * sizeof(int64_t),
                                         cudaMemcpyDeviceToDevice, s));
      ND_CUDA_TRY(cudaMemsetAsync(nfb, 0, sizeof(int), s));
      if (n) k_fallback<<<nd_grid(n, 256), 256, 0, s>>>(nnz, n, m, fb, nfb);
      int hn = 0;
      ND_TRY(nd_d2h(&hn, nfb, sizeof(int), s));
      ND_CUDA_TRY(cudaStreamSynchronize(s));
      n_flagged = hn;
      nd_free(sd.npt, s);
      nd_free(sd.npsid, s);
      nd_free(sd.nptix, s);
      sd.npt = reinterpret_cast<uint32_t*>(uval);
      sd.npsid = usid;
      sd.nptix = utix;
      sd.nnext = um;
      sd.dedup = true;
    }
    if (n) k_tot_add<<<nd_grid(n, 256), 256, 0, s>>>(tot, nnz, n);
    nd_free(flags, s);
    nd_free(sc, s);
    nd_free(spo, s);
    spo = spo_next;
    // the next step's pairs are this step's compacted list (kept for the final
    // rows; freed with the step data at the end)
    pt = sd.npt;
    psid = sd.npsid;
    ptix = sd.nptix;
    P = sd.nnext;
    steps.push_back(sd);
    step++;
  }
  const int64_t n_steps = step;
  // ---- outputs ------------------------------------------------------------------
  int32_t* final_ids = nullptr;  // int32 vertex ids (F_FINAL_IDS32; int64 derived on request)
  int32_t* step_vals = nullptr;  // int32 (F_STEP_VALS32; int64 derived on request)
  int64_t *flen = nullptr, *final_off = nullptr, *roots_out = nullptr, *roots_off = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, n * R, s));
  ND_CUDA_TRY(nd_alloc(&roots_off, n + 1, s));
  ND_CUDA_TRY(cudaMemcpyAsync(flen, tot, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  ND_CUDA_TRY(cudaMemsetAsync(flen + n, 0, sizeof(int64_t), s));
  if (n) k_plus_r<<<nd_grid(n, 256), 256, 0, s>>>(flen, n, R);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flen, final_off, n + 1, s);
    void* tmp;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flen, final_off, n + 1, s));
    nd_free(tmp, s);
  }
  ND_TRY(nd_d2h(h_tmp, final_off + n, sizeof(int64_t), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t total = h_tmp[0];
  nd_trace("ind:final-scan(synced)");
  ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
  if (n * R) {
    if (roots)
      k_ind_roots<int64_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots, n, R, final_off, final_ids,
                                                              roots_out, roots_off);
    else
      k_ind_roots<int32_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots32, n, R, final_off,
                                                              final_ids, roots_out, roots_off);
  } else {
    ND_CUDA_TRY(cudaMemsetAsync(roots_off, 0, (n + 1) * sizeof(int64_t), s));
  }
  int64_t total_items = 0;
  for (auto& sd : steps) total_items += sd.dedup ? sd.nnext : sd.items;
  ND_CUDA_TRY(nd_alloc(&step_vals, total_items, s));
  int64_t pos = 0;
  for (auto& sd : steps) {
    if (sd.nnext)
      k_ind_final<<<nd_grid(sd.nnext, 256), 256, 0, s>>>(sd.npt, sd.npsid, sd.nptix, sd.nnext,
                                                          final_off, sd.cum, R, final_ids);
    if (sd.dedup) {
      if (sd.nnext)
        ND_CUDA_TRY(cudaMemcpyAsync(step_vals + pos, sd.npt, sd.nnext * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, s));
      pos += sd.nnext;
    } else {
      if (sd.items)
        ND_CUDA_TRY(cudaMemcpyAsync(step_vals + pos, sd.out, sd.items * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, s));
      pos += sd.items;
    }
  }
  ND_CUDA_TRY(cudaGetLastError());
  int h_stall = 0;
  unsigned long long h_ctr[4];
  ND_TRY(nd_d2h(&h_stall, stall, sizeof(int), s));
  ND_TRY(nd_d2h(h_ctr, ctr, sizeof(h_ctr), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  nd_trace("ind:done(synced)");
  for (auto& sd : steps) {
    nd_free(sd.out, s);
    nd_free(sd.cum, s);
    nd_free(sd.npt, s);
    nd_free(sd.npsid, s);
    nd_free(sd.nptix, s);
  }
  nd_free(pt0, s); nd_free(psid0, s); nd_free(ptix0, s);
  nd_free(spo, s); nd_free(tot, s); nd_free(nnz, s); nd_free(ctr, s); nd_free(stall, s);
  nd_free(fb, s); nd_free(nfb, s); nd_free(scratch_stats, s);
  nd_free(flen, s); nd_free(roots32, s);
  if (tp_cap) TS.release(s);
  if (h_stall) {
    nd_free(final_off, s); nd_free(final_ids, s); nd_free(roots_out, s); nd_free(roots_off, s);
    nd_free(step_vals, s); nd_free(step_counts, s); nd_free(stats, s);
    prof.destroy();
    return ND_ERR_STALL;
  }
  nd_result* res = new nd_result();
  res->stream = s;
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n * R;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n * R);
  res->set(ND_F_ROOTS_OFF, roots_off, n + 1);
  res->set(ND_F_STEP_COUNTS, step_counts, n_steps * n);
  res->set(ND_F_STEP_VALS32, step_vals, total_items);
  res->set(ND_F_STATS, stats, 4 * n_steps);
  res->counters[NDC_ITEMS] = total_items;
  res->counters[NDC_SLOT_BYTES] = (int64_t)h_ctr[0];
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

// ---- k-hop minibatch plans: one CUDA graph per (graph, fanouts, batch size) ----
// GraphSAGE trains on many small batches (1,024 roots); a
// batch through nd_run_individual is ~15 launches, stream-ordered
// allocations and one host synchronisation (totals size the outputs), so a
// single batch costs far more than its sampling.  A plan allocates every
// buffer once with upper-bound sizes (final ids: n * (1 + sum of the step
// blocks)), captures the fixed-layout SP run for n samples into a CUDA graph
// whose kernels read the batch's roots and (sample_lo, seed) from device
// memory, and replays it per batch: no allocation, no host synchronisation,
// one graph launch.  Rows equal nd_run_individual's for the same roots and
// sample ids (driver.py:203-235 with keyed draws, tests/test_gpu_khop_plan.py).

struct KhopDyn {
  int64_t sample_lo;
  uint64_t seed;
};

namespace {

__global__ void k_khop_set_dyn(KhopDyn* d, int64_t sample_lo, uint64_t seed) {
  d->sample_lo = sample_lo;
  d->seed = seed;
}

// one thread per (sample, parent, slot) of step s: u % deg over the parent's
// row (_ckernels.pyx:212-223), key (seed, sample, step, rank, slot) read from
// the batch's device parameters; per-sample non-NULL counts as k_fx_sample
__global__ void __launch_bounds__(IND_BLOCK) k_fxg_sample(const int64_t* __restrict__ row,
                                                         const int32_t* __restrict__ col,
                                                         const KhopDyn* __restrict__ dyn, int step,
                                                         int64_t n, FastDiv Bp, FastDiv m,
                                                         const int32_t* __restrict__ prev,
                                                         const int32_t* __restrict__ rank,
                                                         int32_t* __restrict__ out,
                                                         unsigned long long* __restrict__ cnt) {
  const int64_t sample_lo = dyn->sample_lo;
  const uint64_t base0 = key_base(dyn->seed, (uint64_t)step, 0, 0);
  const int64_t total = n * (int64_t)Bp.d * m.d;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x; q0 < total; q0 += stride) {
    const int64_t q = q0 + threadIdx.x;
    int64_t i = -1;
    int32_t o = -1;
    if (q < total) {
      const uint32_t ip = m.div((uint32_t)q), slot = (uint32_t)q - ip * m.d;
      const int32_t v = prev[ip];
      i = Bp.div(ip);
      if (v >= 0) {
        const int64_t lo = __ldg(row + v), deg = __ldg(row + v + 1) - lo;
        if (deg > 0) {
          const uint64_t ik = key_item((uint64_t)(sample_lo + i), (uint64_t)rank[ip], (uint64_t)slot);
          o = __ldg(col + lo + (int64_t)mod_u64(draw_u64(base0, ik), (uint64_t)deg));
        }
      }
      out[q] = o;
    }
    const unsigned act = __ballot_sync(0xffffffffu, o >= 0);
    const unsigned same = __match_any_sync(0xffffffffu, i);
    const unsigned grp = act & same;
    if (o >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(cnt + i, (unsigned long long)__popc(grp));
  }
}

}  // namespace

struct nd_khop_plan {
  const nd_graph* G = nullptr;
  int64_t n = 0, S = 0, cap = 0;
  int64_t B[9] = {}, fan[8] = {};
  int64_t* roots = nullptr;      // int64 [n], filled per batch
  KhopDyn* dyn = nullptr;
  int32_t* blk[9] = {};
  int32_t* rank[8] = {};
  int64_t* nn[8] = {};
  unsigned long long* scnt = nullptr;
  unsigned long long* fetch = nullptr;
  int64_t *flen = nullptr, *final_off = nullptr, *roots_out = nullptr, *roots_off = nullptr;
  int32_t* final_ids = nullptr;
  void* tmp = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern "C" int nd_khop_plan_destroy(nd_khop_plan* p) {
  if (!p) return ND_OK;
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  for (auto* x : p->blk) cudaFree(x);
  for (auto* x : p->rank) cudaFree(x);
  for (auto* x : p->nn) cudaFree(x);
  cudaFree(p->roots); cudaFree(p->dyn); cudaFree(p->scnt); cudaFree(p->fetch);
  cudaFree(p->flen); cudaFree(p->final_off); cudaFree(p->roots_out); cudaFree(p->roots_off);
  cudaFree(p->final_ids); cudaFree(p->tmp);
  delete p;
  return ND_OK;
}

extern "C" int nd_khop_plan_create(const nd_graph* G, const int64_t* host_fanouts, int64_t n_fanouts,
                                   int64_t n_samples, void* stream, nd_khop_plan** out) {
  NvtxRange nvtx("nd_khop_plan_create");
  if (!G || !out || n_samples <= 0 || n_samples >= (1ll << 31) || n_fanouts < 1 || n_fanouts > 8)
    return ND_ERR_ARG;
  auto* p = new nd_khop_plan();
  p->G = G;
  p->n = n_samples;
  p->S = n_fanouts;
  p->B[0] = 1;
  int64_t cells = 1;
  for (int64_t k = 0; k < n_fanouts; k++) {
    if (host_fanouts[k] < 1) { delete p; return ND_ERR_ARG; }
    p->fan[k] = host_fanouts[k];
    p->B[k + 1] = p->B[k] * host_fanouts[k];
    cells += p->B[k + 1];
    if ((double)n_samples * (double)p->B[k + 1] >= 4.0e9) { delete p; return ND_ERR_ARG; }
  }
  const int64_t n = n_samples;
  p->cap = n * cells;  // roots + every slot of every step: the final ids' upper bound
  auto fail = [&](cudaError_t e) {
    nd_set_last_error(cudaGetErrorString(e), __FILE__, __LINE__);
    nd_khop_plan_destroy(p);
    return e == cudaErrorMemoryAllocation ? ND_ERR_NOMEM : ND_ERR_CUDA;
  };
  cudaError_t e = cudaSuccess;
#define PLAN_ALLOC(ptr, count) \
  if ((e = cudaMalloc(&(ptr), (size_t)(count) * sizeof(*(ptr)))) != cudaSuccess) return fail(e)
  PLAN_ALLOC(p->roots, n);
  PLAN_ALLOC(p->dyn, 1);
  for (int64_t k = 0; k <= p->S; k++) PLAN_ALLOC(p->blk[k], n * p->B[k]);
  for (int64_t k = 0; k < p->S; k++) {
    PLAN_ALLOC(p->rank[k], n * p->B[k]);
    PLAN_ALLOC(p->nn[k], n);
  }
  PLAN_ALLOC(p->scnt, n);
  PLAN_ALLOC(p->fetch, 1);
  PLAN_ALLOC(p->flen, n + 1);
  PLAN_ALLOC(p->final_off, n + 1);
  PLAN_ALLOC(p->roots_out, n);
  PLAN_ALLOC(p->roots_off, n + 1);
  PLAN_ALLOC(p->final_ids, p->cap);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, p->flen, p->final_off, n + 1);
  PLAN_ALLOC(*reinterpret_cast<char**>(&p->tmp), tb + 16);
#undef PLAN_ALLOC
  // capture the batch: roots -> blocks -> counts -> offsets -> final rows
  cudaStream_t cs;
  if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  const DevGraph& g = G->g;
  FxSteps FS;
  FS.n_steps = (int)p->S;
  for (int64_t k = 0; k < p->S; k++) { FS.blk[k] = p->blk[k + 1]; FS.B[k] = p->B[k + 1]; }
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    cudaMemsetAsync(p->scnt, 0, n * sizeof(unsigned long long), cs);
    k_fx_narrow_roots<<<nd_grid(n, 256), 256, 0, cs>>>(p->roots, n, p->blk[0]);
    for (int64_t k = 0; k < p->S; k++) {
      k_fx_rank<<<nd_grid(n * 32, 256, 148 * 32), 256, 0, cs>>>(p->blk[k], n, p->B[k], p->rank[k],
                                                                p->nn[k], p->fetch);
      k_fxg_sample<<<nd_grid(n * p->B[k + 1], IND_BLOCK, 148 * 64), IND_BLOCK, 0, cs>>>(
          g.row, g.col, p->dyn, (int)k, n, FastDiv((uint32_t)p->B[k]), FastDiv((uint32_t)p->fan[k]),
          p->blk[k], p->rank[k], p->blk[k + 1], p->scnt);
    }
    k_fx_flen<<<nd_grid(n + 1, 256), 256, 0, cs>>>(p->scnt, n, 1, p->flen);
    cub::DeviceScan::ExclusiveSum(p->tmp, tb, p->flen, p->final_off, n + 1, cs);
    k_fx_final<int32_t><<<nd_grid(n * 32, 256, 148 * 32), 256, 0, cs>>>(FS, p->blk[0], n, 1, p->final_off,
                                                                       p->final_ids, p->roots_out,
                                                                       p->roots_off);
    e = cudaStreamEndCapture(cs, &p->graph);
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&p->exec, p->graph, 0);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess) return fail(e);
  (void)stream;
  *out = p;
  return ND_OK;
}

// One batch: the roots (device int64 [n], copied into the plan; NULL: the
// plan's roots buffer was filled by the caller) with sample ids
// [sample_lo, sample_lo + n) and the seed, then the captured graph.  Fully
// asynchronous on `stream`; outputs (nd_khop_plan_outputs) are valid after it.
extern "C" int nd_khop_plan_run(nd_khop_plan* p, const int64_t* roots, int64_t sample_lo,
                                uint64_t seed, void* stream) {
  if (!p || sample_lo < 0) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  k_khop_set_dyn<<<1, 1, 0, s>>>(p->dyn, sample_lo, seed);
  if (roots && roots != p->roots)
    ND_CUDA_TRY(cudaMemcpyAsync(p->roots, roots, p->n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  ND_CUDA_TRY(cudaGraphLaunch(p->exec, s));
  return ND_OK;
}

// Device views: roots buffer (int64 [n]), final offsets (int64 [n+1]; the
// total is final_off[n]), final ids (int32, capacity `cap`), and step k's
// block (int32 [n * B_{k+1}], NULL slots -1) for k < n_steps.
extern "C" int nd_khop_plan_outputs(const nd_khop_plan* p, int64_t** roots, const int64_t** final_off,
                                    const int32_t** final_ids, int64_t* cap, const int32_t** blocks,
                                    int64_t* block_sizes, int64_t n_max) {
  if (!p) return ND_ERR_ARG;
  if (roots) *roots = p->roots;
  if (final_off) *final_off = p->final_off;
  if (final_ids) *final_ids = p->final_ids;
  if (cap) *cap = p->cap;
  for (int64_t k = 0; k < p->S && k < n_max; k++) {
    if (blocks) blocks[k] = p->blk[k + 1];
    if (block_sizes) block_sizes[k] = p->n * p->B[k + 1];
  }
  return ND_OK;
}
