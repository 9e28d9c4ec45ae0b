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

#include <cstdlib>

#include <vector>

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
  for (int64_t k = 0; k < S; k++) {
    ND_CUDA_TRY(nd_alloc(&rank[k], n * B[k], s));
    ND_CUDA_TRY(nd_alloc(&nn[k], n, s));
    ND_CUDA_TRY(nd_alloc(&blk[k + 1], n * B[k + 1], s));
    const int64_t items = n * B[k + 1];
    if (!tp) {
      k_fx_rank<<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(blk[k], n, B[k], rank[k], nn[k],
                                                              stats + 4 * k + 3);
      k_fx_sample<<<nd_grid(items, IND_BLOCK, 148 * 64), IND_BLOCK, 0, s>>>(
          gv, a, key_base(seed, (uint64_t)k, 0, 0), sample_lo, n, FastDiv((uint32_t)B[k]),
          FastDiv((uint32_t)fan[k]), blk[k], rank[k], blk[k + 1], scnt, stall, ctr);
      continue;
    }
    // transit-parallel order: sort the parent slots by transit, classify the groups
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
    k_fx_sample_tp<<<nd_grid(items, IND_BLOCK, 148 * 64), IND_BLOCK, 0, s>>>(
        gv, a, key_base(seed, (uint64_t)k, 0, 0), sample_lo, N, FastDiv((uint32_t)B[k]),
        FastDiv((uint32_t)fan[k]), sentinel, k1, v1, blk[k + 1], stall, ctr);
    k_fx_block_counts<<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(blk[k + 1], n, B[k + 1], scnt);
    nd_free(k0, s); nd_free(k1, s); nd_free(v0, s); nd_free(v1, s);
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
  ND_CUDA_TRY(cudaGetLastError());
  for (int64_t k = 0; k < S; k++) nd_free(nn[k], s);
  nd_free(flen, s); nd_free(scnt, s); nd_free(ctr, s); nd_free(stall, s); nd_free(tp_scratch, s);
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
      k_ind_small<<<148 * 8, IND_BLOCK, 0, s>>>(c, keys, vals, TS.gstart, TS.med_list,
                                                TS.counters + 1, ctr);
      k_ind_group<<<148 * 4, IND_BLOCK, STAGE_BYTES, s>>>(c, keys, vals, TS.gstart,
                                                          TS.large_units, TS.counters + 2, g, sp,
                                                          ctr);
      ND_CUDA_TRY(cudaGetLastError());
      nd_free(k0, s); nd_free(k1, s); nd_free(v0, s); nd_free(v1, s);
    } else {
      k_ind_flat<<<(unsigned)((items + IND_BLOCK - 1) / IND_BLOCK), IND_BLOCK, 0, s>>>(c, P, ctr);
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
  *out_res = res;
  return ND_OK;
}
