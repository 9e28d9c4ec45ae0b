// nd_walk.cu — whole-run chain walks on device (engine/chain.py:64-179).
//
// DeepWalk / PPR / node2vec: walker state (current transit, packed
// (walker id, previous transit)) lives in HBM; each step either runs the flat
// sample-parallel kernel (SP) or the transit-parallel step of nd_tp.cuh (TP).
// Every item appends a step record (walker, vertex) and, if alive, its next
// state (warp-aggregated compaction); a NULL result records the walker's
// death step (chain.py:152-155: walks die after a NULL pick).  After the loop
// the records are scattered into the compacted final layout
// (roots, then non-NULL vertices in step order; core.py:116-123).
//
// MultiRW (root pick, chain.py:102-108,144-151): every walker is alive every
// step; the transit is roots[key(domain 1) % R]; the sampled vertex replaces
// the first root equal to the transit.  Values go to a dense [steps, N] slab.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "nd_tp.cuh"

using namespace nd;

namespace {

struct ChainAct {
  GView<int32_t> gv;
  NdApp a;
  uint64_t base0;
  int64_t sample_lo;
  int step;
  int32_t* rec_w;
  int32_t* rec_v;
  uint32_t* ncur;
  uint64_t* nwp;
  int* ncount;
  int32_t* dstep;
  int* stall;
  int32_t* rows;  // fixed-length walks: per-walker rows [n, ld] written in place (else records)
  int64_t ld;

  template <class RowT>
  __device__ __forceinline__ void operator()(int64_t i, int64_t v, uint64_t val, const RowT& row,
                                             int64_t deg, ItemStats& st) const {
    const int32_t w = (int32_t)(val >> 32);
    const int64_t t = (int64_t)(int32_t)(uint32_t)(val & 0xFFFFFFFFull);
    int stl = 0;
    const int64_t out = run_item(gv, row, a, v, deg, t, base0,
                                 key_item((uint64_t)(sample_lo + w), 0, 0), st, &stl);
    if (stl) atomicExch(stall, 1);
    if (rows != nullptr) {
      if (out >= 0) rows[(int64_t)w * ld + step] = (int32_t)out;
    } else {
      rec_w[i] = w;
      rec_v[i] = (int32_t)out;
    }
    const int64_t slot = warp_append(out >= 0, ncount);
    if (slot >= 0) {
      ncur[slot] = (uint32_t)out;
      nwp[slot] = ((uint64_t)(uint32_t)w << 32) | (uint32_t)v;
    } else {
      dstep[w] = step;
    }
  }
};

struct RootPickAct {
  GView<int32_t> gv;
  NdApp a;
  uint64_t base0;
  int64_t sample_lo;
  int32_t* roots;  // [N, R] mutated
  int64_t R;
  int32_t* slab;   // this step's [N] values
  int* stall;

  template <class RowT>
  __device__ __forceinline__ void operator()(int64_t i, int64_t v, uint64_t val, const RowT& row,
                                             int64_t deg, ItemStats& st) const {
    const int64_t w = (int64_t)(val >> 32);
    int stl = 0;
    const int64_t out = run_item(gv, row, a, v, deg, -1, base0,
                                 key_item((uint64_t)(sample_lo + w), 0, 0), st, &stl);
    slab[w] = (int32_t)out;
    if (out >= 0) {
      int32_t* rr = roots + w * R;
      for (int64_t c = 0; c < R; c++)
        if (rr[c] == (int32_t)v) { rr[c] = (int32_t)out; break; }
    }
  }
};

__global__ void k_init_chain(const int64_t* __restrict__ roots64, const int32_t* __restrict__ roots32,
                             int64_t n, int64_t R, uint32_t* __restrict__ cur,
                             uint64_t* __restrict__ wp, int32_t* __restrict__ dstep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    cur[i] = roots64 ? (uint32_t)roots64[i * R] : (uint32_t)roots32[i * R];
    wp[i] = ((uint64_t)(uint32_t)i << 32) | 0xFFFFFFFFull;  // prev = NULL
    dstep[i] = -1;
  }
}

// root pick (domain 1): key = roots[w, key_u64(seed, sid, step, 0, 0, 1) % R]
__global__ void k_rootpick_keys(const int32_t* __restrict__ roots, int64_t n, int64_t R,
                                uint64_t base1, int64_t sample_lo, uint32_t* __restrict__ keys,
                                uint64_t* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = draw_u64(base1, key_item((uint64_t)(sample_lo + i), 0, 0));
    const int64_t pick = (int64_t)mod_u64(u, (uint64_t)R);
    keys[i] = (uint32_t)roots[i * R + pick];
    vals[i] = (uint64_t)i << 32;
  }
}

__global__ void k_chain_lengths(const int32_t* __restrict__ dstep, int64_t n, int64_t R,
                                int64_t n_steps, int64_t* __restrict__ flen,
                                int64_t* __restrict__ clen) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { flen[n] = 0; continue; }
    const int32_t d = dstep[i];
    const int64_t nnz = d >= 0 ? d : n_steps;
    flen[i] = R + nnz;
    clen[i] = d >= 0 ? d + 1 : n_steps;
  }
}

template <typename RootT>
__global__ void k_write_roots(const RootT* __restrict__ roots, int64_t n, int64_t R,
                              const int64_t* __restrict__ off, int32_t* __restrict__ ids,
                              int64_t* __restrict__ roots_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * R;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i / R, k = i - w * R;
    const int64_t r = (int64_t)roots[i];
    ids[off[w] + k] = (int32_t)r;
    if (roots_out) roots_out[i] = r;
  }
}

__global__ void k_scatter_records(const int32_t* __restrict__ rec_w, const int32_t* __restrict__ rec_v,
                                  int64_t total, const int64_t* __restrict__ step_base,
                                  int64_t n_steps, const int64_t* __restrict__ off, int64_t R,
                                  int32_t* __restrict__ ids) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < total;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = rec_v[r];
    if (v < 0) continue;
    int64_t lo = 0, hi = n_steps;  // last step s with step_base[s] <= r
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (step_base[mid] <= r) lo = mid; else hi = mid;
    }
    ids[off[rec_w[r]] + R + lo] = v;
  }
}

// fixed-length TP walks: each walker's first min(len, steps) values from its row
__global__ void k_rows_emit(const int32_t* __restrict__ rows, int64_t ld,
                            const int32_t* __restrict__ dstep, int64_t n, int64_t n_steps,
                            int64_t steps, const int64_t* __restrict__ off, int64_t R,
                            int32_t* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < n; w += nw) {
    const int32_t d = dstep[w];
    int64_t len = d >= 0 ? d : n_steps;
    if (len > steps) len = steps;
    const int32_t* src = rows + w * ld;
    int32_t* dst = ids + off[w] + R;
    for (int64_t k = lane; k < len; k += 32) dst[k] = src[k];
  }
}

// multirw: per-walker non-NULL counts over the slab, then the final rows
__global__ void k_slab_counts(const int32_t* __restrict__ slab, int64_t n, int64_t S, int64_t R,
                              int64_t* __restrict__ flen) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= n;
       w += (int64_t)gridDim.x * blockDim.x) {
    if (w == n) { flen[n] = 0; continue; }
    int64_t c = 0;
    for (int64_t s = 0; s < S; s++) c += slab[s * n + w] >= 0;
    flen[w] = R + c;
  }
}

__global__ void k_slab_write(const int32_t* __restrict__ slab, int64_t n, int64_t S, int64_t R,
                             const int64_t* __restrict__ off, int32_t* __restrict__ ids,
                             int64_t* __restrict__ chain) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n;
       w += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = off[w] + R;
    for (int64_t s = 0; s < S; s++) {
      const int32_t v = slab[s * n + w];
      if (chain) chain[w * S + s] = v;
      if (v >= 0) ids[p++] = v;
    }
  }
}

__global__ void k_stats_fetch(unsigned long long* stats, unsigned long long n) { stats[3] += n; }


// ---- walker-major persistent kernel (SP) ------------------------------------------
// Each lane owns one walker at a time and advances it step after step with the
// walker state in registers (no per-step state traffic, no global sync); when
// its walker dies or leaves the step window it takes the next walker from a
// warp-aggregated work queue, so divergent walk lengths (PPR) keep every lane
// busy.  Values go to a row-major window [rows, Lw] (one row per walker).
struct PWArgs {
  GView<int32_t> gv;
  NdApp a;
  uint64_t seed;
  int64_t sample_lo;
  int64_t n;                 // rows this window
  const int32_t* wid;        // row -> walker (nullptr: identity)
  const int32_t* v0;         // row start transit (nullptr: roots)
  const int32_t* t0;         // row previous vertex
  const int64_t* roots64;
  const int32_t* roots32;
  int64_t R;
  int64_t step0, step_end;
  int64_t Lw;                // row stride of `out` (window length padded to 8)
  int32_t* out;              // [n, Lw]
  int32_t* nnz;              // per row: non-NULL values written
  int32_t* died;             // per walker: 1 when its walk ended with NULL
  int32_t* cont_wid;         // continuation (alive at step_end)
  int32_t* cont_v;
  int32_t* cont_t;
  int* cont_n;
  int* queue;
  int* max_len;
  int* stall;
  unsigned long long* ctr;
  const VRec* vrec;   // packed vertex records (or null)
  const NbrW* nbw;    // neighbour records (or null)
  const NbrP* nbp;
  const NbrU* nbu;
  const PickLine* pl;    // line-packed pick rows (DeepWalk / PPR on weighted graphs) or null
  const int32_t* vline;  // first line of each row (with pl)
  int chunk;             // walkers a warp claims per queue atomic (32 or 64)
};

// one 32-byte sector: row bounds, max weight and prefix total of v
__device__ __forceinline__ void load_vertex(const PWArgs& A, int64_t v, int64_t& lo, int64_t& deg,
                                            double& mx, double& tot) {
  if (A.vrec != nullptr) {
    int4 a, b;
    ld32B(A.vrec + v, a, b);
    lo = ((int64_t)(uint32_t)a.y << 32) | (uint32_t)a.x;
    deg = ((int64_t)(uint32_t)a.w << 32) | (uint32_t)a.z;
    mx = __longlong_as_double(((long long)(uint32_t)b.y << 32) | (uint32_t)b.x);
    tot = __longlong_as_double(((long long)(uint32_t)b.w << 32) | (uint32_t)b.z);
  } else {
    lo = __ldg(A.gv.row + v);
    deg = __ldg(A.gv.row + v + 1) - lo;
    mx = -1.0;
    tot = -1.0;
  }
}

// accept/reject of one node2vec try whose pick (nb, w) is known; -2 = rejected.
// t's row is probed only when the decision depends on it (n2v_accept).
__device__ __forceinline__ int64_t n2v_decide(const PWArgs& A, int64_t nb, double w, int64_t t,
                                              int64_t tlo, int64_t thi, double env, uint64_t b,
                                              uint64_t ik, ItemStats& st) {
  st.tries++;
  st.bytes += 2 * SECTOR;
  const double u01 = to_unit(draw_u64(b + C_DRAW, ik));
  bool probed = false;
  const bool acc = n2v_accept(A.a, nb, t, w, u01, env, [&] {
    if (A.gv.hset != nullptr && thi - tlo > HASH_MIN_DEG)
      return hset_contains(A.gv.hset + 4 * tlo, hset_size(thi - tlo), (int32_t)nb, &st.sect);
    st.sect += 1 + search_sectors(thi - tlo);
    return has_edge(A.gv.col, tlo, thi, nb);
  }, probed);
  if (probed) st.bytes += SECTOR * search_sectors(thi - tlo);
  return acc ? nb : -2;
}

// node2vec rejection try j for a walker at v with previous vertex t
// (_ckernels.pyx:243-262); returns the neighbour on acceptance, -2 on reject.
template <class RowT>
__device__ __forceinline__ int64_t n2v_try(const PWArgs& A, const RowT& r, int64_t deg, int64_t t,
                                           int64_t tlo, int64_t thi, double env, uint64_t b,
                                           uint64_t ik, ItemStats& st) {
  const int64_t k = (int64_t)mod_u64(draw_u64(b, ik), (uint64_t)deg);
  int64_t nb;
  double w;
  r.cw(k, nb, w, A.gv.unit);
  return n2v_decide(A, nb, w, t, tlo, thi, env, b, ik, st);
}


// ---- neighbour-record step: the record that selects the next
// vertex carries its header (row start, degree, max weight / prefix total).
struct NextHdr {
  int64_t lo = -1;
  int64_t deg = 0;
  double mx = -1.0;
  double tot = -1.0;
};

// 32-byte record / 16-byte loads from global memory (read-only path) or from
// a row staged in shared memory (SH) by the transit-parallel hub kernels
template <bool SH>
__device__ __forceinline__ void ldrec32(const void* p, int4& a, int4& b) {
  if (SH) {
    a = reinterpret_cast<const int4*>(p)[0];
    b = reinterpret_cast<const int4*>(p)[1];
  } else {
    ld32B(p, a, b);
  }
}
template <bool SH>
__device__ __forceinline__ int4 ldrec16(const void* p) {
  return SH ? *reinterpret_cast<const int4*>(p) : __ldg(reinterpret_cast<const int4*>(p));
}
template <bool SH>
__device__ __forceinline__ double ldf64(const double* p) {
  return SH ? *p : __ldg(p);
}

// weighted pick over a row's neighbour records rp[0, deg) (or unit records
// ru); gd = the row's guide table (global) or null
template <bool SH>
__device__ __forceinline__ int64_t rec_pick_at(const NbrP* rp, const NbrU* ru, const int32_t* gd0,
                                               int64_t deg, double tot, double u01, NextHdr& nh,
                                               ItemStats& st) {
  if (ru != nullptr) {  // unit weights: floor identity
    int64_t k = (int64_t)__dmul_rn(u01, (double)deg);
    if (k > deg - 1) k = deg - 1;
    const int4 r = ldrec16<SH>(ru + k);
    nh.deg = r.y;
    nh.lo = (int64_t)(((uint64_t)(uint32_t)r.w << 32) | (uint32_t)r.z);
    nh.mx = nh.deg > 0 ? 1.0 : 0.0;
    nh.tot = (double)nh.deg;
    st.bytes += SECTOR + 8;
    st.sect += 1;
    return r.x;
  }
  const double x = __dmul_rn(u01, tot);
  int64_t a = 0, b = deg;
  if (gd0 != nullptr && deg > GUIDE_MIN_DEG) {
    const int64_t j = guide_bucket(x, tot, deg);
    if (j >= 0) {  // guide[j], guide[j+1]: adjacent, one sector unless they straddle
      const int32_t* gd = gd0 + j;
      a = __ldg(gd);
      b = j + 1 < deg ? (int64_t)__ldg(gd + 1) : deg;
      st.sect += 1 + (j + 1 < deg && (reinterpret_cast<uintptr_t>(gd) >> 5) !=
                                         (reinterpret_cast<uintptr_t>(gd + 1) >> 5));
    }
  }
  // upper bound over [a, b) with whole-record (32-byte) probes: the probe
  // that proves the answer is usually the selected record itself
  int64_t have = -1;
  int4 h0 = make_int4(0, 0, 0, 0), h1 = h0;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    int4 q0, q1;
    ldrec32<SH>(rp + mid, q0, q1);
    st.sect += 1;
    const double pre = __longlong_as_double(((long long)(uint32_t)q0.y << 32) | (uint32_t)q0.x);
    if (pre <= x) {
      a = mid + 1;
    } else {
      b = mid;
      have = mid;
      h0 = q0;
      h1 = q1;
    }
  }
  const int64_t k = a < deg - 1 ? a : deg - 1;
  if (k != have) {
    ldrec32<SH>(rp + k, h0, h1);
    st.sect += 1;
  }
  nh.deg = h0.w;
  nh.lo = ((int64_t)(uint32_t)h1.y << 32) | (uint32_t)h1.x;
  nh.tot = __longlong_as_double(((long long)(uint32_t)h1.w << 32) | (uint32_t)h1.z);
  nh.mx = -1.0;
  st.bytes += SECTOR + SECTOR * search_sectors(deg) + SECTOR + 8;
  return h0.z;
}

__device__ __forceinline__ int64_t rec_pick(const PWArgs& A, int64_t lo, int64_t deg, double tot,
                                            double u01, NextHdr& nh, ItemStats& st) {
  return rec_pick_at<false>(A.nbu ? nullptr : A.nbp + lo, A.nbu ? A.nbu + lo : nullptr,
                            A.gv.guide ? A.gv.guide + lo : nullptr, deg, tot, u01, nh, st);
}

// weighted pick over the line-packed rows (PickLine, nd_common.cuh): the
// exact bucket's bracket guide[j], guide[j+1] sits in the line of bucket j,
// next to the records around j (the upper-bound probes and the selected
// record are usually sectors of that same line).  L = the row's first line.
template <bool SH>
__device__ __forceinline__ int64_t line_pick_at(const PickLine* L, int64_t deg, double tot,
                                                double u01, NextHdr& nh, ItemStats& st) {
  const double x = __dmul_rn(u01, tot);
  int64_t a = 0, b = deg;
  const int64_t j = guide_bucket(x, tot, deg);
  int64_t line = -1;
  if (j >= 0) {
    const int4 g = ldrec16<SH>(L[j / 3].g);  // 16-byte aligned
    const int sidx = (int)(j % 3);
    a = sidx == 0 ? g.x : sidx == 1 ? g.y : g.z;
    b = sidx == 0 ? g.y : sidx == 1 ? g.z : g.w;
    line = j / 3;
    st.sect += 1;
  }
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (mid / 3 != line) { line = mid / 3; st.sect += 1; }
    if (ldf64<SH>(&L[mid / 3].r[mid % 3].pre) <= x) a = mid + 1; else b = mid;
  }
  const int64_t k = a < deg - 1 ? a : deg - 1;
  if (k / 3 != line) st.sect += 1;
  int4 h0, h1;
  ldrec32<SH>(&L[k / 3].r[k % 3], h0, h1);
  nh.tot = __longlong_as_double(((long long)(uint32_t)h0.w << 32) | (uint32_t)h0.z);
  nh.deg = h1.y;
  nh.lo = h1.z;
  nh.mx = -1.0;
  st.bytes += SECTOR + SECTOR * search_sectors(deg) + SECTOR + 8;
  return h1.x;
}

__device__ __forceinline__ int64_t line_pick(const PWArgs& A, int64_t llo, int64_t deg, double tot,
                                             double u01, NextHdr& nh, ItemStats& st) {
  return line_pick_at<false>(A.pl + llo, deg, tot, u01, nh, st);
}

// one node2vec rejection try over the row's neighbour records rw (or unit
// records ru); -2 = rejected
template <bool SH>
__device__ __forceinline__ int64_t rec_try_at(const PWArgs& A, const NbrW* rw, const NbrU* ru,
                                              int64_t deg, int64_t t, int64_t tlo, int64_t thi,
                                              double env, uint64_t b, uint64_t ik, NextHdr& nh,
                                              ItemStats& st) {
  const int64_t k = (int64_t)mod_u64(draw_u64(b, ik), (uint64_t)deg);
  int64_t nb;
  double w;
  st.sect += 1;
  if (ru != nullptr) {
    const int4 r = ldrec16<SH>(ru + k);
    nb = r.x;
    w = 1.0;
    nh.deg = r.y;
    nh.lo = (int64_t)(((uint64_t)(uint32_t)r.w << 32) | (uint32_t)r.z);
    nh.mx = nh.deg > 0 ? 1.0 : 0.0;
  } else {
    int4 r0, r1;
    ldrec32<SH>(rw + k, r0, r1);  // the whole record in one 32-byte request
    nb = r0.x;
    nh.deg = r0.y;
    nh.lo = (int64_t)(((uint64_t)(uint32_t)r0.w << 32) | (uint32_t)r0.z);
    w = __longlong_as_double(((long long)(uint32_t)r1.y << 32) | (uint32_t)r1.x);
    nh.mx = __longlong_as_double(((long long)(uint32_t)r1.w << 32) | (uint32_t)r1.z);
  }
  nh.tot = -1.0;
  return n2v_decide(A, nb, w, t, tlo, thi, env, b, ik, st);
}

__device__ __forceinline__ int64_t rec_try(const PWArgs& A, int64_t lo, int64_t deg, int64_t t,
                                           int64_t tlo, int64_t thi, double env, uint64_t b,
                                           uint64_t ik, NextHdr& nh, ItemStats& st) {
  return rec_try_at<false>(A, A.nbu ? nullptr : A.nbw + lo, A.nbu ? A.nbu + lo : nullptr, deg, t,
                           tlo, thi, env, b, ik, nh, st);
}


template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_walk_persistent(PWArgs A) {
  ItemStats st;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1;
  int64_t row = -1, w = 0, v = 0, t = -1, s = 0, lo = 0, deg = 0, tlo = -1, thi = -1;
  double mx = -1.0, tot = -1.0;
  int64_t j = 0;          // node2vec try index of the current step
  uint64_t ik = 0;
  int32_t* orow = nullptr;
  int64_t wbeg = 0, wend = 0;  // this warp's claimed walker range (warp-uniform)
  const bool n2v = A.a.code == ND_NODE2VEC;
  while (true) {
    // ---- hand out walkers from the warp's chunk (one atomic per A.chunk)
    const bool need = row < 0;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
      const int c = __popc(m);
      const int rank = __popc(m & lt_mask);
      int64_t rem = wend - wbeg, nbeg = 0;
      if (rem < c) {
        int base = 0;
        if (lane == 0) base = atomicAdd(A.queue, A.chunk);
        nbeg = __shfl_sync(0xffffffffu, base, 0);
      }
      if (need) {
        row = rank < rem ? wbeg + rank : nbeg + (rank - rem);
        if (row < A.n) {
          w = A.wid ? A.wid[row] : row;
          if (A.v0) {
            v = A.v0[row];
            t = A.t0[row];
          } else {
            v = A.roots64 ? A.roots64[w * A.R] : A.roots32[w * A.R];
            t = -1;
          }
          tlo = thi = -1;
          s = A.step0;
          j = 0;
          ik = key_item((uint64_t)(A.sample_lo + w), 0, 0);
          orow = A.out + row * A.Lw;
          load_vertex(A, v, lo, deg, mx, tot);
          if (A.pl) lo = __ldg(A.vline + v);  // line-packed rows: lo is v's first line
          st.bytes += SECTOR + 8;
          st.sect += 1;
          if (n2v && t >= 0) {  // continuing node2vec walker: t's row for the probes
            tlo = __ldg(A.gv.row + t);
            thi = __ldg(A.gv.row + t + 1);
            if (mx < 0.0) mx = __ldg(A.gv.mx + v);
            st.sect += 1;
          }
        }
      }
      if (rem < c) {
        wbeg = nbeg + (c - rem);
        wend = nbeg + A.chunk;
      } else {
        wbeg += c;
      }
    }
    if (__all_sync(0xffffffffu, row >= A.n)) break;
    if (row >= A.n) continue;
    // ---- one unit of work: a node2vec try (step >= 1) or a whole step
    int stl = 0;
    int64_t o;
    NextHdr nh;
    const uint64_t base0 = key_base(A.seed, (uint64_t)s, 0, 0);
    const bool recs = (A.nbp != nullptr || A.nbu != nullptr) && (!n2v || A.nbw || A.nbu);
    if (recs) {
      if (deg <= 0) {
        o = -1;
      } else if (n2v && t >= 0) {
        if (j == 0) st.bytes += 2 * SECTOR;  // t offsets + max_w (§8 d pair term)
        const double env = __dmul_rn(mx, A.a.f_max);
        o = rec_try(A, lo, deg, t, tlo, thi, env, base0 + 2 * C_DRAW * (uint64_t)j, ik, nh, st);
        if (o == -2) {
          if (++j >= N2V_MAX_TRIES) {
            atomicExch(A.stall, 1);
            o = -1;
          } else {
            continue;  // rejected: the lane tries again next iteration
          }
        }
      } else if (A.a.code == ND_PPR) {
        if (to_unit(draw_u64(base0, ik)) < A.a.term) o = -1;
        else if (A.pl) o = line_pick(A, lo, deg, tot, to_unit(draw_u64(base0 + C_DRAW, ik)), nh, st);
        else o = rec_pick(A, lo, deg, tot, to_unit(draw_u64(base0 + C_DRAW, ik)), nh, st);
      } else {  // DeepWalk, node2vec step 0: draw 0 weighted pick
        o = A.pl ? line_pick(A, lo, deg, tot, to_unit(draw_u64(base0, ik)), nh, st)
                 : rec_pick(A, lo, deg, tot, to_unit(draw_u64(base0, ik)), nh, st);
      }
    } else if (n2v && t >= 0 && deg > 0) {
      if (j == 0) st.bytes += 2 * SECTOR;  // t offsets + max_w (§8 d pair term)
      const double env = __dmul_rn(mx >= 0.0 ? mx : __ldg(A.gv.mx + v), A.a.f_max);
      o = n2v_try(A, grow(A.gv, lo), deg, t, tlo, thi, env, base0 + 2 * C_DRAW * (uint64_t)j, ik,
                  st);
      if (o == -2) {
        if (++j >= N2V_MAX_TRIES) {
          atomicExch(A.stall, 1);
          o = -1;
        } else {
          continue;  // rejected: the lane tries again next iteration
        }
      }
    } else {  // plain CSR rows (records not built: ND_NO_PACK)
      o = run_item(A.gv, grow(A.gv, lo), A.a, v, deg, t, base0, ik, st, &stl, tlo, thi, mx, tot);
    }
    if (stl) atomicExch(A.stall, 1);
    orow[s - A.step0] = (int32_t)o;
    s++;
    j = 0;
    if (o < 0) {
      A.nnz[row] = (int32_t)(s - 1 - A.step0);
      A.died[w] = 1;
      atomicMax(A.max_len, (int)s);
      row = -1;
    } else if (s == A.step_end) {
      A.nnz[row] = (int32_t)(s - A.step0);
      atomicMax(A.max_len, (int)s);
      const int slot = atomicAdd(A.cont_n, 1);
      A.cont_wid[slot] = (int32_t)w;
      A.cont_v[slot] = (int32_t)o;
      A.cont_t[slot] = (int32_t)v;
      row = -1;
    } else {
      tlo = lo;
      thi = lo + deg;
      t = v;
      v = o;
      if (nh.lo >= 0) {  // header delivered by the selecting record
        lo = nh.lo;
        deg = nh.deg;
        mx = nh.mx;
        tot = nh.tot;
        if (n2v && mx < 0.0) { mx = __ldg(A.gv.mx + v); st.sect += 1; }  // after node2vec's step-0 pick
      } else {
        load_vertex(A, v, lo, deg, mx, tot);
        if (A.pl) lo = __ldg(A.vline + v);
        st.sect += 1;
      }
      st.bytes += SECTOR + 8;
    }
  }
  flush_stats(st, A.ctr);
}

// per-walker totals across windows
__global__ void k_pw_accum(const int32_t* __restrict__ wid, const int32_t* __restrict__ nnz,
                           int64_t n, int64_t* __restrict__ tot) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    tot[wid ? wid[r] : r] += nnz[r];
}

__global__ void k_pw_lengths(const int64_t* __restrict__ tot, const int32_t* __restrict__ died,
                             int64_t n, int64_t R, int64_t* __restrict__ flen,
                             int64_t* __restrict__ clen, unsigned long long* __restrict__ hist,
                             int64_t hist_len) {
  // chain-length histogram (per-step alive counts for RunStats): shared-memory
  // bins for short lengths, global atomics beyond
  constexpr int SH = 4096;
  __shared__ unsigned int sh[SH];
  for (int k = threadIdx.x; k < SH; k += blockDim.x) sh[k] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { flen[n] = 0; continue; }
    flen[i] = R + tot[i];
    const int64_t c = tot[i] + died[i];
    clen[i] = c;
    if (c < SH) atomicAdd(sh + c, 1u);
    else if (c < hist_len) atomicAdd(hist + c, 1ull);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < SH && k < hist_len; k += blockDim.x)
    if (sh[k]) atomicAdd(hist + k, (unsigned long long)sh[k]);
}

// copy one window's rows into the final layout: one warp per row, lanes
// stream the row's non-NULL prefix (int32 reads and writes, both coalesced)
__global__ void k_pw_emit(const int32_t* __restrict__ wid, const int32_t* __restrict__ out,
                          const int32_t* __restrict__ nnz, int64_t n, int64_t Lw, int64_t step0,
                          const int64_t* __restrict__ off, int64_t R, int32_t* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nw) {
    const int64_t k_end = nnz[r];
    const int64_t w = wid ? wid[r] : r;
    int32_t* dst = ids + off[w] + R + step0;
    const int32_t* src = out + r * Lw;
    for (int64_t k = lane; k < k_end; k += 32) dst[k] = src[k];
  }
}

// per-step fetch stats (SP): alive at step s = #{walkers: chain length > s}
__global__ void k_pw_stats(const unsigned long long* __restrict__ hist, int64_t n_steps,
                           int64_t n, unsigned long long* __restrict__ stats) {
  if (blockIdx.x || threadIdx.x) return;
  unsigned long long alive = (unsigned long long)n;
  for (int64_t s = 0; s < n_steps; s++) {
    alive -= hist[s];  // walkers with chain length == s stop before step s
    stats[4 * s + 3] = alive;
  }
}
}  // namespace

static int g_profile = 0;
int nd_profiling() { return g_profile; }
// persisting-L2 set-aside shared by concurrent TP walk runs (nd_walk_hub engine)
static std::mutex g_l2_mu;
static int g_l2_users = 0;
static size_t g_l2_prev = 0;
extern "C" int nd_set_profiling(int on) {
  g_profile = on;
  return ND_OK;
}

// Runs started by the calling host thread share the GPU with k-1 others
// (engine.submit_device_concurrent, HostPipeline, ShardedJob: one host thread
// per concurrent job).  The persistent walk kernels then launch their share
// of every SM's CTA slots instead of all of them: a persistent grid holds its
// slots until its walker queue drains, so a full grid makes a concurrent
// job's kernels wait behind it instead of running beside it.
static thread_local int t_share = 1;
extern "C" int nd_set_concurrency(int k) {
  if (k < 1) return ND_ERR_ARG;
  t_share = k;
  return ND_OK;
}
int nd_concurrency() { return t_share; }



// One walker-major window: rows [n] (row -> walker wid, or the identity),
// entering step step0 at vertex vin (previous vertex tin; both null: the roots).
struct PWindow {
  int32_t *wid, *out, *nnz, *vin, *tin;
  int64_t n, step0, Lw, ld;  // Lw = steps this window covers, ld = row stride
};

static int pw_run_windows(const nd_graph* G, const NdApp& a, uint64_t seed, int64_t sample_lo,
                          int64_t rows, int32_t* cwid, int32_t* cv, int32_t* ct,
                          const int64_t* roots, const int32_t* roots32, int64_t R, int64_t step0,
                          int64_t limit, int64_t Lw_base, int32_t* died, int* ctl,
                          unsigned long long* ctr, bool keep_inputs, cudaStream_t s,
                          std::vector<PWindow>& wins, int* h, double* sample_ms);
static void pw_free_windows(std::vector<PWindow>& wins, cudaStream_t s);

// ---- TP tail: once few walkers remain, TP groups are (nearly) singletons and a
// step costs its launch chain; the remaining steps run in walker-major windows
// (identical outputs: every draw is keyed by (sample, step)), and each tail
// step's TP class statistics are computed exactly afterwards from the logged
// transits (a radix sort of (step, transit) keys + run lengths).
__global__ void k_tail_init(const uint32_t* __restrict__ cur, const uint64_t* __restrict__ wp,
                            int64_t n, int32_t* __restrict__ wid, int32_t* __restrict__ v,
                            int32_t* __restrict__ t) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = wp[i];
    wid[i] = (int32_t)(x >> 32);
    v[i] = (int32_t)cur[i];
    t[i] = (int32_t)(uint32_t)(x & 0xFFFFFFFFull);
  }
}

// per row: steps it entered (non-NULL values + the NULL that ended it) and,
// for walkers that died in the window, their death step
__global__ void k_tail_rows(const int32_t* __restrict__ wid, const int32_t* __restrict__ nnz,
                            int64_t n, int64_t step0, int64_t Lw, int32_t* __restrict__ dstep,
                            int64_t* __restrict__ ent) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = nnz[r];
    if (e < Lw) {
      if (dstep) dstep[wid[r]] = (int32_t)(step0 + e);
      e += 1;
    }
    ent[r] = e;
  }
}

// (step - tail0, transit) keys of every step a row entered, warp per row
__global__ void k_tail_keys(const int32_t* __restrict__ vin, const int32_t* __restrict__ out,
                            const int64_t* __restrict__ ent, const int64_t* __restrict__ koff,
                            int64_t n, int64_t ld, int64_t rel0, int key_bits,
                            uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int64_t e = ent[r];
    uint64_t* dst = keys + koff[r];
    for (int64_t i = lane; i < e; i += 32) {
      const int32_t v = i == 0 ? vin[r] : out[r * ld + i - 1];
      dst[i] = ((uint64_t)(rel0 + i) << key_bits) | (uint32_t)v;
    }
  }
}

// TP tail class statistics of small graphs by counting (no sort): per window,
// chunks of K steps count every entry (row r, window step i < ent[r], transit
// v = i ? out[r][i-1] : vin[r]) into cnt[(i - j0) * V + v], K*V counters small
// enough to stay in L2.  The atomic's old value marks the member that opens
// its group (0), makes it medium (31: the 32nd) or large (1024: the 1025th):
// transit_parallel.py:86-101's classes with m = 1.  A second pass zeroes the
// counters it touched.
constexpr int TAIL_K_MAX = 64;
template <bool CLEAR>
__global__ void k_tail_count(const int32_t* __restrict__ vin, const int32_t* __restrict__ out,
                             const int64_t* __restrict__ ent, int64_t n, int64_t ld, int64_t j0,
                             int logK, int kk, int64_t V, int32_t* __restrict__ cnt,
                             unsigned long long* __restrict__ cls) {
  __shared__ unsigned int sc[TAIL_K_MAX * 3];
  if (!CLEAR) {
    for (int i = threadIdx.x; i < 3 * kk; i += blockDim.x) sc[i] = 0;
    __syncthreads();
  }
  const int64_t total = n << logK;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q >> logK;
    const int j = (int)(q & ((1 << logK) - 1));
    const int64_t i = j0 + j;
    if (j >= kk || i >= ent[r]) continue;
    const int32_t v = i == 0 ? vin[r] : out[r * ld + i - 1];
    int32_t* c = cnt + (int64_t)j * V + v;
    if (CLEAR) {
      *c = 0;
    } else {
      const int32_t old = atomicAdd(c, 1);
      const int k = old == 0 ? 0 : old == 31 ? 1 : old == 1024 ? 2 : -1;
      if (k >= 0) atomicAdd(&sc[3 * j + k], 1u);
    }
  }
  if (!CLEAR) {
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * kk; i += blockDim.x)
      if (sc[i]) atomicAdd(cls + i, (unsigned long long)sc[i]);
  }
}

// chunk counts -> per-step stats {small, medium, large, groups}; clears cls
__global__ void k_tail_flush(unsigned long long* __restrict__ cls, int K, int64_t step,
                             unsigned long long* __restrict__ stats) {
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const unsigned long long g = cls[3 * j], med = cls[3 * j + 1], lg = cls[3 * j + 2];
    if (g) {
      unsigned long long* st = stats + 4 * (step + j);
      st[0] += g - med;
      st[1] += med - lg;
      st[2] += lg;
      st[3] += g;
    }
    cls[3 * j] = cls[3 * j + 1] = cls[3 * j + 2] = 0;
  }
}

__global__ void k_sum_i64(const int64_t* __restrict__ x, int64_t n, unsigned long long* __restrict__ sum) {
  unsigned long long t = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    t += (unsigned long long)x[i];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0 && t) atomicAdd(sum, t);
}

// class counts per tail step from the (step, transit) runs: each thread walks
// a contiguous range of runs (sorted by step) and flushes per step
__global__ void k_tail_classes(const uint64_t* __restrict__ ukeys, const int* __restrict__ counts,
                               const int* __restrict__ n_runs, int key_bits, int64_t tail0,
                               unsigned long long* __restrict__ stats) {
  constexpr int64_t PER = 64;
  const int64_t G = *n_runs;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * PER; b < G;
       b += (int64_t)gridDim.x * blockDim.x * PER) {
    const int64_t e = b + PER < G ? b + PER : G;
    int64_t cs = -1;
    unsigned long long c[3] = {0, 0, 0};
    for (int64_t i = b; i <= e; i++) {
      const int64_t si = i < e ? tail0 + (int64_t)(ukeys[i] >> key_bits) : -2;
      if (si != cs) {
        if (cs >= 0) {
          unsigned long long* st = stats + 4 * cs;
          for (int k = 0; k < 3; k++)
            if (c[k]) atomicAdd(st + k, c[k]);
          atomicAdd(st + 3, c[0] + c[1] + c[2]);
        }
        cs = si;
        c[0] = c[1] = c[2] = 0;
      }
      if (i < e) {
        const int64_t work = counts[i];  // members * m, m = 1 for walks
        c[work < SMALL_MAX_WORK ? 0 : (work <= LARGE_MIN_WORK ? 1 : 2)]++;
      }
    }
  }
}

static int run_tp_tail(const nd_graph* G, const NdApp& a, uint64_t seed, int64_t sample_lo,
                       int64_t n, int64_t A, const uint32_t* cur, const uint64_t* wp, int64_t R,
                       int64_t step, int64_t limit, int64_t Lw_base, int key_bits, int32_t* dstep,
                       int* stall, unsigned long long* ctr, unsigned long long* stats,
                       cudaStream_t s, std::vector<PWindow>& wins, int64_t& n_steps,
                       int64_t& items, double& sample_ms, int32_t* wid_in = nullptr,
                       int32_t* v_in = nullptr, int32_t* t_in = nullptr,
                       int32_t* died_ext = nullptr);

// TP chain walk (SP chain walks run in run_chain_walk_sp).  Byte-model
// counters (see nd_item.cuh): ctr[0]=bytes, ctr[1]=tries
static int run_chain_walk(const nd_graph* G, const NdApp& a, int64_t sample_lo, int64_t n,
                          const int64_t* roots, int64_t R, uint64_t seed, int64_t steps,
                          int64_t step_cap, int paradigm, cudaStream_t s, nd_result* res) {
  if (paradigm != ND_TP) return ND_ERR_ARG;
  const DevGraph& g = G->g;
  const int key_bits = key_bits_for(g.V);
  uint32_t *cur0 = nullptr, *cur1 = nullptr;
  uint64_t *wp0 = nullptr, *wp1 = nullptr;
  int32_t *dstep = nullptr, *rec_w = nullptr, *rec_v = nullptr, *roots32 = nullptr;
  int* ncount = nullptr;
  int* stall = nullptr;
  unsigned long long* ctr = nullptr;
  unsigned long long* stats = nullptr;
  const int64_t max_steps = steps >= 0 ? (steps < step_cap ? steps : step_cap) : step_cap;
  int64_t rec_cap = 0;
  TPScratch S;
  ND_CUDA_TRY(nd_alloc(&cur0, n, s));
  ND_CUDA_TRY(nd_alloc(&cur1, n, s));
  ND_CUDA_TRY(nd_alloc(&wp0, n, s));
  ND_CUDA_TRY(nd_alloc(&wp1, n, s));
  ND_CUDA_TRY(nd_alloc(&dstep, n, s));
  ND_CUDA_TRY(nd_alloc(&ncount, 1, s));
  ND_CUDA_TRY(nd_alloc(&stall, 1, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 4, s));
  ND_CUDA_TRY(nd_alloc(&stats, 4 * (max_steps + 1), s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * (max_steps + 1) * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stall, 0, sizeof(int), s));
  ND_TRY(S.alloc(n, key_bits, s));
  if (!roots) {
    ND_CUDA_TRY(nd_alloc(&roots32, n * R, s));
    ND_TRY(nd_uniform_roots_i32(g, R, seed, sample_lo, n, roots32, s));
  }
  if (n) k_init_chain<<<nd_grid(n, 256), 256, 0, s>>>(roots, roots32, n, R, cur0, wp0, dstep);
  // fixed-length walks write each value into its walker's row (one random
  // 4-byte store, then a coalesced emission); INF-length walks keep per-step
  // records scattered at the end
  int32_t* rows = nullptr;
  const bool direct = steps >= 0 && max_steps > 0;
  if (direct) ND_CUDA_TRY(nd_alloc(&rows, n * max_steps, s));
  rec_cap = direct ? 0 : (steps >= 0 ? n * max_steps : n * 128);
  ND_CUDA_TRY(nd_alloc(&rec_w, rec_cap, s));
  ND_CUDA_TRY(nd_alloc(&rec_v, rec_cap, s));

  Profiler prof(s);
  std::vector<int64_t> step_base;
  int64_t A = n, rec_base = 0, step = 0;
  uint32_t* cur_in = cur0;
  uint64_t* wp_in = wp0;
  uint32_t* cur_alt = cur1;
  uint64_t* wp_alt = wp1;
  int* h_count = reinterpret_cast<int*>(nd_pinned_scratch());
  double sched_ms = 0, sample_ms = 0;
  // TP tail threshold (ND_TP_TAIL=0: every step through the TP class kernels)
  const int64_t tail_T = getenv("ND_TP_TAIL") ? atoll(getenv("ND_TP_TAIL")) : 131072;
  bool tail = false;
  while (A > 0) {
    if (steps >= 0 && step >= steps) break;
    if (step >= step_cap) break;
    if (paradigm == ND_TP && A <= tail_T && A * (max_steps - step) < (1ll << 31)) {
      tail = true;
      break;
    }
    if (!direct && rec_base + A > rec_cap) {
      int64_t nc = rec_cap * 2 > rec_base + A ? rec_cap * 2 : rec_base + A;
      int32_t *nw = nullptr, *nv = nullptr;
      ND_CUDA_TRY(nd_alloc(&nw, nc, s));
      ND_CUDA_TRY(nd_alloc(&nv, nc, s));
      ND_CUDA_TRY(cudaMemcpyAsync(nw, rec_w, rec_base * 4, cudaMemcpyDeviceToDevice, s));
      ND_CUDA_TRY(cudaMemcpyAsync(nv, rec_v, rec_base * 4, cudaMemcpyDeviceToDevice, s));
      nd_free(rec_w, s);
      nd_free(rec_v, s);
      rec_w = nw;
      rec_v = nv;
      rec_cap = nc;
    }
    ND_CUDA_TRY(cudaMemsetAsync(ncount, 0, sizeof(int), s));
    size_t e0 = prof.ev.size();
    prof.mark();
    const int need_pre = !g.unit && (a.code == ND_DEEPWALK || a.code == ND_PPR ||
                                     (a.code == ND_NODE2VEC && step == 0));
    const int need_w = !g.unit && a.code == ND_NODE2VEC && step > 0;
    unsigned long long* st_step = stats + 4 * step;
    {
      cub::DoubleBuffer<uint32_t> dk(cur_in, cur_alt);
      cub::DoubleBuffer<uint64_t> dv(wp_in, wp_alt);
      ND_TRY(tp_sort(dk, dv, A, key_bits, S, s));
      prof.mark();
      // the sorted state is Current(); the next state is written to Alternate()
      ChainAct act{view(g), a, key_base(seed, (uint64_t)step, 0, 0), sample_lo, (int)step,
                   rec_w + rec_base, rec_v + rec_base, dk.Alternate(), dv.Alternate(), ncount,
                   dstep, stall, rows, max_steps};
      ND_TRY(tp_run_sorted(dk.Current(), dv.Current(), A, 1, g, stage_spec(need_pre, need_w), act,
                           S, ctr, st_step, s));
      cur_in = dk.Alternate();
      wp_in = dv.Alternate();
      cur_alt = dk.Current();
      wp_alt = dv.Current();
    }
    prof.mark();
    ND_TRY(nd_d2h(h_count, ncount, sizeof(int), s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    if (prof.on) {
      sched_ms += prof.between(e0, e0 + 1);
      sample_ms += prof.between(e0 + 1, e0 + 2);
      prof.steps.push_back({e0, e0 + 1, e0 + 2, 1});
    }
    step_base.push_back(rec_base);
    rec_base += A;
    A = *h_count;
    step++;
  }
  const int64_t tp_steps = step;
  int64_t n_steps = step, tail_items = 0;
  step_base.push_back(rec_base);
  std::vector<PWindow> tail_wins;
  if (tail) {
    ND_TRY(run_tp_tail(G, a, seed, sample_lo, n, A, cur_in, wp_in, R, step, max_steps,
                       steps >= 0 ? max_steps - step : 128, key_bits, dstep, stall, ctr, stats, s,
                       tail_wins, n_steps, tail_items, sample_ms));
  }
  // ---- output compaction -----------------------------------------------------------
  prof.mark();
  const size_t ef = prof.ev.size() - 1;
  int32_t* final_ids = nullptr;  // int32 vertex ids (F_FINAL_IDS32; int64 derived on request)
  int64_t *flen = nullptr, *final_off = nullptr, *clen = nullptr,
          *roots_out = nullptr, *d_step_base = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&clen, n, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, n * R, s));
  ND_CUDA_TRY(nd_alloc(&d_step_base, tp_steps + 1, s));
  ND_CUDA_TRY(cudaMemcpyAsync(d_step_base, step_base.data(), (tp_steps + 1) * sizeof(int64_t),
                              cudaMemcpyHostToDevice, s));
  k_chain_lengths<<<nd_grid(n + 1, 256), 256, 0, s>>>(dstep, n, R, n_steps, flen, clen);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flen, final_off, n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flen, final_off, n + 1, s));
    nd_free(tmp, s);
  }
  int64_t total = 0;
  ND_TRY(nd_d2h(&total, final_off + n, sizeof(int64_t), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
  if (n) {
    if (roots)
      k_write_roots<int64_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots, n, R, final_off, final_ids,
                                                                roots_out);
    else
      k_write_roots<int32_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots32, n, R, final_off,
                                                                final_ids, roots_out);
  }
  if (direct && n && tp_steps)
    k_rows_emit<<<nd_grid(n * 32, 256, 148 * 32), 256, 0, s>>>(rows, max_steps, dstep, n, n_steps,
                                                               tp_steps, final_off, R, final_ids);
  else if (!direct && rec_base)
    k_scatter_records<<<nd_grid(rec_base, 256, 148 * 64), 256, 0, s>>>(
        rec_w, rec_v, rec_base, d_step_base, tp_steps, final_off, R, final_ids);
  for (auto& W : tail_wins)
    if (W.n * W.Lw)
      k_pw_emit<<<nd_grid(W.n * 32, 256, 148 * 32), 256, 0, s>>>(W.wid, W.out, W.nnz, W.n, W.ld,
                                                                W.step0, final_off, R, final_ids);
  pw_free_windows(tail_wins, s);
  prof.mark();
  ND_CUDA_TRY(cudaGetLastError());
  int h_stall = 0;
  unsigned long long h_ctr[4];
  ND_TRY(nd_d2h(&h_stall, stall, sizeof(int), s));
  ND_TRY(nd_d2h(h_ctr, ctr, sizeof(h_ctr), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  if (prof.on) res->counters[NDC_STEPS] = 0;
  double final_ms = prof.on ? prof.between(ef, ef + 1) : 0.0;
  prof.to_result(res);
  prof.destroy();

  // stats as int64 (unsigned long long has the same layout)
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n * R;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n * R);
  res->set(ND_F_CHAIN_LEN, clen, n);
  res->set(ND_F_STATS, stats, 4 * n_steps);
  res->counters[NDC_ITEMS] = rec_base + tail_items;
  res->counters[NDC_PAIRS] = rec_base + tail_items;
  res->counters[NDC_N2V_TRIES] = (int64_t)h_ctr[1];
  res->counters[NDC_SLOT_BYTES] = (int64_t)h_ctr[0];
  res->counters[NDC_STEPS] = n_steps;
  res->prof_ms[0] = sched_ms;
  res->prof_ms[1] = sample_ms;
  res->prof_ms[2] = final_ms;

  nd_free(cur0, s); nd_free(cur1, s); nd_free(wp0, s); nd_free(wp1, s);
  nd_free(dstep, s); nd_free(ncount, s); nd_free(stall, s); nd_free(ctr, s);
  nd_free(rec_w, s); nd_free(rec_v, s); nd_free(rows, s); nd_free(roots32, s); nd_free(flen, s);
  nd_free(d_step_base, s);
  if (paradigm == ND_TP) S.release(s);
  return h_stall ? ND_ERR_STALL : ND_OK;
}

__global__ void k_narrow(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}


// A per-app integer knob from the environment: "K" for every app, or
// "code=K,code=K" per app code (ND_DEEPWALK 0, ND_PPR 1, ND_NODE2VEC 2, ...);
// apps not named keep their default.  Parsed per call (no shared state).
static int app_knob(const char* name, int code, int dflt) {
  const char* e = getenv(name);
  if (!e || !*e) return dflt;
  if (!strchr(e, '=')) return atoi(e);
  for (const char* p = e; *p;) {
    const int c = atoi(p);
    const char* q = strchr(p, '=');
    if (!q) break;
    if (c == code) return atoi(q + 1);
    p = strchr(q, ',');
    if (!p) break;
    ++p;
  }
  return dflt;
}

// resident CTAs per SM requested from ptxas for an app's persistent walk
// kernel; shared with concurrent jobs, 4 (64 registers), so that each of
// them holds half of every SM's slots (C2: node2vec || PPR at 2 + 2 CTAs per
// SM 19.3-19.5 ms, against 23.3 at 3 per SM each with the grids queued)
static int walk_minb(int code, int share, bool big) {
  return app_knob("ND_WALK_MINB", code,
                  share > 1 ? 4 : (big || code == ND_PPR || code == ND_NODE2VEC) ? 3 : 4);
}

// A graph whose resident structures exceed ND_WALK_BIG_GB (default 32 GB):
// its random reads spread over more memory than the translation caches
// cover, and with every CTA slot busy the walk kernel's time turns bimodal
// from run to run (C5 DeepWalk alone: 16.2 or 21.7-22.5 ms at 4 CTAs per SM);
// at 2 CTAs per SM (built for 3) it is a steady 17.6 ms.
static bool walk_big_graph(const nd_graph* G) {
  const char* e = getenv("ND_WALK_BIG_GB");
  const double gb = e ? atof(e) : 32.0;
  return (double)G->bytes > gb * 1e9;
}

// Run persistent-kernel windows from step0 until no walker continues or
// `limit`.  Walkers that continue past a window re-enter the next one with
// their (vertex, previous vertex); later windows get proportionally more
// steps so a geometric tail runs in one or two launches.  ctl = [queue,
// cont_n, max_len, stall] (max_len/stall accumulate).  keep_inputs keeps each
// window's vin/tin (the TP tail derives its transits from them).
static int pw_run_windows(const nd_graph* G, const NdApp& a, uint64_t seed, int64_t sample_lo,
                          int64_t rows, int32_t* cwid, int32_t* cv, int32_t* ct,
                          const int64_t* roots, const int32_t* roots32, int64_t R, int64_t step0,
                          int64_t limit, int64_t Lw_base, int32_t* died, int* ctl,
                          unsigned long long* ctr, bool keep_inputs, cudaStream_t s,
                          std::vector<PWindow>& wins, int* h, double* sample_ms) {
  const DevGraph& g = G->g;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // register/occupancy variant of the persistent kernel: resident CTAs per SM
  // requested from ptxas.  Default per app, measured on C2:
  // node2vec and PPR 3 (PPR 6% faster alone, node2vec equal alone, and the
  // two run concurrently in 21.2-21.8 vs 23.2-23.8 ms at 4 on 4 of 5 boxes),
  // DeepWalk 4 (22% slower at 3).  ND_WALK_MINB = "3" sets every app,
  // "1=3,2=4" per app code.
  const int share = nd_concurrency();
  const bool big = share == 1 && walk_big_graph(G);
  const int minb = walk_minb(a.code, share, big);
  void (*kern)(PWArgs) = minb >= 8 ? k_walk_persistent<8>
                         : minb == 6 ? k_walk_persistent<6>
                         : minb == 5 ? k_walk_persistent<5>
                         : minb == 3 ? k_walk_persistent<3> : k_walk_persistent<4>;
  int occ = 4;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
  if (occ < 1) occ = 1;
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (g_profile) {
    cudaEventCreate(&pe0);
    cudaEventCreate(&pe1);
  }
  const int64_t budget = (rows * Lw_base > (1ll << 24)) ? rows * Lw_base : (1ll << 24);
  const int64_t first = step0;
  int rc = ND_OK;
  while (rows > 0 && step0 < limit) {
    int64_t Lw = step0 == first ? Lw_base : budget / rows;
    if (Lw < Lw_base) Lw = Lw_base;
    if (Lw > limit - step0) Lw = limit - step0;
    // row stride padded to 8 values: the kernels flush 32-byte aligned chunks
    const int64_t ld = (Lw + 7) & ~int64_t(7);
    PWindow W{cwid, nullptr, nullptr, cv, ct, rows, step0, Lw, ld};
    nd_trace("sp:window-begin");
    int32_t *nw = nullptr, *nv = nullptr, *nt = nullptr;
    if (nd_alloc(&W.out, rows * ld, s) != cudaSuccess || nd_alloc(&W.nnz, rows, s) != cudaSuccess ||
        nd_alloc(&nw, rows, s) != cudaSuccess || nd_alloc(&nv, rows, s) != cudaSuccess ||
        nd_alloc(&nt, rows, s) != cudaSuccess) {
      rc = ND_ERR_CUDA;
    }
    if (rc == ND_OK && cudaMemsetAsync(ctl, 0, 2 * sizeof(int), s) != cudaSuccess) rc = ND_ERR_CUDA;
    if (rc != ND_OK) {
      nd_free(W.out, s); nd_free(W.nnz, s); nd_free(nw, s); nd_free(nv, s); nd_free(nt, s);
      break;
    }
    PWArgs A{view(g), a, seed, sample_lo, rows, cwid, cv, ct, roots, roots32, R, step0,
             step0 + Lw, ld, W.out, W.nnz, died, nw, nv, nt, ctl + 1, ctl, ctl + 2, ctl + 3, ctr,
             g.vrec, g.nbw, g.nbp, g.nbu,
             (a.code == ND_DEEPWALK || a.code == ND_PPR) ? g.pl : nullptr, g.vline};
    // small windows (few walkers per lane, e.g. L2-resident graphs or the
    // PPR tail): 128-thread CTAs spread over every SM, one walker per lane
    int64_t tpb = 256, grid = (int64_t)nsm * occ;
    // CTAs per SM of this app's windows (ND_WALK_GRID, per app code): below
    // the occupancy, concurrent jobs share every SM instead of queueing
    // behind each other's persistent grids
    {
      int cps = app_knob("ND_WALK_GRID", a.code, 0);
      if (cps <= 0 && share > 1) cps = std::max(1, occ / share);
      if (cps <= 0 && big) cps = 2;
      if (cps > 0 && cps < occ) grid = (int64_t)nsm * cps;
    }
    if (rows < grid * 256) {
      tpb = 128;
      grid = std::min<int64_t>(grid * 2, (rows + 127) / 128);
    }
    A.chunk = rows <= grid * tpb * 2 ? 32 : 64;
    nd_trace("sp:allocs");
    if (g_profile) cudaEventRecord(pe0, s);
    kern<<<(unsigned)grid, (unsigned)tpb, 0, s>>>(A);
    if (g_profile) cudaEventRecord(pe1, s);
    if (cudaGetLastError() != cudaSuccess || nd_d2h(h, ctl, 4 * sizeof(int), s) != ND_OK)
      rc = ND_ERR_CUDA;
    nd_trace("sp:window-synced");
    if (getenv("ND_TRACE") && getenv("ND_TRACE")[0] == '1')
      fprintf(stderr, "[nd_trace]   window step0=%lld Lw=%lld rows=%lld -> continuing %d\n",
              (long long)step0, (long long)Lw, (long long)rows, h[1]);
    if (g_profile && rc == ND_OK) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pe0, pe1);
      *sample_ms += ms;
    }
    if (!keep_inputs) {
      nd_free(cv, s);
      nd_free(ct, s);
      W.vin = W.tin = nullptr;
    }
    wins.push_back(W);
    cwid = nw;
    cv = nv;
    ct = nt;
    rows = h[1];
    step0 += Lw;
    if (rc != ND_OK) break;
  }
  nd_free(cwid, s); nd_free(cv, s); nd_free(ct, s);
  if (g_profile) {
    cudaEventDestroy(pe0);
    cudaEventDestroy(pe1);
  }
  return rc;
}

static void pw_free_windows(std::vector<PWindow>& wins, cudaStream_t s) {
  for (auto& W : wins) {
    nd_free(W.out, s); nd_free(W.nnz, s); nd_free(W.wid, s); nd_free(W.vin, s); nd_free(W.tin, s);
  }
  wins.clear();
}

__global__ void k_or_flag(int* __restrict__ dst, const int* __restrict__ src) {
  if (*src) *dst = 1;
}

static int bits_for(int64_t x) {
  int b = 1;
  while ((1ll << b) <= x) b++;
  return b;
}

// TP tail (see k_tail_init): the A alive walkers (cur, wp) continue from
// `step` in walker-major windows; dstep/stall/ctr/stats are updated as the TP
// steps would have; the windows are returned for the final emission.
static int run_tp_tail(const nd_graph* G, const NdApp& a, uint64_t seed, int64_t sample_lo,
                       int64_t n, int64_t A, const uint32_t* cur, const uint64_t* wp, int64_t R,
                       int64_t step, int64_t limit, int64_t Lw_base, int key_bits, int32_t* dstep,
                       int* stall, unsigned long long* ctr, unsigned long long* stats,
                       cudaStream_t s, std::vector<PWindow>& wins, int64_t& n_steps,
                       int64_t& items, double& sample_ms, int32_t* wid_in,
                       int32_t* v_in, int32_t* t_in,
                       int32_t* died_ext) {
  nd_trace("tp:tail-begin");
  // inputs: the sort engine's (cur, wp) state, or (wid, v, t) rows handed over
  // (the windows take ownership of them)
  int32_t *wid = wid_in, *v = v_in, *t = t_in, *died = died_ext;
  int* ctl = nullptr;
  if (!cur) {
    if (!wid || !v || !t) return ND_ERR_ARG;
  } else {
    ND_CUDA_TRY(nd_alloc(&wid, A, s));
    ND_CUDA_TRY(nd_alloc(&v, A, s));
    ND_CUDA_TRY(nd_alloc(&t, A, s));
  }
  if (!died_ext) ND_CUDA_TRY(nd_alloc(&died, n, s));
  ND_CUDA_TRY(nd_alloc(&ctl, 4, s));
  ND_CUDA_TRY(cudaMemsetAsync(ctl, 0, 4 * sizeof(int), s));
  if (cur) k_tail_init<<<nd_grid(A, 256), 256, 0, s>>>(cur, wp, A, wid, v, t);
  int* h = reinterpret_cast<int*>(nd_pinned_scratch());
  h[1] = h[2] = h[3] = 0;
  int rc = pw_run_windows(G, a, seed, sample_lo, A, wid, v, t, nullptr, nullptr, R, step, limit,
                          Lw_base, died, ctl, ctr, true, s, wins, h, &sample_ms);
  if (rc == ND_OK) {
    k_or_flag<<<1, 1, 0, s>>>(stall, ctl + 3);
    if ((int64_t)h[2] > n_steps) n_steps = h[2];
  }
  if (!died_ext) nd_free(died, s);
  nd_free(ctl, s);
  if (rc != ND_OK) return rc;
  nd_trace("tp:tail-windows");
  {
    // small graphs: the class counts by counting into L2-resident counters
    const int64_t V = G->g.V;
    int64_t K = TAIL_K_MAX;
    while (K > 1 && K * V * 4 > (32ll << 20)) K >>= 1;
    static const bool force_sort = getenv("ND_TAIL_SORT") && getenv("ND_TAIL_SORT")[0] == '1';
    if (K >= 16 && !force_sort) {
      int logK = 0;
      while ((1ll << logK) < K) logK++;
      int32_t* cnt = nullptr;
      unsigned long long *cls = nullptr, *dsum = nullptr;
      int64_t* ent = nullptr;
      int64_t max_n = 1;
      for (const PWindow& W : wins) max_n = std::max(max_n, W.n);
      if (nd_alloc(&cnt, K * V, s) != cudaSuccess || nd_alloc(&cls, 3 * TAIL_K_MAX, s) != cudaSuccess ||
          nd_alloc(&ent, max_n + 1, s) != cudaSuccess || nd_alloc(&dsum, 1, s) != cudaSuccess)
        rc = ND_ERR_CUDA;
      if (rc == ND_OK) {
        cudaMemsetAsync(cnt, 0, K * V * sizeof(int32_t), s);
        cudaMemsetAsync(cls, 0, 3 * TAIL_K_MAX * sizeof(unsigned long long), s);
        cudaMemsetAsync(dsum, 0, sizeof(unsigned long long), s);
      }
      for (size_t k = 0; k < wins.size() && rc == ND_OK; k++) {
        const PWindow& W = wins[k];
        k_tail_rows<<<nd_grid(W.n, 256), 256, 0, s>>>(W.wid, W.nnz, W.n, W.step0, W.Lw, dstep, ent);
        k_sum_i64<<<nd_grid(W.n, 256), 256, 0, s>>>(ent, W.n, dsum);
        for (int64_t j0 = 0; j0 < W.Lw; j0 += K) {
          const int kk = (int)std::min<int64_t>(K, W.Lw - j0);
          const int grid = nd_grid(W.n << logK, 256, 148 * 16);
          k_tail_count<false><<<grid, 256, 0, s>>>(W.vin, W.out, ent, W.n, W.ld, j0, logK, kk, V,
                                                  cnt, cls);
          // the chunk's counters back to zero: one contiguous memset of kk * V
          // (<= 32 MB, L2-resident) instead of a second pass over the rows
          cudaMemsetAsync(cnt, 0, (size_t)kk * V * sizeof(int32_t), s);
          k_tail_flush<<<1, 64, 0, s>>>(cls, kk, W.step0 + j0, stats);
        }
        if (cudaGetLastError() != cudaSuccess) rc = ND_ERR_CUDA;
      }
      if (rc == ND_OK) {
        unsigned long long* hs = reinterpret_cast<unsigned long long*>(nd_pinned_scratch() + 8);
        if (nd_d2h(hs, dsum, sizeof(unsigned long long), s) != ND_OK) rc = ND_ERR_CUDA;
        else items = (int64_t)*hs;
      }
      nd_free(cnt, s); nd_free(cls, s); nd_free(ent, s); nd_free(dsum, s);
      nd_trace("tp:tail-stats");
      return rc;
    }
  }
  // entries per row, death steps, key offsets
  std::vector<int64_t*> ent(wins.size(), nullptr), koff(wins.size(), nullptr);
  std::vector<int64_t> kbase(wins.size(), 0);
  int64_t E = 0;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  auto need_tmp = [&](size_t b) -> int {
    if (b <= tmp_bytes) return ND_OK;
    nd_free(tmp, s);
    tmp = nullptr;
    tmp_bytes = b;
    return nd_alloc((char**)&tmp, b, s) == cudaSuccess ? ND_OK : ND_ERR_CUDA;
  };
  for (size_t k = 0; k < wins.size() && rc == ND_OK; k++) {
    const PWindow& W = wins[k];
    if (nd_alloc(&ent[k], W.n + 1, s) != cudaSuccess || nd_alloc(&koff[k], W.n + 1, s) != cudaSuccess) {
      rc = ND_ERR_CUDA;
      break;
    }
    cudaMemsetAsync(ent[k] + W.n, 0, sizeof(int64_t), s);
    k_tail_rows<<<nd_grid(W.n, 256), 256, 0, s>>>(W.wid, W.nnz, W.n, W.step0, W.Lw, dstep, ent[k]);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, ent[k], koff[k], W.n + 1, s);
    if ((rc = need_tmp(tb)) != ND_OK) break;
    if (cub::DeviceScan::ExclusiveSum(tmp, tb, ent[k], koff[k], W.n + 1, s) != cudaSuccess) {
      rc = ND_ERR_CUDA;
      break;
    }
    int64_t* hk = nd_pinned_scratch() + 8;
    if (nd_d2h(hk, koff[k] + W.n, sizeof(int64_t), s) != ND_OK) {
      rc = ND_ERR_CUDA;
      break;
    }
    kbase[k] = E;
    E += *hk;
  }
  uint64_t *keys = nullptr, *sorted = nullptr, *ukeys = nullptr;
  int *counts = nullptr, *n_runs = nullptr;
  if (rc == ND_OK && E > 0) {
    const int end_bit = key_bits + bits_for(n_steps - step);
    if (end_bit > 64 || E >= (1ll << 31)) rc = ND_ERR_ARG;
    if (rc == ND_OK && (nd_alloc(&keys, E, s) != cudaSuccess || nd_alloc(&sorted, E, s) != cudaSuccess ||
                        nd_alloc(&ukeys, E, s) != cudaSuccess || nd_alloc(&counts, E, s) != cudaSuccess ||
                        nd_alloc(&n_runs, 1, s) != cudaSuccess))
      rc = ND_ERR_CUDA;
    for (size_t k = 0; k < wins.size() && rc == ND_OK; k++) {
      const PWindow& W = wins[k];
      k_tail_keys<<<nd_grid(W.n * 32, 256, 148 * 32), 256, 0, s>>>(
          W.vin, W.out, ent[k], koff[k], W.n, W.ld, W.step0 - step, key_bits, keys + kbase[k]);
    }
    if (rc == ND_OK) {
      size_t tb = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, (int)E, 0, end_bit, s);
      size_t tb2 = 0;
      cub::DeviceRunLengthEncode::Encode(nullptr, tb2, sorted, ukeys, counts, n_runs, (int)E, s);
      if ((rc = need_tmp(tb > tb2 ? tb : tb2)) == ND_OK) {
        if (cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, (int)E, 0, end_bit, s) != cudaSuccess ||
            cub::DeviceRunLengthEncode::Encode(tmp, tb2, sorted, ukeys, counts, n_runs, (int)E, s) !=
                cudaSuccess)
          rc = ND_ERR_CUDA;
      }
    }
    if (rc == ND_OK)
      k_tail_classes<<<nd_grid(E / 64 + 1, 256), 256, 0, s>>>(ukeys, counts, n_runs, key_bits, step,
                                                               stats);
  }
  items = E;
  for (size_t k = 0; k < wins.size(); k++) {
    nd_free(ent[k], s);
    nd_free(koff[k], s);
  }
  nd_free(tmp, s); nd_free(keys, s); nd_free(sorted, s); nd_free(ukeys, s); nd_free(counts, s);
  nd_free(n_runs, s);
  if (rc == ND_OK && cudaGetLastError() != cudaSuccess) rc = ND_ERR_CUDA;
  nd_trace("tp:tail-stats");
  return rc;
}

// SP chain walk: walker-major persistent kernel over step windows of Lw.
static int run_chain_walk_sp(const nd_graph* G, const NdApp& a, int64_t sample_lo, int64_t n,
                             const int64_t* roots, int64_t R, uint64_t seed, int64_t steps,
                             int64_t step_cap, cudaStream_t s, nd_result* res) {
  const DevGraph& g = G->g;
  nd_trace("sp:enter");
  const int64_t limit = steps >= 0 ? (steps < step_cap ? steps : step_cap) : step_cap;
  const int64_t Lw_base = steps >= 0 ? (limit > 0 ? limit : 1) : 128;
  int32_t *roots32 = nullptr, *died = nullptr;
  int64_t* tot = nullptr;
  int* ctl = nullptr;  // [0]=queue [1]=cont_n [2]=max_len [3]=stall
  unsigned long long* ctr = nullptr;
  ND_CUDA_TRY(nd_alloc(&died, n, s));
  ND_CUDA_TRY(nd_alloc(&tot, n, s));
  ND_CUDA_TRY(nd_alloc(&ctl, 4, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 4, s));
  ND_CUDA_TRY(cudaMemsetAsync(died, 0, n * sizeof(int32_t), s));
  ND_CUDA_TRY(cudaMemsetAsync(tot, 0, n * sizeof(int64_t), s));
  ND_CUDA_TRY(cudaMemsetAsync(ctl, 0, 4 * sizeof(int), s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), s));
  if (!roots) {
    ND_CUDA_TRY(nd_alloc(&roots32, n * R, s));
    ND_TRY(nd_uniform_roots_i32(g, R, seed, sample_lo, n, roots32, s));
  }
  std::vector<PWindow> wins;
  int* h = reinterpret_cast<int*>(nd_pinned_scratch());
  h[1] = h[2] = h[3] = 0;
  int64_t launches = roots ? 0 : 1;
  double sample_ms = 0.0;
  {
    const int rc = pw_run_windows(G, a, seed, sample_lo, limit > 0 ? n : 0, nullptr, nullptr,
                                  nullptr, roots, roots32, R, 0, limit, Lw_base, died, ctl, ctr,
                                  false, s, wins, h, &sample_ms);
    if (rc != ND_OK) {
      pw_free_windows(wins, s);
      return rc;
    }
  }
  for (auto& W : wins) {
    k_pw_accum<<<nd_grid(W.n, 256), 256, 0, s>>>(W.wid, W.nnz, W.n, tot);
    launches += 2;
  }
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (g_profile) {
    cudaEventCreate(&pe0);
    cudaEventCreate(&pe1);
  }
  const int h_stall = h[3];
  const int64_t n_steps = h[2];
  // ---- compaction into the final layout -------------------------------------------
  nd_trace("sp:windows-done");
  if (g_profile) cudaEventRecord(pe0, s);
  int32_t* final_ids = nullptr;  // int32 vertex ids (F_FINAL_IDS32; int64 derived on request)
  int64_t *flen = nullptr, *final_off = nullptr, *clen = nullptr,
          *roots_out = nullptr;
  unsigned long long *hist = nullptr, *stats = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&clen, n, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, n * R, s));
  ND_CUDA_TRY(nd_alloc(&hist, limit + 2, s));
  ND_CUDA_TRY(nd_alloc(&stats, 4 * (n_steps + 1), s));
  ND_CUDA_TRY(cudaMemsetAsync(hist, 0, (limit + 2) * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * (n_steps + 1) * sizeof(unsigned long long), s));
  k_pw_lengths<<<nd_grid(n + 1, 256, 148 * 4), 256, 0, s>>>(tot, died, n, R, flen, clen, hist, limit + 2);
  k_pw_stats<<<1, 1, 0, s>>>(hist, n_steps, n, stats);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flen, final_off, n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flen, final_off, n + 1, s));
    nd_free(tmp, s);
  }
  int64_t total = 0;
  ND_TRY(nd_d2h(&total, final_off + n, sizeof(int64_t), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  nd_trace("sp:scan-synced");
  ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
  if (n * R) {
    if (roots)
      k_write_roots<int64_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots, n, R, final_off, final_ids,
                                                                roots_out);
    else
      k_write_roots<int32_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots32, n, R, final_off,
                                                                final_ids, roots_out);
  }
  int64_t items = 0;
  for (auto& W : wins) {
    if (W.n * W.Lw)
      k_pw_emit<<<nd_grid(W.n * 32, 256, 148 * 32), 256, 0, s>>>(W.wid, W.out, W.nnz, W.n, W.ld,
                                                                W.step0, final_off, R, final_ids);
    items += W.n;  // rows touched (upper bound of pairs)
    launches += 1;
  }
  launches += 2 /*lengths, stats*/ + 2 /*scan*/ + (n * R ? 1 : 0);
  if (g_profile) cudaEventRecord(pe1, s);
  unsigned long long h_ctr[4];
  ND_TRY(nd_d2h(h_ctr, ctr, sizeof(h_ctr), s));
  ND_CUDA_TRY(cudaGetLastError());
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  pw_free_windows(wins, s);
  if (g_profile) {
    float ms = 0;
    cudaEventElapsedTime(&ms, pe0, pe1);
    res->prof_ms[1] = sample_ms;
    res->prof_ms[2] = ms;
    cudaEventDestroy(pe0);
    cudaEventDestroy(pe1);
  }
  res->counters[NDC_LAUNCHES] = launches;
  nd_trace("sp:done");
  nd_free(died, s); nd_free(tot, s); nd_free(ctl, s); nd_free(ctr, s); nd_free(roots32, s);
  nd_free(flen, s); nd_free(hist, s);
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n * R;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n * R);
  res->set(ND_F_CHAIN_LEN, clen, n);
  res->set(ND_F_STATS, stats, 4 * n_steps);
  res->counters[NDC_N2V_TRIES] = (int64_t)h_ctr[1];
  res->counters[NDC_SLOT_BYTES] = (int64_t)h_ctr[0];
  res->counters[NDC_RAND_SECTORS] = (int64_t)h_ctr[2];
  res->counters[NDC_STEPS] = n_steps;
  return h_stall ? ND_ERR_STALL : ND_OK;
}

static int run_rootpick_walk(const nd_graph* G, const NdApp& a, int64_t sample_lo, int64_t n,
                             const int64_t* roots, int64_t R, uint64_t seed, int64_t steps,
                             int64_t step_cap, int paradigm, cudaStream_t s, nd_result* res) {
  const DevGraph& g = G->g;
  const int key_bits = key_bits_for(g.V);
  const int64_t S_ = steps >= 0 ? (steps < step_cap ? steps : step_cap) : step_cap;
  const int64_t n_steps = (n > 0 && R > 0) ? S_ : 0;
  int32_t *roots32 = nullptr, *slab = nullptr;
  uint32_t *k0 = nullptr, *k1 = nullptr;
  uint64_t *v0 = nullptr, *v1 = nullptr;
  int* stall = nullptr;
  unsigned long long *ctr = nullptr, *stats = nullptr;
  TPScratch S;
  ND_CUDA_TRY(nd_alloc(&roots32, n * R, s));
  ND_CUDA_TRY(nd_alloc(&slab, n * (n_steps ? n_steps : 1), s));
  ND_CUDA_TRY(nd_alloc(&k0, n, s));
  ND_CUDA_TRY(nd_alloc(&k1, n, s));
  ND_CUDA_TRY(nd_alloc(&v0, n, s));
  ND_CUDA_TRY(nd_alloc(&v1, n, s));
  ND_CUDA_TRY(nd_alloc(&stall, 1, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 4, s));
  ND_CUDA_TRY(nd_alloc(&stats, 4 * (n_steps + 1), s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * (n_steps + 1) * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stall, 0, sizeof(int), s));
  if (roots) {
    if (n * R) k_narrow<<<nd_grid(n * R, 256), 256, 0, s>>>(roots, n * R, roots32);
  } else {
    ND_TRY(nd_uniform_roots_i32(g, R, seed, sample_lo, n, roots32, s));
  }
  if (paradigm == ND_TP) ND_TRY(S.alloc(n, key_bits, s));
  Profiler prof(s);
  double sched_ms = 0, sample_ms = 0;
  for (int64_t step = 0; step < n_steps; step++) {
    size_t e0 = prof.ev.size();
    prof.mark();
    k_rootpick_keys<<<nd_grid(n, 256), 256, 0, s>>>(roots32, n, R, key_base(seed, step, 1, 0),
                                                     sample_lo, k0, v0);
    RootPickAct act{view(g), a, key_base(seed, (uint64_t)step, 0, 0), sample_lo, roots32, R,
                    slab + step * n, stall};
    unsigned long long* st_step = stats + 4 * step;
    if (paradigm == ND_TP) {
      cub::DoubleBuffer<uint32_t> dk(k0, k1);
      cub::DoubleBuffer<uint64_t> dv(v0, v1);
      ND_TRY(tp_sort(dk, dv, n, key_bits, S, s));
      prof.mark();
      ND_TRY(tp_run_sorted(dk.Current(), dv.Current(), n, 1, g, stage_spec(0, 0), act, S, ctr,
                           st_step, s));
    } else {
      prof.mark();
      ND_TRY(sp_step(k0, v0, n, g, act, ctr, st_step, s));
      k_stats_fetch<<<1, 1, 0, s>>>(st_step, (unsigned long long)n);
    }
    prof.mark();
    if (prof.on) {
      ND_CUDA_TRY(cudaStreamSynchronize(s));
      sched_ms += prof.between(e0, e0 + 1);
      sample_ms += prof.between(e0 + 1, e0 + 2);
      prof.steps.push_back({e0, e0 + 1, e0 + 2, 1});
    }
  }
  prof.mark();
  const size_t ef = prof.ev.size() - 1;
  int32_t* final_ids = nullptr;  // int32 vertex ids (F_FINAL_IDS32; int64 derived on request)
  int64_t *flen = nullptr, *final_off = nullptr, *roots_out = nullptr,
          *chain = nullptr, *clen = nullptr;
  ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&roots_out, n * R, s));
  ND_CUDA_TRY(nd_alloc(&chain, n * n_steps, s));
  ND_CUDA_TRY(nd_alloc(&clen, n, s));
  k_slab_counts<<<nd_grid(n + 1, 256), 256, 0, s>>>(slab, n, n_steps, R, flen);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flen, final_off, n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flen, final_off, n + 1, s));
    nd_free(tmp, s);
  }
  int64_t total = 0;
  ND_TRY(nd_d2h(&total, final_off + n, sizeof(int64_t), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
  if (n * R)
    k_write_roots<int32_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots32, n, R, final_off, final_ids,
                                                              roots_out);
  if (n) k_slab_write<<<nd_grid(n, 128), 128, 0, s>>>(slab, n, n_steps, R, final_off, final_ids, chain);
  {
    std::vector<int64_t> h(n, n_steps);
    if (n) ND_CUDA_TRY(cudaMemcpyAsync(clen, h.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    prof.mark();
    unsigned long long h_ctr[4];
    ND_TRY(nd_d2h(h_ctr, ctr, sizeof(h_ctr), s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    res->counters[NDC_N2V_TRIES] = (int64_t)h_ctr[1];
    res->counters[NDC_SLOT_BYTES] = (int64_t)h_ctr[0];
  }
  ND_CUDA_TRY(cudaGetLastError());
  res->prof_ms[0] = sched_ms;
  res->prof_ms[1] = sample_ms;
  res->prof_ms[2] = prof.on ? prof.between(ef, ef + 1) : 0.0;
  prof.to_result(res);
  prof.destroy();
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n * R;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n * R);
  res->set(ND_F_CHAIN_LEN, clen, n);
  res->set(ND_F_CHAIN_VALS, chain, n * n_steps);
  res->set(ND_F_STATS, stats, 4 * n_steps);
  res->counters[NDC_ITEMS] = n * n_steps;
  res->counters[NDC_PAIRS] = n * n_steps;
  res->counters[NDC_STEPS] = n_steps;
  nd_free(roots32, s); nd_free(slab, s); nd_free(k0, s); nd_free(k1, s); nd_free(v0, s);
  nd_free(v1, s); nd_free(stall, s); nd_free(ctr, s); nd_free(flen, s);
  if (paradigm == ND_TP) S.release(s);
  return ND_OK;
}

#include "nd_bulk.cuh"
#include "nd_walk_hub.cuh"

// dynamic shared memory above 48 KB for the hub kernel (once per process)
static int tw_attrs() {
  static int rc = -1;
  if (rc < 0)
    rc = cudaFuncSetAttribute(k_tw_hub<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)TW_HUB_SMEM) == cudaSuccess ? ND_OK : ND_ERR_CUDA;
  return rc;
}

// The hub engine applies when the walker-major records exist (the SP kernel's
// record paths) and edge offsets fit the 32-bit state.
static bool tw_applicable(const DevGraph& g, const NdApp& a) {
  if (getenv("ND_TP_ENGINE") && strcmp(getenv("ND_TP_ENGINE"), "sort") == 0) return false;
  if (g.E >= (1ll << 32) || !g.vrec) return false;
  const bool n2v = a.code == ND_NODE2VEC;
  if (a.code != ND_DEEPWALK && a.code != ND_PPR && !n2v) return false;
  if (g.unit) return g.nbu != nullptr;
  return g.nbp != nullptr && (!n2v || g.nbw != nullptr);
}

// TP chain walk through the hub-bucket inversion (nd_walk_hub.cuh): windows of
// per-step kernels over the alive walkers' rows; walks still alive at a
// window's end continue in the next window, and once at most ND_TP_TAIL
// walkers are alive the rest runs in the walker-major tail (run_tp_tail).
static int run_chain_walk_hub(const nd_graph* G, const NdApp& a, int64_t sample_lo, int64_t n,
                              const int64_t* roots, int64_t R, uint64_t seed, int64_t steps,
                              int64_t step_cap, cudaStream_t s, nd_result* res) {
  const DevGraph& g = G->g;
  ND_TRY(tw_attrs());
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int occ = 4;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tw_sample<4>, TW_BLOCK, 0);
  if (occ < 1) occ = 1;
  int hocc = 4;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hocc, k_tw_hub<4>, TW_BLOCK, TW_HUB_SMEM);
  if (hocc < 1) hocc = 1;
  // k_tw_multi's resident CTAs per SM requested from ptxas (ND_TW_MINB 3 | 4)
  void (*kmul)(TwArgs) = app_knob("ND_TW_MINB", a.code, 4) == 3 ? k_tw_multi<3> : k_tw_multi<4>;
  int mocc = 4;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&mocc, kmul, TW_BLOCK, 0);
  if (mocc < 1) mocc = 1;
  {  // concurrent jobs (nd_set_concurrency): this run's share of the CTA slots
    const int share = nd_concurrency();
    occ = std::max(1, occ / share);
    hocc = std::max(1, hocc / share);
    mocc = std::max(1, mocc / share);
  }
  // steps per launch once the staged tiers are off (k_tw_multi; ND_TW_MULTI,
  // 1: one step per launch through k_tw_sample)
  const int kmulti = [&] {
    const int k = app_knob("ND_TW_MULTI", a.code, 3);
    return k < 1 ? 1 : (k > TW_KMAX ? TW_KMAX : k);
  }();
  const int64_t max_steps = steps >= 0 ? (steps < step_cap ? steps : step_cap) : step_cap;
  const int64_t tail_T = getenv("ND_TP_TAIL") ? atoll(getenv("ND_TP_TAIL")) : 131072;
  const int key_bits = key_bits_for(g.V);
  const bool n2v = a.code == ND_NODE2VEC;
  const int64_t V = g.V;
  const int64_t hcap = n / TW_TM + 2;                 // hubs per step
  const int64_t ucap = hcap + n / TW_UNIT + 2;        // CTA units per step
  int32_t *roots32 = nullptr, *died = nullptr, *maxlen = nullptr;
  TwRec* hrec = nullptr;
  int32_t *pos = nullptr, *cnt[2] = {}, *vhub[2] = {}, *hubs[2] = {};
  int32_t *cur[2] = {}, *dg[2] = {};
  uint32_t* lo[2] = {};
  double* hd[2] = {};
  TwCtl* ctl = nullptr;
  TwUnit *wunits = nullptr, *cunits = nullptr;
  int64_t* tot = nullptr;
  unsigned long long *ctr = nullptr, *stats = nullptr;
  int* stall = nullptr;
  ND_CUDA_TRY(nd_alloc(&died, n, s));
  ND_CUDA_TRY(nd_alloc(&tot, n, s));
  ND_CUDA_TRY(nd_alloc(&maxlen, 1, s));
  ND_CUDA_TRY(nd_alloc(&stall, 1, s));
  ND_CUDA_TRY(nd_alloc(&ctr, 6, s));  // [0..2] byte model, [4] staged, [5] in place
  ND_CUDA_TRY(nd_alloc(&stats, 4 * (max_steps + 1), s));
  ND_CUDA_TRY(nd_alloc(&ctl, 2, s));
  ND_CUDA_TRY(nd_alloc(&wunits, hcap, s));
  ND_CUDA_TRY(nd_alloc(&cunits, ucap, s));
  ND_CUDA_TRY(nd_alloc(&hrec, n, s));
  ND_CUDA_TRY(nd_alloc(&pos, n, s));
  // member counts: both parities (k_tw_sample), or k_tw_multi's kmulti
  // per-step arrays over the same memory, behind its row queue; one L2 window
  const int64_t ncnt = std::max<int64_t>(2, kmulti) * V;
  int32_t* karena = nullptr;
  ND_CUDA_TRY(nd_alloc(&karena, 32 + ncnt, s));
  int* kqueue = karena;
  cnt[0] = karena + 32;
  cnt[1] = cnt[0] + V;
  ND_CUDA_TRY(cudaMemsetAsync(karena, 0, (32 + ncnt) * sizeof(int32_t), s));
  for (int b = 0; b < 2; b++) {
    ND_CUDA_TRY(nd_alloc(&vhub[b], V, s));
    ND_CUDA_TRY(nd_alloc(&hubs[b], hcap, s));
  }
  for (int b = 0; b < 2; b++) {
    ND_CUDA_TRY(nd_alloc(&cur[b], n, s));
    ND_CUDA_TRY(nd_alloc(&lo[b], n, s));
    ND_CUDA_TRY(nd_alloc(&dg[b], n, s));
    ND_CUDA_TRY(nd_alloc(&hd[b], n, s));
  }
  ND_CUDA_TRY(cudaMemsetAsync(died, 0, n * sizeof(int32_t), s));
  ND_CUDA_TRY(cudaMemsetAsync(tot, 0, n * sizeof(int64_t), s));
  ND_CUDA_TRY(cudaMemsetAsync(maxlen, 0, sizeof(int32_t), s));
  ND_CUDA_TRY(cudaMemsetAsync(stall, 0, sizeof(int), s));
  ND_CUDA_TRY(cudaMemsetAsync(ctr, 0, 6 * sizeof(unsigned long long), s));
  ND_CUDA_TRY(cudaMemsetAsync(stats, 0, 4 * (max_steps + 1) * sizeof(unsigned long long), s));
  if (!roots) {
    ND_CUDA_TRY(nd_alloc(&roots32, n * R, s));
    ND_TRY(nd_uniform_roots_i32(g, R, seed, sample_lo, n, roots32, s));
  }
  // The member counts take one random atomic per (tile, transit) and one
  // random read per walker every step: keep them resident in L2 (persisting
  // window over cnt) so the walk's record traffic does not evict them.
  cudaStreamAttrValue l2win{}, l2off{};
  bool l2set = false, l2pin = false;
  {
    int max_persist = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    const size_t want = (size_t)ncnt * sizeof(int32_t);
    if (max_persist > 0 && !getenv("ND_TW_NO_L2PIN")) {
      // The set-aside is device-wide and outlives the run: the first of any
      // concurrent TP runs records the previous limit, the last one restores
      // it, so later kernels get the whole L2 back.
      size_t lim = 0;
      {
        std::lock_guard<std::mutex> lk(g_l2_mu);
        cudaDeviceGetLimit(&lim, cudaLimitPersistingL2CacheSize);
        if (g_l2_users++ == 0) g_l2_prev = lim;
      }
      const size_t setaside = std::min<size_t>((size_t)max_persist, std::max(lim, want));
      if (lim < setaside) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside);
      l2win.accessPolicyWindow.base_ptr = cnt[0];
      l2win.accessPolicyWindow.num_bytes = want;
      l2win.accessPolicyWindow.hitRatio = want <= setaside ? 1.0f : (float)setaside / (float)want;
      l2win.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      l2win.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      l2set = cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &l2win) == cudaSuccess;
      l2pin = true;
      cudaGetLastError();
    }
  }

  PWArgs P{};
  P.gv = view(g);
  P.a = a;
  P.seed = seed;
  P.sample_lo = sample_lo;
  P.R = R;
  P.stall = stall;
  P.ctr = ctr;
  P.vrec = g.vrec;
  P.nbw = g.nbw;
  P.nbp = g.nbp;
  P.nbu = g.nbu;
  P.pl = (a.code == ND_DEEPWALK || a.code == ND_PPR) ? g.pl : nullptr;
  P.vline = g.vline;

  // bytes per edge of the records a hub's members read (k_tw_prep's rmode)
  auto rmode = [&](int tries) {
    if (tries || !P.pl) return g.unit ? 1 : 0;
    return 2;
  };
  int64_t next_Lw = 1;
  // ND_TW_PROFILE=1 (development): event-timed phases of every step, summed
  struct TwPhases {
    bool on = getenv("ND_TW_PROFILE") != nullptr;
    std::vector<cudaEvent_t> ev;
    std::vector<int> ph;
    void mark(cudaStream_t st, int p) {
      if (!on) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      ev.push_back(e);
      ph.push_back(p);
    }
    void report() {
      if (!on) return;
      cudaEventSynchronize(ev.empty() ? nullptr : ev.back());
      double t[8] = {};
      for (size_t i = 1; i < ev.size(); i++)
        if (ph[i] == ph[i - 1] + 1) {
          float ms = 0;
          cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
          t[ph[i - 1]] += ms;
        }
      fprintf(stderr, "[tw-profile] prep %.3f sample %.3f hub %.3f ms\n", t[0], t[1], t[2]);
      for (auto e : ev) cudaEventDestroy(e);
    }
  } tp;
  struct TWin {
    int32_t *wid, *out, *nnz;
    int64_t rows, step0, Lw;
  };
  std::vector<TWin> twins;
  std::vector<PWindow> tail_wins;
  int32_t *wid = nullptr, *v0 = nullptr, *t0 = nullptr;
  int64_t rows = max_steps > 0 ? n : 0, step = 0, n_steps = 0, tail_items = 0;
  int* h = reinterpret_cast<int*>(nd_pinned_scratch());
  Profiler prof(s);
  const size_t e_run = prof.mark();
  bool tail = false;
  int rc = ND_OK;
  // staged hub tiers on until a window shows they do not engage (ND_TW_STAGE=1:
  // always on, 0: always off; development)
  const bool tw_debug = getenv("ND_TW_DEBUG") != nullptr;
  const char* stg_env = getenv("ND_TW_STAGE");
  bool staging = !(stg_env && stg_env[0] == '0');
  const bool stage_fixed = stg_env != nullptr;
  unsigned long long hubs_prev = 0, staged_prev = 0;
  bool ctl_clean = false;  // the next step's control was zeroed by a sampling kernel
  unsigned int* done = nullptr;
  ND_CUDA_TRY(nd_alloc(&done, 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(done, 0, sizeof(unsigned int), s));
  if (!staging)
    for (int b = 0; b < 2; b++) ND_CUDA_TRY(cudaMemsetAsync(vhub[b], 0xFF, V * sizeof(int32_t), s));
  while (rows > 0 && step < max_steps) {
    if (rows <= tail_T && rows * (max_steps - step) < (1ll << 31)) {
      tail = true;
      break;
    }
    // windows of 1, 4, 16, 64, 256 steps (32 for walks of unbounded length,
    // whose alive count falls every step): the alive walkers are compacted
    // between windows and the tail hand-off is checked there
    const int64_t Lw = std::min<int64_t>(max_steps - step, next_Lw);
    next_Lw = std::min<int64_t>(next_Lw * 4, steps >= 0 ? 256 : 32);
    TWin W{wid, nullptr, nullptr, rows, step, Lw};
    int32_t *cw = nullptr, *cv = nullptr, *ct = nullptr;
    int* cont_n = nullptr;
    ND_CUDA_TRY(nd_alloc(&W.out, Lw * rows, s));
    ND_CUDA_TRY(nd_alloc(&W.nnz, rows, s));
    ND_CUDA_TRY(nd_alloc(&cw, rows, s));
    ND_CUDA_TRY(nd_alloc(&cv, rows, s));
    ND_CUDA_TRY(nd_alloc(&ct, rows, s));
    ND_CUDA_TRY(nd_alloc(&cont_n, 1, s));
    ND_CUDA_TRY(cudaMemsetAsync(cont_n, 0, sizeof(int), s));
    ND_CUDA_TRY(cudaMemsetAsync(ctl, 0, 2 * sizeof(TwCtl), s));
    TwArgs A{};
    A.P = P;
    A.rows = rows;
    A.wid = wid;
    A.Lw = Lw;
    A.pos = pos;
    A.tier = ctr + 4;
    A.out = W.out;
    A.nnz = W.nnz;
    A.died = died;
    A.cont_wid = cw;
    A.cont_v = cv;
    A.cont_t = ct;
    A.cont_n = cont_n;
    A.max_len = maxlen;
    A.hrec = hrec;
    A.hcap = n;
    A.hubs_seen = ctr + 3;
    A.done = done;
    A.no_hub_list = !staging;
    ctl_clean = false;  // the window start zeroed both controls; count0 fills the first

    A.wunits = wunits;
    A.cunits = cunits;
    // window start: state of every row
    A.s = step;
    A.cur = cur[0]; A.lo = lo[0]; A.deg = dg[0]; A.hd = hd[0];
    A.ncur = cur[1]; A.nlo = lo[1]; A.ndeg = dg[1]; A.nhd = hd[1];
    k_tw_init<<<nd_grid(rows, TW_BLOCK, nsm * 8), TW_BLOCK, 0, s>>>(A, roots, roots32, R, v0, t0);
    // staged tiers off: K steps per launch (k_tw_multi), counts in zeroed
    // per-step arrays instead of the parity pair the sampling kernel clears
    const bool multi = !staging && kmulti > 1;
    {
      const int b = (int)(step & 1);
      A.nctl = ctl + b; A.ncnt = cnt[b]; A.nhubs = hubs[b];
      if (multi) {
        A.ncnt = cnt[0];
        ND_CUDA_TRY(cudaMemsetAsync(cnt[0], 0, V * sizeof(int32_t), s));
      }
      A.nstats = stats + 4 * step;
      k_tw_count0<<<nd_grid(rows, TW_BLOCK, nsm * 8), TW_BLOCK, 0, s>>>(A);
    }
    {
      const int64_t thr = (int64_t)nsm * occ * TW_BLOCK;
      A.P.chunk = rows > 8 * thr ? 128 : rows > 2 * thr ? 64 : 32;
    }
    for (int64_t k = 0; multi && k < Lw;) {
      const int Ke = (int)std::min<int64_t>(kmulti, Lw - k);
      const int64_t st_ = step + k;
      const int in = (int)(k & 1), ou = in ^ 1;
      A.s = st_;
      A.k = k;
      A.K = Ke;
      A.cur = cur[in]; A.lo = lo[in]; A.deg = dg[in]; A.hd = hd[in];
      A.ncur = cur[ou]; A.nlo = lo[ou]; A.ndeg = dg[ou]; A.nhd = hd[ou];
      A.kcnt = cnt[0];
      A.kV = V;
      A.kqueue = kqueue;
      A.nstats = stats + 4 * (st_ + 1);
      prof.step_begin(Ke);
      ND_CUDA_TRY(cudaMemsetAsync(karena, 0, (32 + Ke * V) * sizeof(int32_t), s));
      prof.step_built();
      kmul<<<nsm * mocc, TW_BLOCK, 0, s>>>(A);
      prof.step_sampled();
      if (cudaGetLastError() != cudaSuccess) { rc = ND_ERR_CUDA; break; }
      k += Ke;
    }
    for (int64_t k = 0; !multi && k < Lw; k++) {
      const int64_t st_ = step + k;
      const int b = (int)(st_ & 1), pb = b ^ 1;
      const int in = (int)(k & 1), ou = in ^ 1;
      A.s = st_;
      A.k = k;
      A.last = k == Lw - 1;
      A.tries = n2v && st_ > 0;
      A.cur = cur[in]; A.lo = lo[in]; A.deg = dg[in]; A.hd = hd[in];
      A.ncur = cur[ou]; A.nlo = lo[ou]; A.ndeg = dg[ou]; A.nhd = hd[ou];
      A.ctl = ctl + b; A.cnt = cnt[b]; A.vhub = vhub[b]; A.hubs = hubs[b];
      A.nctl = ctl + pb; A.ncnt = cnt[pb]; A.nhubs = hubs[pb];
      A.nstats = stats + 4 * (st_ + 1);
      A.rmode = rmode(A.tries);
      {
        const int64_t thr = (int64_t)nsm * occ * TW_BLOCK;
        A.P.chunk = rows > 8 * thr ? 128 : rows > 2 * thr ? 64 : 32;
      }
      tp.mark(s, 0);
      prof.step_begin();
      A.reset_self = nullptr;
      if (staging) {
        k_tw_prep<<<nd_grid(rows / TW_TM + 1, 256, nsm * 4), 256, 0, s>>>(A);
        ctl_clean = false;
      } else {
        // every hub in the grid tier; the prep's other duty, zeroing the step
        // control the emission fills, is done by the previous step's last CTA
        // (its own control), except at the first step of a window or after
        // a staged step
        if (!ctl_clean) ND_CUDA_TRY(cudaMemsetAsync(A.nctl, 0, sizeof(TwCtl), s));
        A.reset_self = A.ctl;
        ctl_clean = true;
      }
      prof.step_built();
      tp.mark(s, 1);
      k_tw_sample<4><<<nsm * occ, TW_BLOCK, 0, s>>>(A);
      tp.mark(s, 2);
      if (staging) k_tw_hub<4><<<nsm * hocc, TW_BLOCK, TW_HUB_SMEM, s>>>(A);
      prof.step_sampled();
      tp.mark(s, 3);
      if (cudaGetLastError() != cudaSuccess) { rc = ND_ERR_CUDA; break; }
      if (tw_debug && (st_ % 10 == 1)) {  // development: per-step tier sizes
        TwCtl hc;
        if (nd_d2h(&hc, ctl + b, sizeof(TwCtl), s) == ND_OK)
          fprintf(stderr, "[tw] step %lld hubs %d groups %d small %d warp-hubs %d cta-units %d "
                  "grid-members %d staged-members %d\n", (long long)st_, hc.nhub, 0, 0,
                  hc.nwarp, hc.nunit, 0, hc.front);
      }
    }
    k_pw_accum<<<nd_grid(rows, 256), 256, 0, s>>>(wid, W.nnz, rows, tot);
    if (rc == ND_OK && nd_d2h(h, cont_n, sizeof(int), s) != ND_OK) rc = ND_ERR_CUDA;
    nd_free(cont_n, s);
    nd_free(v0, s);
    nd_free(t0, s);
    twins.push_back(W);
    if (rc != ND_OK) {
      nd_free(cw, s); nd_free(cv, s); nd_free(ct, s);
      wid = v0 = t0 = nullptr;
      break;
    }
    wid = cw;
    v0 = cv;
    t0 = ct;
    rows = h[0];
    step += Lw;
    // Staged tiers that never engage: when this window's prep kernels classed
    // hubs but none of their members was sampled from a staged row (rows too
    // long for their members to pay, PAPER.md:832-838's trade-off), the
    // remaining windows run every hub in the grid tier and skip the prep and
    // hub launches.  Which tier samples a member does not change any row;
    // the class statistics come from the count crossings either way.
    if (staging && !stage_fixed) {
      unsigned long long hc[2];
      if (nd_d2h(hc, ctr + 3, sizeof(hc), s) != ND_OK) { rc = ND_ERR_CUDA; break; }
      if (hc[0] > hubs_prev && hc[1] == staged_prev) {
        staging = false;
        for (int b = 0; b < 2; b++)
          ND_CUDA_TRY(cudaMemsetAsync(vhub[b], 0xFF, V * sizeof(int32_t), s));
      }
      hubs_prev = hc[0];
      staged_prev = hc[1];
    }
  }
  double sample_ms = 0.0;
  if (rc == ND_OK && tail && step == 0) {  // every walker in the tail: rows from the roots
    if (nd_alloc(&wid, rows, s) != cudaSuccess || nd_alloc(&v0, rows, s) != cudaSuccess ||
        nd_alloc(&t0, rows, s) != cudaSuccess)
      rc = ND_ERR_CUDA;
    else
      k_tw_rows0<<<nd_grid(rows, 256), 256, 0, s>>>(roots, roots32, R, rows, wid, v0, t0);
  }
  if (rc == ND_OK && tail) {
    // the remaining walkers (rows of wid/v0/t0) continue walker-major
    int64_t ns = 0;
    rc = run_tp_tail(G, a, seed, sample_lo, n, rows, nullptr, nullptr, R, step, max_steps,
                     steps >= 0 ? max_steps - step : 128, key_bits, nullptr, stall, ctr, stats, s,
                     tail_wins, ns, tail_items, sample_ms, wid, v0, t0, died);
    if (ns > n_steps) n_steps = ns;
    wid = v0 = t0 = nullptr;  // owned by the tail windows
    for (auto& W : tail_wins) k_pw_accum<<<nd_grid(W.n, 256), 256, 0, s>>>(W.wid, W.nnz, W.n, tot);
  } else {
    nd_free(v0, s);
    nd_free(t0, s);
  }
  tp.report();
  if (l2set) {  // back to normal caching for the stream; release the persisting lines
    l2off.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &l2off);
    cudaGetLastError();
  }
  if (l2pin) {
    std::lock_guard<std::mutex> lk(g_l2_mu);
    if (--g_l2_users == 0) {
      cudaStreamSynchronize(s);
      cudaCtxResetPersistingL2Cache();
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_prev);
    }
    cudaGetLastError();
  }
  const size_t e_sampled = prof.mark();
  int h_stall = 0;
  if (rc == ND_OK) {
    int mlen = 0;
    if (nd_d2h(&mlen, maxlen, sizeof(int), s) != ND_OK) rc = ND_ERR_CUDA;
    if (mlen > n_steps) n_steps = mlen;
  }
  // ---- compaction into the final layout -------------------------------------------
  int32_t* final_ids = nullptr;
  int64_t *flen = nullptr, *final_off = nullptr, *clen = nullptr, *roots_out = nullptr;
  unsigned long long* hist = nullptr;
  int64_t total = 0;
  if (rc == ND_OK) {
    const int64_t hl = max_steps + 2;
    ND_CUDA_TRY(nd_alloc(&flen, n + 1, s));
    ND_CUDA_TRY(nd_alloc(&final_off, n + 1, s));
    ND_CUDA_TRY(nd_alloc(&clen, n, s));
    ND_CUDA_TRY(nd_alloc(&roots_out, n * R, s));
    ND_CUDA_TRY(nd_alloc(&hist, hl, s));
    ND_CUDA_TRY(cudaMemsetAsync(hist, 0, hl * sizeof(unsigned long long), s));
    k_pw_lengths<<<nd_grid(n + 1, 256, nsm * 4), 256, 0, s>>>(tot, died, n, R, flen, clen, hist, hl);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flen, final_off, n + 1, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flen, final_off, n + 1, s));
    nd_free(tmp, s);
    ND_TRY(nd_d2h(&total, final_off + n, sizeof(int64_t), s));
    ND_CUDA_TRY(nd_alloc(&final_ids, total, s));
    if (n * R) {
      if (roots)
        k_write_roots<int64_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots, n, R, final_off,
                                                                  final_ids, roots_out);
      else
        k_write_roots<int32_t><<<nd_grid(n * R, 256), 256, 0, s>>>(roots32, n, R, final_off,
                                                                  final_ids, roots_out);
    }
    for (auto& W : twins)
      if (W.rows * W.Lw)
        k_tw_emit<<<nd_grid((W.rows + 31) / 32 * ((W.Lw + 31) / 32) * 32, 256, nsm * 16), 256, 0, s>>>(
            W.out, W.rows, W.Lw, W.nnz, W.wid, W.step0, final_off, R, final_ids);
    for (auto& W : tail_wins)
      if (W.n * W.Lw)
        k_pw_emit<<<nd_grid(W.n * 32, 256, nsm * 32), 256, 0, s>>>(W.wid, W.out, W.nnz, W.n, W.ld,
                                                                  W.step0, final_off, R, final_ids);
    unsigned long long h_ctr[6];
    ND_TRY(nd_d2h(&h_stall, stall, sizeof(int), s));
    ND_TRY(nd_d2h(h_ctr, ctr, sizeof(h_ctr), s));
    ND_CUDA_TRY(cudaGetLastError());
    res->counters[NDC_N2V_TRIES] = (int64_t)h_ctr[1];
    res->counters[NDC_SLOT_BYTES] = (int64_t)h_ctr[0];
    res->counters[NDC_RAND_SECTORS] = (int64_t)h_ctr[2];
    res->counters[NDC_TP_STAGED] = (int64_t)h_ctr[4];
    res->counters[NDC_TP_INPLACE] = (int64_t)h_ctr[5];
  }
  const size_t e_done = prof.mark();
  if (prof.on && rc == ND_OK) {
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    const auto st = prof.to_result(res);
    res->prof_ms[0] = st[0];
    res->prof_ms[1] = prof.between(e_run, e_sampled) - st[0];
    res->prof_ms[2] = prof.between(e_sampled, e_done);
  }
  prof.destroy();
  for (auto& W : twins) { nd_free(W.wid, s); nd_free(W.out, s); nd_free(W.nnz, s); }
  pw_free_windows(tail_wins, s);
  nd_free(wid, s);
  nd_free(roots32, s); nd_free(died, s); nd_free(tot, s); nd_free(maxlen, s); nd_free(stall, s);
  nd_free(ctr, s); nd_free(ctl, s); nd_free(wunits, s); nd_free(cunits, s);
  nd_free(hrec, s); nd_free(pos, s); nd_free(flen, s); nd_free(hist, s);
  nd_free(karena, s);
  for (int b = 0; b < 2; b++) { nd_free(vhub[b], s); nd_free(hubs[b], s); }
  nd_free(done, s);
  for (int b = 0; b < 2; b++) { nd_free(cur[b], s); nd_free(lo[b], s); nd_free(dg[b], s); nd_free(hd[b], s); }
  if (rc != ND_OK) {
    nd_free(stats, s); nd_free(final_off, s); nd_free(final_ids, s); nd_free(clen, s); nd_free(roots_out, s);
    return rc;
  }
  res->n = n;
  res->n_steps = n_steps;
  res->total_sampled = total - n * R;
  res->set(ND_F_FINAL_OFF, final_off, n + 1);
  res->set(ND_F_FINAL_IDS32, final_ids, total);
  res->set(ND_F_ROOTS, roots_out, n * R);
  res->set(ND_F_CHAIN_LEN, clen, n);
  res->set(ND_F_STATS, stats, 4 * n_steps);
  res->counters[NDC_ITEMS] = total - n * R;
  res->counters[NDC_PAIRS] = res->counters[NDC_ITEMS];
  res->counters[NDC_STEPS] = n_steps;
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  return h_stall ? ND_ERR_STALL : ND_OK;
}

extern "C" int nd_run_walk(const nd_graph* g, int app_code, const double* host_params,
                           int64_t n_params, int64_t sample_lo, int64_t n_samples,
                           const int64_t* roots, int64_t roots_per_sample, uint64_t seed,
                           int64_t steps, int64_t step_cap, int paradigm, void* stream,
                           nd_result** out) {
  NvtxRange nvtx_run("nd_run_walk");
  NdApp a;
  ND_TRY(nd_make_app(app_code, host_params, n_params, &a));
  if (!g || n_samples < 0 || roots_per_sample < 1 || step_cap < 0 || sample_lo < 0)
    return ND_ERR_ARG;
  if (n_samples >= (1ll << 31)) return ND_ERR_ARG;
  if (app_code == ND_KHOP) return ND_ERR_ARG;  // multi-slot: nd_run_individual
  cudaStream_t s = (cudaStream_t)stream;
  // exact search indexes (built once per graph): guide tables for weighted
  // picks, hash sets for node2vec membership
  ND_TRY(nd_graph_ensure_index(const_cast<nd_graph*>(g), app_code == ND_NODE2VEC,
                               app_code != ND_MULTIRW, s));
  // packed records: the walker-major kernel and the TP hub engine read them
  if (app_code != ND_MULTIRW)
    ND_TRY(nd_graph_ensure_records(const_cast<nd_graph*>(g), app_code == ND_NODE2VEC, s));
  if (app_code == ND_DEEPWALK || app_code == ND_PPR)
    ND_TRY(nd_graph_ensure_lines(const_cast<nd_graph*>(g), s));
  nd_result* res = new nd_result();
  res->stream = s;
  int rc;
  if (app_code == ND_MULTIRW)
    rc = run_rootpick_walk(g, a, sample_lo, n_samples, roots, roots_per_sample, seed, steps,
                           step_cap, paradigm, s, res);
  else if (paradigm == ND_SP)
    rc = run_chain_walk_sp(g, a, sample_lo, n_samples, roots, roots_per_sample, seed, steps,
                           step_cap, s, res);
  else if (tw_applicable(g->g, a))
    rc = run_chain_walk_hub(g, a, sample_lo, n_samples, roots, roots_per_sample, seed, steps,
                            step_cap, s, res);
  else
    rc = run_chain_walk(g, a, sample_lo, n_samples, roots, roots_per_sample, seed, steps,
                        step_cap, paradigm, s, res);
  if (rc != ND_OK) {
    cudaStreamSynchronize(s);
    nd_result_destroy(res);
    return rc;
  }
  *out = res;
  return ND_OK;
}

extern "C" int nd_result_profile(const nd_result* r, double* ms, int64_t n) {
  if (!r) return ND_ERR_ARG;
  for (int64_t i = 0; i < n && i < 4; i++) ms[i] = r->prof_ms[i];
  return ND_OK;
}

extern "C" int nd_result_step_times(const nd_result* r, double* build_ms, double* sample_ms,
                                    int64_t n_max, int64_t* n_out) {
  if (!r || !n_out) return ND_ERR_ARG;
  const int64_t k = (int64_t)r->step_build_ms.size();
  *n_out = k;
  for (int64_t i = 0; i < k && i < n_max; i++) {
    if (build_ms) build_ms[i] = r->step_build_ms[i];
    if (sample_ms) sample_ms[i] = r->step_sample_ms[i];
  }
  return ND_OK;
}
