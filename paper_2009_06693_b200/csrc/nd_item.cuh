// nd_item.cuh — the per-slot `next` of every individual app, on device.
//
// One work item = (transit v, previous vertex t, sample id, transit index,
// slot) exactly as in individual_batch (_ckernels.pyx:184-265, draw protocol
// _pykernels.py:161-167):
//   deepwalk  draw 0 -> weighted pick
//   ppr       draw 0 < term -> NULL, else draw 1 -> weighted pick
//   khop/mrw  draw 0 -> col[lo + u % deg]
//   node2vec  t < 0: draw 0 weighted pick; else tries j: draw 2j pick,
//             draw 2j+1 accept test r*env < w*factor (no FMA: products only)
// v's row is read through a row source: global memory (GRow) or a copy
// staged in shared memory by the transit-parallel class kernels (SRow).
// t's row (node2vec membership) is always read from the global CSR.
#pragma once

#include "nd_common.cuh"
#include "nd_internal.h"

namespace nd {

template <typename ColT>
struct GView {
  const int64_t* row;
  const ColT* col;
  const double* w;    // may be null when unit
  const double* pre;  // may be null when unit
  const double* mx;
  int unit;
  const int32_t* hset;   // optional exact membership index (int32 CSR only)
  const int32_t* guide;  // optional guide table
};

__host__ __device__ inline GView<int32_t> view(const DevGraph& g) {
  return GView<int32_t>{g.row, g.col, g.w, g.pre, g.mx, g.unit, g.hset, g.guide};
}

// v's row in global memory, indexed relative to its start
template <typename ColT>
struct GRow {
  const ColT* col;
  const double* pre;
  const double* w;
  const int32_t* gd;  // guide table of this row (or null)
  __device__ __forceinline__ int64_t c(int64_t k) const { return (int64_t)__ldg(col + k); }
  __device__ __forceinline__ double p(int64_t k) const { return __ldg(pre + k); }
  __device__ __forceinline__ double wt(int64_t k) const { return __ldg(w + k); }
  __device__ __forceinline__ void cw(int64_t k, int64_t& c_, double& w_, int unit) const {
    c_ = (int64_t)__ldg(col + k);
    w_ = unit ? 1.0 : __ldg(w + k);
  }
};

template <typename ColT>
__device__ __forceinline__ GRow<ColT> grow(const GView<ColT>& g, int64_t lo) {
  return GRow<ColT>{g.col + lo, g.unit ? nullptr : g.pre + lo, g.unit ? nullptr : g.w + lo,
                    g.guide ? g.guide + lo : nullptr};
}

// v's row staged in shared memory
struct SRow {
  const int32_t* col;
  const double* pre;
  const double* w;
  const int32_t* gd = nullptr;
  __device__ __forceinline__ int64_t c(int64_t k) const { return (int64_t)col[k]; }
  __device__ __forceinline__ double p(int64_t k) const { return pre[k]; }
  __device__ __forceinline__ double wt(int64_t k) const { return w[k]; }
  __device__ __forceinline__ void cw(int64_t k, int64_t& c_, double& w_, int unit) const {
    c_ = (int64_t)col[k];
    w_ = unit ? 1.0 : w[k];
  }
};

// Exact guide bucket of a pick target x (guide tables: nd_index.cu).  The
// build stores guide[j] = upper_bound(prefix row, y_j) with
// y_j = rn(rn(total/deg) * j).  For the bucket j with y_j <= x < y_{j+1},
// found here by exact comparisons against those same rounded products, every
// entry before guide[j] is <= y_j <= x and prefix[guide[j+1]] > y_{j+1} > x:
// the upper bound of x lies in [guide[j], guide[j+1]] (for j = deg-1 in
// [guide[deg-1], deg]), the same entry the full-row search finds.  Returns -1
// when the bucket width is not positive (search the whole row).
__device__ __forceinline__ int64_t guide_bucket(double x, double total, int64_t deg) {
  const double width = __ddiv_rn(total, (double)deg);
  if (!(width > 0.0) || !(x >= 0.0)) return -1;
  const double q = __ddiv_rn(x, width);
  int64_t j = q < (double)(deg - 1) ? (int64_t)q : deg - 1;
  while (j > 0 && __dmul_rn(width, (double)j) > x) j--;
  while (j + 1 < deg && __dmul_rn(width, (double)(j + 1)) <= x) j++;
  return j;
}

// upper-bound inverse-CDF pick (_ckernels.pyx:65-74, 90-100); returns k in [0, deg).
// With a guide table the search runs over the exact bucket's bracket.
template <typename RowT>
__device__ __forceinline__ int64_t pick_rel(const RowT& r, int unit, int64_t deg, double u01,
                                            double total_known = -1.0) {
  if (unit) {
    double x = __dmul_rn(u01, (double)deg);
    int64_t k = (int64_t)x;
    return k < deg - 1 ? k : deg - 1;
  }
  const double total = total_known >= 0.0 ? total_known : r.p(deg - 1);
  const double x = __dmul_rn(u01, total);
  int64_t lo = 0, hi = deg;
  if (r.gd != nullptr && deg > GUIDE_MIN_DEG) {
    const int64_t j = guide_bucket(x, total, deg);
    if (j >= 0) {
      lo = __ldg(r.gd + j);
      hi = j + 1 < deg ? (int64_t)__ldg(r.gd + j + 1) : deg;
    }
  }
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (r.p(mid) <= x) lo = mid + 1; else hi = mid;
  }
  return lo < deg - 1 ? lo : deg - 1;
}

// exact membership through the per-row hash set (open addressing, linear probe)
__device__ __forceinline__ bool hset_contains(const int32_t* __restrict__ tab, int64_t size,
                                              int32_t u, int64_t* loads = nullptr) {
  const uint32_t mask = (uint32_t)size - 1;
  const int sh = 32 - (63 - __clzll(size));  // log2(size) top bits
  uint32_t p = size > 1 ? (hset_hash((uint32_t)u) >> sh) : 0;
  while (true) {
    if (loads) ++*loads;
    const int32_t x = __ldg(tab + p);
    if (x == u) return true;
    if (x < 0) return false;
    p = (p + 1) & mask;
  }
}

template <typename ColT>
__device__ __forceinline__ bool has_edge(const ColT* __restrict__ a, int64_t lo, int64_t hi,
                                         int64_t t) {
  int64_t end = hi;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(a + mid) < t) lo = mid + 1; else hi = mid;
  }
  return lo < end && (int64_t)__ldg(a + lo) == t;
}

// node2vec acceptance of one try (_ckernels.pyx:249-261):
//   factor = f_ret if nbr == t, f_adj if nbr in adj(t), else f_far;
//   accept iff env <= 0 or r*env < w*factor   (two rounded products, no FMA)
// For nbr != t the membership test only matters when r*env falls between
// w*f_adj and w*f_far: rounding is monotone, so r*env below both products
// accepts and r*env at or above both rejects whatever has_edge(t, nbr) says.
// `member()` (the probe into t's row) runs only in the band; `probed` reports
// it for the byte model.
template <class Member>
__device__ __forceinline__ bool n2v_accept(const NdApp& a, int64_t nb, int64_t t, double w,
                                           double u01, double env, Member member, bool& probed) {
  if (env <= 0.0) return true;
  const double lhs = __dmul_rn(u01, env);
  if (nb == t) return lhs < __dmul_rn(w, a.f_ret);
  const double pa = __dmul_rn(w, a.f_adj), pf = __dmul_rn(w, a.f_far);
  if (lhs < pa && lhs < pf) return true;
  if (!(lhs < pa) && !(lhs < pf)) return false;
  probed = true;
  return lhs < (member() ? pa : pf);
}

// ceil(log2(ceil(deg/4))): binary-search sectors over 8-byte entries (SURVEY §8 d)
__device__ __forceinline__ int search_sectors(int64_t deg) {
  int64_t s = (deg + 3) >> 2;
  if (s <= 1) return 0;
  return 64 - __clzll(s - 1);
}

// Algorithmic-byte model of SURVEY §8(d) (S = 32-byte sector): accumulated by
// the kernels so the roofline numerator is counted, not estimated.
struct ItemStats {
  int64_t bytes = 0;
  int64_t tries = 0;
  int64_t sect = 0;  // random 32-byte sector reads issued (gather-ceiling comparison)
};
constexpr int64_t SECTOR = 32;

// Evaluate one item.  `base0` = key_base(seed, step, 0, 0); `ik` =
// key_item(sid, tix, slot).  `deg` is v's degree.  Returns the vertex or -1.
template <typename ColT, typename RowT>
__device__ __forceinline__ int64_t run_item(const GView<ColT>& g, const RowT& r, const NdApp& a,
                                            int64_t v, int64_t deg, int64_t t, uint64_t base0,
                                            uint64_t ik, ItemStats& st, int* stall,
                                            int64_t t_lo_known = -1, int64_t t_hi_known = -1,
                                            double mx_known = -1.0, double tot_known = -1.0) {
  if (deg <= 0) return -1;
  const int64_t wsec = g.unit ? 0 : SECTOR * search_sectors(deg);
  switch (a.code) {
    case ND_DEEPWALK: {
      st.bytes += SECTOR + wsec + SECTOR + 8;
      return r.c(pick_rel(r, g.unit, deg, to_unit(draw_u64(base0, ik)), tot_known));
    }
    case ND_PPR: {
      if (to_unit(draw_u64(base0, ik)) < a.term) return -1;
      st.bytes += SECTOR + wsec + SECTOR + 8;
      return r.c(pick_rel(r, g.unit, deg, to_unit(draw_u64(base0 + C_DRAW, ik)), tot_known));
    }
    case ND_KHOP:
    case ND_MULTIRW: {
      st.bytes += SECTOR + 8;
      return r.c((int64_t)mod_u64(draw_u64(base0, ik), (uint64_t)deg));
    }
    case ND_NODE2VEC: {
      if (t < 0) {
        st.bytes += SECTOR + wsec + SECTOR + 8;
        return r.c(pick_rel(r, g.unit, deg, to_unit(draw_u64(base0, ik)), tot_known));
      }
      const int64_t t_lo = t_lo_known >= 0 ? t_lo_known : __ldg(g.row + t);
      const int64_t t_hi = t_lo_known >= 0 ? t_hi_known : __ldg(g.row + t + 1);
      const double env = __dmul_rn(mx_known >= 0.0 ? mx_known : __ldg(g.mx + v), a.f_max);
      const int64_t probe = SECTOR * search_sectors(t_hi - t_lo);
      st.bytes += 2 * SECTOR + 8;
      uint64_t b = base0;
      for (int64_t j = 0; j < N2V_MAX_TRIES; j++) {
        const int64_t k = (int64_t)mod_u64(draw_u64(b, ik), (uint64_t)deg);
        int64_t nb;
        double w;
        r.cw(k, nb, w, g.unit);
        st.tries++;
        st.bytes += 2 * SECTOR;
        const double u01 = to_unit(draw_u64(b + C_DRAW, ik));
        bool probed = false;
        const bool acc = n2v_accept(a, nb, t, w, u01, env, [&] {
          if (g.hset != nullptr && t_hi - t_lo > HASH_MIN_DEG)
            return hset_contains(g.hset + 4 * t_lo, hset_size(t_hi - t_lo), (int32_t)nb);
          return has_edge(g.col, t_lo, t_hi, nb);
        }, probed);
        if (probed) st.bytes += probe;
        if (acc) return nb;
        b += 2 * C_DRAW;
      }
      *stall = 1;
      return -1;
    }
  }
  return -1;
}

}  // namespace nd
