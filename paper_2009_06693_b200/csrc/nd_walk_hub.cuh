// nd_walk_hub.cuh — transit-parallel chain walks without a sort (included by
// nd_walk.cu after the walker-major kernel, whose per-walker step functions
// it shares).
//
// The reference's TP step (transit_parallel.py:185-230) inverts the alive
// (walker, transit) pairs into transit groups (:71-83), classes the groups by
// work = members*m with m = 1 for walks (small < 32, medium 32..1024, large
// > 1024; :86-101) and runs each class with its own kernel.
// Here that step is built from member counts instead of a radix sort:
//
//   count     — one streaming pass over the window's rows: the walkers of a
//               1024-row tile are counted per distinct transit in a shared-
//               memory hash table, then one atomicAdd per (tile, transit) on
//               cnt[v] returns the tile's base position in the group (a hub's
//               many members cost one global atomic per tile); each walker's
//               position = base + its rank in the tile.  The group count
//               (0 -> 1 crossings), the medium and large class counts
//               (crossings of 32 and 1025 members) and the hub list (groups
//               reaching 32 members: every medium and large group) fall out
//               of the same atomics, exactly;
//   prep      — one thread per hub: its tier and its member slots (disjoint
//               ranges reserved by atomics, staged tiers from the front of the
//               member array, the grid tier from the back);
//   place     — a second streaming pass writes every hub member's record at
//               its group position and lists the small-class walkers;
//   small     — the sub-warp class (m = 1: one lane per member): a
//               persistent kernel steps the listed walkers (rejection tries
//               refill lanes as in the walker-major kernel);
//   hub tiers — warp (one warp per hub, row staged), thread block (one CTA per
//               unit of a hub's members, row staged) and grid (the members of
//               every hub whose row does not fit or does not pay, spread over
//               the whole grid, rows read from global memory).  Staging is one
//               bulk copy (cp.async.bulk + mbarrier, nd_bulk.cuh) of the
//               transit's record row into shared memory, awaited after the
//               first members' records are in flight.
// The sampling kernels clear cnt[v] of the transits they step, so the next
// step's count starts from zero without a separate pass.
//
// Walker state is held per window row in HBM as structure-of-arrays
// (vertex, row start, degree, max weight or prefix total), double-buffered:
// node2vec reads its previous vertex's row from the buffer it is about to
// overwrite.  Values are written step-major ([Lw, rows], coalesced) and
// transposed into the final rows at the end.  Windows compact the alive
// walkers between them.  Every draw is keyed by (sample, step), so the rows
// equal the walker-major engine's and the reference's.

namespace {

constexpr int TW_BLOCK = 256;
constexpr int TW_TM = 32;           // members at which a walk group is medium (work >= 32)
constexpr int TW_TL = 1025;         // members at which it is large (work > 1024)
constexpr int TW_WARP_MAX = 256;    // members of a warp-tier hub
constexpr int TW_UNIT = 2048;       // members per CTA unit
constexpr int TW_STAGE_W = 4096;    // staged row bytes per warp
constexpr int TW_STAGE_C = 96 * 1024;  // staged row bytes per CTA
constexpr int TW_PAY = 64;          // stage when row bytes <= members * TW_PAY
constexpr int TW_Q = 4;             // tiles of 32 rows per warp in the streaming passes
constexpr int TW_TILE = TW_BLOCK * TW_Q;  // rows per CTA tile
constexpr int TW_HT = 2048;         // hash slots per tile (>= 2 * TW_TILE)
constexpr int TW_PLACE_ROWS = 4096; // rows per place CTA chunk (small list staged in smem)

struct TwCtl {  // per step (alternating by step parity)
  int nhub, nsmall, queue, nwarp, nunit, front, back, pad;
};

struct __align__(16) TwUnit {
  int32_t v, m0, m1, j;  // hub vertex, member slots [m0, m1), hub index
};

// A hub member as the hub kernels read it (48 bytes, two loads): its row,
// walker, transit with the transit's row header, group position and
// (node2vec) previous vertex with that vertex's row bounds.
struct __align__(16) TwRec {
  int32_t row, w, v, deg;
  uint32_t lo;
  int32_t t, tdeg;
  uint32_t tlo;
  double hd;
  int32_t pos, j;
};

struct TwArgs {
  PWArgs P;             // graph records, app, seed, sample_lo, ctr, stall
  int64_t rows;
  const int32_t* wid;   // row -> walker (null: identity)
  int64_t s, k, Lw;     // absolute step, step within the window, window length
  int last;             // s is the window's last step (continuations instead of state)
  int tries;            // node2vec tries this step (t >= 0 for every walker)
  int rmode;            // bytes per edge of the hub rows read: 0: 32, 1: 16, 2: lines
  // state of step s and of step s+1 (node2vec: t's fields are read from the
  // step s+1 buffer before it is written)
  const int32_t* cur;
  const uint32_t* lo;
  const int32_t* deg;
  const double* hd;
  int32_t* ncur;
  uint32_t* nlo;
  int32_t* ndeg;
  double* nhd;
  int32_t* pos;         // group position of the row's walker this step
  int32_t* out;         // [Lw, rows]
  int32_t* nnz;         // per row: non-NULL values of the window
  int32_t* died;        // per walker: ended with a NULL
  int32_t* cont_wid;
  int32_t* cont_v;
  int32_t* cont_t;
  int* cont_n;
  int* max_len;
  // this step's groups
  TwCtl* ctl;
  TwCtl* nctl;          // the next step's (reset by prep)
  int32_t* cnt;         // member counts (zero between steps)
  int32_t* vhub;        // hub index of a vertex (valid while cnt >= TW_TM)
  int32_t* hubs;
  unsigned long long* stats;
  int32_t* hoff;        // per hub: first member slot
  TwRec* hrec;          // hub members in group order
  int64_t hcap;         // member slots
  int32_t* slist;       // small-class rows
  TwUnit* wunits;
  TwUnit* cunits;
};

struct TwCounts {
  unsigned long long ng = 0, nm = 0, nl = 0;
};

struct TwLane {
  int64_t row = -1;
  int64_t w = 0;
  int32_t v = 0, t = -1;
  int64_t lo = 0, tlo = 0;
  int32_t deg = 0, tdeg = 0;
  double hd = 0.0;
  int32_t j = 0;
  uint64_t ik = 0;
};

// ---- count: member positions, class counts and the hub list ------------------
struct TwTable {
  int32_t key[TW_HT];
  int32_t num[TW_HT];
  int32_t base[TW_HT];
};

// warp-aggregated append of the lanes with f set; returns each lane's slot
__device__ __forceinline__ int tw_warp_append(bool f, int* gcount) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if (!m) return -1;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(gcount, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  return f ? base + __popc(m & ((1u << lane) - 1)) : -1;
}

// One CTA tile of TW_TILE rows (every thread calls it; v[q] >= 0 are alive
// walkers at transit v).
template <int Q>
__device__ __forceinline__ void tw_count_tile(const TwArgs& A, const int32_t (&v)[Q], int64_t b0,
                                              TwCounts& cc, TwTable& T) {
  const int lane = threadIdx.x & 31;
  int slot[Q], loc[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    slot[q] = -1;
    loc[q] = 0;
    if (v[q] < 0) continue;
    uint32_t h = hset_hash((uint32_t)v[q]) >> (32 - 11);
    while (true) {
      const int32_t k = atomicCAS(&T.key[h], -1, v[q]);
      if (k == -1 || k == v[q]) break;
      h = (h + 1) & (TW_HT - 1);
    }
    slot[q] = (int)h;
    loc[q] = atomicAdd(&T.num[h], 1);
  }
  __syncthreads();
  // one global atomic per distinct transit of the tile, all in flight together
  constexpr int PER = TW_HT / TW_BLOCK;
  int32_t kv[PER], c[PER], o[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const int sl = k * TW_BLOCK + threadIdx.x;
    kv[k] = T.key[sl];
    c[k] = T.num[sl];
    o[k] = kv[k] >= 0 ? atomicAdd(A.cnt + kv[k], c[k]) : 0;
  }
#pragma unroll
  for (int k = 0; k < PER; k++) {
    bool hm = false;
    if (kv[k] >= 0) {
      T.base[k * TW_BLOCK + threadIdx.x] = o[k];
      cc.ng += o[k] == 0;
      hm = o[k] < TW_TM && o[k] + c[k] >= TW_TM;
      cc.nm += hm;
      cc.nl += o[k] < TW_TL && o[k] + c[k] >= TW_TL;
    }
    const int idx = tw_warp_append(hm, &A.ctl->nhub);  // rare: a group becomes a hub
    if (hm) {
      A.hubs[idx] = kv[k];
      A.vhub[kv[k]] = idx;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < Q; q++)
    if (slot[q] >= 0) A.pos[b0 + q * 32 + lane] = T.base[slot[q]] + loc[q];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PER; k++) {
    T.key[k * TW_BLOCK + threadIdx.x] = -1;
    T.num[k * TW_BLOCK + threadIdx.x] = 0;
  }
  __syncthreads();
}

// per-warp class deltas (a tile can cross a threshold of a group another tile
// opened: the signed deltas sum to the exact counts over the grid)
__device__ __forceinline__ void tw_flush_classes(TwCounts cc, unsigned long long* stats) {
  for (int o = 16; o > 0; o >>= 1) {
    cc.ng += __shfl_down_sync(0xffffffffu, cc.ng, o);
    cc.nm += __shfl_down_sync(0xffffffffu, cc.nm, o);
    cc.nl += __shfl_down_sync(0xffffffffu, cc.nl, o);
  }
  if ((threadIdx.x & 31) == 0 && (cc.ng | cc.nm | cc.nl)) {
    if (cc.ng != cc.nm) atomicAdd(stats + 0, cc.ng - cc.nm);
    if (cc.nm != cc.nl) atomicAdd(stats + 1, cc.nm - cc.nl);
    if (cc.nl) atomicAdd(stats + 2, cc.nl);
    if (cc.ng) atomicAdd(stats + 3, cc.ng);
  }
}

__global__ void __launch_bounds__(TW_BLOCK) k_tw_count(TwArgs A) {
  __shared__ TwTable T;
  for (int k = threadIdx.x; k < TW_HT; k += TW_BLOCK) {
    T.key[k] = -1;
    T.num[k] = 0;
  }
  __syncthreads();
  TwCounts cc;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int64_t t0 = blockIdx.x * (int64_t)TW_TILE; t0 < A.rows; t0 += (int64_t)gridDim.x * TW_TILE) {
    const int64_t b0 = t0 + wib * 32 * TW_Q;
    int32_t v[TW_Q];
#pragma unroll
    for (int q = 0; q < TW_Q; q++) {
      const int64_t row = b0 + q * 32 + lane;
      v[q] = row < A.rows ? A.cur[row] : -1;
    }
    tw_count_tile<TW_Q>(A, v, b0, cc, T);
  }
  tw_flush_classes(cc, A.stats);
}

// ---- prep: hub tiers and member slots (one thread per hub) --------------------
// A hub's members read its record row; staging pays when the row is at most
// TW_PAY bytes per member.  Tiers:
//   warp   <= TW_WARP_MAX members, row <= TW_STAGE_W bytes: one warp, staged;
//   CTA    row <= TW_STAGE_C bytes: units of <= TW_UNIT members, one CTA each,
//          staged;
//   grid   rows too large to stage (or not worth it): the members of every
//          such hub spread over the whole grid, rows read from global memory.
// Member slots: disjoint ranges reserved with warp-aggregated atomics, the
// staged tiers from the front of the member array, the grid tier from the
// back, so the grid tier's members are one contiguous range.
__device__ __forceinline__ uint32_t tw_rbytes(int rmode, int64_t deg) {
  if (deg <= 0) return 0;
  const int64_t b = rmode == 2 ? (deg + 2) / 3 * 128 : deg * (rmode == 1 ? 16 : 32);
  return b > 0x7fffffff ? 0x7fffffffu : (uint32_t)b;
}
__device__ __forceinline__ int tw_tier(int c, uint32_t bytes) {
  const bool pays = bytes > 0 && (uint64_t)bytes <= (uint64_t)c * TW_PAY;
  if (pays && c <= TW_WARP_MAX && bytes <= TW_STAGE_W) return 0;
  if (pays && bytes <= TW_STAGE_C) return 1;
  return 2;
}

// reserve n (per lane) from a counter with one atomic per warp
__device__ __forceinline__ int tw_warp_reserve(int n, int* gcount) {
  const int lane = threadIdx.x & 31;
  int x = n;  // inclusive scan
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const int total = __shfl_sync(0xffffffffu, x, 31);
  int base = 0;
  if (lane == 31 && total) base = atomicAdd(gcount, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + x - n;
}

__global__ void __launch_bounds__(256) k_tw_prep(TwArgs A) {
  const int H = A.ctl->nhub;
  if (blockIdx.x == 0 && threadIdx.x == 0) *A.nctl = TwCtl{};
  for (int jb = blockIdx.x * blockDim.x; jb < H; jb += gridDim.x * blockDim.x) {
    const int j = jb + threadIdx.x;
    int32_t v = -1, c = 0, t = -1, nu = 0;
    if (j < H) {
      v = A.hubs[j];
      c = A.cnt[v];
      const int64_t r0 = __ldg(A.P.gv.row + v), r1 = __ldg(A.P.gv.row + v + 1);
      t = tw_tier(c, tw_rbytes(A.rmode, r1 - r0));
      if (t == 1) nu = (c + TW_UNIT - 1) / TW_UNIT;
    }
    const int mf = tw_warp_reserve(t == 0 || t == 1 ? c : 0, &A.ctl->front);
    const int mg = tw_warp_reserve(t == 2 ? c : 0, &A.ctl->back);
    const int wu = tw_warp_reserve(t == 0 ? 1 : 0, &A.ctl->nwarp);
    const int cu = tw_warp_reserve(nu, &A.ctl->nunit);
    if (j < H) {
      const int m0 = t == 2 ? (int)(A.hcap - mg - c) : mf;
      A.hoff[j] = m0;
      if (t == 0) A.wunits[wu] = TwUnit{v, m0, m0 + c, j};
      for (int q = 0; q < nu; q++)
        A.cunits[cu + q] = TwUnit{v, m0 + q * TW_UNIT, m0 + min(c, (q + 1) * TW_UNIT), j};
    }
  }
}

// ---- place: hub member records at their group positions, the small list -------
// Each CTA takes chunks of TW_PLACE_ROWS consecutive rows, collects its small
// rows in shared memory and reserves their list slots with one atomic.
__global__ void __launch_bounds__(TW_BLOCK) k_tw_place(TwArgs A) {
  __shared__ int32_t s_small[TW_PLACE_ROWS];
  __shared__ int s_n, s_base;
  const int lane = threadIdx.x & 31;
  for (int64_t c0 = blockIdx.x * (int64_t)TW_PLACE_ROWS; c0 < A.rows;
       c0 += (int64_t)gridDim.x * TW_PLACE_ROWS) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int64_t c1 = A.rows < c0 + TW_PLACE_ROWS ? A.rows : c0 + TW_PLACE_ROWS;
    for (int64_t r0 = c0 + (threadIdx.x & ~31) * TW_Q; r0 < c1; r0 += TW_TILE) {
      int32_t v[TW_Q], c[TW_Q];
#pragma unroll
      for (int q = 0; q < TW_Q; q++) {
        const int64_t row = r0 + q * 32 + lane;
        v[q] = row < c1 ? A.cur[row] : -2;
      }
#pragma unroll
      for (int q = 0; q < TW_Q; q++) c[q] = v[q] >= 0 ? A.cnt[v[q]] : 0;
#pragma unroll
      for (int q = 0; q < TW_Q; q++) {
        const int64_t row = r0 + q * 32 + lane;
        if (v[q] == -1) A.ncur[row] = -1;  // ended earlier in the window
        const bool hub = v[q] >= 0 && c[q] >= TW_TM;
        if (hub) {
          const int32_t j = A.vhub[v[q]], p = A.pos[row];
          TwRec r;
          r.row = (int32_t)row;
          r.w = A.wid ? A.wid[row] : (int32_t)row;
          r.v = v[q];
          r.deg = A.deg[row];
          r.lo = A.lo[row];
          r.hd = A.hd[row];
          r.t = -1;
          r.tdeg = 0;
          r.tlo = 0;
          if (A.tries) {
            r.t = A.ncur[row];
            r.tlo = A.nlo[row];
            r.tdeg = A.ndeg[row];
          }
          r.pos = p;
          r.j = j;
          A.hrec[A.hoff[j] + p] = r;
        }
        const bool sm = v[q] >= 0 && c[q] < TW_TM;
        const unsigned m = __ballot_sync(0xffffffffu, sm);
        if (m) {
          int base = 0;
          if (lane == 0) base = atomicAdd(&s_n, __popc(m));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (sm) s_small[base + __popc(m & ((1u << lane) - 1))] = (int32_t)row;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_n ? atomicAdd(&A.ctl->nsmall, s_n) : 0;
    __syncthreads();
    for (int k = threadIdx.x; k < s_n; k += TW_BLOCK) A.slist[s_base + k] = s_small[k];
    __syncthreads();
  }
}

__device__ __forceinline__ void tw_flush_len(int mlen, int* max_len) {
  for (int o = 16; o > 0; o >>= 1) mlen = max(mlen, __shfl_down_sync(0xffffffffu, mlen, o));
  if ((threadIdx.x & 31) == 0 && mlen > 0) atomicMax(max_len, mlen);
}

// ---- sampling ---------------------------------------------------------------------
// One unit of work of a lane's walker at step s: a node2vec try or a whole
// pick (the walker-major kernel's protocol, k_walk_persistent).  `srec` is
// the transit's record row staged in shared memory (SH).  Returns true when
// the step is decided (o = next vertex or NULL).
template <bool SH>
__device__ __forceinline__ bool tw_work(const TwArgs& A, TwLane& L, const unsigned char* srec,
                                        uint64_t base0, int64_t& o, NextHdr& nh, ItemStats& st) {
  const PWArgs& P = A.P;
  if (L.deg <= 0) {
    o = -1;
    return true;
  }
  if (A.tries) {
    if (L.j == 0) st.bytes += 2 * SECTOR;  // t offsets + max_w (§8 d pair term)
    const double env = __dmul_rn(L.hd, P.a.f_max);
    const NbrW* rw = P.nbu ? nullptr : (SH ? reinterpret_cast<const NbrW*>(srec) : P.nbw + L.lo);
    const NbrU* ru = P.nbu ? (SH ? reinterpret_cast<const NbrU*>(srec) : P.nbu + L.lo) : nullptr;
    o = rec_try_at<SH>(P, rw, ru, L.deg, L.t, L.tlo, L.tlo + L.tdeg, env,
                       base0 + 2 * C_DRAW * (uint64_t)L.j, L.ik, nh, st);
    if (o == -2) {
      if (++L.j >= N2V_MAX_TRIES) {
        atomicExch(P.stall, 1);
        o = -1;
        return true;
      }
      return false;
    }
    return true;
  }
  double u;
  if (P.a.code == ND_PPR) {
    if (to_unit(draw_u64(base0, L.ik)) < P.a.term) {
      o = -1;
      return true;
    }
    u = to_unit(draw_u64(base0 + C_DRAW, L.ik));
  } else {
    u = to_unit(draw_u64(base0, L.ik));
  }
  if (P.pl) {
    o = line_pick_at<SH>(SH ? reinterpret_cast<const PickLine*>(srec) : P.pl + L.lo, L.deg, L.hd,
                         u, nh, st);
  } else {
    const NbrP* rp = P.nbu ? nullptr : (SH ? reinterpret_cast<const NbrP*>(srec) : P.nbp + L.lo);
    const NbrU* ru = P.nbu ? (SH ? reinterpret_cast<const NbrU*>(srec) : P.nbu + L.lo) : nullptr;
    o = rec_pick_at<SH>(rp, ru, P.gv.guide ? P.gv.guide + L.lo : nullptr, L.deg, L.hd, u, nh, st);
  }
  return true;
}

// Emission of a decided step (warp-uniform call; fin marks the lanes whose
// walker decided): the value and the next state, or the walk's end (NULL) /
// the window's continuation list.
__device__ __forceinline__ void tw_emit(const TwArgs& A, bool fin, const TwLane& L, int64_t o,
                                        const NextHdr& nh, int& mlen, ItemStats& st) {
  if (fin) {
    A.out[A.k * A.rows + L.row] = (int32_t)o;
    mlen = max(mlen, (int)A.s + 1);
    if (o < 0) {
      A.nnz[L.row] = (int32_t)A.k;
      A.died[L.w] = 1;
      A.ncur[L.row] = -1;
    } else if (A.last) {
      A.nnz[L.row] = (int32_t)A.k + 1;
    } else {
      double nhd = A.P.a.code == ND_NODE2VEC ? nh.mx : nh.tot;
      if (nhd < 0.0) {  // node2vec after its step-0 pick: max weight of the new vertex
        nhd = __ldg(A.P.gv.mx + o);
        st.sect += 1;
      }
      A.ncur[L.row] = (int32_t)o;
      A.nlo[L.row] = (uint32_t)nh.lo;
      A.ndeg[L.row] = (int32_t)nh.deg;
      A.nhd[L.row] = nhd;
    }
  }
  if (A.last) {
    const bool c = fin && o >= 0;
    const int slot = tw_warp_append(c, A.cont_n);
    if (c) {
      A.cont_wid[slot] = (int32_t)L.w;
      A.cont_v[slot] = (int32_t)o;
      A.cont_t[slot] = L.v;
    }
  }
}

__device__ __forceinline__ void tw_lane_start(const TwArgs& A, TwLane& L, ItemStats& st) {
  L.j = 0;
  L.ik = key_item((uint64_t)(A.P.sample_lo + L.w), 0, 0);
  st.bytes += SECTOR + 8;  // §8(d) pair term: offsets pair + transit id
}

// lane state of a hub member record (48 bytes); the group's first member
// clears the transit's count for the next step
__device__ __forceinline__ void tw_load_rec(const TwArgs& A, TwLane& L, const TwRec* r,
                                            ItemStats& st) {
  const int4* q = reinterpret_cast<const int4*>(r);  // 16-byte aligned (48-byte records)
  const int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  L.row = a.x;
  L.w = a.y;
  L.v = a.z;
  L.deg = a.w;
  L.lo = (uint32_t)b.x;
  L.t = b.y;
  L.tdeg = b.z;
  L.tlo = (uint32_t)b.w;
  L.hd = __longlong_as_double(((long long)(uint32_t)c.y << 32) | (uint32_t)c.x);
  if (c.z == 0) A.cnt[L.v] = 0;
  tw_lane_start(A, L, st);
}

// Persistent lane loop over N work items: `load(i, L)` fills a lane from item
// i; lanes refill from a warp-claimed chunk of a global queue as their walker
// decides (node2vec's rejection tries keep every lane busy).
template <bool SH, class Load>
__device__ __forceinline__ void tw_lanes(const TwArgs& A, int64_t N, int* queue, int chunk,
                                         const unsigned char* srec, Load load, ItemStats& st,
                                         int& mlen) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1;
  const uint64_t base0 = key_base(A.P.seed, (uint64_t)A.s, 0, 0);
  TwLane L;
  int64_t wbeg = 0, wend = 0, i = -1;
  while (true) {
    const bool need = i < 0;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
      const int c = __popc(m);
      const int rank = __popc(m & lt_mask);
      const int64_t rem = wend - wbeg;
      int64_t nbeg = 0;
      if (rem < c) {
        int base = 0;
        if (lane == 0) base = atomicAdd(queue, chunk);
        nbeg = __shfl_sync(0xffffffffu, base, 0);
      }
      if (need) {
        i = rank < rem ? wbeg + rank : nbeg + (rank - rem);
        if (i < N) load(i, L);
      }
      if (rem < c) {
        wbeg = nbeg + (c - rem);
        wend = nbeg + chunk;
      } else {
        wbeg += c;
      }
    }
    if (__all_sync(0xffffffffu, i >= N)) break;
    bool fin = false;
    int64_t o = -1;
    NextHdr nh;
    if (i < N) fin = tw_work<SH>(A, L, srec, base0, o, nh, st);
    tw_emit(A, fin, L, o, nh, mlen, st);
    if (fin) i = -1;
  }
}

// ---- small class and grid tier: one persistent kernel --------------------------
// Items [0, nsmall) are the small-class walkers (the sub-warp kernel, m = 1:
// one lane per member); items [nsmall, nsmall + back) are the members of
// every hub whose row is not staged (the grid kernel: one hub's members over
// the whole grid, the row read from global memory).  One queue feeds both.
template <int MINB>
__global__ void __launch_bounds__(TW_BLOCK, MINB) k_tw_sample(TwArgs A) {
  ItemStats st;
  int mlen = 0;
  const int64_t NS = A.ctl->nsmall, NG = A.ctl->back, M0 = A.hcap - NG;
  tw_lanes<false>(A, NS + NG, &A.ctl->queue, A.P.chunk, nullptr,
                  [&](int64_t i, TwLane& L) {
                    if (i >= NS) {
                      tw_load_rec(A, L, A.hrec + M0 + (i - NS), st);
                      return;
                    }
                    const int64_t row = A.slist[i];
                    L.row = row;
                    L.w = A.wid ? A.wid[row] : row;
                    L.v = A.cur[row];
                    L.lo = A.lo[row];
                    L.deg = A.deg[row];
                    L.hd = A.hd[row];
                    if (A.tries) {
                      L.t = A.ncur[row];
                      L.tlo = A.nlo[row];
                      L.tdeg = A.ndeg[row];
                    }
                    A.cnt[L.v] = 0;  // the next step counts from zero
                    tw_lane_start(A, L, st);
                  },
                  st, mlen);
  flush_stats(st, A.P.ctr);
  tw_flush_len(mlen, A.max_len);
}

// bytes and source of the records a hub's members read this step
__device__ __forceinline__ uint32_t tw_row_bytes(const TwArgs& A, int64_t lo, int32_t deg,
                                                 const void** src) {
  const PWArgs& P = A.P;
  if (deg <= 0) return 0;
  if (A.tries) {
    if (P.nbu) { *src = P.nbu + lo; return (uint32_t)deg * 16u; }
    *src = P.nbw + lo;
    return (uint32_t)deg * 32u;
  }
  if (P.pl) { *src = P.pl + lo; return (uint32_t)((deg + 2) / 3) * 128u; }
  if (P.nbu) { *src = P.nbu + lo; return (uint32_t)deg * 16u; }
  *src = P.nbp + lo;
  return (uint32_t)deg * 32u;
}

// The members [m0, m1) of one staged hub unit, lanes refilled from a shared
// cursor; the staged row (bar) is awaited after the first members' records
// are in flight.
__device__ __forceinline__ void tw_hub_members(const TwArgs& A, const TwUnit& d,
                                               const unsigned char* srec, uint64_t* bar,
                                               uint32_t parity, int* cursor, ItemStats& st,
                                               int& mlen) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1;
  const uint64_t base0 = key_base(A.P.seed, (uint64_t)A.s, 0, 0);
  TwLane L;
  bool done = false, waited = false;
  while (true) {
    const bool need = L.row < 0 && !done;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
      int base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(cursor, __popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (need) {
        const int mem = d.m0 + base + __popc(m & lt_mask);
        if (mem < d.m1) tw_load_rec(A, L, A.hrec + mem, st);
        else done = true;
      }
    }
    if (__all_sync(0xffffffffu, L.row < 0 && done)) break;
    if (!waited) {
      mbar_wait(bar, parity);
      waited = true;
    }
    bool fin = false;
    int64_t o = -1;
    NextHdr nh;
    if (L.row >= 0) fin = tw_work<true>(A, L, srec, base0, o, nh, st);
    tw_emit(A, fin, L, o, nh, mlen, st);
    if (fin) L.row = -1;
  }
  if (!waited) mbar_wait(bar, parity);  // keep the barrier's phases in step
}

// ---- warp tier: one warp per hub of <= TW_WARP_MAX members, row staged --------
__global__ void __launch_bounds__(TW_BLOCK) k_tw_hub_warp(TwArgs A) {
  extern __shared__ __align__(128) unsigned char dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm) + wib;
  int* cursor = reinterpret_cast<int*>(dsm + 8 * (TW_BLOCK / 32)) + wib;
  unsigned char* buf = dsm + 128 * ((12 * (TW_BLOCK / 32) + 127) / 128) + (size_t)wib * TW_STAGE_W;
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncwarp();
  ItemStats st;
  int mlen = 0;
  const int64_t U = A.ctl->nwarp;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t ph = 0;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < U; u += nw) {
    const TwUnit d = A.wunits[u];
    if (lane == 0) {
      *cursor = 0;
      const TwRec* r0 = A.hrec + d.m0;
      const void* src = nullptr;
      const uint32_t bytes = tw_row_bytes(A, r0->lo, r0->deg, &src);
      mbar_arrive_expect_tx(bar, bytes);
      bulk_g2s(buf, src, bytes, bar);
    }
    __syncwarp();
    tw_hub_members(A, d, buf, bar, ph, cursor, st, mlen);
    ph ^= 1u;
    __syncwarp();
  }
  flush_stats(st, A.P.ctr);
  tw_flush_len(mlen, A.max_len);
}

// ---- thread-block tier: one CTA per unit of <= TW_UNIT members, row staged ----
__global__ void __launch_bounds__(TW_BLOCK) k_tw_hub_cta(TwArgs A) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint64_t bar;
  __shared__ int cursor;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  ItemStats st;
  int mlen = 0;
  const int64_t U = A.ctl->nunit;
  uint32_t ph = 0;
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    const TwUnit d = A.cunits[u];
    if (threadIdx.x == 0) {
      cursor = 0;
      const TwRec* r0 = A.hrec + d.m0;
      const void* src = nullptr;
      const uint32_t bytes = tw_row_bytes(A, r0->lo, r0->deg, &src);
      mbar_arrive_expect_tx(&bar, bytes);
      bulk_g2s(dsm, src, bytes, &bar);
    }
    __syncthreads();
    tw_hub_members(A, d, dsm, &bar, ph, &cursor, st, mlen);
    ph ^= 1u;
    __syncthreads();
  }
  flush_stats(st, A.P.ctr);
  tw_flush_len(mlen, A.max_len);
}

// ---- window start: lane state of every row -------------------------------------
__global__ void __launch_bounds__(TW_BLOCK) k_tw_init(TwArgs A, const int64_t* __restrict__ roots64,
                                                      const int32_t* __restrict__ roots32, int64_t R,
                                                      const int32_t* __restrict__ v0,
                                                      const int32_t* __restrict__ t0) {
  const bool n2v = A.P.a.code == ND_NODE2VEC;
  int32_t* cur = const_cast<int32_t*>(A.cur);
  uint32_t* lo_ = const_cast<uint32_t*>(A.lo);
  int32_t* deg_ = const_cast<int32_t*>(A.deg);
  double* hd_ = const_cast<double*>(A.hd);
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < A.rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = A.wid ? A.wid[row] : row;
    const int32_t v = v0 ? v0[row] : (int32_t)(roots64 ? roots64[w * R] : roots32[w * R]);
    const int32_t t = t0 ? t0[row] : -1;
    int64_t lo, deg;
    double mx, tot;
    load_vertex(A.P, v, lo, deg, mx, tot);
    if (A.P.pl) lo = __ldg(A.P.vline + v);
    double hd = tot;
    if (n2v && t >= 0) hd = mx >= 0.0 ? mx : __ldg(A.P.gv.mx + v);
    cur[row] = v;
    lo_[row] = (uint32_t)lo;
    deg_[row] = (int32_t)deg;
    hd_[row] = hd;
    if (n2v) {
      A.ncur[row] = t;
      A.nlo[row] = t >= 0 ? (uint32_t)__ldg(A.P.gv.row + t) : 0u;
      A.ndeg[row] = t >= 0 ? (int32_t)(__ldg(A.P.gv.row + t + 1) - __ldg(A.P.gv.row + t)) : 0;
    }
  }
}

// rows of a run that starts in the walker-major tail
__global__ void k_tw_rows0(const int64_t* __restrict__ roots64, const int32_t* __restrict__ roots32,
                           int64_t R, int64_t n, int32_t* __restrict__ wid,
                           int32_t* __restrict__ v, int32_t* __restrict__ t) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    wid[i] = (int32_t)i;
    v[i] = roots64 ? (int32_t)roots64[i * R] : roots32[i * R];
    t[i] = -1;
  }
}

// Final rows of a step-major window [Lw, rows]: 32 x 32 tiles through shared
// memory, loads coalesced over rows, stores coalesced over a row's steps.
__global__ void __launch_bounds__(256) k_tw_emit(const int32_t* __restrict__ out, int64_t rows,
                                                 int64_t Lw, const int32_t* __restrict__ nnz,
                                                 const int32_t* __restrict__ wid, int64_t step0,
                                                 const int64_t* __restrict__ off, int64_t R,
                                                 int32_t* __restrict__ ids) {
  __shared__ int32_t tile[8][32][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t rt = (rows + 31) / 32, kt = (Lw + 31) / 32;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < rt * kt; t += nw) {
    const int64_t r0 = (t / kt) * 32, k0 = (t % kt) * 32;
    const int64_t r = r0 + lane;
    int32_t n = 0;
    int64_t base = 0;
    if (r < rows) {
      n = nnz[r];
      base = off[wid ? wid[r] : r] + R + step0;
    }
    const int32_t nmax = __reduce_max_sync(0xffffffffu, n);
    const int64_t kr = (int64_t)nmax - k0;
    const int kend = kr < 32 ? (int)kr : 32;
    for (int i = 0; i < kend; i++)
      tile[wib][i][lane] = r < rows ? out[(k0 + i) * rows + r] : 0;
    __syncwarp();
    for (int i = 0; i < 32 && r0 + i < rows; i++) {
      const int32_t ni = __shfl_sync(0xffffffffu, n, i);
      const int64_t bi = __shfl_sync(0xffffffffu, base, i);
      if (k0 + lane < ni) ids[bi + k0 + lane] = tile[wib][lane][i];
    }
    __syncwarp();
  }
}

constexpr size_t TW_WARP_SMEM = 128 * ((12 * (TW_BLOCK / 32) + 127) / 128) + (size_t)(TW_BLOCK / 32) * TW_STAGE_W;
constexpr size_t TW_CTA_SMEM = TW_STAGE_C;

}  // namespace
