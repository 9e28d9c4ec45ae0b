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
//   count     — fused into the previous step's emission: a walker landing on
//               vertex o does atomicAdd(cnt_{s+1}[o], 1) (its result consumed
//               one lane iteration later, behind the next walker's loads); the
//               returned old count is its position in o's group, and the +1
//               crossings of 0, 32 and 1025 members give the group count, the
//               medium and large class counts and the hub list (groups
//               reaching 32 members: every medium and large group), exactly;
//   prep      — one thread per hub: its tier and, for the staged tiers, its
//               member slots (disjoint ranges reserved by atomics);
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
// Counts alternate between two buffers by step parity: the sampling kernels
// of step s clear cnt_s[v] of the transits they step while counting into
// cnt_{s+1}, so no separate clearing pass is needed.
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
constexpr int TW_STAGE_W = 2048;    // staged row bytes per warp
constexpr int TW_STAGE_C = 32 * 1024;  // staged row bytes per CTA
constexpr int TW_PAY = 64;          // stage when row bytes <= members * TW_PAY

struct TwCtl {  // per step (alternating by step parity)
  int nhub, queue, nwarp, nunit, front, wq, uq, pad;
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
  unsigned long long* tier;  // [0] staged hub members stepped, [1] walkers stepped in place
  unsigned long long* hubs_seen;  // hubs the prep kernels have classed (all steps)
  TwCtl* reset_self;    // staged tiers off: the sampling kernel's last CTA zeroes its own
                        // step control (the next-but-one step's), no prep launch needed
  unsigned int* done;   // CTAs finished (last-CTA detection; reset by the last one)
  int no_hub_list;      // staged tiers off for good: skip the hub list appends
  int32_t* out;         // [Lw, rows]
  int32_t* nnz;         // per row: non-NULL values of the window
  int32_t* died;        // per walker: ended with a NULL
  int32_t* cont_wid;
  int32_t* cont_v;
  int32_t* cont_t;
  int* cont_n;
  int* max_len;
  // this step's groups (counted by the previous step's emission)
  TwCtl* ctl;
  int32_t* cnt;         // member counts (cleared by this step's sampling)
  int32_t* vhub;        // staged hub's first member slot, -1 grid tier (valid while cnt >= TW_TM)
  int32_t* hubs;
  // the next step's, counted by this step's emission
  TwCtl* nctl;          // (reset by prep)
  int32_t* ncnt;
  int32_t* nhubs;
  unsigned long long* nstats;
  TwRec* hrec;          // hub members in group order
  int64_t hcap;         // member slots
  TwUnit* wunits;
  TwUnit* cunits;
  // k_tw_multi (staged tiers off): K steps per launch, step j's member counts
  // in kcnt + j * V (zeroed before the launch), rows claimed from *kqueue
  int32_t* kcnt;
  int64_t kV;
  int* kqueue;
  int K;
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

// ---- member counting ------------------------------------------------------------
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

// A walker counted at vertex o of the next step (the emission's atomicAdd
// on ncnt[o]; its result is consumed after the lane's next pick, so the
// atomic's latency hides behind that pick's loads).  The returned old count is
// the walker's position in its group; +1 crossings of 0, 32 and 1025 members
// give the group count, the medium / large class counts and the hub list,
// exactly.
struct TwPend {
  bool on = false;
  int32_t o = 0, old = 0;
  int64_t row = 0;
};

__device__ __forceinline__ void tw_count_issue(const TwArgs& A, TwPend& p, bool live, int32_t o,
                                               int64_t row) {
  if (live) {
    p.on = true;
    p.o = o;
    p.row = row;
    p.old = atomicAdd(A.ncnt + o, 1);
  }
}

// warp-uniform call
__device__ __forceinline__ void tw_count_take(const TwArgs& A, TwPend& p, TwCounts& cc) {
  bool hm = false;
  if (p.on) {
    A.pos[p.row] = p.old;
    cc.ng += p.old == 0;
    hm = p.old == TW_TM - 1;
    cc.nm += hm;
    cc.nl += p.old == TW_TL - 1;
  }
  // the hub list feeds the prep kernel only: with the staged tiers off it is
  // not built (its single counter is the most contended address of a step)
  if (!A.no_hub_list) {
    const int idx = tw_warp_append(hm, &A.nctl->nhub);  // a group becomes a hub
    if (hm) A.nhubs[idx] = p.o;
  }
  p.on = false;
}

// per-warp class deltas (a walker can cross a threshold of a group another
// warp opened: the signed deltas sum to the exact counts over the grid)
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

// ---- prep: hub tiers and member slots (one thread per hub) --------------------
// A hub's members read its record row; staging pays when the row is at most
// TW_PAY bytes per member.  Tiers:
//   warp   <= TW_WARP_MAX members, row <= TW_STAGE_W bytes: one warp, staged;
//   CTA    row <= TW_STAGE_C bytes: units of <= TW_UNIT members, one CTA each,
//          staged;
//   grid   rows too large to stage (or not worth it): the members of every
//          such hub spread over the whole grid, rows read from global memory.
// Member slots: disjoint ranges reserved with warp-aggregated atomics for the
// staged tiers; the grid tier needs none (its members are stepped where the
// sampling kernel meets them, each carrying its own row header).
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
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *A.nctl = TwCtl{};
    if (H) atomicAdd(A.hubs_seen, (unsigned long long)H);
  }
  for (int jb = blockIdx.x * blockDim.x; jb < H; jb += gridDim.x * blockDim.x) {
    const int j = jb + threadIdx.x;
    int32_t v = -1, c = 0, t = 2, nu = 0;
    if (j < H) {
      v = A.hubs[j];
      // the hub's members past its first TW_TM are staged (the first ones are
      // stepped in place by the sampling kernel, which reads no count)
      c = A.cnt[v] - TW_TM;
      const int64_t r0 = __ldg(A.P.gv.row + v), r1 = __ldg(A.P.gv.row + v + 1);
      t = c > 0 ? tw_tier(c, tw_rbytes(A.rmode, r1 - r0)) : 2;
      if (t == 1) nu = (c + TW_UNIT - 1) / TW_UNIT;
    }
    const int m0 = tw_warp_reserve(t < 2 ? c : 0, &A.ctl->front);
    const int wu = tw_warp_reserve(t == 0 ? 1 : 0, &A.ctl->nwarp);
    const int cu = tw_warp_reserve(nu, &A.ctl->nunit);
    if (j < H) {
      // the sampling kernel reads vhub of a hub member's transit: the staged
      // hub's first member slot, or -1 (grid tier: stepped in place)
      A.vhub[v] = t < 2 ? m0 : -1;
      if (t == 0) A.wunits[wu] = TwUnit{v, m0, m0 + c, j};
      for (int q = 0; q < nu; q++)
        A.cunits[cu + q] = TwUnit{v, m0 + q * TW_UNIT, m0 + min(c, (q + 1) * TW_UNIT), j};
    }
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
__device__ __forceinline__ bool tw_work(const TwArgs& A, bool tries, TwLane& L,
                                        const unsigned char* srec, uint64_t base0, int64_t& o,
                                        NextHdr& nh, ItemStats& st) {
  const PWArgs& P = A.P;
  if (L.deg <= 0) {
    o = -1;
    return true;
  }
  if (tries) {
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
                                        const NextHdr& nh, int& mlen, ItemStats& st, TwPend& pd) {
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
      tw_count_issue(A, pd, true, (int32_t)o, L.row);
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

__device__ __forceinline__ void tw_flush_tier(unsigned long long n, unsigned long long* dst) {
  for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(dst, n);
}

__device__ __forceinline__ void tw_lane_start(const TwArgs& A, TwLane& L, ItemStats& st) {
  L.j = 0;
  L.ik = key_item((uint64_t)(A.P.sample_lo + L.w), 0, 0);
  st.bytes += SECTOR + 8;  // §8(d) pair term: offsets pair + transit id
}

// lane state of a hub member record (48 bytes); the group's first member
// a staged hub member's record into a lane
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
  tw_lane_start(A, L, st);
}

// Persistent lane loop over N work items: `load(i, L)` fills a lane from item
// i (false: nothing to sample, the lane takes the next item); lanes refill
// from a warp-claimed chunk of a global queue as their walker decides
// (node2vec's rejection tries keep every lane busy).
template <bool SH, class Load>
__device__ __forceinline__ void tw_lanes(const TwArgs& A, int64_t N, int* queue, int chunk,
                                         const unsigned char* srec, Load load, ItemStats& st,
                                         int& mlen) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1;
  const uint64_t base0 = key_base(A.P.seed, (uint64_t)A.s, 0, 0);
  TwLane L;
  TwPend pd;
  TwCounts cc;
  int64_t wbeg = 0, wend = 0, i = -1;
  bool has = false;
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
        if (i < N) {
          has = load(i, L);
          if (!has) i = -1;
        }
      }
      if (rem < c) {
        wbeg = nbeg + (c - rem);
        wend = nbeg + chunk;
      } else {
        wbeg += c;
      }
    }
    if (__all_sync(0xffffffffu, i >= N)) {
      tw_count_take(A, pd, cc);
      break;
    }
    bool fin = false;
    int64_t o = -1;
    NextHdr nh;
    if (has) fin = tw_work<SH>(A, A.tries, L, srec, base0, o, nh, st);
    tw_count_take(A, pd, cc);  // the previous iteration's count, after this one's picks
    tw_emit(A, fin, L, o, nh, mlen, st, pd);
    if (fin) {
      i = -1;
      has = false;
    }
  }
  tw_flush_classes(cc, A.nstats);
}

// ---- small class and grid tier: persistent over the window's rows ---------------
// The sub-warp kernel (m = 1: one lane per member) and the grid kernel (a
// hub's members over the whole grid, its row read from global memory).  A
// lane takes a row: a walker of the small class or of a grid-tier hub is
// stepped right away, a member of a staged hub has its record written at its
// group position for the hub kernel, an ended row is skipped.
template <int MINB>
__global__ void __launch_bounds__(TW_BLOCK, MINB) k_tw_sample(TwArgs A) {
  ItemStats st;
  int mlen = 0;
  unsigned long long inplace = 0;
  tw_lanes<false>(A, A.rows, &A.ctl->queue, A.P.chunk, nullptr,
                  [&](int64_t row, TwLane& L) -> bool {
                    const int32_t v = A.cur[row];
                    if (v < 0) {  // ended earlier in the window
                      A.ncur[row] = -1;
                      return false;
                    }
                    const uint32_t lo = A.lo[row];
                    const int32_t deg = A.deg[row];
                    const double hd = A.hd[row];
                    int32_t t = -1, tdeg = 0;
                    uint32_t tlo = 0;
                    if (A.tries) {
                      t = A.ncur[row];
                      tlo = A.nlo[row];
                      tdeg = A.ndeg[row];
                    }
                    const int32_t w = A.wid ? A.wid[row] : (int32_t)row;
                    // the walker's position in its group (the previous emission's
                    // count): members past the 32nd belong to a hub (its group
                    // reached TW_TM members), the first TW_TM of every group are
                    // stepped here -- no read of the group's count per walker
                    const int32_t p = A.pos[row];
                    if (p >= TW_TM) {
                      const int32_t m0 = A.vhub[v];
                      if (m0 >= 0) {  // staged tier: the record at its staged slot
                        A.hrec[m0 + p - TW_TM] =
                            TwRec{(int32_t)row, w, v, deg, lo, t, tdeg, tlo, hd, p, 0};
                        return false;
                      }
                    }
                    // stepped here (first members, small class, grid tier); the
                    // group's first member clears its count for step s+2 (prep,
                    // the only reader of this step's counts, ran before)
                    if (p == 0) A.cnt[v] = 0;
                    L.row = row;
                    L.w = w;
                    L.v = v;
                    L.lo = lo;
                    L.deg = deg;
                    L.hd = hd;
                    L.t = t;
                    L.tlo = tlo;
                    L.tdeg = tdeg;
                    tw_lane_start(A, L, st);
                    inplace++;
                    return true;
                  },
                  st, mlen);
  flush_stats(st, A.P.ctr);
  tw_flush_len(mlen, A.max_len);
  tw_flush_tier(inplace, A.tier + 1);
  if (A.reset_self) {  // every CTA is past the step's work queue: the last one resets it
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(A.done, 1u) == gridDim.x - 1) {
        *A.reset_self = TwCtl{};
        *A.done = 0;
        __threadfence();
      }
    }
  }
}

// ---- staged tiers off: K steps per launch ----------------------------------------
// When no hub is staged (every member is stepped in place by k_tw_sample; on
// C2 the staged tiers never pay), a step's only TP duty
// besides sampling is its exact class statistics, and those come from the
// count crossings at emission time -- in whatever order the walkers are
// counted.  So K consecutive steps run in one launch with the walker state in
// registers between them (one state round trip per K steps instead of per
// step): step j's landings are counted into their own zeroed array kcnt + j*V
// and its crossings summed per CTA in shared memory, then flushed as signed
// deltas to the statistics of step s+j+1.  No later kernel reads the counts
// (no tier prep), so the host zeroes the arrays before the next launch.
// Rows and statistics equal the one-step launches' (every draw is keyed by
// (walker, step)).
constexpr int TW_KMAX = 8;

template <int MINB>
__global__ void __launch_bounds__(TW_BLOCK, MINB) k_tw_multi(TwArgs A) {
  __shared__ unsigned int scls[TW_KMAX][3];  // per step: groups opened, medium, large
  for (int q = threadIdx.x; q < TW_KMAX * 3; q += blockDim.x) (&scls[0][0])[q] = 0;
  __syncthreads();
  const PWArgs& P = A.P;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1;
  const bool n2v = P.a.code == ND_NODE2VEC;
  const int K = A.K;
  // the state after the launch: buffer parity of step k + K
  int32_t* fcur = (K & 1) ? A.ncur : const_cast<int32_t*>(A.cur);
  uint32_t* flo = (K & 1) ? A.nlo : const_cast<uint32_t*>(A.lo);
  int32_t* fdeg = (K & 1) ? A.ndeg : const_cast<int32_t*>(A.deg);
  double* fhd = (K & 1) ? A.nhd : const_cast<double*>(A.hd);
  int32_t* tcur = (K & 1) ? const_cast<int32_t*>(A.cur) : A.ncur;
  uint32_t* tlo = (K & 1) ? const_cast<uint32_t*>(A.lo) : A.nlo;
  int32_t* tdeg = (K & 1) ? const_cast<int32_t*>(A.deg) : A.ndeg;
  const bool has_last = A.k + K == A.Lw;  // the launch ends the window
  ItemStats st;
  int mlen = 0;
  unsigned long long inplace = 0;
  TwLane L;
  int jj = 0;            // the lane walker's step within the launch
  uint64_t base0 = 0;
  bool pon = false;      // a count whose result is taken one iteration later
  int pold = 0, pj = 0;
  int64_t wbeg = 0, wend = 0, i = -1;
  bool has = false;
  const int64_t N = A.rows;
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
        if (lane == 0) base = atomicAdd(A.kqueue, P.chunk);
        nbeg = __shfl_sync(0xffffffffu, base, 0);
      }
      if (need) {
        i = rank < rem ? wbeg + rank : nbeg + (rank - rem);
        if (i < N) {
          const int64_t row = i;
          const int32_t v = A.cur[row];
          if (v < 0) {  // ended earlier in the window
            if (K & 1) A.ncur[row] = -1;
            has = false;
            i = -1;
          } else {
            L.row = row;
            L.w = A.wid ? A.wid[row] : (int32_t)row;
            L.v = v;
            L.lo = A.lo[row];
            L.deg = A.deg[row];
            L.hd = A.hd[row];
            if (n2v) {
              L.t = A.ncur[row];
              L.tlo = A.nlo[row];
              L.tdeg = A.ndeg[row];
            } else {
              L.t = -1;
            }
            jj = 0;
            base0 = key_base(P.seed, (uint64_t)A.s, 0, 0);
            tw_lane_start(A, L, st);
            has = true;
          }
        }
      }
      if (rem < c) {
        wbeg = nbeg + (c - rem);
        wend = nbeg + P.chunk;
      } else {
        wbeg += c;
      }
    }
    const bool all_done = __all_sync(0xffffffffu, i >= N);
    bool fin = false;
    int64_t o = -1;
    NextHdr nh;
    if (!all_done && has) fin = tw_work<false>(A, n2v && A.s + jj > 0, L, nullptr, base0, o, nh, st);
    if (pon) {  // the previous landing's count: class crossings of its step
      if (pold == 0) atomicAdd(&scls[pj][0], 1u);
      if (pold == TW_TM - 1) atomicAdd(&scls[pj][1], 1u);
      if (pold == TW_TL - 1) atomicAdd(&scls[pj][2], 1u);
      pon = false;
    }
    if (all_done) break;
    bool cont = false;
    if (fin) {
      const int64_t ks = A.k + jj;  // step within the window
      const int64_t row = L.row;
      A.out[ks * A.rows + row] = (int32_t)o;
      mlen = max(mlen, (int)(A.s + jj) + 1);
      inplace++;
      if (o < 0) {
        A.nnz[row] = (int32_t)ks;
        A.died[L.w] = 1;
        fcur[row] = -1;
        i = -1;
        has = false;
      } else if (ks == A.Lw - 1) {
        A.nnz[row] = (int32_t)ks + 1;
        cont = true;
        i = -1;
        has = false;
      } else {
        double nhd = n2v ? nh.mx : nh.tot;
        if (nhd < 0.0) {  // node2vec after its step-0 pick: max weight of the new vertex
          nhd = __ldg(P.gv.mx + o);
          st.sect += 1;
        }
        pold = atomicAdd(A.kcnt + (int64_t)jj * A.kV + o, 1);
        pon = true;
        pj = jj;
        if (jj + 1 == K) {  // the launch's last step: state for the next launch
          fcur[row] = (int32_t)o;
          flo[row] = (uint32_t)nh.lo;
          fdeg[row] = (int32_t)nh.deg;
          fhd[row] = nhd;
          if (n2v) {
            tcur[row] = L.v;
            tlo[row] = (uint32_t)L.lo;
            tdeg[row] = L.deg;
          }
          i = -1;
          has = false;
        } else {  // next step in registers
          L.t = L.v;
          L.tlo = L.lo;
          L.tdeg = L.deg;
          L.v = (int32_t)o;
          L.lo = nh.lo;
          L.deg = (int32_t)nh.deg;
          L.hd = nhd;
          jj++;
          base0 = key_base(P.seed, (uint64_t)(A.s + jj), 0, 0);
          tw_lane_start(A, L, st);
        }
      }
    }
    if (has_last) {
      const int slot = tw_warp_append(cont, A.cont_n);
      if (cont) {
        A.cont_wid[slot] = (int32_t)L.w;
        A.cont_v[slot] = (int32_t)o;
        A.cont_t[slot] = L.v;
      }
    }
  }
  flush_stats(st, P.ctr);
  tw_flush_len(mlen, A.max_len);
  tw_flush_tier(inplace, A.tier + 1);
  __syncthreads();
  if (threadIdx.x < K) {
    const unsigned long long ng = scls[threadIdx.x][0], nm = scls[threadIdx.x][1],
                             nl = scls[threadIdx.x][2];
    unsigned long long* stt = A.nstats + 4 * threadIdx.x;  // statistics of step s + j + 1
    if (ng != nm) atomicAdd(stt + 0, ng - nm);
    if (nm != nl) atomicAdd(stt + 1, nm - nl);
    if (nl) atomicAdd(stt + 2, nl);
    if (ng) atomicAdd(stt + 3, ng);
  }
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
  TwPend pd;
  TwCounts cc;
  unsigned long long staged = 0;
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
        if (mem < d.m1) {
          tw_load_rec(A, L, A.hrec + mem, st);
          staged++;
        } else {
          done = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, L.row < 0 && done)) {
      tw_count_take(A, pd, cc);
      break;
    }
    if (!waited) {
      mbar_wait(bar, parity);
      waited = true;
    }
    bool fin = false;
    int64_t o = -1;
    NextHdr nh;
    if (L.row >= 0) fin = tw_work<true>(A, A.tries, L, srec, base0, o, nh, st);
    tw_count_take(A, pd, cc);
    tw_emit(A, fin, L, o, nh, mlen, st, pd);
    if (fin) L.row = -1;
  }
  if (!waited) mbar_wait(bar, parity);  // keep the barrier's phases in step
  tw_flush_classes(cc, A.nstats);
  tw_flush_tier(staged, A.tier);
}

// ---- hub kernel: thread-block and warp tiers --------------------------------------
// Every CTA first takes thread-block units (the whole CTA on one unit of a
// hub's members, the row staged in the CTA's stage), then each warp takes
// warp-tier hubs (row staged in the warp's stage).
constexpr size_t TW_HUB_HDR = 128;  // barriers and cursors
constexpr size_t TW_HUB_SMEM = TW_HUB_HDR + TW_STAGE_C + (size_t)(TW_BLOCK / 32) * TW_STAGE_W;

template <int MINB>
__global__ void __launch_bounds__(TW_BLOCK, MINB) k_tw_hub(TwArgs A) {
  extern __shared__ __align__(128) unsigned char dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint64_t* cbar = reinterpret_cast<uint64_t*>(dsm);
  uint64_t* wbar = cbar + 1 + wib;
  int* ccur = reinterpret_cast<int*>(dsm + 8 * (1 + TW_BLOCK / 32));
  int* wcur = ccur + 1 + wib;
  int* s_u = ccur + 1 + TW_BLOCK / 32;
  unsigned char* cbuf = dsm + TW_HUB_HDR;
  unsigned char* wbuf = cbuf + TW_STAGE_C + (size_t)wib * TW_STAGE_W;
  if (threadIdx.x == 0) mbar_init(cbar, 1);
  if (lane == 0) mbar_init(wbar, 1);
  if (threadIdx.x == 0) mbar_fence_init();
  __syncthreads();
  ItemStats st;
  int mlen = 0;
  // thread-block tier
  const int U = A.ctl->nunit;
  uint32_t ph = 0;
  while (true) {
    if (threadIdx.x == 0) *s_u = U ? atomicAdd(&A.ctl->uq, 1) : U;
    __syncthreads();
    const int u = *s_u;
    if (u >= U) break;
    const TwUnit d = A.cunits[u];
    if (threadIdx.x == 0) {
      *ccur = 0;
      const TwRec* r0 = A.hrec + d.m0;
      const void* src = nullptr;
      const uint32_t bytes = tw_row_bytes(A, r0->lo, r0->deg, &src);
      mbar_arrive_expect_tx(cbar, bytes);
      bulk_g2s(cbuf, src, bytes, cbar);
    }
    __syncthreads();
    tw_hub_members(A, d, cbuf, cbar, ph, ccur, st, mlen);
    ph ^= 1u;
    __syncthreads();
  }
  // warp tier
  const int W = A.ctl->nwarp;
  uint32_t wph = 0;
  while (true) {
    int u = W;
    if (lane == 0 && W) u = atomicAdd(&A.ctl->wq, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= W) break;
    const TwUnit d = A.wunits[u];
    if (lane == 0) {
      *wcur = 0;
      const TwRec* r0 = A.hrec + d.m0;
      const void* src = nullptr;
      const uint32_t bytes = tw_row_bytes(A, r0->lo, r0->deg, &src);
      mbar_arrive_expect_tx(wbar, bytes);
      bulk_g2s(wbuf, src, bytes, wbar);
    }
    __syncwarp();
    tw_hub_members(A, d, wbuf, wbar, wph, wcur, st, mlen);
    wph ^= 1u;
    __syncwarp();
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

// the window's first step: members counted (into the n* buffers) per row
__global__ void __launch_bounds__(TW_BLOCK) k_tw_count0(TwArgs A) {
  TwCounts cc;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < A.rows; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = b + threadIdx.x;
    TwPend pd;
    if (row < A.rows) tw_count_issue(A, pd, true, A.cur[row], row);
    tw_count_take(A, pd, cc);
  }
  tw_flush_classes(cc, A.nstats);
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


}  // namespace
