// nd_common.cuh — shared device primitives for the NextDoor B200 engine.
//
// Keyed counter RNG (bit-identical to trawl/rng.py:43-77 and
// _ckernels.pyx:38-62), exact weighted pick / membership searches
// (_ckernels.pyx:65-100), the device CSR layout, status codes and the
// stream-ordered allocator helpers used by every translation unit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nextdoor_b200.h"

namespace nd {

// ---- RNG constants (rng.py:22-30) -----------------------------------------
constexpr uint64_t C_SAMPLE = 0x9E3779B97F4A7C15ull;
constexpr uint64_t C_STEP = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t C_TRANSIT = 0x165667B19E3779F9ull;
constexpr uint64_t C_SLOT = 0x27D4EB2F165667C5ull;
constexpr uint64_t C_DOMAIN = 0x85EBCA77C2B2AE63ull;
constexpr uint64_t C_DRAW = 0xD6E8FEB86659FD93ull;
constexpr uint64_t MIX_A = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t MIX_B = 0x94D049BB133111EBull;

constexpr int32_t NULLV = -1;
constexpr int64_t N2V_MAX_TRIES = 1000000;   // apps.py:35
constexpr int64_t SMALL_MAX_WORK = 32;       // transit_parallel.py:37
constexpr int64_t LARGE_MIN_WORK = 1024;     // transit_parallel.py:38

__host__ __device__ __forceinline__ uint64_t fin64(uint64_t z) {
  z = (z ^ (z >> 30)) * MIX_A;
  z = (z ^ (z >> 27)) * MIX_B;
  return z ^ (z >> 31);
}

// Step/domain/draw part of the Weyl key (seed + C_STEP(step+1) +
// C_DOMAIN(dom+1) + C_DRAW(draw+1)); _ckernels.pyx:56-58.
__host__ __device__ __forceinline__ uint64_t key_base(uint64_t seed, uint64_t step,
                                                      uint64_t domain, uint64_t draw) {
  return seed + C_STEP * (step + 1) + C_DOMAIN * (domain + 1) + C_DRAW * (draw + 1);
}

// Per-item part (sample, transit index, slot); _ckernels.pyx:47-53.
__host__ __device__ __forceinline__ uint64_t key_item(uint64_t sid, uint64_t tix, uint64_t slot) {
  return C_SAMPLE * (sid + 1) + C_TRANSIT * (tix + 1) + C_SLOT * (slot + 1);
}

__host__ __device__ __forceinline__ uint64_t draw_u64(uint64_t base, uint64_t item) {
  return fin64(fin64(base + item));
}

// (u >> 11) * 2^-53, exact (rng.py:74-77)
__device__ __forceinline__ double to_unit(uint64_t u) {
  return __ull2double_rn(u >> 11) * (1.0 / 9007199254740992.0);
}

// Exact u % d (the reference's uint64 modulo, _ckernels.pyx:222) without the
// ~70-instruction 64-bit division routine: for d < 2^32 two fp64 quotient
// estimates (hi word, then the 64-bit remainder-extended low word), each off by
// at most one and corrected exactly.  Fuzzed against `%` in tests/test_gpu_kernels.py.
__device__ __forceinline__ uint64_t mod_u64(uint64_t u, uint64_t d) {
  if (d > 0xFFFFFFFFull) return u % d;
  const double inv = __drcp_rn((double)d);
  const int64_t sd = (int64_t)d;
  uint64_t hi = u >> 32;
  uint64_t q1 = (uint64_t)__dmul_rz(__ull2double_rn(hi), inv);
  int64_t r1 = (int64_t)(hi - q1 * d);
  if (r1 < 0) r1 += sd; else if (r1 >= sd) r1 -= sd;
  uint64_t x = ((uint64_t)r1 << 32) | (u & 0xFFFFFFFFull);
  uint64_t q2 = (uint64_t)__dmul_rz(__ull2double_rn(x), inv);
  int64_t r2 = (int64_t)(x - q2 * d);
  if (r2 < 0) r2 += sd; else if (r2 >= sd) r2 -= sd;
  return (uint64_t)r2;
}

// Division by a run-constant 32-bit divisor d >= 1 for numerators < 2^32
// (round-up multiplier method): q = (umulhi(x, m) + x) >> l, exact.
struct FastDiv {
  uint32_t d = 1, m = 0;
  int l = 0;
  FastDiv() = default;
  __host__ explicit FastDiv(uint32_t dv) : d(dv) {
    while ((1ull << l) < d) l++;
    m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    return (uint32_t)(((uint64_t)__umulhi(x, m) + x) >> l);
  }
};

// Exact u % d for a run-constant divisor d >= 1 (a hub's degree): with
// M = floor((2^64-1)/d) >= 2^64/d - 1, q = umulhi(u, M) satisfies
// u/d - 1 < q <= u/d, so one conditional subtraction gives the remainder.
struct ModU64 {
  uint64_t d = 1, M = ~0ull;
  ModU64() = default;
  __host__ __device__ explicit ModU64(uint64_t dv) : d(dv), M(dv ? ~0ull / dv : 0) {}
  __device__ __forceinline__ uint64_t mod(uint64_t u) const {
    const uint64_t q = __umul64hi(u, M);
    const uint64_t r = u - q * d;
    return r >= d ? r - d : r;
  }
};

// one 32-byte load (LDG.E.256): a whole record / hash-set chunk per request
__device__ __forceinline__ void ld32B(const void* p, int4& lo, int4& hi) {
  unsigned long long a, b, c, d;
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  lo = make_int4((int)(uint32_t)a, (int)(uint32_t)(a >> 32), (int)(uint32_t)b, (int)(uint32_t)(b >> 32));
  hi = make_int4((int)(uint32_t)c, (int)(uint32_t)(c >> 32), (int)(uint32_t)d, (int)(uint32_t)(d >> 32));
}

// ---- device CSR -------------------------------------------------------------
// Layout in HBM: int64 row offsets, int32 column ids (V <
// 2^31), f64 weights / inclusive per-row prefix / per-row max.  Unit-weight
// graphs keep neither weights nor prefix: the upper-bound search over the
// integer prefix 1..deg reduces exactly to floor(r*deg).
// Optional exact indexes (built on first use, see nd_index.cu):
//   hset  — per-row open-addressing hash set of the row's neighbours, table of
//           next_pow2(2*deg) int32 slots at offset 4*row[v] (rows with
//           deg > HASH_MIN_DEG); answers has_edge (node2vec) in ~1 probe.
//   guide — per-row guide table of deg int32 entries at offset row[v]:
//           guide[j] = upper_bound(prefix row, j*(total/deg)) (rows with
//           deg > GUIDE_MIN_DEG); narrows the inverse-CDF search to ~3 entries.
// Both return exactly what the reference's binary searches return.
constexpr int64_t HASH_MIN_DEG = 0;  // every non-empty row (the table space is allocated anyway)
constexpr int64_t GUIDE_MIN_DEG = 4;

// Packed records for the walker-major kernels: the fields one step reads
// together share one 32-byte sector.
struct __align__(32) VRec {   // per vertex
  int64_t lo;                 // row start
  int64_t deg;
  double mx;                  // per-row max weight (node2vec envelope)
  double total;               // prefix[hi-1] (weighted pick); deg for unit rows
};
// Neighbour records for the walker-major kernel: each edge record also
// carries its destination's row header, so the record that selects the next
// vertex delivers that vertex's header in the same sector (no separate
// vertex-record load per step).
struct __align__(32) NbrW {   // node2vec try: neighbour, its weight, its header
  int32_t col;
  int32_t deg;
  int64_t lo;
  double w;
  double mx;
};
struct __align__(32) NbrP {   // weighted pick: prefix, neighbour, its header
  double pre;
  int32_t col;
  int32_t deg;
  int64_t lo;
  double total;
};
struct __align__(16) NbrU {   // unit-weight graphs: neighbour + its header
  int32_t col;
  int32_t deg;
  int64_t lo;
};

// Line-packed weighted-pick rows (DeepWalk / PPR).  A random read pulls a
// 128-byte line from HBM anyway, so each line carries three consecutive pick
// records of a row AND the guide entries of those three buckets (plus the
// next bucket's): the exact-bucket bracket and the records around it are
// usually in the line the bucket lands in.  Rows start on a line boundary
// (vline[v] = first line of v).
struct __align__(32) PickRec {
  double pre;     // inclusive prefix of this edge
  double total;   // prefix total of col's row (its pick target scale)
  int32_t col;
  int32_t deg;    // col's degree
  int32_t llo;    // col's first line
  int32_t pad;
};
struct __align__(128) PickLine {
  PickRec r[3];   // edges 3L .. 3L+2 of the row (+inf prefix past its end)
  int32_t g[4];   // guide[3L .. 3L+3] (deg past the row's end)
  int32_t spare[4];
};

struct DevGraph {
  int64_t V = 0, E = 0;
  const int64_t* row = nullptr;
  const int32_t* col = nullptr;
  const double* w = nullptr;     // null when unit
  const double* pre = nullptr;   // null when unit
  const double* mx = nullptr;
  const int32_t* hset = nullptr;  // optional, 4E slots
  const int32_t* guide = nullptr; // optional, E entries
  const VRec* vrec = nullptr;     // optional packed vertex records
  const NbrW* nbw = nullptr;      // optional neighbour records (node2vec tries)
  const NbrP* nbp = nullptr;      // optional neighbour records (weighted picks)
  const NbrU* nbu = nullptr;      // optional neighbour records (unit graphs)
  const PickLine* pl = nullptr;   // optional line-packed pick rows (weighted graphs)
  const int32_t* vline = nullptr; // [V] first line of each row (with pl)
  int unit = 0;
};

__host__ __device__ __forceinline__ int64_t hset_size(int64_t deg) {
  // next_pow2(2*deg) <= 4*deg
  int64_t t = 1;
  while (t < 2 * deg) t <<= 1;
  return t;
}

__device__ __forceinline__ uint32_t hset_hash(uint32_t u) { return u * 0x9E3779B1u; }

// first index in [lo, hi) with a[i] > x (upper bound; _ckernels.pyx:65-74)
__device__ __forceinline__ int64_t upper_bound_f64(const double* __restrict__ a, int64_t lo,
                                                   int64_t hi, double x) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// lower-bound membership over a sorted int32 row (_ckernels.pyx:77-87)
__device__ __forceinline__ bool row_contains(const int32_t* __restrict__ a, int64_t lo, int64_t hi,
                                             int32_t t) {
  int64_t end = hi;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < t) lo = mid + 1; else hi = mid;
  }
  return lo < end && __ldg(a + lo) == t;
}

// Weighted pick (_ckernels.pyx:90-100): idx = upper_bound(prefix, r*total),
// clamped to the last entry.  Unit weights: prefix[lo+k] = k+1 exactly, so the
// first entry > r*deg is floor(r*deg).
__device__ __forceinline__ int64_t weighted_index(const DevGraph& g, int64_t lo, int64_t deg,
                                                  double r) {
  if (g.unit) {
    double x = __dmul_rn(r, (double)deg);
    int64_t k = (int64_t)x;  // x >= 0, floor
    return lo + (k < deg - 1 ? k : deg - 1);
  }
  double total = __ldg(g.pre + lo + deg - 1);
  int64_t idx = upper_bound_f64(g.pre, lo, lo + deg, __dmul_rn(r, total));
  return idx < lo + deg - 1 ? idx : lo + deg - 1;
}

}  // namespace nd

// ---- error plumbing -----------------------------------------------------------
#define ND_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) {                                \
      nd_set_last_error(cudaGetErrorString(_e), __FILE__, __LINE__); \
      return ND_ERR_CUDA;                                   \
    }                                                       \
  } while (0)

#define ND_TRY(expr)                  \
  do {                                \
    int _rc = (expr);                 \
    if (_rc != ND_OK) return _rc;     \
  } while (0)

void nd_set_last_error(const char* msg, const char* file, int line);
// host-side phase trace (ND_TRACE=1): prints milliseconds since the previous mark
void nd_trace(const char* what);

// stream-ordered scratch allocation (cudaMallocAsync from the device pool)
template <typename T>
inline cudaError_t nd_alloc(T** p, size_t n, cudaStream_t s) {
  return cudaMallocAsync((void**)p, (n ? n : 1) * sizeof(T), s);
}
inline void nd_free(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

// column array entries to allocate: a multiple of 4 plus 4 of slack, so the
// 16-byte-aligned superset of any row (nd_bulk.cuh row_span) is inside it
inline int64_t nd_col_alloc(int64_t E) { return ((E + 3) & ~(int64_t)3) + 4; }

inline int nd_grid(int64_t n, int block, int cap = 148 * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}
