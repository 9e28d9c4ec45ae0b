// nd_ingest.cu — edge-list ingestion on device.
//
// The reference parses edge lists line by line in Python (load_edge_list,
// graph.py:132-188) and builds the CSR with a host lexsort (from_edges,
// graph.py:107-129): minutes for a billion-edge file.  Here the raw bytes go
// to HBM once and the whole parse is data-parallel:
//
//   1. line split with Python's universal newlines ("\n", "\r\n", lone "\r"),
//      1-based line numbers as enumerate(fh, start=1) assigns them;
//   2. one thread per line: strip, '#' comments, whitespace split into 2 or 3
//      fields, int(field) for the ids (sign, digits, PEP 515 underscores),
//      float(field) for a weight (Clinger's exact fast path: <= 19 significant
//      digits, mantissa <= 2^53, |exp10| <= 22; inf/nan), or the keyed default
//      weight lo + (hi - lo) * key_uniform(seed, line_no, domain 3) without FMA;
//   3. lines the device cannot decide bit-exactly (non-ASCII bytes, long
//      mantissas, ids >= 2^63) are listed for the host, which parses exactly
//      those lines with the reference's own rules and patches their values;
//      malformed lines report their first line number (the host re-parses that
//      line for the reference's exact message);
//   4. edges in line order (undirected lines emit (s, d), (d, s)), ids
//      compacted onto [0, n) through a device sort + unique (the remap), then
//      the device from_edges build (stable by (src, dst)).
#include <cub/cub.cuh>

#include <vector>

#include "nd_internal.h"

using namespace nd;

int nd_build_from_edges_dev(const int64_t* src, const int64_t* dst, const double* w, int64_t E,
                            int64_t V, cudaStream_t s, nd_graph** out);

struct nd_text {
  int64_t n_lines = 0;
  int64_t* start = nullptr;   // [n_lines] content start byte
  int64_t* end = nullptr;     // [n_lines] content end byte (terminator excluded)
  uint8_t* kind = nullptr;    // [n_lines] 0 skip, 1 edge, 2 error, 3 host
  uint8_t* code = nullptr;    // [n_lines] error code (kind 2)
  int64_t* src = nullptr;     // [n_lines]
  int64_t* dst = nullptr;
  double* w = nullptr;
  int64_t* remap = nullptr;   // [V] after finish
  int64_t V = 0;
  int weighted = 0;
  cudaStream_t stream = nullptr;
};

namespace {

enum : int { K_SKIP = 0, K_EDGE = 1, K_ERR = 2, K_HOST = 3 };
// error codes (the host re-parses the line for the reference's message)
enum : int { E_FIELDS = 1, E_BAD_ID = 2, E_NEG_ID = 3, E_BAD_W = 4, E_NEG_W = 5 };

__device__ __forceinline__ bool py_space(uint8_t c) {  // ASCII str.isspace()
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

// line ends: '\n', or '\r' not followed by '\n'
__global__ void k_line_ends(const uint8_t* __restrict__ t, int64_t n, uint8_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t c = t[i];
    f[i] = c == '\n' || (c == '\r' && (i + 1 == n || t[i + 1] != '\n'));
  }
}

__global__ void k_line_bounds(const uint8_t* __restrict__ t, const int64_t* __restrict__ ends,
                              int64_t n_ends, int64_t n, int64_t n_lines,
                              int64_t* __restrict__ start, int64_t* __restrict__ end) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_lines;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = k == 0 ? 0 : ends[k - 1] + 1;
    int64_t b = k < n_ends ? ends[k] : n;  // the unterminated last line
    if (k < n_ends && t[b] == '\n' && b > a && t[b - 1] == '\r') b--;  // "\r\n"
    start[k] = a;
    end[k] = b;
  }
}

// int(field): [sign] digit (["_"] digit)*  ->  0 ok, 1 malformed, 2 >= 2^63 (host)
__device__ int parse_int(const uint8_t* t, int64_t a, int64_t b, int64_t& out) {
  bool neg = false;
  if (a < b && (t[a] == '+' || t[a] == '-')) { neg = t[a] == '-'; a++; }
  if (a >= b) return 1;
  uint64_t v = 0;
  bool big = false, prev_digit = false;
  for (int64_t i = a; i < b; i++) {
    const uint8_t c = t[i];
    if (c >= '0' && c <= '9') {
      if (v > (0x7FFFFFFFFFFFFFFFull - (c - '0')) / 10) big = true;
      else v = v * 10 + (c - '0');
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < b && t[i + 1] >= '0' && t[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return 1;
    }
  }
  if (big) return 2;
  out = neg ? -(int64_t)v : (int64_t)v;
  return 0;
}

__device__ __forceinline__ bool ieq(const uint8_t* t, int64_t a, int64_t b, const char* s) {
  int64_t i = a;
  for (; *s; s++, i++) {
    if (i >= b) return false;
    uint8_t c = t[i];
    if (c >= 'A' && c <= 'Z') c += 32;
    if (c != (uint8_t)*s) return false;
  }
  return i == b;
}

// float(field), Python's grammar over ASCII; 0 ok, 1 malformed, 2 host (inexact
// fast path).  Clinger: m <= 2^53 and |e| <= 22 -> one correctly rounded op.
__device__ int parse_float(const uint8_t* t, int64_t a, int64_t b, double& out) {
  bool neg = false;
  if (a < b && (t[a] == '+' || t[a] == '-')) { neg = t[a] == '-'; a++; }
  if (a >= b) return 1;
  if (ieq(t, a, b, "inf") || ieq(t, a, b, "infinity")) {
    out = neg ? -__longlong_as_double(0x7FF0000000000000ll) : __longlong_as_double(0x7FF0000000000000ll);
    return 0;
  }
  if (ieq(t, a, b, "nan")) {  // CPython: negate ? -Py_NAN : Py_NAN
    out = __longlong_as_double(neg ? (long long)0xFFF8000000000000ull : 0x7FF8000000000000ll);
    return 0;
  }
  uint64_t m = 0;
  int sig = 0;        // significant digits accumulated into m
  int frac = 0;       // digits after the point that went into m
  int dropped = 0;    // integer-part digits beyond 19 (host)
  int n_int = 0, n_frac = 0;
  int64_t i = a;
  bool prev_digit = false;
  // integer digitpart
  for (; i < b; i++) {
    const uint8_t c = t[i];
    if (c >= '0' && c <= '9') {
      if (m == 0 && c == '0') {
      } else if (sig < 19) { m = m * 10 + (c - '0'); sig++; }
      else dropped++;
      n_int++;
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < b && t[i + 1] >= '0' && t[i + 1] <= '9') {
      prev_digit = false;
    } else {
      break;
    }
  }
  if (i < b && t[i] == '.') {
    i++;
    prev_digit = false;
    for (; i < b; i++) {
      const uint8_t c = t[i];
      if (c >= '0' && c <= '9') {
        if (m == 0 && c == '0') frac++;
        else if (sig < 19) { m = m * 10 + (c - '0'); sig++; frac++; }
        else dropped = dropped > 0 ? dropped : -1;  // fraction digits beyond 19: inexact
        n_frac++;
        prev_digit = true;
      } else if (c == '_' && prev_digit && i + 1 < b && t[i + 1] >= '0' && t[i + 1] <= '9') {
        prev_digit = false;
      } else {
        break;
      }
    }
  }
  if (n_int == 0 && n_frac == 0) return 1;  // "." or sign alone
  int64_t e = 0;
  if (i < b && (t[i] == 'e' || t[i] == 'E')) {
    i++;
    bool eneg = false;
    if (i < b && (t[i] == '+' || t[i] == '-')) { eneg = t[i] == '-'; i++; }
    if (i >= b) return 1;
    int n_exp = 0;
    prev_digit = false;
    for (; i < b; i++) {
      const uint8_t c = t[i];
      if (c >= '0' && c <= '9') {
        if (e < 100000) e = e * 10 + (c - '0');
        n_exp++;
        prev_digit = true;
      } else if (c == '_' && prev_digit && i + 1 < b && t[i + 1] >= '0' && t[i + 1] <= '9') {
        prev_digit = false;
      } else {
        return 1;
      }
    }
    if (n_exp == 0) return 1;
    if (eneg) e = -e;
  }
  if (i != b) return 1;
  if (m == 0) {  // every digit zero (any exponent)
    out = neg ? -0.0 : 0.0;
    return 0;
  }
  if (dropped != 0) return 2;
  const int64_t e10 = e - frac;
  if (m > (1ull << 53) || e10 > 22 || e10 < -22) return 2;
  const double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                          1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
  const double dm = (double)m;  // exact: m <= 2^53
  double v = e10 >= 0 ? __dmul_rn(dm, p10[e10]) : __ddiv_rn(dm, p10[-e10]);
  out = neg ? -v : v;
  return 0;
}

__global__ void k_parse_lines(const uint8_t* __restrict__ t, int64_t n_lines,
                              const int64_t* __restrict__ start, const int64_t* __restrict__ end,
                              int weighted, double lo_w, double span_w, uint64_t wbase,
                              uint8_t* __restrict__ kind, uint8_t* __restrict__ code,
                              int64_t* __restrict__ src, int64_t* __restrict__ dst,
                              double* __restrict__ w, unsigned long long* __restrict__ first_err,
                              unsigned long long* __restrict__ n_host) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_lines;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = start[k], b = end[k];
    uint8_t kd = K_SKIP, cd = 0;
    bool ascii = true;
    for (int64_t i = a; i < b; i++)
      if (t[i] >= 0x80) { ascii = false; break; }
    // strip (raw.strip(): the terminator is already excluded)
    while (a < b && py_space(t[a])) a++;
    while (b > a && py_space(t[b - 1])) b--;
    int64_t s = 0, d = 0;
    double we = 1.0;
    if (!ascii) {
      kd = K_HOST;
    } else if (a < b && t[a] != '#') {
      int64_t fa[3], fb[3];
      int nf = 0;
      for (int64_t i = a; i < b;) {
        while (i < b && py_space(t[i])) i++;
        if (i >= b) break;
        const int64_t f0 = i;
        while (i < b && !py_space(t[i])) i++;
        if (nf < 3) { fa[nf] = f0; fb[nf] = i; }
        nf++;
      }
      if (nf != 2 && nf != 3) {
        kd = K_ERR; cd = E_FIELDS;
      } else {
        const int r0 = parse_int(t, fa[0], fb[0], s);
        const int r1 = r0 == 0 ? parse_int(t, fa[1], fb[1], d) : 0;
        if (r0 == 1 || (r0 == 0 && r1 == 1)) { kd = K_ERR; cd = E_BAD_ID; }
        else if (r0 == 2 || r1 == 2) kd = K_HOST;
        else if (s < 0 || d < 0) { kd = K_ERR; cd = E_NEG_ID; }
        else {
          kd = K_EDGE;
          if (weighted) {
            if (nf == 3) {
              const int rw = parse_float(t, fa[2], fb[2], we);
              if (rw == 1) { kd = K_ERR; cd = E_BAD_W; }
              else if (rw == 2) kd = K_HOST;
              else if (we < 0.0) { kd = K_ERR; cd = E_NEG_W; }
            } else {  // lo + (hi - lo) * key_uniform(seed, sample_id=line_no, domain=3)
              const double u = to_unit(draw_u64(wbase, key_item((uint64_t)(k + 1), 0, 0)));
              we = __dadd_rn(lo_w, __dmul_rn(span_w, u));
            }
          }
        }
      }
    }
    kind[k] = kd;
    code[k] = cd;
    src[k] = s;
    dst[k] = d;
    w[k] = we;
    if (kd == K_ERR) atomicMin(first_err, (unsigned long long)(k + 1));
    if (kd == K_HOST) atomicAdd(n_host, 1ull);
  }
}

__global__ void k_host_list(const uint8_t* __restrict__ kind, int64_t n_lines,
                            const int64_t* __restrict__ pos, int64_t* __restrict__ lines) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_lines;
       k += (int64_t)gridDim.x * blockDim.x)
    if (kind[k] == K_HOST) lines[pos[k]] = k;
}

struct U8ToI64 {
  __device__ __forceinline__ int64_t operator()(uint8_t f) const { return f; }
};
struct IsHost {
  __device__ __forceinline__ int64_t operator()(uint8_t k) const { return k == K_HOST ? 1 : 0; }
};
struct IsEdge {
  __device__ __forceinline__ int64_t operator()(uint8_t k) const { return k == K_EDGE ? 1 : 0; }
};

__global__ void k_apply_patches(const int64_t* __restrict__ line, const int64_t* __restrict__ ps,
                                const int64_t* __restrict__ pd, const double* __restrict__ pw,
                                const uint8_t* __restrict__ pk, int64_t np, uint8_t* __restrict__ kind,
                                int64_t* __restrict__ src, int64_t* __restrict__ dst,
                                double* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = line[i];
    kind[k] = pk[i];
    src[k] = ps[i];
    dst[k] = pd[i];
    w[k] = pw[i];
  }
}

// edges in line order; undirected lines emit (s, d) then (d, s)
__global__ void k_emit_edges(const uint8_t* __restrict__ kind, int64_t n_lines,
                             const int64_t* __restrict__ pos, const int64_t* __restrict__ src,
                             const int64_t* __restrict__ dst, const double* __restrict__ w,
                             int undirected, int64_t* __restrict__ es, int64_t* __restrict__ ed,
                             double* __restrict__ ew, int64_t* __restrict__ ids) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_lines;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (kind[k] != K_EDGE) continue;
    const int64_t p = pos[k] * (undirected ? 2 : 1);
    es[p] = src[k]; ed[p] = dst[k];
    if (ew) ew[p] = w[k];
    if (undirected) {
      es[p + 1] = dst[k]; ed[p + 1] = src[k];
      if (ew) ew[p + 1] = w[k];
    }
    ids[2 * pos[k]] = src[k];
    ids[2 * pos[k] + 1] = dst[k];
  }
}

// searchsorted(original, x) over the sorted unique ids
__global__ void k_compact_ids(const int64_t* __restrict__ uniq, int64_t V, int64_t* __restrict__ a,
                              int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = a[i];
    int64_t lo = 0, hi = V;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (uniq[mid] < x) lo = mid + 1; else hi = mid;
    }
    a[i] = lo;
  }
}

template <class Op>
int scan_op(const uint8_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  cub::TransformInputIterator<int64_t, Op, const uint8_t*> it(in, Op());
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, it, out, n, s);
  void* tmp = nullptr;
  ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
  ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, it, out, n, s));
  nd_free(tmp, s);
  return ND_OK;
}

}  // namespace

extern "C" int nd_text_destroy(nd_text* T);

static int text_parse(const char* host_text, const char* dev_text, int64_t n_bytes, int weighted,
                      double lo_w, double hi_w, uint64_t seed, void* stream, nd_text** out,
                      int64_t* host_info) {
  if (!out || !host_info || n_bytes < 0 || (n_bytes > 0 && !host_text && !dev_text))
    return ND_ERR_ARG;
  nd_pool_init();
  cudaStream_t s = (cudaStream_t)stream;
  nd_text* T = new nd_text();
  T->weighted = weighted;
  T->stream = s;
  uint8_t *text = nullptr, *flags = nullptr;
  int64_t* ends = nullptr;
  int64_t* n_ends_d = nullptr;
  unsigned long long* ctl = nullptr;  // [0] first error line (1-based), [1] host lines
  int64_t h[2] = {0, 0};
  auto fail = [&](int rc) {
    nd_free(text, s); nd_free(flags, s); nd_free(ends, s); nd_free(n_ends_d, s); nd_free(ctl, s);
    cudaStreamSynchronize(s);
    nd_text_destroy(T);
    return rc;
  };
  if ((!dev_text && nd_alloc(&text, n_bytes + 1, s)) || nd_alloc(&flags, n_bytes + 1, s) ||
      nd_alloc(&n_ends_d, 1, s) || nd_alloc(&ctl, 2, s))
    return fail(ND_ERR_NOMEM);
  if (n_bytes && !dev_text) cudaMemcpyAsync(text, host_text, n_bytes, cudaMemcpyHostToDevice, s);
  const uint8_t* tx = dev_text ? reinterpret_cast<const uint8_t*>(dev_text) : text;
  int64_t n_ends = 0, last_end = -1;
  if (n_bytes) {
    // count the terminators, then list their positions (no n_bytes-sized index array)
    k_line_ends<<<nd_grid(n_bytes, 256, 148 * 32), 256, 0, s>>>(tx, n_bytes, flags);
    cub::TransformInputIterator<int64_t, U8ToI64, const uint8_t*> fl(flags, U8ToI64());
    size_t tb = 0;
    cub::DeviceReduce::Sum(nullptr, tb, fl, n_ends_d, n_bytes, s);
    void* tmp = nullptr;
    if (nd_alloc((char**)&tmp, tb, s)) return fail(ND_ERR_NOMEM);
    cub::DeviceReduce::Sum(tmp, tb, fl, n_ends_d, n_bytes, s);
    nd_free(tmp, s);
    cudaMemcpyAsync(&n_ends, n_ends_d, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return fail(ND_ERR_CUDA);
    if (nd_alloc(&ends, n_ends > 0 ? n_ends : 1, s)) return fail(ND_ERR_NOMEM);
    if (n_ends) {
      cub::CountingInputIterator<int64_t> idx(0);
      tb = 0;
      cub::DeviceSelect::Flagged(nullptr, tb, idx, flags, ends, n_ends_d, n_bytes, s);
      if (nd_alloc((char**)&tmp, tb, s)) return fail(ND_ERR_NOMEM);
      cub::DeviceSelect::Flagged(tmp, tb, idx, flags, ends, n_ends_d, n_bytes, s);
      nd_free(tmp, s);
      cudaMemcpyAsync(&last_end, ends + n_ends - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) return fail(ND_ERR_CUDA);
    }
  }
  // lines: one per terminator, plus an unterminated tail
  const int64_t n_lines = n_ends + ((n_bytes > 0 && last_end != n_bytes - 1) ? 1 : 0);
  T->n_lines = n_lines;
  const int64_t L = n_lines > 0 ? n_lines : 1;
  if (nd_alloc(&T->start, L, s) || nd_alloc(&T->end, L, s) || nd_alloc(&T->kind, L, s) ||
      nd_alloc(&T->code, L, s) || nd_alloc(&T->src, L, s) || nd_alloc(&T->dst, L, s) ||
      nd_alloc(&T->w, L, s))
    return fail(ND_ERR_NOMEM);
  const unsigned long long init[2] = {~0ull, 0ull};
  cudaMemcpyAsync(ctl, init, sizeof(init), cudaMemcpyHostToDevice, s);
  if (n_lines) {
    k_line_bounds<<<nd_grid(n_lines, 256), 256, 0, s>>>(tx, ends, n_ends, n_bytes, n_lines,
                                                        T->start, T->end);
    k_parse_lines<<<nd_grid(n_lines, 128, 148 * 64), 128, 0, s>>>(
        tx, n_lines, T->start, T->end, weighted, lo_w, hi_w - lo_w,
        key_base(seed, 0, 3, 0), T->kind, T->code, T->src, T->dst, T->w, ctl, ctl + 1);
  }
  unsigned long long hc[2];
  cudaMemcpyAsync(hc, ctl, sizeof(hc), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return fail(ND_ERR_CUDA);
  nd_free(text, s); nd_free(flags, s); nd_free(ends, s); nd_free(n_ends_d, s); nd_free(ctl, s);
  h[0] = hc[0] == ~0ull ? 0 : (int64_t)hc[0];
  h[1] = (int64_t)hc[1];
  host_info[0] = n_lines;
  host_info[1] = h[0];  // first malformed line (1-based), 0 = none
  host_info[2] = 0;
  if (h[0]) {
    uint8_t c = 0;
    cudaMemcpy(&c, T->code + (h[0] - 1), 1, cudaMemcpyDeviceToHost);
    host_info[2] = c;
  }
  host_info[3] = h[1];  // lines for the host (non-ASCII / inexact numbers)
  *out = T;
  return ND_OK;
}

extern "C" int nd_text_parse(const char* host_text, int64_t n_bytes, int weighted, double lo_w,
                             double hi_w, uint64_t seed, void* stream, nd_text** out,
                             int64_t* host_info) {
  return text_parse(host_text, nullptr, n_bytes, weighted, lo_w, hi_w, seed, stream, out, host_info);
}

extern "C" int nd_text_parse_device(const char* dev_text, int64_t n_bytes, int weighted,
                                    double lo_w, double hi_w, uint64_t seed, void* stream,
                                    nd_text** out, int64_t* host_info) {
  return text_parse(nullptr, dev_text, n_bytes, weighted, lo_w, hi_w, seed, stream, out, host_info);
}

extern "C" int nd_text_host_lines(const nd_text* T, int64_t* host_lines) {
  if (!T || !host_lines) return ND_ERR_ARG;
  if (!T->n_lines) return ND_OK;
  cudaStream_t s = T->stream;
  int64_t *pos = nullptr, *lines = nullptr;
  ND_CUDA_TRY(nd_alloc(&pos, T->n_lines + 1, s));
  ND_TRY(scan_op<IsHost>(T->kind, T->n_lines, pos, s));
  int64_t cnt = 0;
  uint8_t lastkind = 0;
  cudaMemcpyAsync(&cnt, pos + T->n_lines - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&lastkind, T->kind + T->n_lines - 1, 1, cudaMemcpyDeviceToHost, s);
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  cnt += lastkind == K_HOST;
  ND_CUDA_TRY(nd_alloc(&lines, cnt > 0 ? cnt : 1, s));
  k_host_list<<<nd_grid(T->n_lines, 256), 256, 0, s>>>(T->kind, T->n_lines, pos, lines);
  if (cnt) ND_CUDA_TRY(cudaMemcpyAsync(host_lines, lines, cnt * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  nd_free(pos, s);
  nd_free(lines, s);
  return ND_OK;
}

extern "C" int nd_text_line_bounds(const nd_text* T, int64_t line_index, int64_t* host_lo_hi) {
  if (!T || line_index < 0 || line_index >= T->n_lines || !host_lo_hi) return ND_ERR_ARG;
  ND_CUDA_TRY(cudaMemcpy(host_lo_hi, T->start + line_index, sizeof(int64_t), cudaMemcpyDeviceToHost));
  ND_CUDA_TRY(cudaMemcpy(host_lo_hi + 1, T->end + line_index, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return ND_OK;
}

extern "C" int nd_text_finish(nd_text* T, const int64_t* host_line, const int64_t* host_src,
                              const int64_t* host_dst, const double* host_w,
                              const uint8_t* host_kind, int64_t n_patch, int undirected,
                              void* stream, nd_graph** out, int64_t* n_vertices) {
  if (!T || !out || !n_vertices || n_patch < 0) return ND_ERR_ARG;
  cudaStream_t s = stream ? (cudaStream_t)stream : T->stream;
  const int64_t NL = T->n_lines;
  if (n_patch) {
    int64_t *pl = nullptr, *ps = nullptr, *pd = nullptr;
    double* pw = nullptr;
    uint8_t* pk = nullptr;
    ND_CUDA_TRY(nd_alloc(&pl, n_patch, s));
    ND_CUDA_TRY(nd_alloc(&ps, n_patch, s));
    ND_CUDA_TRY(nd_alloc(&pd, n_patch, s));
    ND_CUDA_TRY(nd_alloc(&pw, n_patch, s));
    ND_CUDA_TRY(nd_alloc(&pk, n_patch, s));
    cudaMemcpyAsync(pl, host_line, n_patch * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(ps, host_src, n_patch * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(pd, host_dst, n_patch * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(pw, host_w, n_patch * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(pk, host_kind, n_patch, cudaMemcpyHostToDevice, s);
    k_apply_patches<<<nd_grid(n_patch, 256), 256, 0, s>>>(pl, ps, pd, pw, pk, n_patch, T->kind,
                                                          T->src, T->dst, T->w);
    nd_free(pl, s); nd_free(ps, s); nd_free(pd, s); nd_free(pw, s); nd_free(pk, s);
  }
  int64_t* pos = nullptr;
  ND_CUDA_TRY(nd_alloc(&pos, NL + 1, s));
  int64_t n_edge_lines = 0;
  if (NL) {
    ND_TRY(scan_op<IsEdge>(T->kind, NL, pos, s));
    int64_t last = 0;
    uint8_t lk = 0;
    cudaMemcpyAsync(&last, pos + NL - 1, 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&lk, T->kind + NL - 1, 1, cudaMemcpyDeviceToHost, s);
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    n_edge_lines = last + (lk == 1);
  }
  if (n_edge_lines == 0) {
    nd_free(pos, s);
    *n_vertices = 0;
    return ND_ERR_EMPTY;
  }
  const int64_t E = n_edge_lines * (undirected ? 2 : 1);
  int64_t *es = nullptr, *ed = nullptr, *ids = nullptr, *ids_sorted = nullptr, *uniq = nullptr,
          *n_uniq = nullptr;
  double* ew = nullptr;
  ND_CUDA_TRY(nd_alloc(&es, E, s));
  ND_CUDA_TRY(nd_alloc(&ed, E, s));
  if (T->weighted) ND_CUDA_TRY(nd_alloc(&ew, E, s));
  ND_CUDA_TRY(nd_alloc(&ids, 2 * n_edge_lines, s));
  ND_CUDA_TRY(nd_alloc(&ids_sorted, 2 * n_edge_lines, s));
  ND_CUDA_TRY(nd_alloc(&uniq, 2 * n_edge_lines, s));
  ND_CUDA_TRY(nd_alloc(&n_uniq, 1, s));
  k_emit_edges<<<nd_grid(NL, 256), 256, 0, s>>>(T->kind, NL, pos, T->src, T->dst, T->w, undirected,
                                                es, ed, ew, ids);
  {  // original = np.unique(concatenate([src, dst])): sort + unique (ids >= 0)
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, ids, ids_sorted, 2 * n_edge_lines, 0, 63, s);
    size_t tb2 = 0;
    cub::DeviceSelect::Unique(nullptr, tb2, ids_sorted, uniq, n_uniq, 2 * n_edge_lines, s);
    void* tmp = nullptr;
    ND_CUDA_TRY(nd_alloc((char**)&tmp, tb > tb2 ? tb : tb2, s));
    ND_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, tb, ids, ids_sorted, 2 * n_edge_lines, 0, 63, s));
    ND_CUDA_TRY(cub::DeviceSelect::Unique(tmp, tb2, ids_sorted, uniq, n_uniq, 2 * n_edge_lines, s));
    nd_free(tmp, s);
  }
  int64_t V = 0;
  cudaMemcpyAsync(&V, n_uniq, 8, cudaMemcpyDeviceToHost, s);
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  k_compact_ids<<<nd_grid(E, 256, 148 * 64), 256, 0, s>>>(uniq, V, es, E);
  k_compact_ids<<<nd_grid(E, 256, 148 * 64), 256, 0, s>>>(uniq, V, ed, E);
  ND_CUDA_TRY(cudaGetLastError());
  int rc = nd_build_from_edges_dev(es, ed, ew, E, V, s, out);
  nd_free(es, s); nd_free(ed, s); nd_free(ew, s); nd_free(ids, s); nd_free(ids_sorted, s);
  nd_free(n_uniq, s); nd_free(pos, s);
  if (T->remap) nd_free(T->remap, s);
  T->remap = uniq;
  T->V = V;
  *n_vertices = V;
  return rc;
}

extern "C" int nd_text_remap(const nd_text* T, int64_t* host_remap) {
  if (!T || !host_remap || !T->remap) return ND_ERR_ARG;
  ND_CUDA_TRY(cudaMemcpyAsync(host_remap, T->remap, T->V * sizeof(int64_t), cudaMemcpyDeviceToHost,
                              T->stream));
  ND_CUDA_TRY(cudaStreamSynchronize(T->stream));
  return ND_OK;
}

extern "C" int nd_text_destroy(nd_text* T) {
  if (!T) return ND_OK;
  cudaStream_t s = T->stream;
  nd_free(T->start, s); nd_free(T->end, s); nd_free(T->kind, s); nd_free(T->code, s);
  nd_free(T->src, s); nd_free(T->dst, s); nd_free(T->w, s); nd_free(T->remap, s);
  cudaStreamSynchronize(s);
  delete T;
  return ND_OK;
}
