// nd_format.cu — text rows on the device ("a C++ or
// vectorised formatter is needed for ~5e8-id outputs").
//
// The reference's text writer (output.py:72-92, `render_text`) prints one line
// per sample, "<sample id>: <v0> <v1> ...", the ids in decimal and remapped to
// the input's original vertex labels (output.py:145-150).  In Python that is
// a per-row str() join: minutes for C2's 257M ids.  Here the rows are printed
// where they live: one warp per row sums its ids' decimal widths (pass 1), an
// exclusive scan places the lines, and the same warp writes every id's digits
// at its offset (pass 2, a warp prefix sum over the widths of each 32-id
// chunk).  Byte-for-byte the reference's text: an empty row prints "<sid>: ".

#include <cub/cub.cuh>

#include "nd_internal.h"

using namespace nd;

namespace {

__device__ __forceinline__ int dec_width(int64_t v) {
  uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1u : (uint64_t)v;
  int d = 1;
  while (u >= 10000) { u /= 10000; d += 4; }
  while (u >= 10) { u /= 10; d++; }
  return d + (v < 0);
}

// digits of v ending just before `end` (width w, from dec_width)
__device__ __forceinline__ void dec_write(char* p, int64_t v, int w) {
  uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1u : (uint64_t)v;
  char* q = p + w;
  do {
    *--q = (char)('0' + (int)(u % 10));
    u /= 10;
  } while (u);
  if (v < 0) *--q = '-';
}

template <typename IdT>
__device__ __forceinline__ int64_t id_at(const IdT* ids, const int64_t* remap, int64_t k) {
  const int64_t x = (int64_t)ids[k];
  return remap ? remap[x] : x;
}

// pass 1: bytes of each line ("sid: " + ids joined by ' ' + '\n')
template <typename IdT>
__global__ void k_fmt_len(const int64_t* __restrict__ off, const IdT* __restrict__ ids,
                          const int64_t* __restrict__ sid, const int64_t* __restrict__ remap,
                          int64_t n, int64_t* __restrict__ len) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int64_t a = off[i], b = off[i + 1];
    int64_t w = 0;
    for (int64_t k = a + lane; k < b; k += 32) w += dec_width(id_at(ids, remap, k));
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if (lane == 0) {
      const int64_t c = b - a;
      len[i] = dec_width(sid[i]) + 2 + w + (c > 0 ? c - 1 : 0) + 1;
    }
  }
}

// pass 2: the lines at their scanned offsets
template <typename IdT>
__global__ void k_fmt_write(const int64_t* __restrict__ off, const IdT* __restrict__ ids,
                            const int64_t* __restrict__ sid, const int64_t* __restrict__ remap,
                            int64_t n, const int64_t* __restrict__ lpos, char* __restrict__ text) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int64_t a = off[i], b = off[i + 1];
    char* line = text + lpos[i];
    const int sw = dec_width(sid[i]);
    if (lane == 0) {
      dec_write(line, sid[i], sw);
      line[sw] = ':';
      line[sw + 1] = ' ';
    }
    int64_t pos = sw + 2;  // next id's first byte (warp-uniform)
    for (int64_t k0 = a; k0 < b; k0 += 32) {
      const int64_t k = k0 + lane;
      int64_t v = 0;
      int w = 0;
      if (k < b) {
        v = id_at(ids, remap, k);
        w = dec_width(v) + (k > a);  // a separating space before every id but the first
      }
      int x = w;  // inclusive warp scan of the widths
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (k < b) {
        char* p = line + pos + x - w;
        if (k > a) *p++ = ' ';
        dec_write(p, v, w - (k > a));
      }
      pos += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) line[pos] = '\n';
  }
}

template <typename IdT>
int format_rows(const int64_t* off, const IdT* ids, const int64_t* sid, const int64_t* remap,
                int64_t n, cudaStream_t s, char* host_out, int64_t cap, int64_t* text_len) {
  int64_t *len = nullptr, *lpos = nullptr;
  ND_CUDA_TRY(nd_alloc(&len, n + 1, s));
  ND_CUDA_TRY(nd_alloc(&lpos, n + 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(len + n, 0, sizeof(int64_t), s));
  const int grid = nd_grid(n * 32, 256, 148 * 32);
  if (n) k_fmt_len<IdT><<<grid, 256, 0, s>>>(off, ids, sid, remap, n, len);
  int rc = ND_OK;
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, len, lpos, n + 1, s);
    char* tmp = nullptr;
    if (nd_alloc(&tmp, tb, s) != cudaSuccess ||
        cub::DeviceScan::ExclusiveSum(tmp, tb, len, lpos, n + 1, s) != cudaSuccess)
      rc = ND_ERR_CUDA;
    nd_free(tmp, s);
  }
  int64_t total = 0;
  if (rc == ND_OK) {
    int64_t* h = nd_pinned_scratch();
    if (nd_d2h(h, lpos + n, sizeof(int64_t), s) != ND_OK) rc = ND_ERR_CUDA;
    else total = *h;
  }
  if (rc == ND_OK) *text_len = total;
  if (rc == ND_OK && host_out) {
    if (cap < total) {
      rc = ND_ERR_ARG;
    } else if (total > 0) {
      char* text = nullptr;
      if (nd_alloc(&text, total, s) != cudaSuccess) {
        rc = ND_ERR_CUDA;
      } else {
        k_fmt_write<IdT><<<grid, 256, 0, s>>>(off, ids, sid, remap, n, lpos, text);
        if (cudaGetLastError() != cudaSuccess ||
            cudaMemcpyAsync(host_out, text, total, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
          rc = ND_ERR_CUDA;
        nd_free(text, s);
      }
    }
  }
  nd_free(len, s);
  nd_free(lpos, s);
  if (rc == ND_OK && cudaGetLastError() != cudaSuccess) rc = ND_ERR_CUDA;
  return rc;
}

}  // namespace

extern "C" int nd_format_rows(const int64_t* off, const void* ids, int id_bytes,
                              const int64_t* sample_ids, int64_t n, const int64_t* remap,
                              void* stream, char* host_out, int64_t cap, int64_t* text_len) {
  if (!off || !sample_ids || !text_len || n < 0 || (id_bytes != 4 && id_bytes != 8))
    return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  NvtxRange r("nd_format_rows");
  return id_bytes == 4
             ? format_rows(off, (const int32_t*)ids, sample_ids, remap, n, s, host_out, cap, text_len)
             : format_rows(off, (const int64_t*)ids, sample_ids, remap, n, s, host_out, cap, text_len);
}
