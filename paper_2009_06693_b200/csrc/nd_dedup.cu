// nd_dedup.cu — unique() steps on device.
//
// dedup_step (output.py:27-31) replaces a sample's step slots with their
// sorted distinct non-NULL values; finish_step (driver.py:165-172) applies it
// to every alive sample after a unique step.  On device the step's non-NULL
// (sample, vertex) pairs — already compacted in sample-major order by the
// engines — are radix sorted on the 64-bit key (sample << 32 | vertex), the
// adjacent duplicates dropped (flag + exclusive scan), and the per-sample
// distinct counts recovered from the segment boundaries.
#include <cub/cub.cuh>

#include "nd_internal.h"

using namespace nd;

namespace {

__global__ void k_pack(const int32_t* __restrict__ sid, const int32_t* __restrict__ val, int64_t n,
                       uint64_t* __restrict__ key) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    key[j] = ((uint64_t)(uint32_t)sid[j] << 32) | (uint32_t)val[j];
}

__global__ void k_uflags(const uint64_t* __restrict__ key, int64_t n, int64_t* __restrict__ f) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= n;
       j += (int64_t)gridDim.x * blockDim.x)
    f[j] = (j < n && (j == 0 || key[j] != key[j - 1])) ? 1 : 0;
}

__global__ void k_uwrite(const uint64_t* __restrict__ key, const int64_t* __restrict__ f,
                         const int64_t* __restrict__ pos, int64_t n, int32_t* __restrict__ osid,
                         int32_t* __restrict__ oval, unsigned long long* __restrict__ counts) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (!f[j]) continue;
    const uint64_t k = key[j];
    const int32_t sm = (int32_t)(k >> 32);
    osid[pos[j]] = sm;
    oval[pos[j]] = (int32_t)(k & 0xFFFFFFFFull);
    atomicAdd(counts + sm, 1ull);
  }
}

int bits_for(int64_t x) {
  int b = 1;
  while ((1ll << b) <= x) b++;
  return b;
}

}  // namespace

// Sorted-distinct per sample.  Inputs: m (sample, vertex) pairs (vertex >= 0).
// Outputs (allocated here): out_sid/out_val (sample-major, vertices ascending),
// *out_m; counts[n_samples] (device int64, overwritten).
int nd_dedup_segments(const int32_t* sid, const int32_t* val, int64_t m, int64_t n_samples,
                      int64_t n_vertices, int32_t** out_sid, int32_t** out_val, int64_t* out_m,
                      int64_t* counts, cudaStream_t s) {
  ND_CUDA_TRY(cudaMemsetAsync(counts, 0, (n_samples ? n_samples : 1) * sizeof(int64_t), s));
  if (m == 0) {
    *out_m = 0;
    ND_CUDA_TRY(nd_alloc(out_sid, 1, s));
    ND_CUDA_TRY(nd_alloc(out_val, 1, s));
    return ND_OK;
  }
  uint64_t *k0, *k1;
  int64_t *f, *pos;
  ND_CUDA_TRY(nd_alloc(&k0, m, s));
  ND_CUDA_TRY(nd_alloc(&k1, m, s));
  ND_CUDA_TRY(nd_alloc(&f, m + 1, s));
  ND_CUDA_TRY(nd_alloc(&pos, m + 1, s));
  k_pack<<<nd_grid(m, 256), 256, 0, s>>>(sid, val, m, k0);
  const int end_bit = 32 + bits_for(n_samples);
  const int begin_bit = 0;
  size_t tb = 0, tb2 = 0;
  cub::DoubleBuffer<uint64_t> dk(k0, k1);
  cub::DeviceRadixSort::SortKeys(nullptr, tb, dk, m, begin_bit, end_bit > 64 ? 64 : end_bit, s);
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, f, pos, m + 1, s);
  if (tb2 > tb) tb = tb2;
  void* tmp;
  ND_CUDA_TRY(nd_alloc((char**)&tmp, tb, s));
  size_t t = tb;
  ND_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, t, dk, m, begin_bit, end_bit > 64 ? 64 : end_bit, s));
  (void)n_vertices;
  k_uflags<<<nd_grid(m + 1, 256), 256, 0, s>>>(dk.Current(), m, f);
  t = tb;
  ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, t, f, pos, m + 1, s));
  int64_t* h = nd_pinned_scratch();
  ND_TRY(nd_d2h(h, pos + m, sizeof(int64_t), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t u = h[0];
  ND_CUDA_TRY(nd_alloc(out_sid, u, s));
  ND_CUDA_TRY(nd_alloc(out_val, u, s));
  k_uwrite<<<nd_grid(m, 256), 256, 0, s>>>(dk.Current(), f, pos, m, *out_sid, *out_val,
                                            reinterpret_cast<unsigned long long*>(counts));
  ND_CUDA_TRY(cudaGetLastError());
  nd_free(k0, s);
  nd_free(k1, s);
  nd_free(f, s);
  nd_free(pos, s);
  nd_free(tmp, s);
  *out_m = u;
  return ND_OK;
}
