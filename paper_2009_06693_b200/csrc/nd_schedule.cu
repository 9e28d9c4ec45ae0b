// nd_schedule.cu — exact export of the transit-parallel schedule.
//
// build_transit_map + partition_work_classes (transit_parallel.py:71-101)
// on device: a stable radix sort of (transit, pair id) inverts the step's
// sample-major pairs into transit groups (members stay sample-major), group
// boundaries come from a flag scan, and the per-class scheduling index is the
// exclusive scan of each class's indicator in transit-ascending order.  The
// engines run the same sort + classes on every step; this entry exists so the
// schedule itself can be compared with the reference bit for bit.
#include <cub/cub.cuh>

#include "nd_internal.h"

using namespace nd;

namespace {

__global__ void k_iota_keys(const int64_t* __restrict__ pt, int64_t n, uint64_t* __restrict__ keys,
                            int64_t* __restrict__ ids, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (pt[i] < 0) atomicExch(bad, 1);
    keys[i] = (uint64_t)pt[i];
    ids[i] = i;
  }
}

__global__ void k_flags64(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_groups(const int64_t* __restrict__ flags, const int64_t* __restrict__ gid,
                         const uint64_t* __restrict__ keys, int64_t n,
                         int64_t* __restrict__ gstart, int64_t* __restrict__ gtransit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flags[i]) {
      gstart[gid[i] - 1] = i;
      gtransit[gid[i] - 1] = (int64_t)keys[i];
    }
    if (i == n - 1) gstart[gid[i]] = n;
  }
}

__global__ void k_class_ind(const int64_t* __restrict__ gstart, int64_t G, int64_t m,
                            int32_t* __restrict__ gclass, int64_t* __restrict__ ind) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t work = (gstart[g + 1] - gstart[g]) * m;
    const int c = work < SMALL_MAX_WORK ? 0 : (work <= LARGE_MIN_WORK ? 1 : 2);
    gclass[g] = c;
    for (int k = 0; k < 3; k++) ind[k * G + g] = (k == c);
  }
}

__global__ void k_sched_pick(const int32_t* __restrict__ gclass, const int64_t* __restrict__ ranks,
                             int64_t G, int64_t* __restrict__ sched) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G;
       g += (int64_t)gridDim.x * blockDim.x)
    sched[g] = ranks[gclass[g] * G + g];
}

}  // namespace

extern "C" int nd_transit_schedule(const int64_t* pair_transit, int64_t n_pairs, int64_t m,
                                   int64_t* order, int64_t* group_start, int64_t* group_transit,
                                   int32_t* group_class, int64_t* sched_index, int64_t* n_groups,
                                   void* stream) {
  if (n_pairs < 0 || m < 1) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_pairs == 0) {
    *n_groups = 0;
    int64_t z = 0;
    ND_CUDA_TRY(cudaMemcpyAsync(group_start, &z, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    ND_CUDA_TRY(cudaStreamSynchronize(s));
    return ND_OK;
  }
  const int64_t n = n_pairs;
  uint64_t *k0, *k1;
  int64_t *i1, *flags, *gid, *ind, *ranks;
  int* bad;
  ND_CUDA_TRY(nd_alloc(&k0, n, s));
  ND_CUDA_TRY(nd_alloc(&k1, n, s));
  ND_CUDA_TRY(nd_alloc(&i1, n, s));
  ND_CUDA_TRY(nd_alloc(&flags, n, s));
  ND_CUDA_TRY(nd_alloc(&gid, n, s));
  ND_CUDA_TRY(nd_alloc(&bad, 1, s));
  ND_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), s));
  k_iota_keys<<<nd_grid(n, 256), 256, 0, s>>>(pair_transit, n, k0, order, bad);
  cub::DoubleBuffer<uint64_t> dk(k0, k1);
  cub::DoubleBuffer<int64_t> dv(order, i1);
  size_t tb = 0, tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, 64, s);
  cub::DeviceScan::InclusiveSum(nullptr, tb2, flags, gid, n, s);
  if (tb2 > tb) tb = tb2;
  void* tmp;
  ND_CUDA_TRY(nd_alloc((char**)&tmp, tb + 3 * 1024, s));
  size_t t = tb;
  ND_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, t, dk, dv, n, 0, 64, s));
  if (dv.Current() != order)
    ND_CUDA_TRY(cudaMemcpyAsync(order, dv.Current(), n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  const uint64_t* keys = dk.Current();
  k_flags64<<<nd_grid(n, 256), 256, 0, s>>>(keys, n, flags);
  t = tb;
  ND_CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp, t, flags, gid, n, s));
  int64_t G = 0;
  ND_TRY(nd_d2h(&G, gid + n - 1, sizeof(int64_t), s));
  k_groups<<<nd_grid(n, 256), 256, 0, s>>>(flags, gid, keys, n, group_start, group_transit);
  int hbad = 0;
  ND_TRY(nd_d2h(&hbad, bad, sizeof(int), s));
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  ND_CUDA_TRY(nd_alloc(&ind, 3 * G, s));
  ND_CUDA_TRY(nd_alloc(&ranks, 3 * G, s));
  k_class_ind<<<nd_grid(G, 256), 256, 0, s>>>(group_start, G, m, group_class, ind);
  size_t tb3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb3, ind, ranks, G, s);
  void* tmp3;
  ND_CUDA_TRY(nd_alloc((char**)&tmp3, tb3, s));
  for (int c = 0; c < 3; c++) {
    size_t t3 = tb3;
    ND_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp3, t3, ind + c * G, ranks + c * G, G, s));
  }
  k_sched_pick<<<nd_grid(G, 256), 256, 0, s>>>(group_class, ranks, G, sched_index);
  ND_CUDA_TRY(cudaGetLastError());
  ND_CUDA_TRY(cudaStreamSynchronize(s));
  nd_free(k0, s); nd_free(k1, s); nd_free(i1, s); nd_free(flags, s); nd_free(gid, s);
  nd_free(ind, s); nd_free(ranks, s); nd_free(tmp, s); nd_free(tmp3, s); nd_free(bad, s);
  *n_groups = G;
  return hbad ? ND_ERR_ARG : ND_OK;
}
