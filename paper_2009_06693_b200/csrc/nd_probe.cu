// nd_probe.cu — the measured random-gather ceiling of this GPU.
//
// The walk kernels are gather-bound: every step reads a few 32-byte sectors
// at data-dependent addresses spread over gigabytes of records.  Such reads
// are limited neither by the streaming copy bandwidth (MEASURED_PEAKS.json)
// nor by DRAM sector counts alone: on B200 a random sector read pulls a
// 128-byte line from HBM and misses the SM's address-translation caches once
// the footprint exceeds a few hundred 2 MB pages (tools/gather_peak.cu,
// profiles/r01_gather_ceiling.json).  nd_gather_ceiling measures the rate of
// dependent random 32-byte sector reads (pointer chasing, one chain per
// thread, like one walker per lane) over a buffer the size of the sampler's
// working set, so bench.py can report the kernels' random-sector rate as a
// fraction of what the hardware sustains for that access pattern.
#include "nd_internal.h"

namespace {

__device__ __forceinline__ uint64_t chase_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_fill_chase(int4* __restrict__ buf, uint64_t n16) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x)
    buf[i] = make_int4((int)chase_mix(i), (int)i, (int)(i >> 32), (int)(chase_mix(i) >> 32));
}

// each thread: `iters` dependent 16-byte reads at hashed 32-byte-sector addresses
__global__ void k_chase(const int4* __restrict__ buf, uint64_t sector_mask, int iters,
                        unsigned long long* __restrict__ sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t g = chase_mix(tid * 0x9E3779B97F4A7C15ull + 1) & sector_mask;
  int acc = 0;
  for (int it = 0; it < iters; it++) {
    const int4 a = __ldg(buf + 2 * g);
    acc ^= a.y;
    g = chase_mix((uint64_t)(uint32_t)a.x + g) & sector_mask;
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

}  // namespace

extern "C" int nd_gather_ceiling(int64_t bytes, int ctas_per_sm, int iters,
                                  double* sectors_per_s, void* stream) {
  if (bytes < (1 << 20) || ctas_per_sm < 1 || iters < 1 || !sectors_per_s) return ND_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t sectors = 1;
  while (sectors * 2 * 32 <= (uint64_t)bytes) sectors *= 2;  // power of two
  int4* buf = nullptr;
  unsigned long long* sink = nullptr;
  ND_CUDA_TRY(nd_alloc(&buf, sectors * 2, s));
  ND_CUDA_TRY(nd_alloc(&sink, 1, s));
  k_fill_chase<<<148 * 8, 256, 0, s>>>(buf, sectors * 2);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = nsm * ctas_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_chase<<<grid, 256, 0, s>>>(buf, sectors - 1, iters, sink);  // warm-up
  cudaEventRecord(e0, s);
  k_chase<<<grid, 256, 0, s>>>(buf, sectors - 1, iters, sink);
  cudaEventRecord(e1, s);
  ND_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  nd_free(buf, s);
  nd_free(sink, s);
  ND_CUDA_TRY(cudaGetLastError());
  *sectors_per_s = (double)grid * 256.0 * iters / (ms * 1e-3);
  return ND_OK;
}
