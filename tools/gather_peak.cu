// gather_peak.cu — measured ceiling of random 32-byte sector gathers from HBM
// on this GPU (the roofline denominator a gather-bound sampler actually
// faces, beside the streaming copy peak in MEASURED_PEAKS.json).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/gather_peak tools/gather_peak.cu
//   gpurun_out/gather_peak [buffer_GiB]
//
// Each thread issues ILP independent loads per iteration at hashed sector
// addresses (uniform over the buffer); variants: 32/64/128-byte granules,
// independent vs. dependent (pointer-chase) chains, buffer 1..N GiB.  Prints
// one JSON line per variant: GB/s of sectors actually requested.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// independent gathers: GRAN bytes (multiple of 16) per access
template <int GRAN, int ILP>
__global__ void k_gather(const int4* __restrict__ buf, uint64_t n_gran, int iters, uint64_t seed,
                         unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  int acc = 0;
  constexpr int V = GRAN / 16;
  for (int it = 0; it < iters; it++) {
    int4 r[ILP][V];
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      const uint64_t g = mix(seed + tid * 0x9E3779B97F4A7C15ull + (uint64_t)(it * ILP + i)) & (n_gran - 1);
#pragma unroll
      for (int k = 0; k < V; k++) r[i][k] = __ldg(buf + g * V + k);
    }
#pragma unroll
    for (int i = 0; i < ILP; i++)
#pragma unroll
      for (int k = 0; k < V; k++) acc ^= r[i][k].x ^ r[i][k].w;
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

// load flavours: 0 __ldg (ld.global.nc), 1 plain ld.global, 2 __ldcg (L2 only),
// 3 ld.global.nc.L1::no_allocate, 4 __ldcs (evict-first)
template <int OP>
__device__ __forceinline__ int4 ld16(const int4* p) {
  if (OP == 0) return __ldg(p);
  if (OP == 1) return *p;
  if (OP == 2) return __ldcg(p);
  if (OP == 3) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
  }
  return __ldcs(p);
}

template <int CHAINS, int OP>
__global__ void k_chase_op(const int4* __restrict__ buf, uint64_t n_gran, int iters, uint64_t seed,
                           unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t g[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; c++) g[c] = mix(seed + tid * 0x9E3779B97F4A7C15ull + c) & (n_gran - 1);
  int acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
      const int4 a = ld16<OP>(buf + 2 * g[c]);
      acc ^= a.y ^ a.z;
      g[c] = mix((uint64_t)(uint32_t)a.x + (uint64_t)a.w + g[c]) & (n_gran - 1);
    }
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

// dependent chains: the next address depends on the loaded value (like a walk)
template <int CHAINS>
__global__ void k_chase(const int4* __restrict__ buf, uint64_t n_gran, int iters, uint64_t seed,
                        unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t g[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; c++) g[c] = mix(seed + tid * 0x9E3779B97F4A7C15ull + c) & (n_gran - 1);
  int acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
      const int4 a = __ldg(buf + 2 * g[c]);
      acc ^= a.y;
      g[c] = mix((uint64_t)(uint32_t)a.x + g[c]) & (n_gran - 1);
    }
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

// dependent chains over a fixed 64 MB (L2-resident) working set scattered
// across the whole buffer: `touch` sectors at the start of every 2 MB page.
// Same L2 footprint, growing page count: isolates address translation.
__global__ void k_chase_sparse(const int4* __restrict__ buf, uint64_t n_pages, uint64_t touch,
                               int iters, uint64_t seed, unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h = mix(seed + tid * 0x9E3779B97F4A7C15ull);
  int acc = 0;
  for (int it = 0; it < iters; it++) {
    const uint64_t page = h % n_pages, off = (h >> 32) % touch;
    const int4 a = __ldg(buf + (page << 17) + 2 * off);  // 2 MB = 2^17 int4
    acc ^= a.y;
    h = mix((uint64_t)(uint32_t)a.x + h);
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// dependent chains where the SM running the thread picks the page subset:
// part = smid / block (contiguous SM blocks) or smid % parts (interleaved);
// each part spans n_pages / parts pages.  Tests whether translation reach is
// per SM / per GPC (partitioned pages scale it) or device-wide.
__global__ void k_chase_part(const int4* __restrict__ buf, uint64_t n_pages, int parts, int mode,
                             int n_sm, int iters, uint64_t seed, unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const unsigned sm = smid();
  const int block = (n_sm + parts - 1) / parts;
  const uint64_t part = mode == 0 ? sm / block : sm % parts;
  const uint64_t ppp = n_pages / parts;
  uint64_t h = mix(seed + tid * 0x9E3779B97F4A7C15ull);
  int acc = 0;
  for (int it = 0; it < iters; it++) {
    const uint64_t page = part * ppp + h % ppp, off = (h >> 32) & 65535;
    const int4 a = __ldg(buf + (page << 17) + 2 * off);
    acc ^= a.y;
    h = mix((uint64_t)(uint32_t)a.x + h);
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

// per-SM page sets with an L2-resident footprint: SM k touches only pages
// [k*pps, (k+1)*pps) (mod n_pages), `touch` sectors at the start of each.
// High rates here with low rates in chase_sparse => translation caching is
// per SM (or per GPC): partitioning pages across SMs multiplies its reach.
__global__ void k_chase_smpages(const int4* __restrict__ buf, uint64_t n_pages, uint64_t pps,
                                uint64_t touch, int iters, uint64_t seed, unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t base = ((uint64_t)smid() * pps) % n_pages;
  uint64_t h = mix(seed + tid * 0x9E3779B97F4A7C15ull);
  int acc = 0;
  for (int it = 0; it < iters; it++) {
    const uint64_t page = (base + h % pps) % n_pages, off = (h >> 32) % touch;
    const int4 a = __ldg(buf + (page << 17) + 2 * off);
    acc ^= a.y;
    h = mix((uint64_t)(uint32_t)a.x + h);
  }
  if (acc == 0x7fffffff) atomicAdd(sink, 1ull);
}

template <class F>
static float time_it(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

__global__ void k_fill(int4* buf, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    buf[i] = make_int4((int)mix(i), (int)i, 0, (int)(mix(i) >> 32));
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 4.0;
  if (getenv("GP_L2FETCH")) {  // cudaLimitMaxL2FetchGranularity (0..128 bytes, a hint)
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(getenv("GP_L2FETCH")));
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity\": %zu, \"set_rc\": %d}\n", v, (int)e);
  }
  const uint64_t bytes = (uint64_t)(gib * (1ull << 30));
  int4* buf = nullptr;
  unsigned long long* sink = nullptr;
  const char* how = argc > 2 ? argv[2] : "malloc";
  if (!strcmp(how, "vmm")) {  // cuMemCreate/cuMemMap in 1 GiB chunks, VA aligned to 1 GiB
    cudaFree(0);
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gmin = 0, grec = 0;
    cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    printf("{\"granularity_min\": %zu, \"granularity_recommended\": %zu}\n", gmin, grec);
    const size_t chunk = 1ull << 30;
    const size_t total = (bytes + chunk - 1) / chunk * chunk;
    CUdeviceptr va = 0;
    if (cuMemAddressReserve(&va, total, chunk, 0, 0) != CUDA_SUCCESS) { printf("reserve failed\n"); return 1; }
    for (size_t off = 0; off < total; off += chunk) {
      CUmemGenericAllocationHandle h;
      if (cuMemCreate(&h, chunk, &prop, 0) != CUDA_SUCCESS) { printf("create failed\n"); return 1; }
      cuMemMap(va + off, chunk, 0, h, 0);
    }
    CUmemAccessDesc ad = {};
    ad.location = prop.location;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cuMemSetAccess(va, total, &ad, 1);
    buf = (int4*)va;
  } else if (!strcmp(how, "async")) {
    if (cudaMallocAsync((void**)&buf, bytes, 0) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  } else if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&sink, 8);
  k_fill<<<148 * 16, 256>>>(buf, bytes / 16);
  cudaDeviceSynchronize();
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 64;
  for (int occ : {2, 4, 8}) {  // 256-thread CTAs per SM (all resident)
    const int grid = nsm * occ;
    const uint64_t threads = (uint64_t)grid * 256;
    auto run_g = [&](auto kern, int gran, int ilp, const char* name) {
      const uint64_t n_gran = bytes / gran;
      float ms = time_it([&] { kern<<<grid, 256>>>(buf, n_gran, iters, 12345, sink); });
      const double req = (double)threads * iters * ilp * gran;
      printf("{\"variant\": \"%s\", \"granule_B\": %d, \"ilp\": %d, \"ctas_per_sm\": %d, \"buffer_GiB\": %.1f, "
             "\"ms\": %.3f, \"GBps\": %.1f, \"Gaccess_per_s\": %.2f}\n",
             name, gran, ilp, occ, gib, ms, req / ms / 1e6, (double)threads * iters * ilp / ms / 1e6);
    };
    {
      run_g(k_gather<32, 1>, 32, 1, "independent");
      run_g(k_gather<32, 2>, 32, 2, "independent");
      run_g(k_gather<32, 4>, 32, 4, "independent");
      run_g(k_gather<64, 2>, 64, 2, "independent");
      run_g(k_gather<128, 1>, 128, 1, "independent");
    }
    auto run_c = [&](auto kern, int chains) {
      const uint64_t n_gran = bytes / 32;
      float ms = time_it([&] { kern<<<grid, 256>>>(buf, n_gran, iters, 777, sink); });
      const double req = (double)threads * iters * chains * 32;
      printf("{\"variant\": \"chase\", \"granule_B\": 32, \"chains\": %d, \"ctas_per_sm\": %d, \"buffer_GiB\": %.1f, "
             "\"ms\": %.3f, \"GBps\": %.1f, \"Gaccess_per_s\": %.2f}\n",
             chains, occ, gib, ms, req / ms / 1e6, (double)threads * iters * chains / ms / 1e6);
    };
    {
      run_c(k_chase<1>, 1);
      run_c(k_chase<2>, 2);
      run_c(k_chase<4>, 4);
    }
  }
  {
    const uint64_t n_pages = bytes >> 21;
    const uint64_t touch = ((64ull << 20) / n_pages) / 32 > 0 ? ((64ull << 20) / n_pages) / 32 : 1;
    const int grid = nsm * 4;
    const uint64_t threads = (uint64_t)grid * 256;
    float ms = time_it([&] { k_chase_sparse<<<grid, 256>>>(buf, n_pages, touch, iters * 4, 99, sink); });
    printf("{\"variant\": \"chase_sparse_64MB\", \"pages_2MB\": %llu, \"sectors_per_page\": %llu, "
           "\"buffer_GiB\": %.2f, \"ms\": %.3f, \"Gaccess_per_s\": %.2f}\n",
           (unsigned long long)n_pages, (unsigned long long)touch, gib, ms,
           (double)threads * iters * 4 / ms / 1e6);
  }
  {
    const int grid = nsm * 4;
    const uint64_t threads = (uint64_t)grid * 256;
    const uint64_t n_gran = bytes / 32;
    auto run_op = [&](auto kern, const char* op) {
      float ms = time_it([&] { kern<<<grid, 256>>>(buf, n_gran, iters, 31, sink); });
      printf("{\"variant\": \"chase_op\", \"op\": \"%s\", \"chains\": 4, \"buffer_GiB\": %.2f, \"ms\": %.3f, "
             "\"Gaccess_per_s\": %.2f}\n", op, gib, ms, (double)threads * iters * 4 / ms / 1e6);
    };
    run_op(k_chase_op<4, 0>, "ldg_nc");
    run_op(k_chase_op<4, 1>, "ld_global");
    run_op(k_chase_op<4, 2>, "ldcg");
    run_op(k_chase_op<4, 3>, "nc_L1_no_allocate");
    run_op(k_chase_op<4, 4>, "ldcs");
  }
  for (uint64_t pps : {4ull, 8ull, 16ull, 32ull, 64ull, 128ull}) {
    const uint64_t n_pages = bytes >> 21;
    const uint64_t used = pps * nsm < n_pages ? pps * nsm : n_pages;
    const uint64_t touch = ((64ull << 20) / used) / 32 > 0 ? ((64ull << 20) / used) / 32 : 1;
    const int grid = nsm * 4;
    const uint64_t threads = (uint64_t)grid * 256;
    float ms = time_it([&] { k_chase_smpages<<<grid, 256>>>(buf, n_pages, pps, touch, iters * 4, 3, sink); });
    printf("{\"variant\": \"chase_smpages_64MB\", \"pages_per_sm\": %llu, \"pages_used\": %llu, "
           "\"buffer_GiB\": %.2f, \"ms\": %.3f, \"Gaccess_per_s\": %.2f}\n",
           (unsigned long long)pps, (unsigned long long)used, gib, ms, (double)threads * iters * 4 / ms / 1e6);
  }
  if (getenv("GP_PART"))
  for (int mode = 0; mode < 2; mode++)
    for (int parts : {1, 2, 4, 8, 16, 37, 74, 148}) {
      const uint64_t n_pages = bytes >> 21;
      if ((uint64_t)parts > n_pages) continue;
      const int grid = nsm * 4;
      const uint64_t threads = (uint64_t)grid * 256;
      float ms = time_it([&] { k_chase_part<<<grid, 256>>>(buf, n_pages, parts, mode, nsm, iters * 4, 5, sink); });
      printf("{\"variant\": \"chase_part\", \"mode\": \"%s\", \"parts\": %d, \"pages_per_part\": %llu, "
             "\"buffer_GiB\": %.2f, \"ms\": %.3f, \"Gaccess_per_s\": %.2f}\n",
             mode == 0 ? "sm_blocks" : "sm_interleaved", parts, (unsigned long long)(n_pages / parts), gib, ms,
             (double)threads * iters * 4 / ms / 1e6);
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
