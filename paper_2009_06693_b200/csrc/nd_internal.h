// nd_internal.h — host-side structs shared by the translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <array>
#include <functional>
#include <vector>

#include "nd_common.cuh"

struct nd_graph {
  nd::DevGraph g;       // device views
  int64_t* row = nullptr;
  int32_t* col = nullptr;
  double* w = nullptr;
  double* pre = nullptr;
  double* mx = nullptr;
  int32_t* hset = nullptr;   // optional exact indexes (nd_index.cu)
  int32_t* guide = nullptr;
  nd::VRec* vrec = nullptr;  // packed records (nd_index.cu)
  nd::NbrW* nbw = nullptr;
  nd::NbrP* nbp = nullptr;
  nd::NbrU* nbu = nullptr;
  nd::PickLine* pl = nullptr;
  int32_t* vline = nullptr;
  int64_t bytes = 0;       // everything resident (CSR + built indexes/records)
  int64_t csr_bytes = 0;   // row/col/weights/prefix/max at creation
  double prep_ms = 0.0;    // host wall time of the lazy index/record builds
  int built = 0;           // ND_IDX_* bits of the structures built
  int skipped = 0;         // ND_IDX_* bits left out for lack of room (plain-CSR path)
  int device = 0;
  // col / w / pre are device views of page-locked host arrays (zero copy,
  // nd_graph_create_mapped): not freed here, unregistered when we registered
  bool host_mapped = false;
  std::vector<const void*> registered;
};

// nd_graph_footprint bits (one per optional structure, nd_index.cu)
enum { ND_IDX_VREC = 1, ND_IDX_NBW = 2, ND_IDX_NBP = 4, ND_IDX_NBU = 8, ND_IDX_GUIDE = 16,
       ND_IDX_HSET = 32, ND_IDX_LINES = 64 };

constexpr int ND_N_FIELDS = 14;
constexpr int ND_N_COUNTERS = 12;

struct nd_result {
  int64_t n = 0;
  int64_t n_steps = 0;
  int64_t total_sampled = 0;
  int64_t total_recorded = 0;
  void* ptr[ND_N_FIELDS] = {};
  int64_t cnt[ND_N_FIELDS] = {};
  int esz[ND_N_FIELDS] = {8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 8, 4, 4};  // bytes per element
  int64_t counters[ND_N_COUNTERS] = {};
  double prof_ms[4] = {};  // schedule, sample, compaction (nd_set_profiling)
  // per-step build (schedule / inversion) and sample times of step-structured
  // runs (nd_set_profiling): RunStats.timings (driver.py:42-48)
  std::vector<float> step_build_ms, step_sample_ms;
  cudaStream_t stream = nullptr;
  // a field the run leaves to be built on first request (step rows of the
  // fixed-layout k-hop): `lazy_field` is filled by `lazy_build`; `lazy_free`
  // releases the device buffers it captured (after building, or at destroy)
  int lazy_field = -1;
  std::function<int(nd_result*)> lazy_build;
  std::function<void()> lazy_free;

  void set(int f, void* p, int64_t c) {
    ptr[f] = p;
    cnt[f] = c;
  }
};

// counters slots (nd_result_counters)
enum { NDC_ITEMS = 0, NDC_PAIRS = 1, NDC_N2V_TRIES = 2, NDC_N2V_PROBES = 3, NDC_SEARCH = 4,
       NDC_PAIR_BYTES = 5, NDC_SLOT_BYTES = 6, NDC_STEPS = 7, NDC_LAUNCHES = 8,
       NDC_RAND_SECTORS = 9, NDC_TP_STAGED = 10, NDC_TP_INPLACE = 11 };

// app parameters as the kernels see them (_ckernels.pyx:157-181)
struct NdApp {
  int code = 0;
  double term = 0.0;
  double f_ret = 0.0, f_adj = 0.0, f_far = 0.0, f_max = 0.0;
};

int nd_make_app(int code, const double* params, int64_t n_params, NdApp* a);
int nd_pool_init();
int64_t* nd_pinned_scratch();
// Small device->host read, synchronous on `s`: a one-block kernel copies the
// bytes into mapped pinned memory, then the stream is synchronised.  Unlike a
// cudaMemcpyAsync it does not queue behind bulk device->host copies on the
// copy engine (the host pipeline's row copies on another stream).
int nd_d2h(void* dst, const void* src, int64_t bytes, cudaStream_t s);
int nd_graph_ensure_index(nd_graph* G, int want_hset, int want_guide, cudaStream_t s);
int nd_graph_ensure_records(nd_graph* G, int want_tries, cudaStream_t s);
int nd_graph_ensure_lines(nd_graph* G, cudaStream_t s);
int nd_dedup_segments(const int32_t* sid, const int32_t* val, int64_t m, int64_t n_samples,
                      int64_t n_vertices, int32_t** out_sid, int32_t** out_val, int64_t* out_m,
                      int64_t* counts, cudaStream_t s);
inline bool nd_unique_at(const uint8_t* mask, int64_t n, int64_t step) {
  if (!mask || n <= 0) return false;
  return mask[step < n ? step : n - 1] != 0;
}

// device counters block reset/read helpers
int nd_uniform_roots_i32(const nd::DevGraph& g, int64_t count, uint64_t seed, int64_t sample_lo,
                         int64_t n, int32_t* roots, cudaStream_t s);

int nd_profiling();  // nd_set_profiling state
int nd_concurrency();  // nd_set_concurrency state of the calling thread

// CUDA-event marks on a run's stream, recorded only under nd_set_profiling(1):
// phase totals (res->prof_ms) and per-step build / sample times
// (StepTiming, transit_parallel.py:204-228).  Read after the run's final sync.
struct Profiler {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<std::array<size_t, 4>> steps;  // event indices: start, built, sampled; steps spanned
  Profiler() = default;
  explicit Profiler(cudaStream_t st) : on(nd_profiling() != 0), s(st) {}
  size_t mark() {  // index of the recorded event (0 when off)
    if (!on) return 0;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
    return ev.size() - 1;
  }
  // span: steps one launch covers (their times split evenly between them)
  void step_begin(size_t span = 1) { if (on) steps.push_back({mark(), 0, 0, span}); }
  void step_built() { if (on && !steps.empty()) steps.back()[1] = mark(); }
  void step_sampled() { if (on && !steps.empty()) steps.back()[2] = mark(); }
  float between(size_t a, size_t b) {
    float ms = 0;
    if (on && a < ev.size() && b < ev.size()) cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return ms;
  }
  // per-step times into the result; returns (sum build, sum sample)
  std::array<double, 2> to_result(nd_result* r) {
    std::array<double, 2> tot{0.0, 0.0};
    if (!on) return tot;
    for (auto& st : steps) {
      const float b = between(st[0], st[1]), m = between(st[1], st[2]);
      for (size_t k = 0; k < st[3]; k++) {
        r->step_build_ms.push_back(b / st[3]);
        r->step_sample_ms.push_back(m / st[3]);
      }
      tot[0] += b;
      tot[1] += m;
    }
    return tot;
  }
  void destroy() {
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
  }
};

// NVTX range over a host scope (the run and its phases show up by name in
// nsys / ncu --nvtx timelines); header-only NVTX v3, no-op without a tool
struct NvtxRange {
  explicit NvtxRange(const char* m) { nvtxRangePushA(m); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
