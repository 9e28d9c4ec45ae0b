// nd_bulk.cuh — Blackwell row staging: 1-D bulk copies (cp.async.bulk, SASS
// UBLKCP) from global into shared memory, completion tracked by an mbarrier
// transaction count (SASS SYNCS), and the hub-bucket transit inversion shared
// by the transit-parallel engines.
//
// Row staging (the paper's thread-block / grid kernels cache the transit's
// adjacency in shared memory): one elected thread arms the
// stage's mbarrier with the byte count and issues one bulk copy of the
// 16-byte-aligned superset of the row; the consumers wait on the barrier's
// phase.  Two stages per CTA (or per warp) let the copy of the next hub's row
// run while the current one is sampled.  The column array is allocated with
// 16 bytes of slack past a multiple of 4 entries (nd_col_alloc) so the aligned
// superset of the last row stays inside the allocation.
#pragma once

#include <stdint.h>

namespace nd {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// make the initialised barriers visible to the async proxy (bulk copies)
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// global -> shared bulk copy; dst/src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The aligned superset of the int32 row [lo, lo+deg): copy start (in
// entries, a multiple of 4), entry count (a multiple of 4) and where the
// row's entry 0 lands in the staged buffer.
struct RowSpan {
  int64_t a;      // first copied entry
  uint32_t n;     // copied entries
  uint32_t skew;  // row entry k is at buf[skew + k]
};
__host__ __device__ __forceinline__ RowSpan row_span(int64_t lo, int64_t deg) {
  RowSpan r;
  r.a = lo & ~(int64_t)3;
  const int64_t b = (lo + deg + 3) & ~(int64_t)3;
  r.n = (uint32_t)(b - r.a);
  r.skew = (uint32_t)(lo - r.a);
  return r;
}

// Elected thread: arm `bar` and copy the row's aligned superset into buf.
__device__ __forceinline__ void stage_row_bulk(int32_t* buf, const int32_t* col, const RowSpan& sp,
                                               uint64_t* bar) {
  mbar_arrive_expect_tx(bar, sp.n * 4u);
  bulk_g2s(buf, col + sp.a, sp.n * 4u, bar);
}

}  // namespace nd
