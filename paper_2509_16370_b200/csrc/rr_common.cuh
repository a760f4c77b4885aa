// rr_common.cuh -- small device helpers shared by the B200 kernels of this library.
// (Product code only; the CPU oracle under oracle/ shares nothing with this file.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rr.h"

#define RR_FULL_MASK 0xffffffffu

namespace rrk {

// Per-instance shared-memory slot stride (doubles) for lane groups of width lg < 16: the 16/lg
// groups of a half-warp (one 64-bit shared wavefront) start lg double-banks apart, so broadcast
// reads of the same offset -- and stride-1 / odd-stride column reads -- of different instances
// fall in disjoint banks instead of serialising.
__host__ __device__ constexpr int group_stride(int slot, int lg) {
  return lg >= 16 ? ((slot + 1) & ~1) : ((slot + 1) & ~1) + ((lg - (((slot + 1) & ~1) % 16) + 16) % 16);
}

// Block index of stage i of a dynamics (A, B) or cost (Q, M, R) operand of instance `inst`
// (include/rr.h RR_FLAG_SHARED_* / RR_FLAG_STAGE_INVARIANT_*): [batch][N] | [N] | [batch] | [1].
__host__ __device__ __forceinline__ int64_t dyn_blk(int fl, int64_t inst, int64_t N, int64_t i) {
  const int64_t b = (fl & RR_FLAG_SHARED_DYN) ? 0 : inst;
  return (fl & RR_FLAG_STAGE_INVARIANT_DYN) ? b : b * N + i;
}
__host__ __device__ __forceinline__ int64_t cost_blk(int fl, int64_t inst, int64_t N, int64_t i) {
  const int64_t b = (fl & RR_FLAG_SHARED_COST) ? 0 : inst;
  return (fl & RR_FLAG_STAGE_INVARIANT_COST) ? b : b * N + i;
}

// LAPACK 'L' packed index of (r, c) with r >= c in an n×n symmetric matrix.
__host__ __device__ __forceinline__ int pidx(int n, int r, int c) { return c * (2 * n - c - 1) / 2 + r; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Ampere-style asynchronous global->shared copies (SASS LDGSTS), L1-bypassing for 16 B.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Copy `cnt` doubles global->shared with the `width` lanes of a lane group (lane index j).
__device__ __forceinline__ void copy_async(double* dst, const double* src, int cnt, int j, int width) {
  const bool vec = (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0) &&
                   ((cnt & 1) == 0);
  if (vec) {
    for (int e = 2 * j; e < cnt; e += 2 * width) cp_async16(dst + e, src + e);
  } else {
    for (int e = j; e < cnt; e += width) cp_async8(dst + e, src + e);
  }
}

// ---- TMA 1-D bulk copies (cp.async.bulk, SASS UBLKCP) completing on a shared-memory mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-byte aligned both sides)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global bulk copy of `bytes` (multiple of 16, 16-byte aligned both sides), bulk-group completion
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// the shared-memory sources of this thread's committed bulk stores have been read (may be reused)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// this thread's committed bulk stores are complete (globally performed)
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// order this thread's prior generic-proxy shared accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Reciprocal for pivots: hardware approximation (rcp.approx.ftz.f64, ~2^-20 relative) refined by
// two Newton steps (error ~2^-80 before rounding, i.e. within 1 ulp of 1/d).  No IEEE slow path:
// d = 0 gives inf/NaN, which the pivot checks (d > 0) report anyway.
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ int32_t mk_status(int code, int stage) { return code | (stage << 8); }

// Status combine key: the failure met first in the backward sweep (highest stage) wins; at
// equal stage the larger code wins (S_NOT_PD is detected before G_NOT_PD, as in the oracle).
__device__ __forceinline__ int64_t status_key(int32_t st) {
  return st == 0 ? -1 : ((int64_t)(st >> 8) << 8) | (st & 0xff);
}

}  // namespace rrk
