// bfp_bulk.cuh -- bulk-async (TMA engine) staged stencil pipeline for the 2-D
// int32 hot path on sm_100a.
//
// A CTA owns a strip of W = 4*T columns and marches R rows.  One elected
// thread streams rows global -> shared with cp.async.bulk (the TMA engine's 1-D
// bulk copy) into a ring of D+3 x-row slots and D+1 y-row slots, signalling a
// ring of mbarriers with complete_tx; the consumers wait on the mbarrier of the
// step, read their 4 points and the 3-row neighbourhood from shared memory,
// and write one int4.  Bytes in flight are bounded by shared memory (D steps
// of (W+8)+W words per CTA), not by registers.  Slots are handed back through
// "empty" mbarriers (one arrival per warp) instead of a block-wide barrier, so
// only the producer waits for the slowest warp and the others run ahead.
#pragma once
#include <cuda.h>  // CUtensorMap (tiled TMA descriptors; encoded through the runtime's driver entry point)

#include "bfp_dev.cuh"

namespace bfpdev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D bulk copy global -> shared (16-B aligned, size multiple of 16), completes tx on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

#ifndef BFP_BULK_T
#define BFP_BULK_T 256
#endif
#ifndef BFP_B2_MINB  // resident CTAs per SM the 2-D pipeline is compiled for
#define BFP_B2_MINB 3    // with D = 3 (tools/ab_b2.sh, profiles/r1_ab_b2.txt)
#endif
// 3-D tiled TMA: box at tensor coordinates (c0, c1, c2) -> shared, completes tx on bar
__device__ __forceinline__ void tma_g2s_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                           int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kBulkT = BFP_BULK_T;      // threads per CTA (one 4-group each)
constexpr int kBulkW = 4 * kBulkT;      // strip width in columns
#ifndef BFP_BULK_D
// C2 4095^2 after the balanced march depth: D = 3 at 3 CTAs/SM residual 0.81, Jacobi 0.77;
// D = 2 at 4/SM 0.78 / 0.75; D = 4 at 3/SM 0.81 / 0.76; D = 4 at 2/SM 0.77 / 0.71
#define BFP_BULK_D 3
#endif
#ifndef BFP_B2_EMPTY  // A/B switch: empty mbarriers (1) or a block barrier (0) per step
#define BFP_B2_EMPTY 1
#endif
constexpr int kBulkD = BFP_BULK_D;      // prefetch depth (steps in flight)
constexpr int kBulkXS = kBulkD + 3;     // x-row slots
constexpr int kBulkYS = kBulkD + 1;     // y-row slots / mbarriers
constexpr int kBulkXW = kBulkW + 8;     // x slot width (4-word halo each side)
// full barriers (tx completion) and empty barriers (one arrival per consumer warp)
constexpr size_t kBulkSmem =
    (size_t)(kBulkXS * kBulkXW + kBulkYS * kBulkW) * 4 + 2 * kBulkYS * 8 + 64;

}  // namespace bfpdev
