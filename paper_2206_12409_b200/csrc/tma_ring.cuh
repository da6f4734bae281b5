// mbarrier + 1-D bulk-copy (cp.async.bulk) helpers of the TMA-streamed apply kernels.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace vsie {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a global range (no shared memory, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// d0 (column j, all lanes) and d1 (column j + 1): after the call lane l holds the full
// column sum of column j + (l >= 16) -- one exchange of the other half's column, then a
// 16-lane butterfly (10 shuffles of 64 bits for two columns instead of 20)
__device__ __forceinline__ cplx pair_reduce(cplx d0, cplx d1, int lane) {
  const bool hi = lane >= 16;
  cplx keep = hi ? d1 : d0, send = hi ? d0 : d1;
  keep.x += __shfl_xor_sync(0xffffffffu, send.x, 16);
  keep.y += __shfl_xor_sync(0xffffffffu, send.y, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    keep.x += __shfl_xor_sync(0xffffffffu, keep.x, o);
    keep.y += __shfl_xor_sync(0xffffffffu, keep.y, o);
  }
  return keep;
}

}  // namespace tma
}  // namespace vsie
