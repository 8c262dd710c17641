// umma.cuh — tcgen05 / TMA tensor-copy helpers shared by the tensor-core
// kernels (coarse_tc.cu: batched coarse quantizer; listscan.cu: list-major
// batched scan). Operands are fp32 tiles in the canonical K-major
// 128-byte-swizzle layout TMA writes; the MMA is kind::tf32 into TMEM.
#pragma once
#include <cuda.h>
#include <cstdint>

#include "dev_common.cuh"

namespace laivg {
namespace dev {

// UMMA shared-memory descriptor of a K-major operand tile in the canonical
// 128-byte-swizzle layout TMA writes (8-row x 128-byte atoms, 1024 B apart).
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
  uint64_t desc = 0;
  desc |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);      // start address
  desc |= static_cast<uint64_t>(1u) << 16;                      // LBO (unused: swizzled K-major)
  desc |= static_cast<uint64_t>(1024u >> 4) << 32;              // SBO: next 8-row atom
  desc |= static_cast<uint64_t>(1u) << 46;                      // descriptor version (sm_100)
  desc |= static_cast<uint64_t>(2u) << 61;                      // SWIZZLE_128B
  return desc;
}

// Instruction descriptor: kind::tf32, fp32 accumulator, both operands K-major.
__host__ __device__ constexpr uint32_t tf32_idesc(uint32_t M, uint32_t N) {
  return (1u << 4)           // D format: F32
         | (2u << 7)         // A format: TF32
         | (2u << 10)        // B format: TF32
         | ((N >> 3) << 17)  // N / 8
         | ((M >> 4) << 24); // M / 16
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x,
                                            int32_t y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

} // namespace dev
} // namespace laivg
