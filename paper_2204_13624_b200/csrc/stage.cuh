// Bulk-async (TMA 1D) staging primitives for the streaming kernels.
//
// A producer warp moves whole component rows of a tile (SoA: one contiguous
// run of cells per component) from HBM into a ring of shared-memory stages
// with cp.async.bulk, completing on an mbarrier transaction count; consumer
// warps wait on the stage's "full" barrier, compute from shared memory and
// release the stage on its "empty" barrier. Memory-level parallelism then
// depends on the stages in flight, not on the consumers' register budget
// (the matvec needs ~200 registers per thread, which caps it at 8 warps/SM).
#pragma once

#include <cstdint>

namespace combo_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

// global -> shared bulk copy (16-byte aligned addresses, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// bulk prefetch of a contiguous range into L2 (no completion tracking); the
// range is trimmed to 16-byte granularity
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, size_t bytes) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~uintptr_t(15);
  if (e <= a) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(uint32_t(e - a)) : "memory");
}

// ring position of the k-th tile a block processes
struct Ring {
  int stages;
  int s = 0;
  uint32_t phase = 0;
  __device__ explicit Ring(int n) : stages(n) {}
  __device__ void next() {
    if (++s == stages) {
      s = 0;
      phase ^= 1u;
    }
  }
};

}  // namespace combo_dev
