// tma.cuh — the Tensor Memory Accelerator and mbarrier helpers shared by the
// TMA-staged volume passes (stencil.cu: the blur; seeds.cu: the MAXIMA pass).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace snk {

static __device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

static __device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

static __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

// One elected thread: arm the barrier for `bytes` and copy the box at (x, y, z).
static __device__ __forceinline__ void tma_load_box(const CUtensorMap* map, void* dst, uint64_t* bar, int x, int y, int z,
                                             uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes to dst (edge fix-up) first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
      : "memory");
}

// u16 volume (nx, ny, nz) x-fastest as a 3D tensor map with box (bx, by, 1);
// out-of-range box elements load as zeros.  On this pool's GPUs the innermost
// box start coordinate must be a multiple of 8 elements (16 bytes) or the load
// faults (profiles/r2_tma_probe.md).
int32_t volume_map(CUtensorMap* map, const uint16_t* base, int nx, int ny, int nz, int bx, int by);
bool tma_available();

}  // namespace snk
