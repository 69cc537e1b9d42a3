// plain bulk copy (cp.async.bulk, non-tensor) global -> shared with mbarrier completion
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint16_t* src, uint16_t* out, int bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(smem)), "l"(src), "r"(bytes), "r"(sa(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(sa(&bar)) : "memory");
  const uint16_t* s = reinterpret_cast<const uint16_t*>(smem);
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = s[i];
}
int main() {
  const int bytes = 16384;
  uint16_t *d, *o; cudaMalloc(&d, bytes); cudaMalloc(&o, bytes);
  uint16_t h[bytes / 2]; for (int i = 0; i < bytes / 2; ++i) h[i] = (uint16_t)(i * 37 + 1);
  cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
  k<<<1, 128, bytes>>>(d, o, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  uint16_t g[bytes / 2]; int bad = -1;
  if (e == cudaSuccess) { cudaMemcpy(g, o, bytes, cudaMemcpyDeviceToHost); bad = 0; for (int i = 0; i < bytes / 2; ++i) bad += g[i] != h[i]; }
  printf("bulk copy: %s mismatches=%d\n", cudaGetErrorString(e), bad);
  return e != cudaSuccess;
}
