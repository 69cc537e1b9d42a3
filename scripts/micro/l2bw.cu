// L2 (and HBM) read-bandwidth microbenchmark for the §8(d)(ii) roofline: a
// read-only streaming kernel (16-byte loads, L1 bypassed with ld.global.cg) over
// a working set of S bytes, repeated until >= 4 GB have been read; CUDA events,
// best of 5.  A working set well inside the 126 MB L2 measures L2 bandwidth;
// 2 GiB measures HBM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw scripts/micro/l2bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void __launch_bounds__(512) rd(const uint4* __restrict__ p, size_t n16, int reps, uint32_t* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t j = i + u * stride;
        if (j < n16) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                                  : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
        else v[u] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d, L2 %d bytes\n", sms, l2);
  const size_t maxb = (size_t)2 << 30;
  uint4* p;
  uint32_t* sink;
  cudaMalloc(&p, maxb);
  cudaMalloc(&sink, 4);
  cudaMemset(p, 1, maxb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t sizes_mb[] = {4, 8, 16, 24, 32, 48, 64, 80, 96, 2048};
  for (size_t mb : sizes_mb) {
    const size_t bytes = mb << 20, n16 = bytes / 16;
    const int reps = (int)std::max<size_t>(1, ((size_t)4 << 30) / bytes);
    for (int bpsm : {4, 8}) {
      const int grid = sms * bpsm, block = 512;
      rd<<<grid, block>>>(p, n16, 1, sink);   // warm (fills L2)
      float best = 1e30f;
      for (int t = 0; t < 5; ++t) {
        cudaEventRecord(a);
        rd<<<grid, block>>>(p, n16, reps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
      }
      printf("working set %5zu MB, %d CTAs/SM: %8.1f GB/s\n", mb, bpsm, (double)bytes * reps / (best * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
