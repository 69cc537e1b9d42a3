// TMA probe, written from scratch (round 2): does cp.async.bulk.tensor work on
// this pool's B200s?  2D and 3D u16 boxes, descriptor passed as a
// __grid_constant__ kernel parameter (the CUTLASS convention), mbarrier
// completion, result compared element by element with the source.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma2 scripts/micro/tma2.cu -lcuda
//   ./tma2
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__constant__ CUtensorMap c_map;
template <int RANK, int SRC>
__global__ void tma_load(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, uint16_t* out, int x, int y, int z, int bytes) {
  const CUtensorMap* mp = SRC == 0 ? &map : (SRC == 1 ? gmap : &c_map);
  if (SRC == 1 && threadIdx.x == 0)
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" :: "l"(gmap) : "memory");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    if (RANK == 2)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sa(smem)),
          "l"(reinterpret_cast<uint64_t>(mp)), "r"(x), "r"(y), "r"(sa(&bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(sa(smem)),
          "l"(reinterpret_cast<uint64_t>(mp)), "r"(x), "r"(y), "r"(z), "r"(sa(&bar))
          : "memory");
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(sa(&bar)) : "memory");
  }
  const uint16_t* s = reinterpret_cast<const uint16_t*>(smem);
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
  const int SRCV = argc > 1 ? atoi(argv[1]) : 0;
  const int n = 96;
  std::vector<uint16_t> h((size_t)n * n * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
  uint16_t *d, *o;
  CK(cudaMalloc(&d, h.size() * 2));
  CK(cudaMalloc(&o, 1 << 20));
  CK(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  int fails = 0;
  for (int rank = 2; rank <= 3; ++rank) {
    for (int bx : {32, 40, 64}) {
      const int by = 16, bz = rank == 3 ? 8 : 1;
      CUtensorMap map;
      cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
      cuuint64_t strides[2] = {(cuuint64_t)n * 2, (cuuint64_t)n * n * 2};
      cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz}, es[3] = {1, 1, 1};
      CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, rank, d, dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int bytes = bx * by * bz * 2;
      const int x = 5, y = 7, z = 9;
      CUtensorMap* gm;
      CK(cudaMalloc(&gm, sizeof(CUtensorMap)));
      CK(cudaMemcpy(gm, &map, sizeof map, cudaMemcpyHostToDevice));
      CK(cudaMemcpyToSymbol(c_map, &map, sizeof map));
      decltype(&tma_load<2, 0>) ks[2][3] = {{tma_load<2, 0>, tma_load<2, 1>, tma_load<2, 2>}, {tma_load<3, 0>, tma_load<3, 1>, tma_load<3, 2>}};
      auto k = ks[rank - 2][SRCV];
      printf("map@host %p aligned64=%d; descriptor source %d (0 param, 1 global, 2 constant)\n", (void*)&map, (int)(((uintptr_t)&map & 63) == 0), SRCV);
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      k<<<1, 128, bytes + 1024>>>(map, gm, o, x, y, z, bytes);
      cudaError_t e = cudaDeviceSynchronize();
      int bad = -1;
      if (e == cudaSuccess) {
        std::vector<uint16_t> g(bytes / 2);
        CK(cudaMemcpy(g.data(), o, bytes, cudaMemcpyDeviceToHost));
        bad = 0;
        for (int zz = 0; zz < bz; ++zz)
          for (int yy = 0; yy < by; ++yy)
            for (int xx = 0; xx < bx; ++xx)
              bad += g[((size_t)zz * by + yy) * bx + xx] !=
                     h[((size_t)(zz + (rank == 3 ? z : 0)) * n + yy + y) * n + xx + x];
      }
      printf("TMA %dD box %dx%dx%d: encode=%d launch=%s mismatches=%d\n", rank, bx, by, bz, (int)r,
             cudaGetErrorString(e), bad);
      if (e != cudaSuccess || bad != 0) ++fails;
      if (e != cudaSuccess) return 2;   // sticky error: stop
    }
  }
  printf("TMA probe: %s\n", fails ? "FAIL" : "OK");
  return fails ? 1 : 0;
}
