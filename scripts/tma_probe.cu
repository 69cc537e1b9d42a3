// Standalone TMA probe: load a 32^3 u16 box with cp.async.bulk.tensor and compare.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe scripts/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE, int VAR>
__global__ void probe(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, uint16_t* out, int x,
                      int y, int z, int bytes) {
  extern __shared__ uint8_t dsm[];
  uint16_t* brick = reinterpret_cast<uint16_t*>(dsm + ((1024u - (smem_u32(dsm) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const void* m = MODE == 0 ? (const void*)&map : (const void*)gmap;
    if (VAR != 4)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes)
                   : "memory");
    if (VAR == 2) asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
    if (VAR == 4) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    if (VAR == 5)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(brick)), "l"(out + 65536), "r"(bytes), "r"(smem_u32(&bar)) : "memory");
    if (VAR == 0 || VAR == 2 || VAR == 3)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(brick)),
          "l"(m), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar))
          : "memory");
    if (VAR == 7)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(brick)),
          "l"(m), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar))
          : "memory");
    if (VAR == 6)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(brick)),
          "l"(m), "r"(x), "r"(y), "r"(smem_u32(&bar))
          : "memory");
    if (VAR == 1)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(brick)),
          "l"(m), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar))
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = brick[i];
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;     // 0 param map, 1 global map
  const int B = argc > 2 ? atoi(argv[2]) : 32;       // box edge (x = y = B), z = BZ
  const int BZ = argc > 3 ? atoi(argv[3]) : B;
  const int n = 64;
  std::vector<uint16_t> h(n * n * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 7 + 3);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 65536 * 4);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  if (argc > 5) enc = cuTensorMapEncodeTiled;   // direct driver call (-lcuda)
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)n * 2, (cuuint64_t)n * n * 2};
  const int BXI = getenv("BX") ? atoi(getenv("BX")) : B;
  const int SW = getenv("SW") ? atoi(getenv("SW")) : 0;
  cuuint32_t box[3] = {(cuuint32_t)BXI, (cuuint32_t)B, (cuuint32_t)BZ}, es[3] = {1, 1, 1};
  const unsigned char* mb = reinterpret_cast<const unsigned char*>(&map);
  const int var0 = argc > 4 ? atoi(argv[4]) : 0;
  const bool f32 = getenv("DT") != nullptr;
  if (f32) { strides[0] *= 2; strides[1] *= 2; }
  CUresult r = enc(&map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, var0 == 6 ? 2 : 3, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)SW, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("var %s mode %d box %dx%dx%d encode: %d (entry %d) map@%p\n", argc > 4 ? argv[4] : "0", mode, B, B, BZ, (int)r, (int)q, (void*)&map);
  for (int i = 0; i < 64; ++i) printf("%02x%s", mb[i], i % 16 == 15 ? "\n" : "");
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  cudaMemcpy(gmap, &map, sizeof map, cudaMemcpyHostToDevice);
  const int bytes = BXI * B * BZ * (getenv("DT") ? 4 : 2);
  const int var = argc > 4 ? atoi(argv[4]) : 0;   // 0 base, 1 shared::cta dst, 2 prefetch, 3 cluster launch
  decltype(&probe<0, 0>) ks[2][8] = {{probe<0, 0>, probe<0, 1>, probe<0, 2>, probe<0, 3>, probe<0, 4>, probe<0, 5>, probe<0, 6>, probe<0, 7>},
                                     {probe<1, 0>, probe<1, 1>, probe<1, 2>, probe<1, 3>, probe<1, 4>, probe<1, 5>, probe<1, 6>, probe<1, 7>}};
  auto k = ks[mode][var];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
  if (var == 3) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = bytes + 256;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, k, map, (const CUtensorMap*)gmap, o, 5, 7, 9, bytes);
    printf("  launchEx: %s\n", cudaGetErrorString(le));
  } else {
    k<<<1, 128, bytes + 2048>>>(map, gmap, o, 5, 7, 9, bytes);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("  result: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<uint16_t> got(bytes / 2);
  cudaMemcpy(got.data(), o, bytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int zz = 0; zz < BZ; ++zz)
    for (int yy = 0; yy < B; ++yy)
      for (int xx = 0; xx < BXI; ++xx)
        bad += got[(zz * B + yy) * BXI + xx] != h[((zz + 9) * n + yy + 7) * n + xx + 5];
  printf("  mismatches %d (BX %d SW %d)\n", bad, BXI, SW);
  return 0;
}
