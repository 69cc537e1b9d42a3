// Gather-throughput microbenchmark for the a5 evolve kernel's 8-tap trilinear
// lookups: shared-memory brick (8 LDS.U16 per sample, the product's path) vs
// texture gathers (2 TLD4 per sample on a layered u16 array: one 2x2 footprint
// per z plane) vs both (alternate samples), at several CTAs per SM.  Sample
// points are uniform in a radius-13 box around a per-CTA centre (C4: r0 = 13),
// the full trilinear arithmetic is done, per-thread sums are written so that
// variants can be compared (the TLD4 component order is checked against the
// brick path).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o texgather scripts/micro/texgather.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NX = 2048, NY = 2048, NZ = 512;
constexpr int S = 33, SX = 34, SP = SX * S;   // brick like the product's (34 x 33 x 33 u16)
constexpr int HALF = 13;

__device__ __forceinline__ uint32_t xs(uint32_t& s) {
  s ^= s << 13; s ^= s >> 17; s ^= s << 5;
  return s;
}
__device__ __forceinline__ float uoff(uint32_t x) {   // [-13, 13)
  return __fmaf_rn(__uint_as_float(0x3F800000u | (x >> 9)) - 1.0f, 2.0f * HALF, -(float)HALF);
}
__device__ __forceinline__ float lerp(float a, float b, float f) { return __fmaf_rn(f, b - a, a); }
__device__ __forceinline__ float mag(uint32_t v) {
  float r;
  asm("cvt.rn.f32.u32 %0, %1;" : "=f"(r) : "r"(v));
  return r;
}

__device__ __forceinline__ void tld4(cudaTextureObject_t t, int layer, float x, float y, uint32_t v[4]) {
  asm volatile("tld4.r.a2d.v4.u32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %8}];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "l"(t), "r"(layer), "f"(x), "f"(y), "f"(0.0f));
}

__device__ __forceinline__ void centre(int b, int& cx, int& cy, int& cz) {
  uint32_t h = (uint32_t)b * 2654435761u + 12345u;
  h ^= h >> 15; h *= 0x2c1b3c6du; h ^= h >> 12;
  cx = 16 + (int)(h % (NX - 40));
  h = h * 0x297a2d39u + 7; h ^= h >> 13;
  cy = 16 + (int)(h % (NY - 40));
  h = h * 0x297a2d39u + 7; h ^= h >> 13;
  cz = 16 + (int)(h % (NZ - 40));
}

// MODE 0: brick, 1: tex, 2: alternate
template <int MODE>
__global__ void __launch_bounds__(128) gather(const uint16_t* __restrict__ img, cudaTextureObject_t tex, int ns,
                                              float* out) {
  extern __shared__ uint16_t brick[];
  int cx, cy, cz;
  centre(blockIdx.x, cx, cy, cz);
  const int bx = (cx - 16) & ~1, by = cy - 16, bz = cz - 16;
  if (MODE != 1) {
    for (int w = threadIdx.x; w < S * S * (SX / 2); w += blockDim.x) {
      const int col = w % (SX / 2), row = w / (SX / 2), ry = row % S, rz = row / S;
      reinterpret_cast<uint32_t*>(brick)[w] =
          *reinterpret_cast<const uint32_t*>(img + ((size_t)(bz + rz) * NY + by + ry) * NX + bx + 2 * col);
    }
    __syncthreads();
  }
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * 128 + threadIdx.x) * 747796405u;
  if (!s) s = 1;
  float acc = 0.f;
#pragma unroll 4
  for (int k = 0; k < ns; ++k) {
    const float px = cx + uoff(xs(s)), py = cy + uoff(xs(s)), pz = cz + uoff(xs(s));
    const float fx0 = floorf(px), fy0 = floorf(py), fz0 = floorf(pz);
    const float fx = px - fx0, fy = py - fy0, fz = pz - fz0;
    const int ix = (int)fx0, iy = (int)fy0, iz = (int)fz0;
    float v000, v100, v010, v110, v001, v101, v011, v111;
    const bool use_tex = MODE == 1 || (MODE == 2 && (k & 1));
    if (!use_tex) {
      const uint16_t* p = brick + (iz - bz) * SP + (iy - by) * SX + (ix - bx);
      v000 = mag(p[0]); v100 = mag(p[1]); v010 = mag(p[SX]); v110 = mag(p[SX + 1]);
      v001 = mag(p[SP]); v101 = mag(p[SP + 1]); v011 = mag(p[SP + SX]); v111 = mag(p[SP + SX + 1]);
    } else {
      uint32_t a[4], b[4];
      tld4(tex, iz, fx0 + 1.0f, fy0 + 1.0f, a);
      tld4(tex, iz + 1, fx0 + 1.0f, fy0 + 1.0f, b);
      // gather order: x = (i0, j1), y = (i1, j1), z = (i1, j0), w = (i0, j0)
      v000 = mag(a[3]); v100 = mag(a[2]); v010 = mag(a[0]); v110 = mag(a[1]);
      v001 = mag(b[3]); v101 = mag(b[2]); v011 = mag(b[0]); v111 = mag(b[1]);
    }
    const float t0 = lerp(lerp(v000, v100, fx), lerp(v010, v110, fx), fy);
    const float t1 = lerp(lerp(v001, v101, fx), lerp(v011, v111, fx), fy);
    acc += lerp(t0, t1, fz);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void order_probe(cudaTextureObject_t tex, uint32_t* o) {
  uint32_t v[4];
  tld4(tex, 3, 5.0f + 1.0f, 7.0f + 1.0f, v);
  for (int i = 0; i < 4; ++i) o[i] = v[i];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, clock %d kHz\n", sms, clk);
  const size_t n = (size_t)NX * NY * NZ;
  std::vector<uint16_t> h(n);
  uint32_t r = 1;
  for (size_t i = 0; i < n; ++i) { r = r * 1664525u + 1013904223u; h[i] = (uint16_t)(r >> 16); }
  uint16_t* img;
  CK(cudaMalloc(&img, n * 2));
  CK(cudaMemcpy(img, h.data(), n * 2, cudaMemcpyHostToDevice));
  cudaChannelFormatDesc cd = cudaCreateChannelDesc(16, 0, 0, 0, cudaChannelFormatKindUnsigned);
  cudaArray_t arr;
  CK(cudaMalloc3DArray(&arr, &cd, make_cudaExtent(NX, NY, NZ), cudaArrayLayered));
  cudaMemcpy3DParms cp;
  memset(&cp, 0, sizeof cp);
  cp.srcPtr = make_cudaPitchedPtr(img, NX * 2, NX, NY);
  cp.dstArray = arr;
  cp.extent = make_cudaExtent(NX, NY, NZ);
  cp.kind = cudaMemcpyDeviceToDevice;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  CK(cudaMemcpy3D(&cp));
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("array copy %.3f ms (%.1f GB/s)\n", ms, 2.0 * n * 2 / ms / 1e6);
  cudaResourceDesc rd;
  memset(&rd, 0, sizeof rd);
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = arr;
  cudaTextureDesc td;
  memset(&td, 0, sizeof td);
  td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  uint32_t* dord;
  CK(cudaMalloc(&dord, 16));
  order_probe<<<1, 1>>>(tex, dord);
  uint32_t ho[4];
  CK(cudaMemcpy(ho, dord, 16, cudaMemcpyDeviceToHost));
  auto at = [&](int x, int y, int z) { return (uint32_t)h[((size_t)z * NY + y) * NX + x]; };
  printf("tld4 (x0=5, y0=7, layer 3): %u %u %u %u ; (5,7)=%u (6,7)=%u (5,8)=%u (6,8)=%u\n", ho[0], ho[1], ho[2],
         ho[3], at(5, 7, 3), at(6, 7, 3), at(5, 8, 3), at(6, 8, 3));

  const int ns = 2048;
  const int smem_brick = SP * S * 2;
  float* out;
  const int maxgrid = sms * 16 * 8;
  CK(cudaMalloc(&out, (size_t)maxgrid * 128 * 4));
  std::vector<float> ref, got;
  for (int mode = 0; mode < 3; ++mode) {
    for (int cps : {2, 3, 4, 6, 8, 12}) {
      int smem = 227 * 1024 / cps - 1024;
      if (mode != 1 && smem < smem_brick) continue;
      if (smem > 48 * 1024) {
        if (mode == 0) cudaFuncSetAttribute(gather<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (mode == 1) cudaFuncSetAttribute(gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (mode == 2) cudaFuncSetAttribute(gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      }
      const int grid = sms * cps * 8;
      auto launch = [&]() {
        if (mode == 0) gather<0><<<grid, 128, smem>>>(img, tex, ns, out);
        if (mode == 1) gather<1><<<grid, 128, smem>>>(img, tex, ns, out);
        if (mode == 2) gather<2><<<grid, 128, smem>>>(img, tex, ns, out);
      };
      launch();
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int t = 0; t < 3; ++t) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      const double samples = (double)grid * 128 * ns;
      const double gs = samples / best / 1e6;
      printf("mode %d (%s) %2d CTAs/SM: %8.3f ms  %7.1f G samples/s  %.3f samples/clk/SM\n", mode,
             mode == 0 ? "brick" : mode == 1 ? "tex  " : "both ", cps, best, gs, gs * 1e9 / (sms * clk * 1e3));
      std::vector<float> hv((size_t)grid * 128);
      CK(cudaMemcpy(hv.data(), out, hv.size() * 4, cudaMemcpyDeviceToHost));
      if (ref.empty() && mode == 0) ref = hv;
      if (!ref.empty()) {
        size_t bad = 0;
        const size_t m = std::min(ref.size(), hv.size());
        for (size_t i = 0; i < m; ++i) bad += ref[i] != hv[i];
        printf("   mismatches vs brick: %zu of %zu\n", bad, m);
      }
    }
  }
  return 0;
}
