// Does every f32x2 intrinsic round each component exactly like its scalar
// counterpart?  Random bit patterns (finite) and near-1 values; prints mismatches.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ float rnd(uint32_t h, int mode) {
  if (mode == 0) { uint32_t b = h & 0x7f7fffff; b |= (h & 0x80000000u); return __uint_as_float(b); }  // any finite-ish
  return __uint_as_float(0x3f000000u | (h & 0x00ffffffu)) * ((h >> 31) ? -1.f : 1.f);            // [0.5, 2)
}
__global__ void k(unsigned long long* cnt, int mode, uint32_t seed) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const float a0 = rnd(hash(i * 6 + seed), mode), b0 = rnd(hash(i * 6 + 1 + seed), mode), c0 = rnd(hash(i * 6 + 2 + seed), mode);
  const float a1 = rnd(hash(i * 6 + 3 + seed), mode), b1 = rnd(hash(i * 6 + 4 + seed), mode), c1 = rnd(hash(i * 6 + 5 + seed), mode);
  const float2 A = make_float2(a0, a1), B = make_float2(b0, b1), C = make_float2(c0, c1);
  float2 r;
  r = __ffma2_rn(A, B, C);
  if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(a0, b0, c0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(a1, b1, c1))) atomicAdd(&cnt[0], 1ull);
  r = __fadd2_rn(A, B);
  if (__float_as_uint(r.x) != __float_as_uint(__fadd_rn(a0, b0)) || __float_as_uint(r.y) != __float_as_uint(__fadd_rn(a1, b1))) atomicAdd(&cnt[1], 1ull);
  r = __fmul2_rn(A, B);
  if (__float_as_uint(r.x) != __float_as_uint(__fmul_rn(a0, b0)) || __float_as_uint(r.y) != __float_as_uint(__fmul_rn(a1, b1))) atomicAdd(&cnt[2], 1ull);
  r = __fadd2_rd(A, B);
  if (__float_as_uint(r.x) != __float_as_uint(__fadd_rd(a0, b0)) || __float_as_uint(r.y) != __float_as_uint(__fadd_rd(a1, b1))) atomicAdd(&cnt[3], 1ull);
  r = __ffma2_rn(make_float2(-a0, -a1), A, A);   // q = u (1 - u) form
  if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(-a0, a0, a0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(-a1, a1, a1))) atomicAdd(&cnt[4], 1ull);
  // immediate / broadcast operand forms used by the evolve kernel
  r = __ffma2_rn(make_float2(2.0f, 2.0f), A, B);
  if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(2.0f, a0, b0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(2.0f, a1, b1))) atomicAdd(&cnt[6], 1ull);
  r = __fadd2_rn(A, make_float2(-1.0f, -1.0f));
  if (__float_as_uint(r.x) != __float_as_uint(__fsub_rn(a0, 1.0f)) || __float_as_uint(r.y) != __float_as_uint(__fsub_rn(a1, 1.0f))) atomicAdd(&cnt[7], 1ull);
  r = __ffma2_rn(make_float2(-2.0f, -2.0f), A, B);
  if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(-2.0f, a0, b0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(-2.0f, a1, b1))) atomicAdd(&cnt[8], 1ull);
  r = __ffma2_rn(make_float2(c0, c0), A, make_float2(-b0, -b1));
  if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(c0, a0, -b0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(c0, a1, -b1))) atomicAdd(&cnt[9], 1ull);
  r = __ffma2_rn(A, B, make_float2(c0, c0));
  if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(a0, b0, c0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(a1, b1, c0))) atomicAdd(&cnt[10], 1ull);
  const float2 km = make_float2(8388608.0f, 8388608.0f);
  const float2 kk = make_float2(fabsf(a0) * 100.f, fabsf(a1) * 100.f);
  r = __fadd2_rn(kk, make_float2(-__fadd2_rn(__fadd2_rd(kk, km), make_float2(-8388608.0f, -8388608.0f)).x,
                                 -__fadd2_rn(__fadd2_rd(kk, km), make_float2(-8388608.0f, -8388608.0f)).y));
  const float fx0 = __fsub_rn(kk.x, __fsub_rn(__fadd_rd(kk.x, 8388608.0f), 8388608.0f));
  const float fx1 = __fsub_rn(kk.y, __fsub_rn(__fadd_rd(kk.y, 8388608.0f), 8388608.0f));
  if (__float_as_uint(r.x) != __float_as_uint(fx0) || __float_as_uint(r.y) != __float_as_uint(fx1)) atomicAdd(&cnt[11], 1ull);
  // subnormal results
  const float2 tiny = make_float2(a0 * 1e-30f, a1 * 1e-30f);
  r = __fmul2_rn(tiny, make_float2(1e-10f, 1e-10f));
  if (__float_as_uint(r.x) != __float_as_uint(__fmul_rn(tiny.x, 1e-10f)) || __float_as_uint(r.y) != __float_as_uint(__fmul_rn(tiny.y, 1e-10f))) atomicAdd(&cnt[5], 1ull);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * sizeof(unsigned long long));
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d, 0, 16 * sizeof(unsigned long long));
    for (int it = 0; it < 16; ++it) k<<<1 << 16, 256>>>(d, mode, it * 0x9e3779b9u);
    unsigned long long h[16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): ffma2 %llu fadd2 %llu fmul2 %llu fadd2_rd %llu q-form %llu subnormal-fmul2 %llu of %d\n", mode,
           mode ? "[0.5,2)" : "random bits", h[0], h[1], h[2], h[3], h[4], h[5], 16 << 24);
    printf("   imm 2 fma %llu  add -1 %llu  imm -2 fma %llu  bcast a %llu  bcast c %llu  magic split %llu\n", h[6], h[7], h[8], h[9], h[10], h[11]);
  }
  return 0;
}
