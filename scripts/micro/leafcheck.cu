// leaves(): scalar vs f32x2 (the evolve kernel's formulas) on random t, R, tri.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ float u01(uint32_t h) { return (h >> 8) * (1.0f / 16777216.0f); }
__device__ float2 bc2(float a) { return make_float2(a, a); }
__device__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
struct L { float a0, cx, aR, S, Sr, SR, qo, qi, s3o, s3i; };
__device__ __forceinline__ L leaf(float t, float a, float inv_dR, float inv_rho_dR, float k2, float tri, float ox) {
  const float uo = __saturatef(__fmaf_rn(t, inv_dR, a));
  const float ui = __saturatef(__fmaf_rn(t, inv_rho_dR, a));
  const float qo = __fmaf_rn(-uo, uo, uo), qi = __fmaf_rn(-ui, ui, ui);
  const float s3o = __fmul_rn(uo, __fmaf_rn(2.0f, qo, uo));
  const float s3i = __fmul_rn(ui, __fmaf_rn(2.0f, qi, ui));
  const float S = __fsub_rn(__fmaf_rn(2.0f, s3i, -s3o), 1.0f);
  const float Sr = __fmaf_rn(k2, qi, -qo);
  const float SR = __fmaf_rn(-2.0f, qi, qo);
  const float w = __fmul_rn(Sr, tri);
  return L{__fmul_rn(S, tri), __fmul_rn(w, ox), __fmul_rn(SR, tri), S, Sr, SR, qo, qi, s3o, s3i};
}
__global__ void k(unsigned long long* cnt, uint32_t seed, float inv_dR, float inv_rho_dR, float k2) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const float R = 5.0f + 15.0f * u01(hsh(i * 7 + seed));
  const float a = __fmul_rn(-__fsub_rn(R, 1.0f), inv_dR);
  const float t0 = (R + 1.0f) * u01(hsh(i * 7 + 1 + seed)), t1 = (R + 1.0f) * u01(hsh(i * 7 + 2 + seed));
  const float tr0 = 65535.f * u01(hsh(i * 7 + 3 + seed)), tr1 = 65535.f * u01(hsh(i * 7 + 4 + seed));
  const float ox0 = 2.f * u01(hsh(i * 7 + 5 + seed)) - 1.f, ox1 = 2.f * u01(hsh(i * 7 + 6 + seed)) - 1.f;
  const L s0 = leaf(t0, a, inv_dR, inv_rho_dR, k2, tr0, ox0), s1 = leaf(t1, a, inv_dR, inv_rho_dR, k2, tr1, ox1);
  const float2 uo = make_float2(__saturatef(__fmaf_rn(t0, inv_dR, a)), __saturatef(__fmaf_rn(t1, inv_dR, a)));
  const float2 ui = make_float2(__saturatef(__fmaf_rn(t0, inv_rho_dR, a)), __saturatef(__fmaf_rn(t1, inv_rho_dR, a)));
  const float2 qo = __ffma2_rn(neg2(uo), uo, uo), qi = __ffma2_rn(neg2(ui), ui, ui);
  const float2 s3o = __fmul2_rn(uo, __ffma2_rn(bc2(2.0f), qo, uo));
  const float2 s3i = __fmul2_rn(ui, __ffma2_rn(bc2(2.0f), qi, ui));
  const float2 Sv = __fadd2_rn(__ffma2_rn(bc2(2.0f), s3i, neg2(s3o)), bc2(-1.0f));
  const float2 Sr = __ffma2_rn(bc2(k2), qi, neg2(qo));
  const float2 SR = __ffma2_rn(bc2(-2.0f), qi, qo);
  const float2 tri = make_float2(tr0, tr1);
  const float2 w = __fmul2_rn(Sr, tri);
  const float2 a0 = __fmul2_rn(Sv, tri), cx = __fmul2_rn(w, make_float2(ox0, ox1)), aR = __fmul2_rn(SR, tri);
#define CHK(j, A, B) if (__float_as_uint(A.x) != __float_as_uint(B##0) || __float_as_uint(A.y) != __float_as_uint(B##1)) atomicAdd(&cnt[j], 1ull);
  const float qo0 = s0.qo, qo1 = s1.qo, qi0 = s0.qi, qi1 = s1.qi, s3o0 = s0.s3o, s3o1 = s1.s3o, s3i0 = s0.s3i, s3i1 = s1.s3i;
  const float S0 = s0.S, S1 = s1.S, Sr0 = s0.Sr, Sr1 = s1.Sr, SR0 = s0.SR, SR1 = s1.SR, A00 = s0.a0, A01 = s1.a0, cx0 = s0.cx, cx1 = s1.cx, aR0 = s0.aR, aR1 = s1.aR;
  CHK(0, qo, qo) CHK(1, qi, qi) CHK(2, s3o, s3o) CHK(3, s3i, s3i) CHK(4, Sv, S) CHK(5, Sr, Sr) CHK(6, SR, SR) CHK(7, a0, A0) CHK(8, cx, cx) CHK(9, aR, aR)
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 8); cudaMemset(d, 0, 16 * 8);
  const double rho = 0.7937005259840998, dR = 2.0;
  for (int it = 0; it < 16; ++it) k<<<1 << 16, 256>>>(d, it * 0x9e3779b9u, (float)(1.0 / dR), (float)(1.0 / (rho * dR)), (float)(2.0 / rho));
  unsigned long long h[16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("qo %llu qi %llu s3o %llu s3i %llu S %llu Sr %llu SR %llu a0 %llu cx %llu aR %llu of %d\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], 16 << 24);
  return 0;
}
