// Throughput of candidate instruction sequences on this GPU (ops per SM per clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ops ops.cu && ./ops
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8, IT = 4096;

template <int OP>
__global__ void __launch_bounds__(256) k(uint32_t* out, uint32_t seed) {
  uint32_t v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = seed + threadIdx.x * 7 + c * 13;
  float f[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) f[c] = __uint_as_float(v[c] & 0x3fffffff);
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) {  // FFMA
        f[c] = __fmaf_rn(f[c], 1.0001f, 0.5f);
      } else if (OP == 1) {  // I2FP.F32.S32 (cvt.rn.f32.s32)
        float r;
        asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(r) : "r"(v[c]));
        v[c] = __float_as_uint(r);
      } else if (OP == 2) {  // IMAD.WIDE.U32 (mul.wide.u32) + fold
        uint64_t p;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(v[c]), "r"(0xD2511F53u));
        v[c] = (uint32_t)(p >> 32);
      } else if (OP == 3) {  // IMAD.HI.U32
        uint32_t r;
        asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(v[c]), "r"(0xD2511F53u));
        v[c] = r;
      } else if (OP == 4) {  // LOP3
        uint32_t r;
        asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(v[c]), "r"(0x1234567u), "r"(seed));
        v[c] = r;
      } else if (OP == 5) {  // IADD3
        uint32_t r;
        asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(v[c]), "r"(0x4B000000u));
        v[c] = r;
      } else if (OP == 6) {  // MUFU.EX2
        float r;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c]));
        f[c] = r;
      } else if (OP == 7) {  // mul.lo.u32 (IMAD)
        uint32_t r;
        asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(v[c]), "r"(0xD2511F53u));
        v[c] = r;
      } else if (OP == 8) {  // full Philox round pair-word: 2 wide muls + 2 xor3 (counted as 1 round)
        uint64_t p0, p1;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p0) : "r"(v[c]), "r"(0xD2511F53u));
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p1) : "r"(v[(c + 1) % CH]), "r"(0xCD9E8D57u));
        v[c] = (uint32_t)(p1 >> 32) ^ (uint32_t)p0 ^ seed;
        v[(c + 1) % CH] = (uint32_t)(p0 >> 32) ^ (uint32_t)p1 ^ 0x9E3779B9u;
      } else if (OP == 9) {  // I2F.U16
        float r;
        asm volatile("cvt.rn.f32.u16 %0, %1;" : "=f"(r) : "h"((unsigned short)v[c]));
        v[c] = __float_as_uint(r);
      } else if (OP == 10) {  // FMNMX
        f[c] = fminf(f[c], 0.75f + f[(c + 1) % CH]);
      } else if (OP == 11) {  // PRMT
        uint32_t r;
        asm volatile("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(v[c]), "r"(0x4B004B00u));
        v[c] = r;
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= v[c] ^ __float_as_uint(f[c]);
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz
  const char* names[] = {"FFMA", "I2FP.F32.S32", "IMAD.WIDE.U32(hi)", "IMAD.HI.U32", "LOP3", "IADD",
                         "MUFU.EX2", "IMAD.LO", "philox-round(2 words)", "I2F.U16", "FMNMX+FADD", "PRMT"};
  void (*ks[])(uint32_t*, uint32_t) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>, k<10>, k<11>};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  for (int o = 0; o < 12; ++o) {
    ks[o]<<<blocks, threads>>>(d, 1);
    cudaEventRecord(a);
    ks[o]<<<blocks, threads>>>(d, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * threads * IT * CH;
    const double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-24s %8.3f ms  %7.1f ops/SM/clk (clock %d MHz)\n", names[o], ms, per_sm_clk, clk / 1000);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
