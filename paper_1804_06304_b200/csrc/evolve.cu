// evolve.cu — a5 + a6: batched Monte-Carlo evolution of independent 3D (2D)
// snakuscules (Eqs. 11-14), the ★ hot loop.
//
// Two kernels compute the same function, bit for bit:
//
//  * evolve_brick_kernel (default; needs an even x extent): one CTA of W warps
//    per cell (the paper's block-per-contour).  The cell's
//    neighbourhood — a (S+2) x S x S brick of the u16 image containing the
//    sampled ball — lives in shared memory, filled by cp.async copies and
//    re-centred only when the ball leaves it, so the per-sample gathers are
//    shared-memory loads with immediate offsets and L2/HBM see a few bricks
//    per cell instead of 8 scattered taps per sample (the warp kernel is
//    L1-bound on C3 and DRAM-bound on C4, profiles/r1_baseline_evolve.md).  A
//    sample ball that cannot fit the brick takes global loads for that
//    iteration (same arithmetic).
//  * evolve_warp_kernel (generic fallback, any shape): W warps per cell,
//    gathers straight from global memory (L1/L2).
//
// Each iteration draws a FIXED number N of samples per cell (no
// divergence), 32 W threads x B = N/(32 W) each.  Per sample: 3 (2D: 2) words
// of the Philox4x32-10 stream (4 samples per 3 blocks) -> (omega, t) -> 8 u16
// taps -> trilinear -> S, S_r, S_R -> 5 leaf products.
// Sums follow one canonical pairwise tree over the N sample positions
// (in-thread binary counter -> xor butterfly over lanes -> pairwise over
// warps), so every W and both kernels give bit-identical results (S:314,
// S:317).  Compiled with -fmad=false: every FMA is explicit.
//
// Reading of the update (G3/G4/G8): E = gamma A0,
// dE/dc = -gamma A_c, dE/dR = gamma (A_R - (d/R) A0), gamma = (2R)^-d;
// (c, R) -= clip((eps0/sqrt(n))/2 * grad, +-max_step); R clamp, leash, domain.
#include <cstdlib>
#include <type_traits>
#include <mutex>

#include "common.cuh"

namespace snk {

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;   // Philox multipliers
constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;   // Weyl key bumps
constexpr float kMagic = 8388608.0f;                        // 2^23
constexpr uint32_t kMagicBits = 0x4B000000u;

// Diagnostic builds (scripts/, never the product): SNK_DIAG_NOCONF makes every
// lane of the fast path gather from one warp-uniform brick address (no bank
// conflicts); SNK_DIAG_PHILOX_ROUNDS < 10 truncates Philox.  Both give wrong
// results on purpose; they bound what conflict-free gathers / fewer
// instructions could buy.
#ifndef SNK_DIAG_NOCONF
#define SNK_DIAG_NOCONF 0
#endif
#ifndef SNK_DIAG_PHILOX_ROUNDS
#define SNK_DIAG_PHILOX_ROUNDS 10
#endif

// diagnostics of the brick kernel: [0] brick (re)loads, [1] cell-iterations
// that took the global-gather path (ball larger than the brick)
__device__ unsigned long long g_evolve_stats[4];

struct EvoParams {
  const uint16_t* img;
  const float* seeds;
  const int64_t* ids;
  snk_cell* out;
  int64_t id_base, n;
  int nx, ny, nz, z_lo, nz_buf;
  float fnx1, fny1, fnz1;        // n - 1
  float mx2, my2, mz2;           // 2^23 + (n - 2): clamp of the magic floor
  float r0, half_dR, inv_dR, inv_rho_dR, eps0, max_step, r_min, r_max, leash, conv_tol;
  float k2_rho, k6_dR;           // 2/rho, 6/dR
  float vscale;                  // iscale * (4/3 pi | pi) / N
  float half_eps0;               // eps0 / 2
  int T;
  int it0, it1;                  // iterations this launch runs (1 .. T + 1 for a whole run)
  const snk_cell* state;         // non-null: continue these records (periodic culling, G25)
  int dom_small;                 // some axis has n - 1 < 2 (r_max + dR/2)
  float isc[3];                  // 1 / scale: physical -> raw grid coordinates (G28)
  float dom1[3];                 // physical extent (n - 1) scale of each axis (= n - 1 isotropic)
  uint32_t rk0[10], rk1[10];     // Philox round keys (seed + r * Weyl)
};

struct Acc {
  float a0, cx, cy, cz, aR;
};

// EST template values: the estimator in bits 0-1 (SNK_EST_MC, _MC_CV, _RAY) and
// bit 2 = anisotropic grid sampled in physical coordinates (G28)
constexpr int kAniso = 4;
// bit 3: no axis of the domain is shorter than a ball (P.dom_small == 0), so the
// update's domain clamp needs no small-axis selects (a launch-time choice)
constexpr int kBig = 8;
#ifndef SNK_BIG
#define SNK_BIG 1
#endif
__host__ __device__ constexpr int est_kind(int e) { return e & 3; }
__host__ __device__ constexpr bool est_aniso(int e) { return (e & kAniso) != 0; }

__device__ __forceinline__ Acc acc_add(const Acc& l, const Acc& r) {
  return Acc{__fadd_rn(l.a0, r.a0), __fadd_rn(l.cx, r.cx), __fadd_rn(l.cy, r.cy),
             __fadd_rn(l.cz, r.cz), __fadd_rn(l.aR, r.aR)};
}

// Per cell-iteration constants.
struct CellIt {
  float cx, cy, cz;
  float rho_s;          // R + dR/2: radius of the sampled ball
  float a;              // -(R - dR/2)/dR: offset of both ramp coordinates
  float lg2_rho_s;      // log2(rho_s)
  uint32_t p0, p1, p3;  // Philox round-1 words that depend only on (n, id)
  // brick: sum over axes of (2^23 + b_a) * stride_a (mod 2^32), so that the
  // brick index of magic-floored coordinates is rx + ry SX + rz SP - boff
  uint32_t boff;
  float ic;             // SNK_EST_MC_CV: the image at the centre, I(c) (u16 units)
#if SNK_DIAG_NOCONF
  uint32_t lic;         // diagnostic build only: a warp-uniform brick index
#endif
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// u = (x >> 9) * 2^-23, exactly, via the mantissa: [1, 2) - 1.
__device__ __forceinline__ float u01(uint32_t x) {
  return __fsub_rn(__uint_as_float(0x3F800000u | (x >> 9)), 1.0f);
}

// u16 value -> float, exact: one I2FP.F32.U32 (ALU pipe; the compiler's own
// conversion of a known-16-bit value is the slow I2F.U16 on the SFU pipe)
__device__ __forceinline__ float mag(uint32_t v) {
  float r;
  asm("cvt.rn.f32.u32 %0, %1;" : "=f"(r) : "r"(v));
  return r;
}

__device__ __forceinline__ float lerp(float a, float b, float f) {
  return __fmaf_rn(f, __fsub_rn(b, a), a);
}

// One axis of the d-linear lookup: clamp k to [0, n-1] (unless the caller
// knows it is inside), i0 = min(floor(k), n-2) by the magic-number floor
// (FADD.RM, no conversions), fraction k - i0.  Returns r = 2^23 + i0 (as bits).
template <bool CLAMP>
__device__ __forceinline__ float split_axis(float k, float n1, float m2, uint32_t* rbits) {
  if (CLAMP) k = fminf(fmaxf(k, 0.0f), n1);
  float r = __fadd_rd(k, kMagic);
  if (CLAMP) r = fminf(r, m2);
  *rbits = __float_as_uint(r);
  return __fsub_rn(k, __fsub_rn(r, kMagic));
}

struct Draw {
  float ox, oy, oz, t;
};

// Philox4x32-10 block b of the cell-iteration stream: ctr = {b, n, id_lo,
// id_hi}, key = seed (G11); round 1's products of the constant words are in C.
__device__ __forceinline__ void philox_block(const EvoParams& P, const CellIt& C, uint32_t b, uint32_t x[4]) {
  const uint64_t pb = (uint64_t)kM0 * b;
  uint32_t c0 = C.p0, c1 = C.p1, c2 = (uint32_t)(pb >> 32) ^ C.p3, c3 = (uint32_t)pb;
#pragma unroll
  for (int r = 1; r < SNK_DIAG_PHILOX_ROUNDS; ++r) {
    const uint64_t p0 = (uint64_t)kM0 * c0;
    const uint64_t p1 = (uint64_t)kM1 * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ P.rk0[r];
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ P.rk1[r];
    c0 = n0;
    c1 = (uint32_t)p1;
    c2 = n2;
    c3 = (uint32_t)p0;
  }
  x[0] = c0; x[1] = c1; x[2] = c2; x[3] = c3;
}

// Words -> the sample's direction (Archimedes, G10) and the radial variate:
// the part of a draw that does not depend on the contour state, so it can be
// computed ahead (evolve_brick_kernel draws iteration n+1 while the update of
// iteration n runs).  3D: (w0, w1, w2) = (u0, u1, u2), L = lg2(u2);
// 2D: (w1, w2) = (u1, u2), L = sqrt(u2).
struct Dir {
  float ox, oy, oz, L;
};

// m = 1 + u in [1, 2): the mantissa word alone (u01 without its subtraction)
__device__ __forceinline__ float m12(uint32_t x) { return __uint_as_float(0x3F800000u | (x >> 9)); }

template <int D>
__device__ __forceinline__ Dir dir_words(uint32_t w0, uint32_t w1, uint32_t w2) {
  const float u2 = u01(w2);
  float sn, cs;
  // phi = 2 pi u1: sin and cos of 2 pi (1 + u1) are the same (period 2 pi), so
  // the mantissa word m1 = 1 + u1 is used directly (one subtraction fewer)
  __sincosf(__fmul_rn(6.2831853071795865f, m12(w1)), &sn, &cs);
  Dir d;
  if (D == 3) {
    // z = 1 - 2 u0 = 3 - 2 m0, exact in fp32 either way (a multiple of 2^-22 in (-1, 1])
    d.oz = __fmaf_rn(-2.0f, m12(w0), 3.0f);
    const float st = sqrt_approx(__fmaf_rn(-d.oz, d.oz, 1.0f));   // sqrt(1 - z^2) = 2 sqrt(u0 (1 - u0))
    d.ox = __fmul_rn(st, cs);
    d.oy = __fmul_rn(st, sn);
    d.L = lg2_approx(u2);
  } else {
    (void)w0;
    d.ox = cs;
    d.oy = sn;
    d.oz = 0.0f;
    d.L = sqrt_approx(u2);
  }
  return d;
}

// The distance: 3D t = rho_s cbrt(u2), 2D t = rho_s sqrt(u2);
// the ray march (EST 3, G27): t = rho_s (m + u) / M with L = (m + u) / M.
template <int D, int EST = 0>
__device__ __forceinline__ Draw finish_draw(const CellIt& C, const Dir& d) {
  Draw r;
  r.ox = d.ox;
  r.oy = d.oy;
  r.oz = d.oz;
  if (est_kind(EST) == SNK_EST_RAY) r.t = __fmul_rn(C.rho_s, d.L);
  else r.t = D == 3 ? ex2_approx(__fmaf_rn(d.L, 0.333333343f, C.lg2_rho_s)) : __fmul_rn(C.rho_s, d.L);
  return r;
}

// The ray march's draws (G27): ray `ray` of the cell-iteration takes the 12
// words of Philox blocks 3 ray .. 3 ray + 2: words 0, 1 give the direction
// (the MC law, G10), words 2 + m the jitter of step m, L = (m + u) / 8.
template <int D>
__device__ __forceinline__ void draw_dirs_ray(const EvoParams& P, const CellIt& C, uint32_t ray, Dir* d) {
  uint32_t a[4], b[4], c[4];
  philox_block(P, C, 3u * ray, a);
  philox_block(P, C, 3u * ray + 1u, b);
  philox_block(P, C, 3u * ray + 2u, c);
  const float u1 = u01(a[1]);
  float sn, cs;
  __sincosf(__fmul_rn(6.2831853071795865f, u1), &sn, &cs);
  Dir o;
  if (D == 3) {
    o.oz = __fmaf_rn(-2.0f, u01(a[0]), 1.0f);
    const float st = sqrt_approx(__fmaf_rn(-o.oz, o.oz, 1.0f));
    o.ox = __fmul_rn(st, cs);
    o.oy = __fmul_rn(st, sn);
  } else {
    o.ox = cs;
    o.oy = sn;
    o.oz = 0.0f;
  }
  const uint32_t w[8] = {a[2], a[3], b[0], b[1], b[2], b[3], c[0], c[1]};
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    d[m] = o;
    d[m].L = __fmul_rn(__fadd_rn((float)m, u01(w[m])), 0.125f);
  }
}

// The image value a sample contributes (u16 units): I(k) (MC, grid), I(k) - I(c)
// (control variate, G21), I(k) t^(d-1) (ray march, the polar volume element).
template <int D, int EST>
__device__ __forceinline__ float est_value(const CellIt& C, float tri, float t) {
  if (est_kind(EST) == SNK_EST_MC_CV) return __fsub_rn(tri, C.ic);
  if (est_kind(EST) == SNK_EST_RAY) return __fmul_rn(tri, D == 3 ? __fmul_rn(t, t) : t);
  return tri;
}

template <int D>
__device__ __forceinline__ Draw draw_words(const CellIt& C, uint32_t w0, uint32_t w1, uint32_t w2) {
  return finish_draw<D>(C, dir_words<D>(w0, w1, w2));
}

// The directions of the CH samples j0 .. j0 + CH - 1 (CH a power of two, j0 %
// CH == 0) of iteration n, keyed through C.p0/p1/p3 only.
template <int D, int CH>
__device__ __forceinline__ void draw_dirs(const EvoParams& P, const CellIt& C, uint32_t j0, Dir* d) {
  constexpr int G = D == 3 ? 4 : 2;
  if constexpr (CH >= G) {
#pragma unroll
    for (int g = 0; g < CH; g += G) {
      uint32_t a[4];
      if (D == 3) {
        uint32_t b[4], c[4];
        const uint32_t b0 = ((j0 + g) >> 2) * 3u;
        philox_block(P, C, b0, a);
        philox_block(P, C, b0 + 1, b);
        philox_block(P, C, b0 + 2, c);
        d[g + 0] = dir_words<3>(a[0], a[1], a[2]);
        d[g + 1] = dir_words<3>(a[3], b[0], b[1]);
        d[g + 2] = dir_words<3>(b[2], b[3], c[0]);
        d[g + 3] = dir_words<3>(c[1], c[2], c[3]);
      } else {
        philox_block(P, C, (j0 + g) >> 1, a);
        d[g + 0] = dir_words<2>(0, a[0], a[1]);
        d[g + 1] = dir_words<2>(0, a[2], a[3]);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const uint32_t j = j0 + k;
      uint32_t x[4];
      if (D == 3) {
        const uint32_t w = 3u * j, o = w & 3u;
        philox_block(P, C, w >> 2, x);
        if (o <= 1) {
          d[k] = o == 0 ? dir_words<3>(x[0], x[1], x[2]) : dir_words<3>(x[1], x[2], x[3]);
        } else {
          uint32_t y[4];
          philox_block(P, C, (w >> 2) + 1, y);
          d[k] = o == 2 ? dir_words<3>(x[2], x[3], y[0]) : dir_words<3>(x[3], y[0], y[1]);
        }
      } else {
        philox_block(P, C, j >> 1, x);
        d[k] = (j & 1u) ? dir_words<2>(0, x[2], x[3]) : dir_words<2>(0, x[0], x[1]);
      }
    }
  }
}

// Sample j alone (G11 word layout: 3D words 3j..3j+2, 2D words 2j, 2j+1).
template <int D>
__device__ __forceinline__ Draw draw(const EvoParams& P, const CellIt& C, uint32_t j) {
  uint32_t x[4];
  if (D == 3) {
    const uint32_t w = 3u * j, o = w & 3u;
    philox_block(P, C, w >> 2, x);
    if (o == 0) return draw_words<3>(C, x[0], x[1], x[2]);
    if (o == 1) return draw_words<3>(C, x[1], x[2], x[3]);
    uint32_t y[4];
    philox_block(P, C, (w >> 2) + 1, y);
    if (o == 2) return draw_words<3>(C, x[2], x[3], y[0]);
    return draw_words<3>(C, x[3], y[0], y[1]);
  }
  philox_block(P, C, j >> 1, x);
  return (j & 1u) ? draw_words<2>(C, 0, x[2], x[3]) : draw_words<2>(C, 0, x[0], x[1]);
}

// The G samples j .. j + G - 1 of one group (j % G == 0; G = 4 in 3D, 2 in 2D):
// 3 (3D) or 1 (2D) Philox blocks.
template <int D>
__device__ __forceinline__ void draw_group(const EvoParams& P, const CellIt& C, uint32_t j, Draw* d) {
  if (D == 3) {
    uint32_t a[4], b[4], c[4];
    const uint32_t b0 = (j >> 2) * 3u;
    philox_block(P, C, b0, a);
    philox_block(P, C, b0 + 1, b);
    philox_block(P, C, b0 + 2, c);
    d[0] = draw_words<3>(C, a[0], a[1], a[2]);
    d[1] = draw_words<3>(C, a[3], b[0], b[1]);
    d[2] = draw_words<3>(C, b[2], b[3], c[0]);
    d[3] = draw_words<3>(C, c[1], c[2], c[3]);
  } else {
    uint32_t a[4];
    philox_block(P, C, j >> 1, a);
    d[0] = draw_words<2>(C, 0, a[0], a[1]);
    d[1] = draw_words<2>(C, 0, a[2], a[3]);
  }
}

// S(t; R) and partials (G1) -> the five leaves for image value tri.
__device__ __forceinline__ Acc leaves(const EvoParams& P, const CellIt& C, const Draw& d, float tri,
                                      bool three) {
  // tau_o = (t - (R - dR/2))/dR,  tau_i = (t - rho (R - dR/2))/(rho dR) = t/(rho dR) + a
  const float uo = __saturatef(__fmaf_rn(d.t, P.inv_dR, C.a));
  const float ui = __saturatef(__fmaf_rn(d.t, P.inv_rho_dR, C.a));
  // q = u (1 - u): s3 = 3u^2 - 2u^3 = u (u + 2q), s3' = 6q
  const float qo = __fmaf_rn(-uo, uo, uo), qi = __fmaf_rn(-ui, ui, ui);
  const float s3o = __fmul_rn(uo, __fmaf_rn(2.0f, qo, uo));
  const float s3i = __fmul_rn(ui, __fmaf_rn(2.0f, qi, ui));
  const float S = __fsub_rn(__fmaf_rn(2.0f, s3i, -s3o), 1.0f);             // (1-s3o) - 2(1-s3i)
  // S_r = (6/dR) (2 qi/rho - qo),  S_R = (6/dR) (qo - 2 qi): the common factor
  // 6/dR is applied once to the sums (cell_update)
  const float Sr = __fmaf_rn(P.k2_rho, qi, -qo);
  const float SR = __fmaf_rn(-2.0f, qi, qo);
  const float w = __fmul_rn(Sr, tri);
  Acc a;
  a.a0 = __fmul_rn(S, tri);
  a.cx = __fmul_rn(w, d.ox);
  a.cy = __fmul_rn(w, d.oy);
  a.cz = three ? __fmul_rn(w, d.oz) : 0.0f;
  a.aR = __fmul_rn(SR, tri);
  return a;
}

// Brick row length: S + 2 rounded down to even (the x origin is even, the
// copies are 4-byte words), so a ball box of width SX - 1 always fits in x.
#ifndef SNK_BRICK_ALIGN
#define SNK_BRICK_ALIGN 2   // brick x origin alignment (elements) = the copy width / 2 bytes
#endif
constexpr int kBA = SNK_BRICK_ALIGN;
__host__ __device__ constexpr int brick_sx(int S) { return (S + 2 * kBA - 2) & ~(kBA - 1); }

// Gather modes
enum { G_GLOBAL = 0, G_GLOBAL_SLAB = 1, G_BRICK_CLAMP = 2, G_BRICK_FAST = 3, G_GLOBAL_FAST = 4 };

// d-linear lookup of the image at k (u16 units), through the brick or global memory.
template <int D, int MODE, int S>
__device__ __forceinline__ float gather_tri(const EvoParams& P, const CellIt& C, float kx, float ky, float kz,
                                            const uint16_t* brick, uint32_t& halo) {
  constexpr bool CLAMP = MODE != G_BRICK_FAST && MODE != G_GLOBAL_FAST;
  uint32_t rx, ry, rz = kMagicBits;
  const float fx = split_axis<CLAMP>(kx, P.fnx1, P.mx2, &rx);
  const float fy = split_axis<CLAMP>(ky, P.fny1, P.my2, &ry);
  float fz = 0.0f;
  if (D == 3) fz = split_axis<CLAMP>(kz, P.fnz1, P.mz2, &rz);
  float v000, v100, v010, v110, v001 = 0, v101 = 0, v011 = 0, v111 = 0;
  if (MODE == G_BRICK_CLAMP || MODE == G_BRICK_FAST) {
    // brick-local index; row stride SX and plane stride SX * S are immediates
    constexpr int SX = brick_sx(S), SP = SX * S;
    uint32_t li = ry * SX + rx;
    if (D == 3) li += rz * SP;
    li -= C.boff;
    asm("" : "+r"(li));   // materialise li: the eight tap offsets become LDS immediates
    const uint16_t* p = brick + li;
    v000 = mag(p[0]);
    v100 = mag(p[1]);
    v010 = mag(p[SX]);
    v110 = mag(p[SX + 1]);
    if (D == 3) {
      v001 = mag(p[SP]);
      v101 = mag(p[SP + 1]);
      v011 = mag(p[SP + SX]);
      v111 = mag(p[SP + SX + 1]);
    }
  } else {
    int iz = (int)(rz - kMagicBits);
    if (MODE == G_GLOBAL_SLAB && D == 3) {
      iz -= P.z_lo;
      if (iz < 0 || iz > P.nz_buf - 2) {
        halo = 1u;
        iz = min(max(iz, 0), P.nz_buf - 2);
      }
    }
    const uint32_t nx = (uint32_t)P.nx;
    const uint32_t base = ((uint32_t)iz * (uint32_t)P.ny + (ry - kMagicBits)) * nx + (rx - kMagicBits);
    const uint16_t* p = P.img + base;
    v000 = mag(__ldg(p));
    v100 = mag(__ldg(p + 1));
    v010 = mag(__ldg(p + nx));
    v110 = mag(__ldg(p + nx + 1));
    if (D == 3) {
      const uint32_t pl = nx * (uint32_t)P.ny;
      v001 = mag(__ldg(p + pl));
      v101 = mag(__ldg(p + pl + 1));
      v011 = mag(__ldg(p + pl + nx));
      v111 = mag(__ldg(p + pl + nx + 1));
    }
  }
  // trilinear: x, then y, then z (G17)
  float tri = lerp(lerp(v000, v100, fx), lerp(v010, v110, fx), fy);
  if (D == 3) tri = lerp(tri, lerp(lerp(v001, v101, fx), lerp(v011, v111, fx), fy), fz);
  return tri;
}

template <int D, int MODE, int S, int EST = 0>
__device__ __forceinline__ Acc sample_leaf(const EvoParams& P, const CellIt& C, const Draw& d,
                                           const uint16_t* brick, uint32_t& halo) {
  float kx = __fmaf_rn(d.t, d.ox, C.cx), ky = __fmaf_rn(d.t, d.oy, C.cy);
  float kz = D == 3 ? __fmaf_rn(d.t, d.oz, C.cz) : 0.0f;
  if (est_aniso(EST)) {   // physical -> raw grid coordinates (G28)
    kx = __fmul_rn(kx, P.isc[0]);
    ky = __fmul_rn(ky, P.isc[1]);
    kz = __fmul_rn(kz, P.isc[2]);
  }
  const float tri = gather_tri<D, MODE, S>(P, C, kx, ky, kz, brick, halo);
  return leaves(P, C, d, est_value<D, EST>(C, tri, d.t), D == 3);
}

// ---------------------------------------------------------------- f32x2 fast path
// Blackwell's packed FP32 instructions (FFMA2 / FADD2 / FMUL2) round each
// component exactly like FFMA / FADD / FMUL, so two samples can share every
// floating-point instruction of sample_leaf<D, G_BRICK_FAST> with bit-identical
// results: half the issue slots for the arithmetic (the kernel is issue-bound).
// The pair is (sample k, sample k + CH/2) of a chunk, so that the chunk's
// pairwise tree is also SIMD: level 1 and 2 adds are FADD2, the last one scalar.
struct Acc2 {
  float2 a0, cx, cy, cz, aR;
};

__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

__device__ __forceinline__ Acc2 acc2_add(const Acc2& l, const Acc2& r) {
  return Acc2{__fadd2_rn(l.a0, r.a0), __fadd2_rn(l.cx, r.cx), __fadd2_rn(l.cy, r.cy),
              __fadd2_rn(l.cz, r.cz), __fadd2_rn(l.aR, r.aR)};
}

// lerp(a, b, f) = fma(f, b - a, a), per component
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 f) {
  return __ffma2_rn(f, __fadd2_rn(b, neg2(a)), a);
}

// split_axis<CLAMP> for two coordinates: r = k + 2^23 rounded down, fraction
// k - (r - 2^23); CLAMP: k clamped to [0, n - 1] and r to 2^23 + (n - 2) first
// (per component, the scalar split_axis<true> operations)
template <bool CLAMP = false>
__device__ __forceinline__ float2 split2(float2 k, uint32_t* r0, uint32_t* r1, float n1 = 0.0f, float m2 = 0.0f) {
  if (CLAMP) {
    k.x = fminf(fmaxf(k.x, 0.0f), n1);
    k.y = fminf(fmaxf(k.y, 0.0f), n1);
  }
  float2 r = __fadd2_rd(k, bc2(kMagic));
  if (CLAMP) {
    r.x = fminf(r.x, m2);
    r.y = fminf(r.y, m2);
  }
  *r0 = __float_as_uint(r.x);
  *r1 = __float_as_uint(r.y);
  return __fadd2_rn(k, neg2(__fadd2_rn(r, bc2(-kMagic))));
}

template <int D, int S, int EST = 0, bool CLAMP = false>
__device__ __forceinline__ Acc2 sample_pair_fast(const EvoParams& P, const CellIt& C, const Draw& d0,
                                                 const Draw& d1, const uint16_t* brick, int salt = 0) {
  constexpr int SX = brick_sx(S), SP = SX * S;
  const float2 t = make_float2(d0.t, d1.t);
  const float2 ox = make_float2(d0.ox, d1.ox), oy = make_float2(d0.oy, d1.oy);
  const float2 oz = make_float2(d0.oz, d1.oz);
  uint32_t rx0, rx1, ry0, ry1, rz0 = kMagicBits, rz1 = kMagicBits;
  float2 kx = __ffma2_rn(t, ox, bc2(C.cx)), ky = __ffma2_rn(t, oy, bc2(C.cy));
  float2 kz = D == 3 ? __ffma2_rn(t, oz, bc2(C.cz)) : bc2(0.0f);
  if (est_aniso(EST)) {   // physical -> raw grid coordinates (G28)
    kx = __fmul2_rn(kx, bc2(P.isc[0]));
    ky = __fmul2_rn(ky, bc2(P.isc[1]));
    kz = __fmul2_rn(kz, bc2(P.isc[2]));
  }
  const float2 fx = split2<CLAMP>(kx, &rx0, &rx1, P.fnx1, P.mx2);
  const float2 fy = split2<CLAMP>(ky, &ry0, &ry1, P.fny1, P.my2);
  float2 fz = bc2(0.0f);
  if (D == 3) fz = split2<CLAMP>(kz, &rz0, &rz1, P.fnz1, P.mz2);
  uint32_t li0 = ry0 * SX + rx0, li1 = ry1 * SX + rx1;
  if (D == 3) { li0 += rz0 * SP; li1 += rz1 * SP; }
  li0 -= C.boff;
  li1 -= C.boff;
#if SNK_DIAG_NOCONF
  li0 = C.lic + (uint32_t)salt;
  li1 = C.lic + 40u + (uint32_t)salt;
#else
  (void)salt;
#endif
  asm("" : "+r"(li0));
  asm("" : "+r"(li1));
  const uint16_t* p = brick + li0;
  const uint16_t* q = brick + li1;
  const float2 v000 = make_float2(mag(p[0]), mag(q[0]));
  const float2 v100 = make_float2(mag(p[1]), mag(q[1]));
  const float2 v010 = make_float2(mag(p[SX]), mag(q[SX]));
  const float2 v110 = make_float2(mag(p[SX + 1]), mag(q[SX + 1]));
  float2 tri = lerp2(lerp2(v000, v100, fx), lerp2(v010, v110, fx), fy);
  if (D == 3) {
    const float2 v001 = make_float2(mag(p[SP]), mag(q[SP]));
    const float2 v101 = make_float2(mag(p[SP + 1]), mag(q[SP + 1]));
    const float2 v011 = make_float2(mag(p[SP + SX]), mag(q[SP + SX]));
    const float2 v111 = make_float2(mag(p[SP + SX + 1]), mag(q[SP + SX + 1]));
    tri = lerp2(tri, lerp2(lerp2(v001, v101, fx), lerp2(v011, v111, fx), fy), fz);
  }
  if (est_kind(EST) == SNK_EST_MC_CV) tri = __fadd2_rn(tri, bc2(-C.ic));
  if (est_kind(EST) == SNK_EST_RAY) tri = __fmul2_rn(tri, D == 3 ? __fmul2_rn(t, t) : t);
  // leaves() per component: ptxas (CUDA 12.9) contracts mul.rn.f32x2 + add.rn.f32x2
  // into FFMA2 in spite of the .rn (the PTX has no contraction), which changed
  // the leaf sums against the scalar path; and the paired leaves measured 3%
  // slower on C4 (845 vs 819 ms) with 9 fewer instructions per sample — the
  // three 64-bit register operands of an FFMA2 cost register-file bandwidth
  // (B300_MICROARCH: rt = max over even/odd banks).  So only the position,
  // magic-floor split and d-linear lerps are paired.
  const Acc la = leaves(P, C, d0, tri.x, D == 3), lb = leaves(P, C, d1, tri.y, D == 3);
  Acc2 a;
  a.a0 = make_float2(la.a0, lb.a0);
  a.cx = make_float2(la.cx, lb.cx);
  a.cy = make_float2(la.cy, lb.cy);
  a.cz = make_float2(la.cz, lb.cz);
  a.aR = make_float2(la.aR, lb.aR);
  return a;
}

// chunk_sum_dirs<D, G_BRICK_FAST, S, CH> (CH = 4, 8) with paired samples: the
// same tree — for CH = 8, ((l0 + l1) + (l2 + l3)) + ((l4 + l5) + (l6 + l7)) —
// with the two halves of the chunk in the two lanes of the f32x2 sums.
template <int N>
__device__ __forceinline__ Acc2 tree_sum2(const Acc2* l) {
  if constexpr (N == 1) return l[0];
  else return acc2_add(tree_sum2<N / 2>(l), tree_sum2<N / 2>(l + N / 2));
}

template <int D, int S, int CH, int EST = 0, bool CLAMP = false>
__device__ __forceinline__ Acc chunk_fast_x2(const EvoParams& P, const CellIt& C, const Dir* d,
                                             const uint16_t* brick) {
  constexpr int H = CH / 2;
  Acc2 l[H];
#pragma unroll
  for (int k = 0; k < H; ++k)
    l[k] = sample_pair_fast<D, S, EST, CLAMP>(P, C, finish_draw<D, EST>(C, d[k]), finish_draw<D, EST>(C, d[k + H]),
                                       brick, k);
  const Acc2 h = tree_sum2<H>(l);
  return Acc{__fadd_rn(h.a0.x, h.a0.y), __fadd_rn(h.cx.x, h.cx.y), __fadd_rn(h.cy.x, h.cy.y),
             __fadd_rn(h.cz.x, h.cz.y), __fadd_rn(h.aR.x, h.aR.y)};
}

// Pairwise sum over CH consecutive samples (CH a power of two).  Groups of G
// samples share their Philox blocks (draw_group); smaller chunks draw alone.
template <int D, int MODE, int S, int CH>
__device__ __forceinline__ Acc chunk_sum(const EvoParams& P, const CellIt& C, uint32_t j0,
                                         const uint16_t* brick, uint32_t& halo) {
  constexpr int G = D == 3 ? 4 : 2;
  if constexpr (CH == 1) {
    return sample_leaf<D, MODE, S>(P, C, draw<D>(P, C, j0), brick, halo);
  } else if constexpr (CH == G) {
    Draw d[G];
    draw_group<D>(P, C, j0, d);
    Acc l[G];
#pragma unroll
    for (int k = 0; k < G; ++k) l[k] = sample_leaf<D, MODE, S>(P, C, d[k], brick, halo);
    if constexpr (G == 4) return acc_add(acc_add(l[0], l[1]), acc_add(l[2], l[3]));
    else return acc_add(l[0], l[1]);
  } else {
    const Acc l = chunk_sum<D, MODE, S, CH / 2>(P, C, j0, brick, halo);
    const Acc r = chunk_sum<D, MODE, S, CH / 2>(P, C, j0 + CH / 2, brick, halo);
    return acc_add(l, r);
  }
}

// Pairwise sum over CH samples with precomputed directions: the same perfect
// binary tree as chunk_sum (leaves in sample order).
template <int N>
__device__ __forceinline__ Acc tree_sum(const Acc* l) {
  if constexpr (N == 1) {
    return l[0];
  } else {
    return acc_add(tree_sum<N / 2>(l), tree_sum<N / 2>(l + N / 2));
  }
}

template <int D, int MODE, int S, int CH, int EST = 0>
__device__ __forceinline__ Acc chunk_sum_dirs(const EvoParams& P, const CellIt& C, const Dir* d,
                                              const uint16_t* brick, uint32_t& halo) {
  Acc l[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k)
    l[k] = sample_leaf<D, MODE, S, EST>(P, C, finish_draw<D, EST>(C, d[k]), brick, halo);
  return tree_sum<CH>(l);
}

// Pairwise sum over CH << L consecutive samples: 2^L chunks combined by a
// binary counter (stack of L partial sums) = a perfect pairwise tree.
template <int D, int MODE, int S, int CH, int L>
__device__ __forceinline__ Acc lane_sum(const EvoParams& P, const CellIt& C, uint32_t j0,
                                        const uint16_t* brick, uint32_t& halo) {
  if constexpr (L == 0) {
    return chunk_sum<D, MODE, S, CH>(P, C, j0, brick, halo);
  } else {
    Acc stk[L];
    Acc res{};
#pragma unroll 1
    for (int i = 0; i < (1 << L); ++i) {
      Acc x = chunk_sum<D, MODE, S, CH>(P, C, j0 + (uint32_t)(i * CH), brick, halo);
      bool carry = true;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        if (carry) {
          if ((i >> l) & 1) x = acc_add(stk[l], x);
          else { stk[l] = x; carry = false; }
        }
      }
      if (carry) res = x;
    }
    return res;
  }
}

__device__ __forceinline__ Acc warp_butterfly(Acc s) {
  // (l, l^1), (l, l^2), ... = pairwise over consecutive lane blocks
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Acc q;
    q.a0 = __shfl_xor_sync(0xffffffffu, s.a0, o);
    q.cx = __shfl_xor_sync(0xffffffffu, s.cx, o);
    q.cy = __shfl_xor_sync(0xffffffffu, s.cy, o);
    q.cz = __shfl_xor_sync(0xffffffffu, s.cz, o);
    q.aR = __shfl_xor_sync(0xffffffffu, s.aR, o);
    s = acc_add(s, q);
  }
  return s;
}

// The same pairwise lane tree as warp_butterfly, as a reduce-scatter: at each
// of the first three levels a lane keeps part of the components (and only
// exchanges the others), so 8 shuffles + 8 adds replace 25 + 25.  Each final
// sum equals warp_butterfly's bit for bit (same pairs; a + b == b + a).  The
// warp's five sums end in lanes 0..4 as components {0, 3, 2, 4, 1}; those lanes
// store them into out[component * stride].
__device__ __forceinline__ void warp_reduce_scatter(const Acc& v, float* out, int lane, int stride) {
  const unsigned F = 0xffffffffu;
  const bool odd = lane & 1, b1 = (lane >> 1) & 1, b2 = (lane >> 2) & 1;
  // level 1 (lanes l, l^1): even lanes keep {a0, cx, cy}, odd lanes {cz, aR}
  const float r0 = __shfl_xor_sync(F, odd ? v.a0 : v.cz, 1);
  const float r1 = __shfl_xor_sync(F, odd ? v.cx : v.aR, 1);
  const float r2 = __shfl_xor_sync(F, v.cy, 1);
  const float k0 = __fadd_rn(odd ? v.cz : v.a0, r0);
  const float k1 = __fadd_rn(odd ? v.aR : v.cx, r1);
  const float k2 = __fadd_rn(v.cy, r2);
  // level 2 (l, l^2): even: b1 = 0 keeps {a0, cx}, b1 = 1 keeps {cy}; odd: b1 = 0 keeps cz, b1 = 1 keeps aR
  const bool e0 = !odd && !b1;
  const float s0 = odd ? (b1 ? k0 : k1) : (b1 ? k0 : k2);
  const float q0 = __shfl_xor_sync(F, s0, 2);
  const float q1 = __shfl_xor_sync(F, k1, 2);
  const float m0 = __fadd_rn(odd ? (b1 ? k1 : k0) : (b1 ? k2 : k0), q0);
  const float m1 = __fadd_rn(k1, q1);   // meaningful on e0 lanes only
  // level 3 (l, l^4): e0 lanes split {a0, cx} by b2; the others hold one component
  const float t0 = __shfl_xor_sync(F, (e0 && !b2) ? m1 : m0, 4);
  float n0 = __fadd_rn((e0 && b2) ? m1 : m0, t0);
  // levels 4, 5: one component per lane
  n0 = __fadd_rn(n0, __shfl_xor_sync(F, n0, 8));
  n0 = __fadd_rn(n0, __shfl_xor_sync(F, n0, 16));
  if (lane < 5) out[((0x14230u >> (4 * lane)) & 0xFu) * stride] = n0;
}

// Pairwise tree over the W warps' partial sums of one component (same pairs as warp_tree).
template <int W>
__device__ __forceinline__ float comp_tree(const float* v) {
  float t[W];
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int w = 0; w < W; w += 4) {
      const float4 q = *reinterpret_cast<const float4*>(v + w);
      t[w] = q.x; t[w + 1] = q.y; t[w + 2] = q.z; t[w + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) t[w] = v[w];
  }
#pragma unroll
  for (int span = 1; span < W; span <<= 1)
#pragma unroll
    for (int w = 0; w + span < W; w += 2 * span) t[w] = __fadd_rn(t[w], t[w + span]);
  return t[0];
}

template <int W>
__device__ __forceinline__ Acc warp_tree(const Acc* v) {
  Acc t[W];
#pragma unroll
  for (int w = 0; w < W; ++w) t[w] = v[w];
#pragma unroll
  for (int span = 1; span < W; span <<= 1)
#pragma unroll
    for (int w = 0; w + span < W; w += 2 * span) t[w] = acc_add(t[w], t[w + span]);
  return t[0];
}

__device__ __forceinline__ float clampf(float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); }

// The per-cell state and the iteration update, shared by both kernels.  The
// state is the displacement u = c - seed (snk_cell.disp): |u| <= leash, so fp32
// resolves it to ~2e-6 voxel, where the absolute centre of a C4 cell (x up to
// 2047) only has 1.2e-4 — stepping c itself let fp32 trajectories drift ~1e-3
// from the fp64 oracle's (profiles/r2_state_precision.md).  The centre used by
// an iteration is c = seed + u, rounded to fp32.
struct CellState {
  float sx, sy, sz;     // seed
  float ux, uy, uz;     // displacement c - seed
  float R, E;
  uint32_t flags;
  int64_t id;
  uint32_t q0, q1, q3;  // Philox round-1 words of the constant counter words (id), keyed
};

__device__ __forceinline__ void cell_begin(const EvoParams& P, int64_t cell, int D, CellState& s) {
  if (P.state) {
    const snk_cell& r = P.state[cell];
    s.sx = r.seed[0];
    s.sy = r.seed[1];
    s.sz = r.seed[2];
    s.id = r.id;
  } else {
    s.sx = P.seeds[3 * cell + 0];
    s.sy = P.seeds[3 * cell + 1];
    s.sz = D == 3 ? P.seeds[3 * cell + 2] : 0.0f;
    s.id = P.ids ? P.ids[cell] : P.id_base + cell;
  }
  const uint32_t id_lo = (uint32_t)((uint64_t)s.id & 0xffffffffu);
  const uint32_t id_hi = (uint32_t)((uint64_t)s.id >> 32);
  // Philox round 1 for ctr = {b, n, id_lo, id_hi}: the M1 * id_lo product and
  // the key words do not depend on (b, n)
  const uint64_t p1 = (uint64_t)kM1 * id_lo;
  s.q0 = (uint32_t)(p1 >> 32) ^ P.rk0[0];
  s.q1 = (uint32_t)p1;
  s.q3 = id_hi ^ P.rk1[0];
  if (P.state) {
    const snk_cell& r = P.state[cell];
    s.ux = r.disp[0]; s.uy = r.disp[1]; s.uz = r.disp[2];
    s.R = r.R;
    s.E = r.energy;
    s.flags = r.flags;
  } else {
    s.ux = 0.0f; s.uy = 0.0f; s.uz = 0.0f;
    s.R = P.r0;
    s.E = 0.0f;
    s.flags = 0;
  }
}

__device__ __forceinline__ CellIt cell_iter(const EvoParams& P, const CellState& s, int it) {
  CellIt C;
  C.cx = __fadd_rn(s.sx, s.ux);
  C.cy = __fadd_rn(s.sy, s.uy);
  C.cz = __fadd_rn(s.sz, s.uz);
  C.rho_s = __fadd_rn(s.R, P.half_dR);
  C.a = __fmul_rn(-__fsub_rn(s.R, P.half_dR), P.inv_dR);
  C.p0 = s.q0 ^ (uint32_t)it;
  C.p1 = s.q1;
  C.p3 = s.q3;
  C.lg2_rho_s = lg2_approx(C.rho_s);
  C.boff = 0;
  return C;
}

// Energy, gradient and the clipped descent step; returns true after E_final.
// GRID: the sums are Eq. 5's voxel sums (unit voxel volume), scaled by iscale
// alone; MC: each sample carries V/N = (4/3 pi | pi) rho_s^d / N.
// RAY (G27): each step carries |S^(d-1)| rho_s t^(d-1) / N, the t^(d-1) already
// in the leaves, so the sums scale by vscale rho_s.
// NB: branch-free form (selects instead of the early return and the uniform
// branches, same arithmetic) so that the compiler can interleave the update
// with independent work of the same basic block (PIPE 3).
template <int D, bool GRID = false, int EST = 0, bool NB = false>
__device__ __forceinline__ bool cell_update(const EvoParams& P, CellState& s, const CellIt& C,
                                            const Acc& sum, int it) {
  const float rs = C.rho_s;
  const float vol = D == 3 ? __fmul_rn(__fmul_rn(rs, rs), rs) : __fmul_rn(rs, rs);
  const float scale = GRID ? P.vscale : (est_kind(EST) == SNK_EST_RAY ? __fmul_rn(P.vscale, rs) : __fmul_rn(P.vscale, vol));
  const float A0 = __fmul_rn(sum.a0, scale);
  const float twoR = __fmul_rn(2.0f, s.R);
  const float gden = D == 3 ? __fmul_rn(__fmul_rn(twoR, twoR), twoR) : __fmul_rn(twoR, twoR);
  const float gamma = rcp_approx(gden);
  s.E = __fmul_rn(gamma, A0);
  if (!NB && it == P.T + 1) return true;
  const float gs = __fmul_rn(__fmul_rn(gamma, scale), P.k6_dR);   // the leaves' 6/dR
  const float gcx = -__fmul_rn(gs, sum.cx), gcy = -__fmul_rn(gs, sum.cy), gcz = -__fmul_rn(gs, sum.cz);
  const float gR = __fmul_rn(gamma, __fsub_rn(__fmul_rn(__fmul_rn(sum.aR, scale), P.k6_dR),
                                              __fmul_rn(__fmul_rn(D == 3 ? 3.0f : 2.0f, rcp_approx(s.R)), A0)));
  // step eps_n / 2 with eps_n = eps0 / sqrt(n), clipped (G8)
  const float h = __fmul_rn(P.half_eps0, rsqrt_approx((float)it));
  const float dcx = clampf(-__fmul_rn(h, gcx), -P.max_step, P.max_step);
  const float dcy = clampf(-__fmul_rn(h, gcy), -P.max_step, P.max_step);
  const float dcz = D == 3 ? clampf(-__fmul_rn(h, gcz), -P.max_step, P.max_step) : 0.0f;
  const float dR = clampf(-__fmul_rn(h, gR), -P.max_step, P.max_step);
  const float ox = s.ux, oy = s.uy, oz = s.uz, oR = s.R;
  const float cx = __fadd_rn(s.ux, dcx), cy = __fadd_rn(s.uy, dcy), cz = __fadd_rn(s.uz, dcz);
  const float R = clampf(__fadd_rn(s.R, dR), P.r_min, P.r_max);
  // leash: |c_a - s_a| = |u_a| <= leash
  const float lx = clampf(cx, -P.leash, P.leash);
  const float ly = clampf(cy, -P.leash, P.leash);
  const float lz = D == 3 ? clampf(cz, -P.leash, P.leash) : cz;
  // domain: c_a = s_a + u_a in [m, L_a - m] (L_a = n_a - 1), m = R + dR/2, i.e.
  // u_a in [m - s_a, (L_a - m) - s_a]; or c_a = L_a / 2 when L_a < 2m (P.dom_small:
  // possible for some axis at all)
  const float m = __fadd_rn(R, P.half_dR);
  float dx, dy, dz = lz;
  if (NB) {
    const float m2 = __fmul_rn(2.0f, m);
    const bool small = !(EST & kBig) && P.dom_small != 0;
    dx = (small && P.dom1[0] < m2) ? __fsub_rn(__fmul_rn(0.5f, P.dom1[0]), s.sx)
                                   : clampf(lx, __fsub_rn(m, s.sx), __fsub_rn(__fsub_rn(P.dom1[0], m), s.sx));
    dy = (small && P.dom1[1] < m2) ? __fsub_rn(__fmul_rn(0.5f, P.dom1[1]), s.sy)
                                   : clampf(ly, __fsub_rn(m, s.sy), __fsub_rn(__fsub_rn(P.dom1[1], m), s.sy));
    if (D == 3)
      dz = (small && P.dom1[2] < m2) ? __fsub_rn(__fmul_rn(0.5f, P.dom1[2]), s.sz)
                                     : clampf(lz, __fsub_rn(m, s.sz), __fsub_rn(__fsub_rn(P.dom1[2], m), s.sz));
  } else if (P.dom_small) {
    const float m2 = __fmul_rn(2.0f, m);
    dx = P.dom1[0] < m2 ? __fsub_rn(__fmul_rn(0.5f, P.dom1[0]), s.sx)
                        : clampf(lx, __fsub_rn(m, s.sx), __fsub_rn(__fsub_rn(P.dom1[0], m), s.sx));
    dy = P.dom1[1] < m2 ? __fsub_rn(__fmul_rn(0.5f, P.dom1[1]), s.sy)
                        : clampf(ly, __fsub_rn(m, s.sy), __fsub_rn(__fsub_rn(P.dom1[1], m), s.sy));
    if (D == 3)
      dz = P.dom1[2] < m2 ? __fsub_rn(__fmul_rn(0.5f, P.dom1[2]), s.sz)
                          : clampf(lz, __fsub_rn(m, s.sz), __fsub_rn(__fsub_rn(P.dom1[2], m), s.sz));
  } else {
    dx = clampf(lx, __fsub_rn(m, s.sx), __fsub_rn(__fsub_rn(P.dom1[0], m), s.sx));
    dy = clampf(ly, __fsub_rn(m, s.sy), __fsub_rn(__fsub_rn(P.dom1[1], m), s.sy));
    if (D == 3) dz = clampf(lz, __fsub_rn(m, s.sz), __fsub_rn(__fsub_rn(P.dom1[2], m), s.sz));
  }
  if (NB) {
    const bool fin = it == P.T + 1;   // E_final only: no update
    s.ux = fin ? ox : dx;
    s.uy = fin ? oy : dy;
    s.uz = fin ? oz : dz;
    s.R = fin ? oR : R;
    if (it == P.T) {   // the flags of the last step (a uniform branch after the update)
      float mv = fabsf(__fsub_rn(R, oR));
      mv = fmaxf(mv, fabsf(__fsub_rn(dx, ox)));
      mv = fmaxf(mv, fabsf(__fsub_rn(dy, oy)));
      mv = fmaxf(mv, fabsf(__fsub_rn(dz, oz)));
      if (mv < P.conv_tol) s.flags |= SNK_F_CONVERGED;
      if ((lx != cx) || (ly != cy) || (lz != cz)) s.flags |= SNK_F_LEASHED;
      if ((dx != lx) || (dy != ly) || (dz != lz)) s.flags |= SNK_F_DOMAIN;
    }
    return fin;
  }
  s.ux = dx; s.uy = dy; s.uz = dz;
  s.R = R;
  if (it == P.T) {
    float mv = fabsf(__fsub_rn(R, oR));
    mv = fmaxf(mv, fabsf(__fsub_rn(s.ux, ox)));
    mv = fmaxf(mv, fabsf(__fsub_rn(s.uy, oy)));
    mv = fmaxf(mv, fabsf(__fsub_rn(s.uz, oz)));
    if (mv < P.conv_tol) s.flags |= SNK_F_CONVERGED;
    if ((lx != cx) || (ly != cy) || (lz != cz)) s.flags |= SNK_F_LEASHED;
    if ((dx != lx) || (dy != ly) || (dz != lz)) s.flags |= SNK_F_DOMAIN;
  }
  return false;
}

// Trivial contours as of the last iteration run.
__device__ __forceinline__ void cell_finish(const EvoParams& P, CellState& s, int64_t cell) {
  s.flags &= ~(uint32_t)(SNK_F_COLLAPSED | SNK_F_RMAX);
  if (s.R <= P.r_min) s.flags |= SNK_F_COLLAPSED;
  if (s.R >= P.r_max) s.flags |= SNK_F_RMAX;
  snk_cell o;
  o.c[0] = __fadd_rn(s.sx, s.ux);
  o.c[1] = __fadd_rn(s.sy, s.uy);
  o.c[2] = __fadd_rn(s.sz, s.uz);
  o.disp[0] = s.ux; o.disp[1] = s.uy; o.disp[2] = s.uz;
  o.reserved = 0;
  o.R = s.R;
  o.seed[0] = s.sx; o.seed[1] = s.sy; o.seed[2] = s.sz;
  o.energy = s.E;
  o.flags = s.flags;
  o.iters = min(P.it1, P.T);
  o.id = s.id;
  P.out[cell] = o;
}

// =========================================================================
// Generic kernel: W warps per cell, gathers from global memory.
template <int D, int W, bool SLAB, int CH, int L>
__global__ void __launch_bounds__(W >= 4 ? 32 * W : 128)
    evolve_warp_kernel(const __grid_constant__ EvoParams P) {
  constexpr int CPB = W >= 4 ? 1 : 4 / W;   // cells per block
  constexpr int B = CH << L;                // samples per thread per iteration
  constexpr int MODE = SLAB ? G_GLOBAL_SLAB : G_GLOBAL;
  __shared__ Acc xch[2][CPB][W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = warp / W, wsub = warp % W;
  const int64_t cell = (int64_t)blockIdx.x * CPB + slot;
  if (cell >= P.n) return;   // uniform per cell group (named barriers below)
  CellState s;
  cell_begin(P, cell, D, s);
  uint32_t halo = 0;
  const uint32_t j0 = (uint32_t)((wsub * 32 + lane) * B);
  for (int it = P.it0; it <= P.it1; ++it) {
    const CellIt C = cell_iter(P, s, it);
    Acc sum = warp_butterfly(lane_sum<D, MODE, 1, CH, L>(P, C, j0, nullptr, halo));
    if constexpr (W > 1) {
      if (lane == 0) xch[it & 1][slot][wsub] = sum;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * W) : "memory");
      sum = warp_tree<W>(xch[it & 1][slot]);
    }
    if (cell_update<D>(P, s, C, sum, it)) break;
  }
  if (SLAB) {
    if (__any_sync(0xffffffffu, halo != 0)) s.flags |= SNK_F_HALO;
    if constexpr (W > 1) {
      __shared__ uint32_t hf[CPB];
      if (wsub == 0 && lane == 0) hf[slot] = 0;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * W) : "memory");
      if (lane == 0 && (s.flags & SNK_F_HALO)) atomicOr(&hf[slot], SNK_F_HALO);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * W) : "memory");
      s.flags |= hf[slot];
    }
  }
  if (wsub == 0 && lane == 0) cell_finish(P, s, cell);
}

// =========================================================================
// Group kernel (small N, C5's sweep): G lanes per cell, 32 / G cells per warp,
// 4 warps per CTA.  A cell's N samples are split G ways (B = N / G per lane,
// contiguous blocks), summed by the in-lane pairwise tree and a butterfly over
// the G lanes — the same canonical tree as the warp kernel (bit-identical
// records) — and every lane takes its cell's update: one instruction stream
// serves 32 / G cells, so the per-iteration reduce and update (the
// occupancy / per-contour overhead the paper measured) are amortised over
// several cells.  No shared memory and no barriers; gathers through L1/L2,
// unclamped when every cell of the warp has its ball inside the volume.
#ifndef SNK_GROUP_MINB
#define SNK_GROUP_MINB 4
#endif
template <int D, int G, bool SLAB, int CH, int L>
__global__ void __launch_bounds__(128, SNK_GROUP_MINB) evolve_group_kernel(const __grid_constant__ EvoParams P) {
  constexpr int CPW = 32 / G;                // cells per warp
  constexpr int B = CH << L;                 // samples per lane per iteration
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cell = ((int64_t)blockIdx.x * 4 + warp) * CPW + lane / G;
  const bool valid = cell < P.n;
  if (((int64_t)blockIdx.x * 4 + warp) * CPW >= P.n) return;   // whole warp past the end
  const int sl = lane % G;
  CellState s;
  cell_begin(P, valid ? cell : P.n - 1, D, s);   // tail lanes shadow the last cell (no write)
  uint32_t halo = 0;
  const uint32_t j0 = (uint32_t)(sl * B);
  const float n1[3] = {P.fnx1, P.fny1, P.fnz1};
  for (int it = P.it0; it <= P.it1; ++it) {
    const CellIt C = cell_iter(P, s, it);
    Acc sum;
    bool fast = false;
    if (!SLAB) {
      // the d-linear taps of the ball [floor(c - ext), floor(c + ext) + 1] inside the volume
      const float ext = __fmaf_rn(C.rho_s, 1.0001f, 0.01f);
      const float c[3] = {C.cx, C.cy, C.cz};
      bool in = true;
#pragma unroll
      for (int a = 0; a < D; ++a) in &= __fsub_rn(c[a], ext) >= 0.0f && __fadd_rn(c[a], ext) + 1.0f <= n1[a];
      fast = __all_sync(0xffffffffu, in);
    }
    if (fast) sum = lane_sum<D, G_GLOBAL_FAST, 1, CH, L>(P, C, j0, nullptr, halo);
    else sum = lane_sum<D, SLAB ? G_GLOBAL_SLAB : G_GLOBAL, 1, CH, L>(P, C, j0, nullptr, halo);
    // the lane tree over the group: (l, l^1), (l, l^2), ... as warp_butterfly's first levels
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      Acc q;
      q.a0 = __shfl_xor_sync(0xffffffffu, sum.a0, o);
      q.cx = __shfl_xor_sync(0xffffffffu, sum.cx, o);
      q.cy = __shfl_xor_sync(0xffffffffu, sum.cy, o);
      q.cz = __shfl_xor_sync(0xffffffffu, sum.cz, o);
      q.aR = __shfl_xor_sync(0xffffffffu, sum.aR, o);
      sum = acc_add(sum, q);
    }
    if (cell_update<D>(P, s, C, sum, it)) break;
  }
  if (SLAB) {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) halo |= __shfl_xor_sync(0xffffffffu, halo, o);
    if (halo) s.flags |= SNK_F_HALO;
  }
  if (valid && sl == 0) cell_finish(P, s, cell);
}

// =========================================================================
// Brick kernel: one CTA (W warps) per cell; the u16 neighbourhood of the cell
// (x: brick_sx(S) columns from an even origin, y and z: S rows/planes) lives in
// shared memory, filled by 4-byte cp.async copies (LDGSTS) when the sampled
// ball leaves it.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int D, int S>
__device__ __forceinline__ void load_brick(uint16_t* brick, const EvoParams& P, int bx, int by, int bz,
                                           int zlo_buf) {
  constexpr int SX = brick_sx(S), WPR = SX / kBA;        // u16 per row, copy words per row
  const int nw = min(WPR, (P.nx - bx + kBA - 1) / kBA);   // words inside the volume (x)
  const int ny = min(S, P.ny - by);
  const int nzl = D == 3 ? min(S, P.z_lo + P.nz_buf - bz) : 1;
  // word (col, ry, rz) of the brick <- word col of volume row (by + ry, bz + rz);
  // offsets from the brick's first word, in 32-bit words (< 2^31: the brick spans <= S planes)
  using Word = typename std::conditional<kBA == 4, uint2, uint32_t>::type;
  const Word* src = reinterpret_cast<const Word*>(P.img) +
                    (((int64_t)(bz - zlo_buf) * P.ny + by) * P.nx + bx) / kBA;   // bx % kBA == 0
  const int rw = P.nx / kBA, pw = rw * P.ny;              // words per volume row / plane
  const uint32_t dst0 = smem_u32(brick);
  // A thread owns the (col, ry) columns p = threadIdx.x, + blockDim.x, ... of a
  // plane and copies each down all nzl planes: the bounds test is per column,
  // and a copy costs the LDGSTS plus two address increments (the per-word
  // (col, ry, rz) stepping took 29 instructions per word).
  constexpr uint32_t kPlaneBytes = (uint32_t)(SX * (D == 3 ? S : 1)) * 2u;
  for (int p = threadIdx.x; p < WPR * S; p += blockDim.x) {
    const int ry = p / WPR, col = p - ry * WPR;
    if (col >= nw || ry >= ny) continue;
    uint32_t dst = dst0 + (uint32_t)(ry * WPR + col) * (2u * kBA);
    const Word* s = src + (ry * rw + col);
    int rz = 0;
#pragma unroll 1
    for (; rz + 4 <= nzl; rz += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst + u * kPlaneBytes), "l"(s + u * pw),
                     "n"(2 * kBA)
                     : "memory");
      dst += 4 * kPlaneBytes;
      s += 4 * pw;
    }
    for (; rz < nzl; ++rz) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst), "l"(s), "n"(2 * kBA) : "memory");
      dst += kPlaneBytes;
      s += pw;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
}

// resident CTAs per SM the register budget is sized for (shared memory allows 3)
#ifndef SNK_BRICK_MINB8
#define SNK_BRICK_MINB8 2
#endif
#ifndef SNK_BRICK_MINB4
#define SNK_BRICK_MINB4 3
#endif
// PIPE (one chunk per thread, L == 0): the state-independent part of the next
// iteration's draws (Philox words -> direction, radial variate) is computed
// while warp 0 alone takes the update step, which it then broadcasts; the
// arithmetic is unchanged, only its placement.
// PIPE 2: every warp then takes the identical update itself — one barrier per
// iteration instead of two (C3/C4 evolve 0.7-0.8% faster).  PIPE 3 (default):
// as 2, with the next draws placed before a branch-free update so the two
// interleave (the Philox words are even hoisted above the barrier; +0.2-0.5%).
#ifndef SNK_BRICK_PIPE
#define SNK_BRICK_PIPE 3
#endif
// the f32x2 fast path (chunk8_fast_x2); 0 = scalar (same results)
#ifndef SNK_F32X2
#define SNK_F32X2 1
#endif
// Brick bookkeeping shared by the MC and grid brick kernels: the brick origin,
// the float bounds of the fast containment test and the index offset.
template <int D, int S, bool SLAB>
struct BrickCtl {
  int b[3];            // brick origin (global voxels)
  float in_lo[3], in_hi[3];
  uint32_t boff;
  int zlo, zhi;        // z range the brick may cover: the slab buffer

  __device__ __forceinline__ void init(const EvoParams& P) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      b[a] = -(1 << 28);   // none yet
      in_lo[a] = INFINITY;
      in_hi[a] = -INFINITY;
    }
    boff = 0;
    zlo = SLAB ? P.z_lo : 0;
    zhi = SLAB ? P.z_lo + P.nz_buf - 1 : P.nz - 1;
  }

  // Make the brick hold the tap box of the ball of radius rho_s around c (the
  // d-linear taps [floor(c - ext), floor(c + ext) + 1], a superset of the grid
  // voxels |k - c| < rho_s), re-loading it if needed.  Returns 0: inside the
  // brick and the volume (no clamps), 1: inside the brick with clamps, 2: the
  // ball does not fit (global gathers).  Called by all threads (uniform).
  //
  // Fast test: the tap box lies in the brick iff c - ext >= in_lo and c + ext <
  // in_hi per axis (exact for the integer bounds); only set for a brick inside
  // the volume, so containment also means no clamping is needed.
  // ANISO (G28): c and rho_s are physical; the box is taken in raw grid units
  template <bool ANISO = false>
  __device__ __forceinline__ int prepare(uint16_t* brick, const EvoParams& P, const float cp[3],
                                         float rho_s) {
    constexpr int EXT[3] = {brick_sx(S), S, S};   // brick extent per axis
    // bounding box of the sampled ball, with a margin for the fp32 rounding of t and k
    float vlo[3], vhi[3];
    bool fast = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const float c = ANISO ? __fmul_rn(cp[a], P.isc[a]) : cp[a];
      const float ext = __fmaf_rn(ANISO ? __fmul_rn(rho_s, P.isc[a]) : rho_s, 1.0001f, 0.01f);
      vlo[a] = __fsub_rn(c, ext);
      vhi[a] = __fadd_rn(c, ext);
      fast &= vlo[a] >= in_lo[a] && vhi[a] < in_hi[a];
    }
    if (fast) return 0;
    const int n[3] = {P.nx, P.ny, P.nz};
    bool interior = true, fits = true, inside = true;
    int lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      lo[a] = (int)floorf(vlo[a]);
      hi[a] = (int)floorf(vhi[a]) + 1;
      interior &= lo[a] >= 0 && hi[a] <= n[a] - 1;
      lo[a] = max(lo[a], 0);
      hi[a] = min(hi[a], n[a] - 1);
      fits &= hi[a] - lo[a] + 1 <= (a == 0 ? EXT[0] - (kBA - 1) : S);
      inside &= lo[a] >= b[a] && hi[a] <= b[a] + EXT[a] - 1;
    }
    if (D == 3 && SLAB) fits &= lo[2] >= zlo && hi[2] <= zhi;
    if (!inside && fits) {
      // re-centre: the ball's box in the middle of the brick, clipped to the
      // volume (z: the slab buffer); the x origin is even (4-byte copies)
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int amin = (a == 2) ? zlo : 0, amax = (a == 2) ? zhi : n[a] - 1;
        int o = lo[a] - (EXT[a] - (hi[a] - lo[a] + 1)) / 2;
        if (a == 0) o &= ~(kBA - 1);
        o = min(o, amax + 1 - EXT[a]);
        if (a == 0) o &= ~(kBA - 1);
        o = max(o, amin);
        b[a] = o;
        const bool in_vol = o >= 0 && o + EXT[a] - 1 <= n[a] - 1;
        in_lo[a] = in_vol ? (float)o : INFINITY;
        in_hi[a] = in_vol ? (float)(o + EXT[a] - 1) : -INFINITY;
      }
      // every read of the old brick finished before last iteration's barrier
      load_brick<D, S>(brick, P, b[0], b[1], D == 3 ? b[2] : 0, zlo);
      boff = (kMagicBits + (uint32_t)b[0]) + (kMagicBits + (uint32_t)b[1]) * (uint32_t)brick_sx(S);
      if (D == 3) boff += (kMagicBits + (uint32_t)b[2]) * (uint32_t)(brick_sx(S) * S);
      inside = true;
      if (threadIdx.x == 0) atomicAdd(&g_evolve_stats[0], 1ull);
    }
    return inside ? (interior ? 0 : 1) : 2;
  }
};

// 2D: an 8.4 KB brick, so registers alone set the occupancy: 4 CTAs (128
// registers) measured C2 evolve 7.34 -> 7.03 ms; 5 CTAs (96 registers) 7.33 ms
#ifndef SNK_BRICK_MINB2D
#define SNK_BRICK_MINB2D 4
#endif
template <int D, int W, int S, bool SLAB, int CH, int L, int EST = 0>
__global__ void __launch_bounds__(32 * W, D == 2 && W == 4 ? SNK_BRICK_MINB2D : (W == 4 ? SNK_BRICK_MINB4 : (W <= 2 ? 5 : SNK_BRICK_MINB8))) evolve_brick_kernel(const __grid_constant__ EvoParams P) {
  constexpr int B = CH << L;
  constexpr bool PIPE = SNK_BRICK_PIPE && L == 0;
  static_assert(EST == 0 || (PIPE && CH == 8), "CV / RAY estimators: 8 samples per thread, pipelined draws");
  extern __shared__ __align__(16) uint16_t brick[];
  __shared__ __align__(16) float xch[2][5][W];      // [parity][component][warp]
  __shared__ float bc[4];                           // PIPE: (ux, uy, uz, R) after warp 0's update
  const int lane = threadIdx.x & 31, wsub = threadIdx.x >> 5;
  const int64_t cell = blockIdx.x;
  CellState s;
  cell_begin(P, cell, D, s);
  uint32_t halo = 0;
  BrickCtl<D, S, SLAB> bk;
  bk.init(P);
  const uint32_t j0 = (uint32_t)((wsub * 32 + lane) * B);
  Dir dir[PIPE ? CH : 1];
  if constexpr (PIPE) {
    if constexpr (est_kind(EST) == SNK_EST_RAY) draw_dirs_ray<D>(P, cell_iter(P, s, P.it0), j0 / 8u, dir);
    else draw_dirs<D, CH>(P, cell_iter(P, s, P.it0), j0, dir);
  }
  for (int it = P.it0; it <= P.it1; ++it) {
    CellIt C = cell_iter(P, s, it);
    const float c[3] = {C.cx, C.cy, C.cz};
    const int mode = bk.template prepare<est_aniso(EST)>(brick, P, c, C.rho_s);
    Acc part;
    C.boff = bk.boff;
#if SNK_DIAG_NOCONF
    {
      constexpr int SX = brick_sx(S);
      C.lic = (uint32_t)((int)C.cx - bk.b[0]) + (uint32_t)((int)C.cy - bk.b[1]) * SX +
              (D == 3 ? (uint32_t)((int)C.cz - bk.b[2]) * (uint32_t)(SX * S) : 0u);
    }
#endif
    if constexpr (est_kind(EST) == SNK_EST_MC_CV) {
      // I(c): the same d-linear lookup as a sample at t = 0
      const float qx = est_aniso(EST) ? __fmul_rn(C.cx, P.isc[0]) : C.cx;
      const float qy = est_aniso(EST) ? __fmul_rn(C.cy, P.isc[1]) : C.cy;
      const float qz = est_aniso(EST) ? __fmul_rn(C.cz, P.isc[2]) : C.cz;
      if (mode == 0) C.ic = gather_tri<D, G_BRICK_FAST, S>(P, C, qx, qy, qz, brick, halo);
      else if (mode == 1) C.ic = gather_tri<D, G_BRICK_CLAMP, S>(P, C, qx, qy, qz, brick, halo);
      else C.ic = gather_tri<D, SLAB ? G_GLOBAL_SLAB : G_GLOBAL, S>(P, C, qx, qy, qz, brick, halo);
    }
    if constexpr (PIPE) {
      if (mode == 0) {
        if constexpr ((CH == 8 || CH == 4) && SNK_F32X2) part = chunk_fast_x2<D, S, CH, EST>(P, C, dir, brick);
        else part = chunk_sum_dirs<D, G_BRICK_FAST, S, CH, EST>(P, C, dir, brick, halo);
        if constexpr (SNK_BRICK_PIPE == 4) {
          // PIPE 4: the next iteration's draws in the same basic block as the
          // gathers, so the Philox rounds fill the shared-load latency
          CellIt Cn;
          Cn.p0 = s.q0 ^ (uint32_t)(it + 1);
          Cn.p1 = s.q1;
          Cn.p3 = s.q3;
          if constexpr (est_kind(EST) == SNK_EST_RAY) draw_dirs_ray<D>(P, Cn, j0 / 8u, dir);
          else draw_dirs<D, CH>(P, Cn, j0, dir);
        }
      } else if (mode == 1) {
        // a ball touching a face: the same f32x2 path with clamped coordinates
        if constexpr ((CH == 8 || CH == 4) && SNK_F32X2) part = chunk_fast_x2<D, S, CH, EST, true>(P, C, dir, brick);
        else part = chunk_sum_dirs<D, G_BRICK_CLAMP, S, CH, EST>(P, C, dir, brick, halo);
      } else {
        part = chunk_sum_dirs<D, SLAB ? G_GLOBAL_SLAB : G_GLOBAL, S, CH, EST>(P, C, dir, brick, halo);
        if (threadIdx.x == 0) atomicAdd(&g_evolve_stats[1], 1ull);
      }
      if constexpr (SNK_BRICK_PIPE == 4) {
        if (mode != 0) {
          CellIt Cn;
          Cn.p0 = s.q0 ^ (uint32_t)(it + 1);
          Cn.p1 = s.q1;
          Cn.p3 = s.q3;
          if constexpr (est_kind(EST) == SNK_EST_RAY) draw_dirs_ray<D>(P, Cn, j0 / 8u, dir);
          else draw_dirs<D, CH>(P, Cn, j0, dir);
        }
      }
    } else {
      if (mode == 0) {
        part = lane_sum<D, G_BRICK_FAST, S, CH, L>(P, C, j0, brick, halo);
      } else if (mode == 1) {
        part = lane_sum<D, G_BRICK_CLAMP, S, CH, L>(P, C, j0, brick, halo);
      } else {
        part = lane_sum<D, SLAB ? G_GLOBAL_SLAB : G_GLOBAL, S, CH, L>(P, C, j0, brick, halo);
        if (threadIdx.x == 0) atomicAdd(&g_evolve_stats[1], 1ull);
      }
    }
    float* xo = &xch[it & 1][0][0];
    warp_reduce_scatter(part, xo + wsub, lane, W);
    __syncthreads();   // also: every brick read of this iteration is done
    if constexpr (PIPE && SNK_BRICK_PIPE == 4) {
      Acc sum;
      sum.a0 = comp_tree<W>(xo + 0 * W);
      sum.cx = comp_tree<W>(xo + 1 * W);
      sum.cy = comp_tree<W>(xo + 2 * W);
      sum.cz = comp_tree<W>(xo + 3 * W);
      sum.aR = comp_tree<W>(xo + 4 * W);
      if (cell_update<D, false, EST, true>(P, s, C, sum, it)) break;
    } else if constexpr (PIPE && SNK_BRICK_PIPE == 3) {
      // PIPE 2 with the next iteration's draws placed before a branch-free
      // update in one basic block, so the two independent streams interleave
      Acc sum;
      sum.a0 = comp_tree<W>(xo + 0 * W);
      sum.cx = comp_tree<W>(xo + 1 * W);
      sum.cy = comp_tree<W>(xo + 2 * W);
      sum.cz = comp_tree<W>(xo + 3 * W);
      sum.aR = comp_tree<W>(xo + 4 * W);
      CellIt Cn;
      Cn.p0 = s.q0 ^ (uint32_t)(it + 1);
      Cn.p1 = s.q1;
      Cn.p3 = s.q3;
      if constexpr (est_kind(EST) == SNK_EST_RAY) draw_dirs_ray<D>(P, Cn, j0 / 8u, dir);
      else draw_dirs<D, CH>(P, Cn, j0, dir);
      if (cell_update<D, false, EST, true>(P, s, C, sum, it)) break;
    } else if constexpr (PIPE && SNK_BRICK_PIPE == 2) {
      // every warp takes the (identical) update itself: one barrier per
      // iteration; xch is double-buffered by parity, and the next brick reload
      // happens after this barrier, i.e. after every read of this iteration
      Acc sum;
      sum.a0 = comp_tree<W>(xo + 0 * W);
      sum.cx = comp_tree<W>(xo + 1 * W);
      sum.cy = comp_tree<W>(xo + 2 * W);
      sum.cz = comp_tree<W>(xo + 3 * W);
      sum.aR = comp_tree<W>(xo + 4 * W);
      if (cell_update<D, false, EST>(P, s, C, sum, it)) break;
      CellIt Cn;
      Cn.p0 = s.q0 ^ (uint32_t)(it + 1);
      Cn.p1 = s.q1;
      Cn.p3 = s.q3;
      if constexpr (est_kind(EST) == SNK_EST_RAY) draw_dirs_ray<D>(P, Cn, j0 / 8u, dir);
      else draw_dirs<D, CH>(P, Cn, j0, dir);
    } else if constexpr (PIPE) {
      const bool done = it == P.T + 1;
      if (wsub == 0) {
        Acc sum;
        sum.a0 = comp_tree<W>(xo + 0 * W);
        sum.cx = comp_tree<W>(xo + 1 * W);
        sum.cy = comp_tree<W>(xo + 2 * W);
        sum.cz = comp_tree<W>(xo + 3 * W);
        sum.aR = comp_tree<W>(xo + 4 * W);
        cell_update<D, false, EST>(P, s, C, sum, it);
        if (lane == 0) { bc[0] = s.ux; bc[1] = s.uy; bc[2] = s.uz; bc[3] = s.R; }
      }
      if (done) break;
      CellIt Cn;   // the next iteration's Philox key words
      Cn.p0 = s.q0 ^ (uint32_t)(it + 1);
      Cn.p1 = s.q1;
      Cn.p3 = s.q3;
      if constexpr (est_kind(EST) == SNK_EST_RAY) draw_dirs_ray<D>(P, Cn, j0 / 8u, dir);
      else draw_dirs<D, CH>(P, Cn, j0, dir);
      __syncthreads();
      if (wsub != 0) { s.ux = bc[0]; s.uy = bc[1]; s.uz = bc[2]; s.R = bc[3]; }
    } else {
      Acc sum;
      sum.a0 = comp_tree<W>(xo + 0 * W);
      sum.cx = comp_tree<W>(xo + 1 * W);
      sum.cy = comp_tree<W>(xo + 2 * W);
      sum.cz = comp_tree<W>(xo + 3 * W);
      sum.aR = comp_tree<W>(xo + 4 * W);
      if (cell_update<D>(P, s, C, sum, it)) break;
    }
  }
  if (SLAB && __syncthreads_or(halo != 0)) s.flags |= SNK_F_HALO;
  if (threadIdx.x == 0) cell_finish(P, s, cell);
}

// =========================================================================
// Grid kernel (SNK_EST_GRID): the paper's original uniform integration, Eq. 5
// — per iteration the sum over the voxels k with |k - c| < R + dR/2
// of S(|k - c|) I(k) and its derivatives (Eqs. 7-10), I(k) read at the voxel (no
// interpolation), unit voxel volume, the radial term 0 at r = 0.  The
// baseline Monte-Carlo integration replaced (Figs. 6-7).  One CTA of W
// warps per cell with the same shared-memory brick as the MC kernel; warp w
// takes the rows (y, z) w, w + W, ... of the voxel box, lane l the voxels x0 +
// l, x0 + l + 32, ... of a row (consecutive u16: conflict-free LDS), rows
// outside the ball skipped whole.  Sums: per thread in row order, then the
// lane and warp trees of the MC kernel — a fixed order, so the result is
// deterministic (it is not the oracle's order: parity is to tolerance).
template <int D, int W, int S, bool SLAB>
__global__ void __launch_bounds__(32 * W, 3) evolve_grid_kernel(const __grid_constant__ EvoParams P) {
  extern __shared__ __align__(16) uint16_t brick[];
  __shared__ __align__(16) float xch[2][5][W];
  constexpr int SX = brick_sx(S), SP = SX * S;
  const int lane = threadIdx.x & 31, wsub = threadIdx.x >> 5;
  const int64_t cell = blockIdx.x;
  CellState s;
  cell_begin(P, cell, D, s);
  uint32_t halo = 0;
  BrickCtl<D, S, SLAB> bk;
  bk.init(P);
  const int n[3] = {P.nx, P.ny, P.nz};
  const float fn1[3] = {P.fnx1, P.fny1, P.fnz1};
  for (int it = P.it0; it <= P.it1; ++it) {
    const CellIt C = cell_iter(P, s, it);
    const float c[3] = {C.cx, C.cy, C.cz};
    const int mode = bk.prepare(brick, P, c, C.rho_s);
    const float rs = C.rho_s, rs2 = __fmul_rn(rs, rs);
    // the voxel box (a superset of the ball: membership is decided by r^2 < rs^2)
    const float ext = __fmaf_rn(rs, 1.0001f, 0.01f);
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      lo[a] = (int)ceilf(fmaxf(__fsub_rn(c[a], ext), 0.0f));
      hi[a] = (int)floorf(fminf(__fadd_rn(c[a], ext), fn1[a]));
    }
    (void)n;
    const int nyb = hi[1] - lo[1] + 1, nzb = D == 3 ? hi[2] - lo[2] + 1 : 1;
    const int nrows = nyb * nzb;
    Acc part{0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    for (int r = wsub; r < nrows; r += W) {
      const int z = D == 3 ? lo[2] + r / nyb : 0;
      const int y = lo[1] + (D == 3 ? r % nyb : r);
      const float dy = __fsub_rn((float)y, c[1]);
      const float dz = D == 3 ? __fsub_rn((float)z, c[2]) : 0.0f;
      const float dyz2 = __fmaf_rn(dz, dz, __fmul_rn(dy, dy));
      if (!(dyz2 < rs2)) continue;   // the row misses the ball (warp-uniform)
      const uint16_t* src;           // the row, indexed by global x
      if (mode != 2) {
        src = brick + ((D == 3 ? (z - bk.b[2]) * SP : 0) + (y - bk.b[1]) * SX - bk.b[0]);
      } else {
        if (SLAB && D == 3 && (z < P.z_lo || z >= P.z_lo + P.nz_buf)) {
          halo = 1u;                 // a voxel of the ball outside the slab buffer
          continue;
        }
        src = P.img + ((int64_t)(z - (SLAB ? P.z_lo : 0)) * P.ny + y) * (int64_t)P.nx;
      }
      for (int x = lo[0] + lane; x <= hi[0]; x += 32) {
        const float dx = __fsub_rn((float)x, c[0]);
        const float r2 = __fmaf_rn(dx, dx, dyz2);
        if (!(r2 < rs2)) continue;
        const float v = mag(src[x]);
        const float rr = __fsqrt_rn(r2);
        const float inv = r2 > 0.0f ? __frcp_rn(rr) : 0.0f;
        Draw d;
        d.t = rr;
        d.ox = __fmul_rn(dx, inv);
        d.oy = __fmul_rn(dy, inv);
        d.oz = __fmul_rn(dz, inv);
        part = acc_add(part, leaves(P, C, d, v, D == 3));
      }
    }
    float* xo = &xch[it & 1][0][0];
    warp_reduce_scatter(part, xo + wsub, lane, W);
    __syncthreads();   // also: every brick read of this iteration is done
    Acc sum;
    sum.a0 = comp_tree<W>(xo + 0 * W);
    sum.cx = comp_tree<W>(xo + 1 * W);
    sum.cy = comp_tree<W>(xo + 2 * W);
    sum.cz = comp_tree<W>(xo + 3 * W);
    sum.aR = comp_tree<W>(xo + 4 * W);
    if (cell_update<D, true>(P, s, C, sum, it)) break;
  }
  if (SLAB && __syncthreads_or(halo != 0)) s.flags |= SNK_F_HALO;
  if (threadIdx.x == 0) cell_finish(P, s, cell);
}

// ------------------------------------------------------------------ launching
template <int D, int W, bool SLAB, int CH, int L>
int32_t launch_warp(const EvoParams& P, cudaStream_t st) {
  constexpr int CPB = W >= 4 ? 1 : 4 / W;
  evolve_warp_kernel<D, W, SLAB, CH, L><<<(unsigned)ceil_div(P.n, CPB), 32 * W * CPB, 0, st>>>(P);
  SNK_LAUNCH_CHECK("evolve_warp_kernel");
  return SNK_OK;
}

template <int D, int G, bool SLAB, int CH, int L>
int32_t launch_group(const EvoParams& P, cudaStream_t st) {
  constexpr int CPB = 4 * (32 / G);
  evolve_group_kernel<D, G, SLAB, CH, L><<<(unsigned)ceil_div(P.n, CPB), 128, 0, st>>>(P);
  SNK_LAUNCH_CHECK("evolve_group_kernel");
  return SNK_OK;
}

template <int D, int G, bool SLAB>
int32_t group_B(const EvoParams& P, int B, cudaStream_t st) {
  switch (B) {
    case 4: return launch_group<D, G, SLAB, 4, 0>(P, st);
    case 8: return launch_group<D, G, SLAB, 4, 1>(P, st);
    case 16: return launch_group<D, G, SLAB, 4, 2>(P, st);
    case 32: return launch_group<D, G, SLAB, 4, 3>(P, st);
    default: return fail(SNK_CONFIG, "group kernel: 4 .. 32 samples per lane");
  }
}

template <int D, bool SLAB>
int32_t group_G(const EvoParams& P, int G, int B, cudaStream_t st) {
  switch (G) {
    case 4: return group_B<D, 4, SLAB>(P, B, st);
    case 8: return group_B<D, 8, SLAB>(P, B, st);
    case 16: return group_B<D, 16, SLAB>(P, B, st);
    default: return fail(SNK_CONFIG, "group kernel: 4, 8 or 16 lanes per cell");
  }
}

// lanes per cell of the group kernel: B = 8 samples per lane (SNK_GROUP_B
// overrides, tuning only; B = 16 measured 15-40% slower on C5); 0 when the
// group kernel does not apply
int group_lanes(int n_samples) {
  // default: as many lanes per cell as allowed (G <= 16, B >= 4 samples per
  // lane) — small N leaves few warps in flight (C5_0 at N = 64: 4 warps per SM
  // with B = 8), so parallelism beats the longer butterfly: B = 4 measured
  // C5_0 1.88 -> 1.36 ms, C5_3 9.56 -> 8.35 ms at N = 64
  const char* e = getenv("SNK_GROUP_B");
  int B = 4;
  while (n_samples / B > 16) B *= 2;
  if (e) B = atoi(e);
  if (B < 4 || B > 32 || (B & (B - 1))) return 0;
  const int G = n_samples / B;
  return (G >= 4 && G <= 16 && G * B == n_samples) ? G : 0;
}

template <int D, int W, int S, bool SLAB, int CH, int L, int EST = 0>
int32_t launch_brick(const EvoParams& P, cudaStream_t st) {
  auto k = evolve_brick_kernel<D, W, S, SLAB, CH, L, EST>;
  const int smem = (D == 3 ? brick_sx(S) * S * S : brick_sx(S) * S) * 2;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] { attr_err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  if (attr_err != cudaSuccess) return cuda_fail(attr_err, "cudaFuncSetAttribute(evolve_brick_kernel)");
  k<<<(unsigned)P.n, 32 * W, smem, st>>>(P);
  SNK_LAUNCH_CHECK("evolve_brick_kernel");
  return SNK_OK;
}

template <int D, int W, int S, bool SLAB>
int32_t launch_grid(const EvoParams& P, cudaStream_t st) {
  auto k = evolve_grid_kernel<D, W, S, SLAB>;
  const int smem = (D == 3 ? brick_sx(S) * S * S : brick_sx(S) * S) * 2;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] { attr_err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  if (attr_err != cudaSuccess) return cuda_fail(attr_err, "cudaFuncSetAttribute(evolve_grid_kernel)");
  k<<<(unsigned)P.n, 32 * W, smem, st>>>(P);
  SNK_LAUNCH_CHECK("evolve_grid_kernel");
  return SNK_OK;
}

// B samples per thread: 1, 2 (one chunk) or 4 << L (chunks of 4, L <= 5).
#define SNK_DISPATCH_B(B, CALL)                              \
  switch (B) {                                               \
    case 1: { constexpr int CH = 1, L = 0; return CALL; }    \
    case 2: { constexpr int CH = 2, L = 0; return CALL; }    \
    case 4: { constexpr int CH = 4, L = 0; return CALL; }    \
    case 8: { constexpr int CH = 4, L = 1; return CALL; }    \
    case 16: { constexpr int CH = 4, L = 2; return CALL; }   \
    case 32: { constexpr int CH = 4, L = 3; return CALL; }   \
    case 64: { constexpr int CH = 4, L = 4; return CALL; }   \
    case 128: { constexpr int CH = 4, L = 5; return CALL; }  \
    default: return fail(SNK_CONFIG, "samples per thread must be a power of two <= 128"); \
  }

template <int D, int W, bool SLAB>
int32_t warp_B(const EvoParams& P, int B, cudaStream_t st) {
  SNK_DISPATCH_B(B, (launch_warp<D, W, SLAB, CH, L>(P, st)))
}

template <int D, bool SLAB>
int32_t warp_W(const EvoParams& P, int W, int B, cudaStream_t st) {
  switch (W) {
    case 1: return warp_B<D, 1, SLAB>(P, B, st);
    case 2: return warp_B<D, 2, SLAB>(P, B, st);
    case 4: return warp_B<D, 4, SLAB>(P, B, st);
    case 8: return warp_B<D, 8, SLAB>(P, B, st);
    default: return fail(SNK_CONFIG, "bad warps per cell");
  }
}

#ifndef SNK_BRICK_S3
#define SNK_BRICK_S3 33
#endif
constexpr int kS3 = SNK_BRICK_S3;

template <int D, int W, int S, bool SLAB>
int32_t brick_B(const EvoParams& P, int B, cudaStream_t st) {
  // 8 samples per chunk: the brick kernel runs 12 warps/SM (shared memory
  // bound), so each warp needs the ILP of 8 independent sample chains
#ifndef SNK_BRICK_CH
#define SNK_BRICK_CH 8
#endif
  constexpr int C8 = SNK_BRICK_CH;
  switch (B) {
    case 1: return launch_brick<D, W, S, SLAB, 1, 0>(P, st);
    case 2: return launch_brick<D, W, S, SLAB, 2, 0>(P, st);
    case 4: return launch_brick<D, W, S, SLAB, 4, 0>(P, st);
    case 8:
      if (SNK_BIG && C8 == 8 && !P.dom_small && SNK_BRICK_PIPE == 3) return launch_brick<D, W, S, SLAB, 8, 0, kBig>(P, st);
      return launch_brick<D, W, S, SLAB, (C8 < 8 ? C8 : 8), (C8 < 8 ? 1 : 0)>(P, st);
    case 16: return launch_brick<D, W, S, SLAB, C8, (C8 < 8 ? 2 : 1)>(P, st);
    case 32: return launch_brick<D, W, S, SLAB, C8, (C8 < 8 ? 3 : 2)>(P, st);
    case 64: return launch_brick<D, W, S, SLAB, C8, (C8 < 8 ? 4 : 3)>(P, st);
    case 128: return launch_brick<D, W, S, SLAB, C8, (C8 < 8 ? 5 : 4)>(P, st);
    default: return fail(SNK_CONFIG, "samples per thread must be a power of two <= 128");
  }
}

// Small N (< 1024) with small contours: 1 or 2 warps per cell keep 8 samples
// per thread (the per-iteration update is paid per warp), and a 28 x 27 x 27
// brick (40.8 KB) lets 5 CTAs share an SM.
#ifndef SNK_BRICK_S3SMALL
#define SNK_BRICK_S3SMALL 27
#endif
constexpr int kS3small = SNK_BRICK_S3SMALL;
template <int W, bool SLAB>
int32_t brick_small_B(const EvoParams& P, int B, cudaStream_t st) {
  switch (B) {
    case 2: return launch_brick<3, W, kS3small, SLAB, 2, 0>(P, st);
    case 4: return launch_brick<3, W, kS3small, SLAB, 4, 0>(P, st);
    case 8: return launch_brick<3, W, kS3small, SLAB, 8, 0>(P, st);
    default: return fail(SNK_INTERNAL, "brick_small_B: 2, 4 or 8 samples per thread");
  }
}

__global__ void cells_init_kernel(const float* seeds, const int64_t* ids, int64_t id_base, int64_t n,
                                  float r0, snk_cell* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  snk_cell o;
  for (int a = 0; a < 3; ++a) {
    o.c[a] = o.seed[a] = seeds[3 * i + a];
    o.disp[a] = 0.0f;
  }
  o.reserved = 0;
  o.R = r0;
  o.energy = 0.0f;
  o.flags = 0;
  o.iters = 0;
  o.id = ids ? ids[i] : id_base + i;
  out[i] = o;
}

}  // namespace

int32_t cells_init_impl(const snk_params* p, const float* d_seeds, const int64_t* d_ids,
                        int64_t id_base, int64_t n, snk_cell* d_cells, cudaStream_t st) {
  if (n == 0) return SNK_OK;
  cells_init_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d_seeds, d_ids, id_base, n,
                                                                 (float)p->r0, d_cells);
  SNK_LAUNCH_CHECK("cells_init_kernel");
  return SNK_OK;
}

int32_t evolve_stats(int64_t out[4], bool reset) {
  unsigned long long h[4];
  SNK_CUDA_CHECK(cudaMemcpyFromSymbol(h, g_evolve_stats, sizeof h));
  for (int i = 0; i < 4; ++i) out[i] = (int64_t)h[i];
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    SNK_CUDA_CHECK(cudaMemcpyToSymbol(g_evolve_stats, z, sizeof z));
  }
  return SNK_OK;
}

int evolve_warps_per_cell(const snk_params* p, int64_t n_cells) {
  int W = p->cta_warps;
  if (W <= 0) {
    // enough warps to fill every SM with >= 32 warps -> warp-per-cell; else
    // spread each cell over more warps (the paper's §II-F fix)
    W = 1;
    while (W < 8 && n_cells * W < 148 * 32 && p->n_samples >= 32 * 2 * W) W *= 2;
  }
  while (p->n_samples / (32 * W) > 128 && W < 8) W *= 2;
  return W;
}

size_t evolve_ws(const snk_grid* g, const snk_params* p, int64_t max_cells) {
  (void)g; (void)p; (void)max_cells;
  return 0;
}

int32_t evolve_impl(const snk_grid* g, const snk_params* p, const uint16_t* d_image,
                    const float* d_seeds, const int64_t* d_ids, int64_t id_base, int64_t n,
                    snk_cell* d_cells, void* d_ws, size_t ws_bytes, cudaStream_t st, int it0, int it1,
                    bool resume) {
  (void)d_ws; (void)ws_bytes;
  if (n == 0) return SNK_OK;
  const int D = g->dim;
  EvoParams P;
  P.img = d_image;
  P.seeds = d_seeds;
  P.ids = d_ids;
  P.out = d_cells;
  P.id_base = id_base;
  P.n = n;
  P.nx = (int)g->n[0];
  P.ny = (int)g->n[1];
  P.nz = (int)g->n[2];
  P.z_lo = (int)g->z_lo;
  P.nz_buf = (int)g->nz_buf;
  P.fnx1 = (float)(g->n[0] - 1);
  P.fny1 = (float)(g->n[1] - 1);
  P.fnz1 = (float)(g->n[2] - 1);
  P.mx2 = 8388608.0f + (float)(g->n[0] - 2);
  P.my2 = 8388608.0f + (float)(g->n[1] - 2);
  P.mz2 = 8388608.0f + (float)std::max<int64_t>(g->n[2] - 2, 0);
  const double rho = rho_of(D);
  P.r0 = (float)p->r0;
  P.half_dR = (float)(p->delta_R / 2.0);
  P.inv_dR = (float)(1.0 / p->delta_R);
  P.inv_rho_dR = (float)(1.0 / (rho * p->delta_R));
  P.k2_rho = (float)(2.0 / rho);
  P.k6_dR = (float)(6.0 / p->delta_R);
  P.eps0 = (float)p->eps0;
  P.half_eps0 = (float)(p->eps0 / 2.0);
  P.max_step = (float)p->max_step;
  P.r_min = (float)p->r_min;
  P.r_max = (float)p->r_max;
  P.leash = (float)p->leash;
  P.conv_tol = (float)p->conv_tol;
  const double pi = 3.14159265358979323846;
  P.vscale = (float)(p->intensity_scale * (D == 3 ? 4.0 / 3.0 * pi : pi) / (double)p->n_samples);
  P.T = p->max_iters;
  P.it0 = it0 > 0 ? it0 : 1;
  P.it1 = it1 > 0 ? it1 : p->max_iters + 1;
  P.state = resume ? d_cells : nullptr;
  for (int a = 0; a < 3; ++a) {
    const double sc = grid_scale(g, a);
    P.isc[a] = (float)(1.0 / sc);
    P.dom1[a] = (float)((double)(g->n[a] - 1) * sc);   // = fn1 exactly when isotropic
  }
  {
    const double m2 = 2.0 * ((double)P.r_max + (double)P.half_dR) * (1.0 + 1e-6) + 1e-3;   // conservative
    P.dom_small = (double)P.dom1[0] < m2 || (double)P.dom1[1] < m2 || (D == 3 && (double)P.dom1[2] < m2);
  }
  uint32_t k0 = (uint32_t)(p->seed & 0xffffffffu), k1 = (uint32_t)(p->seed >> 32);
  for (int r = 0; r < 10; ++r) {
    P.rk0[r] = k0;
    P.rk1[r] = k1;
    k0 += kW0;
    k1 += kW1;
  }
  if (D == 3 && g->n[2] < 2) return fail(SNK_SHAPE, "3D needs nz >= 2");
  if (g->n[0] * g->n[1] * g->nz_buf >= ((int64_t)1 << 32)) return fail(SNK_SHAPE, "buffer too large");
  const bool slab = !(g->z_lo == 0 && g->nz_buf == g->n[2]);
  if (p->estimator == SNK_EST_GRID) {
    // Eq. 5 voxel sums: the brick kernel's brick, 8 warps per cell (rows)
    if (g->n[0] % 2 != 0 || (reinterpret_cast<uintptr_t>(d_image) & 3) != 0 || p->kernel_variant == 1)
      return fail(SNK_CONFIG, "the grid estimator needs the brick kernel (even nx, 4-byte aligned image)");
    P.vscale = (float)p->intensity_scale;
    if (D == 3) return slab ? launch_grid<3, 8, kS3, true>(P, st) : launch_grid<3, 8, kS3, false>(P, st);
    return launch_grid<2, 8, 64, false>(P, st);
  }
  if (grid_aniso(g)) {
    // physical-coordinate sampling on the raw anisotropic grid (G28): the brick
    // kernel, 4 warps x 8 samples per thread, 3D
    if (D != 3 || g->n[0] % 2 != 0 || (reinterpret_cast<uintptr_t>(d_image) & 3) != 0 || p->kernel_variant == 1 ||
        !(p->cta_warps == 0 || p->cta_warps == 4) || p->n_samples != 1024 || p->estimator == SNK_EST_GRID)
      return fail(SNK_CONFIG, "anisotropic grids: 3D brick kernel with 4 warps and n_samples = 1024 (MC / CV / ray)");
    if (p->estimator == SNK_EST_RAY) {
      const double pi = 3.14159265358979323846;
      P.vscale = (float)(p->intensity_scale * 4.0 * pi / (double)p->n_samples);
    }
    constexpr int A0 = kAniso, A2 = kAniso | SNK_EST_MC_CV, A3 = kAniso | SNK_EST_RAY;
    switch (p->estimator) {
      case SNK_EST_MC_CV: return slab ? launch_brick<3, 4, kS3, true, 8, 0, A2>(P, st) : launch_brick<3, 4, kS3, false, 8, 0, A2>(P, st);
      case SNK_EST_RAY: return slab ? launch_brick<3, 4, kS3, true, 8, 0, A3>(P, st) : launch_brick<3, 4, kS3, false, 8, 0, A3>(P, st);
      default: return slab ? launch_brick<3, 4, kS3, true, 8, 0, A0>(P, st) : launch_brick<3, 4, kS3, false, 8, 0, A0>(P, st);
    }
  }
  if (p->estimator == SNK_EST_MC_CV || p->estimator == SNK_EST_RAY) {
    // brick kernel with pipelined draws, 8 samples (one ray) per thread
    const int W = p->cta_warps > 0 ? p->cta_warps : 4;
    if (g->n[0] % 2 != 0 || (reinterpret_cast<uintptr_t>(d_image) & 3) != 0 || p->kernel_variant == 1 ||
        !(W == 4 || W == 8) || p->n_samples != 8 * 32 * W)
      return fail(SNK_CONFIG, "the CV / ray estimators need the brick kernel (even nx) with n_samples = 256 * warps "
                              "per cell (4 warps: N = 1024, 8 warps: N = 2048)");
    if (p->estimator == SNK_EST_RAY) {
      const double pi = 3.14159265358979323846;
      P.vscale = (float)(p->intensity_scale * (D == 3 ? 4.0 * pi : 2.0 * pi) / (double)p->n_samples);
    }
    constexpr int CV = SNK_EST_MC_CV, RY = SNK_EST_RAY;
    const bool ray = p->estimator == SNK_EST_RAY;
    if (D == 3) {
      if (W == 4) {
        if (slab) return ray ? launch_brick<3, 4, kS3, true, 8, 0, RY>(P, st) : launch_brick<3, 4, kS3, true, 8, 0, CV>(P, st);
        return ray ? launch_brick<3, 4, kS3, false, 8, 0, RY>(P, st) : launch_brick<3, 4, kS3, false, 8, 0, CV>(P, st);
      }
      if (slab) return ray ? launch_brick<3, 8, kS3, true, 8, 0, RY>(P, st) : launch_brick<3, 8, kS3, true, 8, 0, CV>(P, st);
      return ray ? launch_brick<3, 8, kS3, false, 8, 0, RY>(P, st) : launch_brick<3, 8, kS3, false, 8, 0, CV>(P, st);
    }
    if (W == 4) return ray ? launch_brick<2, 4, 64, false, 8, 0, RY>(P, st) : launch_brick<2, 4, 64, false, 8, 0, CV>(P, st);
    return ray ? launch_brick<2, 8, 64, false, 8, 0, RY>(P, st) : launch_brick<2, 8, 64, false, 8, 0, CV>(P, st);
  }
  // kernel choice: 0 auto, 1 warp (global gathers), 2 brick (shared memory)
  const uint32_t variant = p->kernel_variant;
  const int Wb = p->cta_warps > 0 ? p->cta_warps : 4;
  const int Bb = p->n_samples / (32 * Wb);
  // the brick kernel copies 4-byte words from an even x origin: needs even nx
  // and a 4-byte aligned image
  const bool brick_ok = variant != 1 && Bb >= 1 && Bb <= 128 && (Wb == 4 || Wb == 8) &&
                        g->n[0] % kBA == 0 && (reinterpret_cast<uintptr_t>(d_image) & (2 * kBA - 1)) == 0;
  if (variant == 2 && !brick_ok) return fail(SNK_CONFIG, "brick kernel unavailable for this volume");
  // small N (C5's sweep): several cells per warp (variant 3; auto for N < 128,
  // where the small-brick kernel would hold one warp per 41 KB brick: C5 at
  // N = 64 1.89 vs 2.19 ms for the warp kernel; from N = 128 the brick wins)
  if (variant == 3 || (variant == 0 && p->cta_warps == 0 && p->n_samples < 128)) {
    const int G = group_lanes(p->n_samples);
    if (G > 0) {
      const int B = p->n_samples / G;
      if (D == 3) return slab ? group_G<3, true>(P, G, B, st) : group_G<3, false>(P, G, B, st);
      return group_G<2, false>(P, G, B, st);
    }
    if (variant == 3) return fail(SNK_CONFIG, "group kernel: n_samples = G x B with G in 4..16, B in 4..32");
  }
  // small N and small contours (C5's sweep): the small-brick kernel, auto warps only
  const bool small_ok = variant != 1 && D == 3 && p->cta_warps == 0 && p->n_samples >= 128 &&
                        p->n_samples < 1024 && p->r0 <= 9.5 && g->n[0] % 2 == 0 &&
                        (reinterpret_cast<uintptr_t>(d_image) & 3) == 0;
  if (small_ok) {
    // 2 warps per cell from N = 256 (C5 at N = 256: 1.95 -> 1.74 ms / 14.9 -> 13.7
    // ms against 1 warp with 8 samples per lane; at N = 128 one warp is faster)
    int Ws = p->n_samples >= 256 ? 2 : 1;
    if (const char* e = getenv("SNK_SMALL_W")) Ws = atoi(e) == 2 ? 2 : 1;   // tuning experiments
    const int Bs = p->n_samples / (32 * Ws);
    if (Ws == 2) return slab ? brick_small_B<2, true>(P, Bs, st) : brick_small_B<2, false>(P, Bs, st);
    return slab ? brick_small_B<1, true>(P, Bs, st) : brick_small_B<1, false>(P, Bs, st);
  }
  if (brick_ok) {
    if (D == 3) {
      // S = 33: 34 x 33 x 33 u16 = 72.3 KB, three CTAs per SM; covers balls up to rho_s ~ 15.5
      if (Wb == 4) return slab ? brick_B<3, 4, kS3, true>(P, Bb, st) : brick_B<3, 4, kS3, false>(P, Bb, st);
      return slab ? brick_B<3, 8, kS3, true>(P, Bb, st) : brick_B<3, 8, kS3, false>(P, Bb, st);
    }
    if (Wb == 4) return brick_B<2, 4, 64, false>(P, Bb, st);
    return brick_B<2, 8, 64, false>(P, Bb, st);
  }
  const int W = evolve_warps_per_cell(p, n);
  const int B = p->n_samples / (32 * W);
  if (B < 1) return fail(SNK_CONFIG, "n_samples < 32 * warps per cell");
  if (D == 3) return slab ? warp_W<3, true>(P, W, B, st) : warp_W<3, false>(P, W, B, st);
  return warp_W<2, false>(P, W, B, st);
}

}  // namespace snk
