// evolve.cu — a5 + a6: batched Monte-Carlo evolution of independent 3D (2D)
// snakuscules (Eqs. 11-14), the ★ hot loop.
//
// Mapping (B200): a cell is owned by W warps (W = 1: warp-per-cell; W > 1:
// the paper's block-per-contour of §II-F) for all T+1 iterations; the
// cell state stays in registers.  Each iteration draws a FIXED number N of
// samples per cell (no divergence), 32 W threads x B = N/(32 W)
// samples each.  Per sample: Philox4x32-10 -> (omega, t) -> 8 u16 gathers ->
// trilinear -> S, S_r, S_R -> 5 leaf products.  Sums follow one canonical
// pairwise tree over the N sample positions (in-thread binary counter ->
// xor-butterfly over lanes -> pairwise over warps), so results are
// bit-identical for every W.  This file is compiled with
// -fmad=false: every FMA is written explicitly, so no schedule can contract
// differently.
//
// Reading of the update (G3/G4/G8): E = gamma A0,
// dE/dc = -gamma A_c, dE/dR = gamma (A_R - (d/R) A0), gamma = (2R)^-d;
// (c, R) -= clip((eps0/sqrt(n))/2 * grad, +-max_step); R clamp, leash, domain.
#include "common.cuh"

namespace snk {

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;   // Philox multipliers
constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;   // Weyl key bumps
constexpr float kMagic = 8388608.0f;                        // 2^23
constexpr uint32_t kMagicBits = 0x4B000000u;

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
  float vscale;                  // iscale * (4/3 pi | pi) / N
  int T;
  uint32_t rk0[10], rk1[10];     // Philox round keys (seed + r * Weyl)
};

struct Acc {
  float a0, cx, cy, cz, aR;
};

__device__ __forceinline__ Acc acc_add(const Acc& l, const Acc& r) {
  return Acc{__fadd_rn(l.a0, r.a0), __fadd_rn(l.cx, r.cx), __fadd_rn(l.cy, r.cy),
             __fadd_rn(l.cz, r.cz), __fadd_rn(l.aR, r.aR)};
}

// Per cell-iteration constants.
struct CellIt {
  float cx, cy, cz;
  float rho_s;        // R + dR/2: radius of the sampled ball
  float a;            // -(R - dR/2)/dR: offset of both ramp coordinates
  uint32_t p0, p1, p3;   // Philox round-1 words that depend only on (n, id)
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
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

// u16 value v as a float offset by 2^23 (exact).
__device__ __forceinline__ float mag(uint32_t v) { return __uint_as_float(kMagicBits | v); }

// clamp k to [0, n-1], i0 = min(floor(k), n-2) (magic-number floor: FADD.RM),
// returns the fraction k - i0 and the integer i0.
__device__ __forceinline__ float split_axis(float k, float n1, float m2, int* i0) {
  k = fminf(fmaxf(k, 0.0f), n1);
  const float r = fminf(__fadd_rd(k, kMagic), m2);
  *i0 = (int)(__float_as_uint(r) - kMagicBits);
  return __fsub_rn(k, __fsub_rn(r, kMagic));
}

__device__ __forceinline__ float lerp_mag(float A, float Bm, float f) {
  // A, Bm are values + 2^23: a + f (b - a), with b - a = Bm - A exact and a = A - 2^23 exact
  return __fmaf_rn(f, __fsub_rn(Bm, A), __fsub_rn(A, kMagic));
}

__device__ __forceinline__ float lerp(float a, float b, float f) {
  return __fmaf_rn(f, __fsub_rn(b, a), a);
}

template <int D, bool SLAB>
__device__ __forceinline__ Acc sample_leaf(const EvoParams& P, const CellIt& C, uint32_t j,
                                           uint32_t& halo) {
  // ---- Philox4x32-10, ctr = {j, n, id_lo, id_hi}, key = seed (G11)
  uint32_t c0 = C.p0, c1 = C.p1, c2 = __umulhi(kM0, j) ^ C.p3, c3 = kM0 * j;
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kM0, c0), lo0 = kM0 * c0;
    const uint32_t hi1 = __umulhi(kM1, c2), lo1 = kM1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ P.rk0[r], n2 = hi0 ^ c3 ^ P.rk1[r];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  const float u0 = u01(c0), u1 = u01(c1), u2 = u01(c2);
  // ---- direction (Archimedes, G10) and distance
  float sn, cs;
  __sincosf(__fmul_rn(6.2831853071795865f, u1), &sn, &cs);
  float ox, oy, oz, t;
  if (D == 3) {
    oz = __fmaf_rn(-2.0f, u0, 1.0f);
    const float st = __fmul_rn(2.0f, sqrt_approx(__fmaf_rn(-u0, u0, u0)));
    ox = __fmul_rn(st, cs);
    oy = __fmul_rn(st, sn);
    t = __fmul_rn(C.rho_s, ex2_approx(__fmul_rn(lg2_approx(u2), 0.333333343f)));
  } else {
    ox = cs;
    oy = sn;
    oz = 0.0f;
    t = __fmul_rn(C.rho_s, sqrt_approx(u2));
  }
  // ---- position k = c + t omega, trilinear (bilinear) gather, clamp-to-edge (G17)
  int ix, iy, iz = 0;
  const float fx = split_axis(__fmaf_rn(t, ox, C.cx), P.fnx1, P.mx2, &ix);
  const float fy = split_axis(__fmaf_rn(t, oy, C.cy), P.fny1, P.my2, &iy);
  float fz = 0.0f;
  if (D == 3) {
    fz = split_axis(__fmaf_rn(t, oz, C.cz), P.fnz1, P.mz2, &iz);
    if (SLAB) {
      iz -= P.z_lo;
      if (iz < 0 || iz > P.nz_buf - 2) { halo = 1u; iz = min(max(iz, 0), P.nz_buf - 2); }
    }
  }
  const uint32_t nx = (uint32_t)P.nx;
  const uint32_t base = ((uint32_t)iz * (uint32_t)P.ny + (uint32_t)iy) * nx + (uint32_t)ix;
  const uint16_t* p = P.img + base;
  const float v00 = lerp_mag(mag(__ldg(p)), mag(__ldg(p + 1)), fx);
  const float v10 = lerp_mag(mag(__ldg(p + nx)), mag(__ldg(p + nx + 1)), fx);
  float tri = lerp(v00, v10, fy);
  if (D == 3) {
    const uint32_t pl = nx * (uint32_t)P.ny;
    const float v01 = lerp_mag(mag(__ldg(p + pl)), mag(__ldg(p + pl + 1)), fx);
    const float v11 = lerp_mag(mag(__ldg(p + pl + nx)), mag(__ldg(p + pl + nx + 1)), fx);
    tri = lerp(tri, lerp(v01, v11, fy), fz);
  }
  // ---- weight S(t; R) and partials (G1): tau_o = (t - (R - dR/2))/dR,
  //      tau_i = (t - rho (R - dR/2))/(rho dR) = t/(rho dR) + a
  const float uo = __saturatef(__fmaf_rn(t, P.inv_dR, C.a));
  const float ui = __saturatef(__fmaf_rn(t, P.inv_rho_dR, C.a));
  const float s3o = __fmul_rn(__fmul_rn(uo, uo), __fmaf_rn(-2.0f, uo, 3.0f));
  const float s3i = __fmul_rn(__fmul_rn(ui, ui), __fmaf_rn(-2.0f, ui, 3.0f));
  const float d3o = __fmul_rn(6.0f, __fmaf_rn(-uo, uo, uo));
  const float d3i = __fmul_rn(6.0f, __fmaf_rn(-ui, ui, ui));
  const float S = __fsub_rn(__fmaf_rn(2.0f, s3i, -s3o), 1.0f);             // (1-s3o) - 2(1-s3i)
  const float Sr = __fmaf_rn(__fmul_rn(2.0f, P.inv_rho_dR), d3i, __fmul_rn(-P.inv_dR, d3o));
  const float SR = __fmul_rn(__fmaf_rn(-2.0f, d3i, d3o), P.inv_dR);
  // ---- leaves (iscale and V/N are applied once per iteration)
  const float w = __fmul_rn(Sr, tri);
  Acc a;
  a.a0 = __fmul_rn(S, tri);
  a.cx = __fmul_rn(w, ox);
  a.cy = __fmul_rn(w, oy);
  a.cz = D == 3 ? __fmul_rn(w, oz) : 0.0f;
  a.aR = __fmul_rn(SR, tri);
  return a;
}

// Pairwise sum over CH consecutive samples (CH a power of two).
template <int D, bool SLAB, int CH>
__device__ __forceinline__ Acc chunk_sum(const EvoParams& P, const CellIt& C, uint32_t j0,
                                         uint32_t& halo) {
  if constexpr (CH == 1) {
    return sample_leaf<D, SLAB>(P, C, j0, halo);
  } else {
    const Acc l = chunk_sum<D, SLAB, CH / 2>(P, C, j0, halo);
    const Acc r = chunk_sum<D, SLAB, CH / 2>(P, C, j0 + CH / 2, halo);
    return acc_add(l, r);
  }
}

// Pairwise sum over CH << L consecutive samples: 2^L chunks combined by a
// binary counter (stack of L partial sums) = a perfect pairwise tree.
template <int D, bool SLAB, int CH, int L>
__device__ __forceinline__ Acc lane_sum(const EvoParams& P, const CellIt& C, uint32_t j0,
                                        uint32_t& halo) {
  if constexpr (L == 0) {
    return chunk_sum<D, SLAB, CH>(P, C, j0, halo);
  } else {
    Acc stk[L];
    Acc res{};
#pragma unroll 1
    for (int i = 0; i < (1 << L); ++i) {
      Acc x = chunk_sum<D, SLAB, CH>(P, C, j0 + (uint32_t)(i * CH), halo);
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

__device__ __forceinline__ float clampf(float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); }

template <int D, int W, bool SLAB, int CH, int L>
__global__ void __launch_bounds__(W >= 4 ? 32 * W : 128)
    evolve_kernel(const __grid_constant__ EvoParams P) {
  constexpr int CPB = W >= 4 ? 1 : 4 / W;   // cells per block
  constexpr int B = CH << L;                // samples per thread per iteration
  __shared__ Acc xch[2][CPB][W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = warp / W, wsub = warp % W;
  const int64_t cell = (int64_t)blockIdx.x * CPB + slot;
  if (cell >= P.n) return;   // uniform per cell group (named barriers below)
  const float sx = P.seeds[3 * cell + 0], sy = P.seeds[3 * cell + 1];
  const float sz = D == 3 ? P.seeds[3 * cell + 2] : 0.0f;
  const int64_t id = P.ids ? P.ids[cell] : P.id_base + cell;
  const uint32_t id_lo = (uint32_t)((uint64_t)id & 0xffffffffu), id_hi = (uint32_t)((uint64_t)id >> 32);
  float cx = sx, cy = sy, cz = sz, R = P.r0, E = 0.0f;
  uint32_t flags = 0, halo = 0;
  const uint32_t j0 = (uint32_t)((wsub * 32 + lane) * B);
  const float inv_d = D == 3 ? 3.0f : 2.0f;
  for (int it = 1; it <= P.T + 1; ++it) {
    CellIt C;
    C.cx = cx; C.cy = cy; C.cz = cz;
    C.rho_s = __fadd_rn(R, P.half_dR);
    C.a = __fmul_rn(-__fsub_rn(R, P.half_dR), P.inv_dR);
    // Philox round 1: words from c1 = n, c2 = id_lo, c3 = id_hi
    C.p0 = __umulhi(kM1, id_lo) ^ (uint32_t)it ^ P.rk0[0];
    C.p1 = kM1 * id_lo;
    C.p3 = id_hi ^ P.rk1[0];
    Acc s = lane_sum<D, SLAB, CH, L>(P, C, j0, halo);
    // butterfly over lanes: (l, l^1), (l, l^2), ... = pairwise over lane blocks
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
    if constexpr (W > 1) {
      if (lane == 0) xch[it & 1][slot][wsub] = s;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * W) : "memory");
      Acc v[W];
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] = xch[it & 1][slot][w];
#pragma unroll
      for (int span = 1; span < W; span <<= 1)
#pragma unroll
        for (int w = 0; w + span < W; w += 2 * span) v[w] = acc_add(v[w], v[w + span]);
      s = v[0];
    }
    // ---- energy and gradient (Eqs. 5-10 in (c, R) form; gamma = (2R)^-d, G3)
    const float rs = C.rho_s;
    const float vol = D == 3 ? __fmul_rn(__fmul_rn(rs, rs), rs) : __fmul_rn(rs, rs);
    const float scale = __fmul_rn(P.vscale, vol);
    const float A0 = __fmul_rn(s.a0, scale);
    const float twoR = __fmul_rn(2.0f, R);
    const float gden = D == 3 ? __fmul_rn(__fmul_rn(twoR, twoR), twoR) : __fmul_rn(twoR, twoR);
    const float gamma = __fdiv_rn(1.0f, gden);
    const float gs = __fmul_rn(gamma, scale);
    E = __fmul_rn(gamma, A0);
    if (it == P.T + 1) break;
    const float gcx = -__fmul_rn(gs, s.cx), gcy = -__fmul_rn(gs, s.cy), gcz = -__fmul_rn(gs, s.cz);
    const float gR = __fmul_rn(gamma, __fsub_rn(__fmul_rn(s.aR, scale), __fmul_rn(__fdiv_rn(inv_d, R), A0)));
    // ---- step eps_n / 2 with eps_n = eps0 / sqrt(n), clipped (G8)
    const float h = __fmul_rn(0.5f, __fdiv_rn(P.eps0, __fsqrt_rn((float)it)));
    const float dcx = clampf(-__fmul_rn(h, gcx), -P.max_step, P.max_step);
    const float dcy = clampf(-__fmul_rn(h, gcy), -P.max_step, P.max_step);
    const float dcz = D == 3 ? clampf(-__fmul_rn(h, gcz), -P.max_step, P.max_step) : 0.0f;
    const float dR = clampf(-__fmul_rn(h, gR), -P.max_step, P.max_step);
    const float ox = cx, oy = cy, oz = cz, oR = R;
    cx = __fadd_rn(cx, dcx);
    cy = __fadd_rn(cy, dcy);
    cz = __fadd_rn(cz, dcz);
    R = clampf(__fadd_rn(R, dR), P.r_min, P.r_max);
    // leash
    const float lx = clampf(cx, __fsub_rn(sx, P.leash), __fadd_rn(sx, P.leash));
    const float ly = clampf(cy, __fsub_rn(sy, P.leash), __fadd_rn(sy, P.leash));
    const float lz = clampf(cz, __fsub_rn(sz, P.leash), __fadd_rn(sz, P.leash));
    const bool leashed = (lx != cx) || (ly != cy) || (lz != cz);
    cx = lx; cy = ly; cz = lz;
    // domain: c_a in [m, n_a - 1 - m], m = R + dR/2, or the axis centre
    const float m = __fadd_rn(R, P.half_dR), m2 = __fmul_rn(2.0f, m);
    const float dx = P.fnx1 < m2 ? __fmul_rn(0.5f, P.fnx1) : clampf(cx, m, __fsub_rn(P.fnx1, m));
    const float dy = P.fny1 < m2 ? __fmul_rn(0.5f, P.fny1) : clampf(cy, m, __fsub_rn(P.fny1, m));
    float dz = cz;
    if (D == 3) dz = P.fnz1 < m2 ? __fmul_rn(0.5f, P.fnz1) : clampf(cz, m, __fsub_rn(P.fnz1, m));
    const bool domained = (dx != cx) || (dy != cy) || (dz != cz);
    cx = dx; cy = dy; cz = dz;
    if (it == P.T) {
      float mv = fabsf(__fsub_rn(R, oR));
      mv = fmaxf(mv, fabsf(__fsub_rn(cx, ox)));
      mv = fmaxf(mv, fabsf(__fsub_rn(cy, oy)));
      mv = fmaxf(mv, fabsf(__fsub_rn(cz, oz)));
      if (mv < P.conv_tol) flags |= SNK_F_CONVERGED;
      if (leashed) flags |= SNK_F_LEASHED;
      if (domained) flags |= SNK_F_DOMAIN;
    }
  }
  if (R <= P.r_min) flags |= SNK_F_COLLAPSED;
  if (R >= P.r_max) flags |= SNK_F_RMAX;
  if (SLAB) {
    if (__any_sync(0xffffffffu, halo != 0)) flags |= SNK_F_HALO;
    if constexpr (W > 1) {
      // combine the halo flag of every warp of the cell
      __shared__ uint32_t hf[CPB];
      if (wsub == 0 && lane == 0) hf[slot] = 0;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * W) : "memory");
      if (lane == 0 && (flags & SNK_F_HALO)) atomicOr(&hf[slot], SNK_F_HALO);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * W) : "memory");
      flags |= hf[slot];
    }
  }
  if (wsub == 0 && lane == 0) {
    snk_cell o;
    o.c[0] = cx; o.c[1] = cy; o.c[2] = cz;
    o.R = R;
    o.seed[0] = sx; o.seed[1] = sy; o.seed[2] = sz;
    o.energy = E;
    o.flags = flags;
    o.iters = P.T;
    o.id = id;
    P.out[cell] = o;
  }
}

template <int D, int W, bool SLAB, int CH, int L>
int32_t launch_one(const EvoParams& P, cudaStream_t st) {
  constexpr int CPB = W >= 4 ? 1 : 4 / W;
  const unsigned grid = (unsigned)ceil_div(P.n, CPB);
  const unsigned block = 32 * W * CPB;
  evolve_kernel<D, W, SLAB, CH, L><<<grid, block, 0, st>>>(P);
  SNK_LAUNCH_CHECK("evolve_kernel");
  return SNK_OK;
}

// B samples per thread: B = 1, 2 (one chunk) or 4 << L (chunks of 4, L <= 5).
template <int D, int W, bool SLAB>
int32_t launch_B(const EvoParams& P, int B, cudaStream_t st) {
  switch (B) {
    case 1: return launch_one<D, W, SLAB, 1, 0>(P, st);
    case 2: return launch_one<D, W, SLAB, 2, 0>(P, st);
    case 4: return launch_one<D, W, SLAB, 4, 0>(P, st);
    case 8: return launch_one<D, W, SLAB, 4, 1>(P, st);
    case 16: return launch_one<D, W, SLAB, 4, 2>(P, st);
    case 32: return launch_one<D, W, SLAB, 4, 3>(P, st);
    case 64: return launch_one<D, W, SLAB, 4, 4>(P, st);
    case 128: return launch_one<D, W, SLAB, 4, 5>(P, st);
    default: return fail(SNK_CONFIG, "samples per thread must be a power of two <= 128");
  }
}

template <int D, bool SLAB>
int32_t launch_W(const EvoParams& P, int W, int B, cudaStream_t st) {
  switch (W) {
    case 1: return launch_B<D, 1, SLAB>(P, B, st);
    case 2: return launch_B<D, 2, SLAB>(P, B, st);
    case 4: return launch_B<D, 4, SLAB>(P, B, st);
    case 8: return launch_B<D, 8, SLAB>(P, B, st);
    default: return fail(SNK_CONFIG, "bad warps per cell");
  }
}

}  // namespace

int evolve_warps_per_cell(const snk_params* p, int64_t n_cells) {
  int W = p->cta_warps;
  if (W <= 0) {
    // enough warps to fill every SM with >= 16 warps -> warp-per-cell; else
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
                    snk_cell* d_cells, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  (void)d_ws; (void)ws_bytes;
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
  P.eps0 = (float)p->eps0;
  P.max_step = (float)p->max_step;
  P.r_min = (float)p->r_min;
  P.r_max = (float)p->r_max;
  P.leash = (float)p->leash;
  P.conv_tol = (float)p->conv_tol;
  const double pi = 3.14159265358979323846;
  P.vscale = (float)(p->intensity_scale * (D == 3 ? 4.0 / 3.0 * pi : pi) / (double)p->n_samples);
  P.T = p->max_iters;
  uint32_t k0 = (uint32_t)(p->seed & 0xffffffffu), k1 = (uint32_t)(p->seed >> 32);
  for (int r = 0; r < 10; ++r) {
    P.rk0[r] = k0;
    P.rk1[r] = k1;
    k0 += kW0;
    k1 += kW1;
  }
  if (D == 3 && g->n[2] < 2) return fail(SNK_SHAPE, "3D needs nz >= 2");
  if (g->n[0] * g->n[1] * g->nz_buf >= ((int64_t)1 << 32)) return fail(SNK_SHAPE, "buffer too large");
  const int W = evolve_warps_per_cell(p, n);
  const int B = p->n_samples / (32 * W);
  if (B < 1) return fail(SNK_CONFIG, "n_samples < 32 * warps per cell");
  const bool slab = !(g->z_lo == 0 && g->nz_buf == g->n[2]);
  if (D == 3) return slab ? launch_W<3, true>(P, W, B, st) : launch_W<3, false>(P, W, B, st);
  return launch_W<2, false>(P, W, B, st);
}

}  // namespace snk
