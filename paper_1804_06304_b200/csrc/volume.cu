// volume.cu — a1 isotropic resampling, a2 separable Q14 Gaussian blur, a3
// gradient magnitude (include/snk.h).  Integer-exact: results are bit-identical
// to the definitions in DESIGN.md §3 (G16, G18, O3).
//
// Layout: u16 x-fastest volumes of nz planes; every kernel is a flat grid over
// output voxels, threadIdx.x along x, so loads and stores are coalesced; the
// stencil neighbours of the y/z passes are the rows/planes above and below and
// are served from L1/L2 (each voxel is read from DRAM about once per pass).
#include <cmath>
#include <vector>

#include "common.cuh"

// 1: the fused TMA-staged blur (stencil.cu) where it applies; 0: the three
// streaming separable passes below (kept for comparison and the fallbacks)
#ifndef SNK_BLUR_TMA
#define SNK_BLUR_TMA 1
#endif

namespace snk {

namespace {

constexpr int kMaxTaps = 65;   // 2 * ceil(4 * 8) + 1
// Q14 taps, passed to the kernels by value (no shared __constant__ state, so
// concurrent calls on different streams with different sigma cannot race)
struct Taps {
  int32_t w[kMaxTaps];
};

// Q14 Gaussian taps (reading G18): h = ceil(4 sigma),
// w_i = round(16384 exp(-i^2 / 2 sigma^2) / sum), centre absorbs the remainder.
int q14_taps(double sigma, std::vector<int32_t>& taps) {
  if (!(sigma > 0.0)) {
    taps.assign(1, 16384);
    return 0;
  }
  const int h = (int)std::ceil(4.0 * sigma);
  std::vector<double> g(2 * h + 1);
  double sum = 0.0;
  for (int i = -h; i <= h; ++i) {
    g[i + h] = std::exp(-(double)(i * i) / (2.0 * sigma * sigma));
    sum += g[i + h];
  }
  taps.assign(2 * h + 1, 0);
  int64_t tot = 0;
  for (int i = 0; i <= 2 * h; ++i) {
    taps[i] = (int32_t)std::floor(16384.0 * g[i] / sum + 0.5);
    tot += taps[i];
  }
  taps[h] += (int32_t)(16384 - tot);
  return h;
}

// One separable pass along AXIS (0 = x, 1 = y, 2 = z): out = (sum w_i in[clamp(p+i)] + 8192) >> 14.
// Two output voxels per thread (x and x+1 share the row) -> 32-bit stores.
template <int AXIS>
__global__ void __launch_bounds__(256) blur_pass_kernel(const uint16_t* __restrict__ in,
                                                        uint16_t* __restrict__ out, int nx, int ny,
                                                        int nz, int h, const __grid_constant__ Taps T) {
  const int64_t pairs_per_row = (nx + 1) >> 1;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = pairs_per_row * ny * nz;
  if (t >= total) return;
  const int x0 = (int)(t % pairs_per_row) * 2;
  const int64_t row = t / pairs_per_row;   // = z * ny + y
  const int y = (int)(row % ny);
  const int z = (int)(row / ny);
  const int64_t plane = (int64_t)nx * ny;
  uint32_t acc0 = 8192, acc1 = 8192;
  const bool two = x0 + 1 < nx;
  if (AXIS == 0) {
    const uint16_t* r = in + row * nx;
    for (int i = -h; i <= h; ++i) {
      const uint32_t w = (uint32_t)T.w[i + h];
      const int xa = min(max(x0 + i, 0), nx - 1);
      const int xb = min(max(x0 + 1 + i, 0), nx - 1);
      acc0 += w * __ldg(r + xa);
      acc1 += w * __ldg(r + xb);
    }
  } else {
    const int p = AXIS == 1 ? y : z;
    const int np = AXIS == 1 ? ny : nz;
    const int64_t stride = AXIS == 1 ? nx : plane;
    const uint16_t* base = in + row * nx - (int64_t)p * stride + x0;
    for (int i = -h; i <= h; ++i) {
      const uint32_t w = (uint32_t)T.w[i + h];
      const int q = min(max(p + i, 0), np - 1);
      const uint16_t* src = base + (int64_t)q * stride;
      acc0 += w * __ldg(src);
      if (two) acc1 += w * __ldg(src + 1);
    }
  }
  uint16_t* o = out + row * nx + x0;
  o[0] = (uint16_t)(acc0 >> 14);
  if (two) o[1] = (uint16_t)(acc1 >> 14);
}

__device__ __forceinline__ float sqrt_approx_f(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// a3: G = (isqrt(gx^2 + gy^2 + gz^2) + 1) >> 1, central differences, clamp-to-edge.
__device__ __forceinline__ uint32_t isqrt_u64(uint64_t v) {
  uint64_t r = (uint64_t)sqrt((double)v);   // exact integer part after correction
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return (uint32_t)r;
}

template <int D>
__global__ void __launch_bounds__(256) gradmag_kernel(const uint16_t* __restrict__ B,
                                                      uint16_t* __restrict__ G, int nx, int ny,
                                                      int nz) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t plane = (int64_t)nx * ny;
  if (t >= plane * nz) return;
  const int x = (int)(t % nx);
  const int y = (int)((t / nx) % ny);
  const int z = (int)(t / plane);
  const int64_t row = t - x;
  const int gx = (int)__ldg(B + row + min(x + 1, nx - 1)) - (int)__ldg(B + row + max(x - 1, 0));
  const int gy = (int)__ldg(B + t + (int64_t)(min(y + 1, ny - 1) - y) * nx) -
                 (int)__ldg(B + t + (int64_t)(max(y - 1, 0) - y) * nx);
  uint64_t s = (uint64_t)((int64_t)gx * gx) + (uint64_t)((int64_t)gy * gy);
  if (D == 3) {
    const int gz = (int)__ldg(B + t + (int64_t)(min(z + 1, nz - 1) - z) * plane) -
                   (int)__ldg(B + t + (int64_t)(max(z - 1, 0) - z) * plane);
    s += (uint64_t)((int64_t)gz * gz);
  }
  G[t] = (uint16_t)((isqrt_u64(s) + 1) >> 1);
}

// a1: one resampling pass along AXIS.  Input dims (ni[0], ni[1], ni[2]) holding
// planes from in_z0 (AXIS 2 only: global raw plane of the buffer's first
// plane); output dims with no[AXIS] = output samples, out_z0 likewise.
// src = (k + 0.5) * ratio - 0.5 in IEEE double, no contraction (G16).
template <int AXIS>
__global__ void __launch_bounds__(256) resample_kernel(const uint16_t* __restrict__ in,
                                                       uint16_t* __restrict__ out, int64_t nix,
                                                       int64_t niy, int64_t noz, int64_t nox,
                                                       int64_t noy, int64_t n_axis, double ratio,
                                                       int64_t in_z0, int64_t out_z0) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nox * noy * noz) return;
  const int64_t x = t % nox, y = (t / nox) % noy, z = t / (nox * noy);
  const int64_t kg = (AXIS == 0 ? x : AXIS == 1 ? y : z + out_z0);   // global output index
  double src = __dadd_rn(__dmul_rn(__dadd_rn((double)kg, 0.5), ratio), -0.5);
  src = fmin(fmax(src, 0.0), (double)(n_axis - 1));
  int64_t i0 = 0, w1 = 0;
  if (n_axis > 1) {
    i0 = min((int64_t)floor(src), n_axis - 2);
    w1 = (int64_t)floor(__dadd_rn(__dmul_rn(16384.0, __dadd_rn(src, -(double)i0)), 0.5));
  }
  int64_t sx = x, sy = y, sz = z, step;
  if (AXIS == 0) { sx = i0; step = 1; }
  else if (AXIS == 1) { sy = i0; step = nix; }
  else { sz = i0 - in_z0; step = nix * niy; }
  const int64_t si = (sz * niy + sy) * nix + sx;
  const uint32_t v0 = __ldg(in + si);
  const uint32_t v1 = n_axis > 1 ? __ldg(in + si + step) : v0;
  out[t] = (uint16_t)((v0 * (uint32_t)(16384 - w1) + v1 * (uint32_t)w1 + 8192u) >> 14);
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)ceil_div(n, block); }

// ---------------------------------------------------------------------------
// Vectorised separable pass: each thread produces 8 consecutive x outputs
// (one 16-byte store) from 16-byte loads; no shared memory, no barriers, so
// the pass streams at HBM rate (stencil neighbours come from L1/L2).
//   OP_BLUR: (sum_i w_i v[clamp(p+i)] + 8192) >> 14 (clamp-to-edge, G18)
//   OP_MAX:  max over the window clipped to [lo, hi] (the MAXIMA box, G20)
// Requires nx % 8 == 0 and 16-byte aligned buffers.
enum { OP_BLUR = 0, OP_MAX = 1 };

__device__ __forceinline__ void unpack8(const uint4 q, uint32_t* v) {
  v[0] = q.x & 0xffffu; v[1] = q.x >> 16; v[2] = q.y & 0xffffu; v[3] = q.y >> 16;
  v[4] = q.z & 0xffffu; v[5] = q.z >> 16; v[6] = q.w & 0xffffu; v[7] = q.w >> 16;
}
__device__ __forceinline__ uint4 pack8(const uint32_t* o) {
  return make_uint4(o[0] | (o[1] << 16), o[2] | (o[3] << 16), o[4] | (o[5] << 16), o[6] | (o[7] << 16));
}

template <int AXIS, int OP, int H>
__global__ void __launch_bounds__(256) sep8_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                                   int nx, int ny, int nz, int lo, int hi,
                                                   const __grid_constant__ Taps T) {
  const int nc = nx >> 3;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * ny * nz) return;
  const int xc = (int)(t % nc);
  const int64_t row = t / nc;                     // z * ny + y
  const int y = (int)(row % ny), z = (int)(row / ny);
  const uint4* rin = reinterpret_cast<const uint4*>(in);
  uint32_t o[8];
  if (AXIS == 0) {
    uint32_t v[24];
    const int64_t rb = row * nc;
    unpack8(__ldg(rin + rb + xc), v + 8);
    if (xc > 0) unpack8(__ldg(rin + rb + xc - 1), v);
    else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = OP == OP_BLUR ? v[8] : 0u;
    }
    if (xc < nc - 1) unpack8(__ldg(rin + rb + xc + 1), v + 16);
    else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[16 + k] = OP == OP_BLUR ? v[15] : 0u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t acc = OP == OP_BLUR ? 8192u : 0u;
#pragma unroll
      for (int i = -H; i <= H; ++i) {
        if (OP == OP_BLUR) acc += (uint32_t)T.w[i + H] * v[8 + k + i];
        else acc = max(acc, v[8 + k + i]);
      }
      o[k] = OP == OP_BLUR ? acc >> 14 : acc;
    }
  } else {
    const int p = AXIS == 1 ? y : z;
    const int np = AXIS == 1 ? ny : nz;
    const int64_t stride = AXIS == 1 ? nc : (int64_t)nc * ny;   // in uint4 units
    const uint4* base = rin + row * nc + xc - (int64_t)p * stride;
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = OP == OP_BLUR ? 8192u : 0u;
#pragma unroll
    for (int i = -H; i <= H; ++i) {
      int q = p + i;
      if (OP == OP_BLUR) q = min(max(q, 0), np - 1);
      else if (q < lo || q > hi) continue;
      uint32_t v[8];
      unpack8(__ldg(base + (int64_t)q * stride), v);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (OP == OP_BLUR) o[k] += (uint32_t)T.w[i + H] * v[k];
        else o[k] = max(o[k], v[k]);
      }
    }
    if (OP == OP_BLUR) {
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] >>= 14;
    }
  }
  reinterpret_cast<uint4*>(out)[t] = pack8(o);
}

// z pass as column streaming: a thread owns one 8-voxel x group of one row
// (xc, y) and walks kZC consecutive output planes with a window of 2H+1 input
// planes held in registers (a ring with static indices: the plane loop is
// unrolled by 2H+1), so every input plane is read (kZC + 2H)/kZC times instead
// of 2H+1 times — the flat z pass re-read its window through L2, which C4's
// 8 MB planes overflow.  Consecutive threads take consecutive x groups of a
// row (16-byte coalesced loads).  Same arithmetic as sep8_kernel<2, OP>:
// blur windows are unpacked once per plane, max windows stay packed (u16x2
// VIMNMX).
constexpr int kZC = 32;
#ifndef ZCOL_AXES
#define ZCOL_AXES 6   // bit 1: y passes, bit 2: z passes
#endif

__device__ __forceinline__ uint4 vmax4(uint4 a, uint4 b) {
  return make_uint4(__vmaxu2(a.x, b.x), __vmaxu2(a.y, b.y), __vmaxu2(a.z, b.z), __vmaxu2(a.w, b.w));
}

// AXIS 2: columns (xc, y) walk z; AXIS 1: columns (xc, z) walk y (the flat y
// pass re-reads 2h+1 rows per output through L1/L2 as well).
template <int AXIS, int OP, int H>
__global__ void __launch_bounds__(256) zcol8_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                                    int nx, int ny, int nzv, int lo, int hi,
                                                    const __grid_constant__ Taps T) {
  constexpr int K = 2 * H + 1;
  const int nc = nx >> 3;
  // "planes" are the walked axis; columns enumerate the other two
  const int nz = AXIS == 2 ? nzv : ny;
  const int64_t ncols = AXIS == 2 ? (int64_t)nc * ny : (int64_t)nc * nzv;
  const int64_t ps = AXIS == 2 ? (int64_t)nc * ny : (int64_t)nc;   // stride of the walked axis (uint4)
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nzc = (nz + kZC - 1) / kZC;
  if (t >= ncols * nzc) return;
  const int64_t col = t % ncols;
  const int z0 = (int)(t / ncols) * kZC, z1 = min(z0 + kZC, nz);
  // column base: AXIS 2: col = y nc + xc; AXIS 1: col = z nc + xc -> (z ny) nc + xc
  const int64_t cb = AXIS == 2 ? col : (col / nc) * (int64_t)ny * nc + col % nc;
  const uint4* rin = reinterpret_cast<const uint4*>(in) + cb;
  uint4* rout = reinterpret_cast<uint4*>(out) + cb;
  auto load = [&](int q) -> uint4 {
    if (OP == OP_BLUR) return __ldg(rin + (int64_t)min(max(q, 0), nz - 1) * ps);
    if (q < lo || q > hi) return make_uint4(0u, 0u, 0u, 0u);   // outside the clipped window
    return __ldg(rin + (int64_t)q * ps);
  };
  // win[j] = plane zb - H + j (j < K - 1); the K planes zb + H .. zb + H + K - 1
  // of a block are loaded together (K loads in flight per thread)
  uint4 win[K - 1];
#pragma unroll
  for (int j = 0; j < K - 1; ++j) win[j] = load(z0 - H + j);
  for (int zb = z0; zb < z1; zb += K) {
    uint4 nxt[K];
#pragma unroll
    for (int s = 0; s < K; ++s) nxt[s] = load(zb + H + s);
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const int z = zb + s;
      if (z < z1) {
        if (OP == OP_BLUR) {
          uint32_t o[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) o[k] = 8192u;
#pragma unroll
          for (int i = 0; i < K; ++i) {     // plane z - H + i
            const int j = s + i;
            uint32_t v[8];
            unpack8(j < K - 1 ? win[j] : nxt[j - (K - 1)], v);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] += (uint32_t)T.w[i] * v[k];
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) o[k] >>= 14;
          rout[(int64_t)z * ps] = pack8(o);
        } else {
          uint4 m = win[s < K - 1 ? s : 0];
          if (s >= K - 1) m = nxt[s - (K - 1)];
#pragma unroll
          for (int i = 1; i < K; ++i) {
            const int j = s + i;
            m = vmax4(m, j < K - 1 ? win[j] : nxt[j - (K - 1)]);
          }
          rout[(int64_t)z * ps] = m;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < K - 1; ++j) win[j] = nxt[j + 1];
  }
}

template <int AXIS, int OP>
int32_t sep8_launch(int h, const uint16_t* in, uint16_t* out, int nx, int ny, int nz, int lo, int hi,
                    const Taps& tp, cudaStream_t st) {
  if (AXIS >= 1 && h > 0 && (AXIS == 2 ? nz : ny) > kZC && ZCOL_AXES & (1 << AXIS)) {
    // y / z: column streaming (the flat passes re-read 2h+1 rows / planes through L1/L2)
    const int64_t cols = AXIS == 2 ? (int64_t)(nx / 8) * ny : (int64_t)(nx / 8) * nz;
    const unsigned zg = (unsigned)ceil_div(cols * ceil_div(AXIS == 2 ? nz : ny, kZC), 256);
    switch (h) {
#define SNK_ZC_CASE(HH) \
      case HH: zcol8_kernel<AXIS, OP, HH><<<zg, 256, 0, st>>>(in, out, nx, ny, nz, lo, hi, tp); break;
      SNK_ZC_CASE(1) SNK_ZC_CASE(2) SNK_ZC_CASE(3) SNK_ZC_CASE(4)
      SNK_ZC_CASE(5) SNK_ZC_CASE(6) SNK_ZC_CASE(7) SNK_ZC_CASE(8)
#undef SNK_ZC_CASE
      default: return fail(SNK_INTERNAL, "zcol8: radius > 8");
    }
    SNK_LAUNCH_CHECK("zcol8_kernel");
    return SNK_OK;
  }
  const unsigned grid = (unsigned)ceil_div((int64_t)(nx / 8) * ny * nz, 256);
  switch (h) {
#define SNK_SEP_CASE(HH) \
    case HH: sep8_kernel<AXIS, OP, HH><<<grid, 256, 0, st>>>(in, out, nx, ny, nz, lo, hi, tp); break;
    SNK_SEP_CASE(0) SNK_SEP_CASE(1) SNK_SEP_CASE(2) SNK_SEP_CASE(3) SNK_SEP_CASE(4)
    SNK_SEP_CASE(5) SNK_SEP_CASE(6) SNK_SEP_CASE(7) SNK_SEP_CASE(8)
#undef SNK_SEP_CASE
    default: return fail(SNK_INTERNAL, "sep8: radius > 8");
  }
  SNK_LAUNCH_CHECK("sep8_kernel");
  return SNK_OK;
}

// ---------------------------------------------------------------------------
// Fused 3D blur: one CTA per 64 x 16 output columns and a 32-plane z-chunk.
// Per input plane: the (16+2H) x (64+2H) tile (clamped coordinates) is
// staged in shared memory, the x pass and the y pass run there (each rounding
// to an integer, exactly as the three separate passes), and the y-passed
// values enter a per-thread register ring of 2H+1 planes, from which the z
// pass produces output plane z - H.  Each voxel is read from HBM ~once and
// written once (the three-pass version moved it 3x each way).
constexpr int kBX = 64, kBY = 16, kBZC = 32, kBThreads = 256;

template <int H>
__global__ void __launch_bounds__(kBThreads) blur3d_fused_kernel(const uint16_t* __restrict__ in,
                                                                 uint16_t* __restrict__ out, int nx,
                                                                 int ny, int nz,
                                                                 const __grid_constant__ Taps T) {
  constexpr int K = 2 * H + 1, RX = kBX + 2 * H, RY = kBY + 2 * H;
  __shared__ uint16_t s_in[RY][RX];
  __shared__ uint16_t s_x[RY][kBX];
  const int x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY, z0 = blockIdx.z * kBZC;
  const int tx = threadIdx.x % kBX, ty = threadIdx.x / kBX;   // 4 rows of outputs per thread
  const int zend = min(z0 + kBZC, nz);
  const int nplanes = (zend - z0) + 2 * H;
  uint32_t ring[K][4];
  // the next plane's tile is prefetched into registers while this plane computes
  constexpr int PER = (RY * RX + kBThreads - 1) / kBThreads;
  uint16_t pf[PER];
  auto fetch = [&](int pi) {
    const int zin = min(max(z0 - H + pi, 0), nz - 1);
    const uint16_t* src = in + (int64_t)zin * nx * ny;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = threadIdx.x + q * kBThreads;
      if (e < RY * RX) {
        const int r = e / RX, c = e % RX;
        const int gy = min(max(y0 - H + r, 0), ny - 1), gx = min(max(x0 - H + c, 0), nx - 1);
        pf[q] = __ldg(src + (int64_t)gy * nx + gx);
      }
    }
  };
  fetch(0);
  for (int base = 0; base < nplanes; base += K) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int pi = base + j;
      if (pi >= nplanes) break;
      __syncthreads();   // previous plane's x pass finished with s_in, y pass with s_x
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int e = threadIdx.x + q * kBThreads;
        if (e < RY * RX) (&s_in[0][0])[e] = pf[q];
      }
      if (pi + 1 < nplanes) fetch(pi + 1);
      __syncthreads();
      for (int e = threadIdx.x; e < RY * kBX; e += kBThreads) {
        const int r = e / kBX, c = e % kBX;
        uint32_t acc = 8192;
#pragma unroll
        for (int i = 0; i < K; ++i) acc += (uint32_t)T.w[i] * s_in[r][c + i];
        s_x[r][c] = (uint16_t)(acc >> 14);
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t acc = 8192;
#pragma unroll
        for (int i = 0; i < K; ++i) acc += (uint32_t)T.w[i] * s_x[ty * 4 + k + i][tx];
        ring[j][k] = acc >> 14;
      }
      if (pi >= 2 * H) {
        const int zo = z0 + pi - 2 * H;
        uint16_t* dst = out + ((int64_t)zo * ny + y0 + ty * 4) * nx + x0 + tx;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t acc = 8192;
#pragma unroll
          for (int i = 0; i < K; ++i) acc += (uint32_t)T.w[i] * ring[(j + 1 + i) % K][k];
          if (x0 + tx < nx && y0 + ty * 4 + k < ny) dst[(int64_t)k * nx] = (uint16_t)(acc >> 14);
        }
      }
    }
  }
}

// 2D: one plane, the same staging for the x and y passes.
template <int H>
__global__ void __launch_bounds__(kBThreads) blur2d_fused_kernel(const uint16_t* __restrict__ in,
                                                                 uint16_t* __restrict__ out, int nx,
                                                                 int ny, const __grid_constant__ Taps T) {
  constexpr int K = 2 * H + 1, RX = kBX + 2 * H, RY = kBY + 2 * H;
  __shared__ uint16_t s_in[RY][RX];
  __shared__ uint16_t s_x[RY][kBX];
  const int x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY;
  const int tx = threadIdx.x % kBX, ty = threadIdx.x / kBX;
  for (int e = threadIdx.x; e < RY * RX; e += kBThreads) {
    const int r = e / RX, c = e % RX;
    const int gy = min(max(y0 - H + r, 0), ny - 1), gx = min(max(x0 - H + c, 0), nx - 1);
    s_in[r][c] = __ldg(in + (int64_t)gy * nx + gx);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < RY * kBX; e += kBThreads) {
    const int r = e / kBX, c = e % kBX;
    uint32_t acc = 8192;
#pragma unroll
    for (int i = 0; i < K; ++i) acc += (uint32_t)T.w[i] * s_in[r][c + i];
    s_x[r][c] = (uint16_t)(acc >> 14);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t acc = 8192;
#pragma unroll
    for (int i = 0; i < K; ++i) acc += (uint32_t)T.w[i] * s_x[ty * 4 + k + i][tx];
    if (x0 + tx < nx && y0 + ty * 4 + k < ny)
      out[(int64_t)(y0 + ty * 4 + k) * nx + x0 + tx] = (uint16_t)(acc >> 14);
  }
}

// Gradient magnitude, tiled: the (16+2) x (64+2) smoothed neighbourhood of
// three consecutive planes is staged in shared memory (plane ring), each
// smoothed voxel is read ~once from L2/HBM.
template <int D>
__global__ void __launch_bounds__(kBThreads) gradmag_tiled_kernel(const uint16_t* __restrict__ B,
                                                                  uint16_t* __restrict__ G, int nx,
                                                                  int ny, int nz) {
  constexpr int RX = kBX + 2, RY = kBY + 2;
  __shared__ uint16_t s[3][RY][RX];
  const int x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY, z0 = blockIdx.z * kBZC;
  const int tx = threadIdx.x % kBX, ty = threadIdx.x / kBX;
  const int zend = D == 3 ? min(z0 + kBZC, nz) : 1;
  auto load = [&](int slot, int zp) {
    const int zc = min(max(zp, 0), nz - 1);
    const uint16_t* src = B + (int64_t)zc * nx * ny;
    for (int e = threadIdx.x; e < RY * RX; e += kBThreads) {
      const int r = e / RX, c = e % RX;
      const int gy = min(max(y0 - 1 + r, 0), ny - 1), gx = min(max(x0 - 1 + c, 0), nx - 1);
      s[slot][r][c] = __ldg(src + (int64_t)gy * nx + gx);
    }
  };
  if (D == 3) load(0, z0 - 1);
  load(1, z0);
  for (int z = z0; z < zend; ++z) {
    const int mid = (z - z0 + 1) % 3, prv = (z - z0) % 3, nxt = (z - z0 + 2) % 3;
    if (D == 3) load(nxt, z + 1);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = ty * 4 + k + 1, c = tx + 1;
      const int gx = (int)s[mid][r][c + 1] - (int)s[mid][r][c - 1];
      const int gy = (int)s[mid][r + 1][c] - (int)s[mid][r - 1][c];
      uint64_t ss = (uint64_t)((int64_t)gx * gx) + (uint64_t)((int64_t)gy * gy);
      if (D == 3) {
        const int gz = (int)s[nxt][r][c] - (int)s[prv][r][c];
        ss += (uint64_t)((int64_t)gz * gz);
      }
      if (x0 + tx < nx && y0 + r - 1 < ny)
        G[((int64_t)z * ny + y0 + r - 1) * nx + x0 + tx] = (uint16_t)((isqrt_u64(ss) + 1) >> 1);
    }
    __syncthreads();
  }
}

// a3, vectorised: 8 consecutive x outputs per thread from 16-byte loads (the
// row, the rows y -+ 1, the planes z -+ 1, and the two x neighbours of the
// group), no shared memory.  isqrt(v) from a float estimate corrected exactly
// in 64-bit integers (the estimate is within 1).
__device__ __forceinline__ uint32_t isqrt_est(uint64_t v, float vf) {
  const float e = sqrt_approx_f(vf);
  uint32_t r = __float_as_uint(__fadd_rz(e, 8388608.0f)) - 0x4B000000u;   // trunc(e), e < 2^23
  if ((uint64_t)r * r > v) --r;
  else if ((uint64_t)(r + 1) * (r + 1) <= v) ++r;
  return r;
}

template <int D>
__global__ void __launch_bounds__(256) gradmag8_kernel(const uint16_t* __restrict__ B, uint16_t* __restrict__ G,
                                                       int nx, int ny, int nz) {
  const int nc = nx >> 3;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nc * ny * nz) return;
  const int xc = (int)(t % nc);
  const int64_t row = t / nc;
  const int y = (int)(row % ny), z = (int)(row / ny);
  const uint4* Bq = reinterpret_cast<const uint4*>(B);
  const int64_t rs = nc, ps = (int64_t)nc * ny;   // row / plane strides in uint4
  uint32_t c[8], ym[8], yp[8], zm[8], zp[8];
  unpack8(__ldg(Bq + t), c);
  unpack8(__ldg(Bq + t - (y > 0 ? rs : 0)), ym);
  unpack8(__ldg(Bq + t + (y < ny - 1 ? rs : 0)), yp);
  if (D == 3) {
    unpack8(__ldg(Bq + t - (z > 0 ? ps : 0)), zm);
    unpack8(__ldg(Bq + t + (z < nz - 1 ? ps : 0)), zp);
  }
  const uint16_t* rowp = B + row * nx + xc * 8;
  const uint32_t l = xc > 0 ? __ldg(rowp - 1) : c[0];
  const uint32_t r = xc < nc - 1 ? __ldg(rowp + 8) : c[7];
  uint32_t o[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int gx = (int)(k < 7 ? c[k + 1] : r) - (int)(k > 0 ? c[k - 1] : l);
    const int gy = (int)yp[k] - (int)ym[k];
    const int gz = D == 3 ? (int)zp[k] - (int)zm[k] : 0;
    const uint64_t v = (uint64_t)((int64_t)gx * gx) + (uint64_t)((int64_t)gy * gy) + (uint64_t)((int64_t)gz * gz);
    const float fx = (float)gx, fy = (float)gy, fz = (float)gz;
    const float vf = __fmaf_rn(fx, fx, __fmaf_rn(fy, fy, __fmul_rn(fz, fz)));
    o[k] = (isqrt_est(v, vf) + 1) >> 1;
  }
  reinterpret_cast<uint4*>(G)[t] = pack8(o);
}

template <int H>
int32_t launch_fused_blur(const snk_grid* g, const uint16_t* d_in, uint16_t* d_out, const Taps& tp,
                          cudaStream_t st) {
  const int nx = (int)g->n[0], ny = (int)g->n[1], nz = (int)g->nz_buf;
  if (g->dim == 3) {
    dim3 grid((unsigned)ceil_div(nx, kBX), (unsigned)ceil_div(ny, kBY), (unsigned)ceil_div(nz, kBZC));
    blur3d_fused_kernel<H><<<grid, kBThreads, 0, st>>>(d_in, d_out, nx, ny, nz, tp);
  } else {
    dim3 grid((unsigned)ceil_div(nx, kBX), (unsigned)ceil_div(ny, kBY));
    blur2d_fused_kernel<H><<<grid, kBThreads, 0, st>>>(d_in, d_out, nx, ny, tp);
  }
  SNK_LAUNCH_CHECK("blur_fused_kernel");
  return SNK_OK;
}


// ---------------------------------------------------------------- a0 ingest
// u8 -> u16 by x257 (an 8-bit volume is promoted exactly; 255 ->
// 65535), 16 voxels per thread with 16-byte loads where aligned.
__global__ void ingest_u8_kernel(const uint8_t* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = t * 16;
  if (i0 >= n) return;
  if (i0 + 16 <= n) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + i0));
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // bytes b0 b1 -> (b0 * 257) | (b1 * 257) << 16: u16 v * 257 = v | v << 8
      const uint32_t lo = __byte_perm(w[k], 0, 0x4140), hi = __byte_perm(w[k], 0, 0x4342);
      o[2 * k] = lo | (lo << 8);
      o[2 * k + 1] = hi | (hi << 8);
    }
    uint4* dst = reinterpret_cast<uint4*>(out + i0);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  } else {
    for (int64_t i = i0; i < n; ++i) out[i] = (uint16_t)(in[i] * 257u);
  }
}

__global__ void ingest_u8_scalar_kernel(const uint8_t* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint16_t)(in[i] * 257u);
}

}  // namespace

size_t preprocess_ws(const snk_grid* g, const snk_params* p) {
  const size_t vol = (size_t)g->n[0] * g->n[1] * g->nz_buf * sizeof(uint16_t) + 256;
  if (grid_aniso(g)) return 2 * vol;   // per-axis passes: two ping-pong buffers
  if (!(p->sigma > 0)) return 0;
  return vol;   // separable ping-pong
}

bool vec8_ok(const snk_grid* g, const void* a, const void* b, const void* c) {
  auto al = [](const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return g->n[0] % 8 == 0 && al(a) && al(b) && al(c);
}

namespace {
int32_t sep_blur(int axis, int h, const Taps& tp, const uint16_t* in, uint16_t* out, int nx, int ny, int nz,
                 cudaStream_t st) {
  if (axis == 0) return sep8_launch<0, OP_BLUR>(h, in, out, nx, ny, nz, 0, 0, tp, st);
  if (axis == 1) return sep8_launch<1, OP_BLUR>(h, in, out, nx, ny, nz, 0, 0, tp, st);
  return sep8_launch<2, OP_BLUR>(h, in, out, nx, ny, nz, 0, 0, tp, st);
}
}  // namespace

int32_t sep_pass(int axis, int op, int h, const uint16_t* in, uint16_t* out, int nx, int ny, int nz,
                 int lo, int hi, cudaStream_t st) {
  if (op != OP_MAX) return fail(SNK_INTERNAL, "sep_pass: blur passes go through preprocess");
  const Taps none{};
  if (axis == 0) return sep8_launch<0, OP_MAX>(h, in, out, nx, ny, nz, lo, hi, none, st);
  if (axis == 1) return sep8_launch<1, OP_MAX>(h, in, out, nx, ny, nz, lo, hi, none, st);
  return sep8_launch<2, OP_MAX>(h, in, out, nx, ny, nz, lo, hi, none, st);
}

int32_t preprocess_impl(const snk_grid* g, const snk_params* p, const uint16_t* d_in,
                        uint16_t* d_smooth, uint16_t* d_gradmag, void* d_ws, size_t ws_bytes,
                        cudaStream_t st) {
  std::vector<int32_t> taps;
  const int h = q14_taps(p->sigma, taps);
  Taps tp{};
  for (size_t i = 0; i < taps.size() && i < (size_t)kMaxTaps; ++i) tp.w[i] = taps[i];
  const int nx = (int)g->n[0], ny = (int)g->n[1], nz = (int)g->nz_buf;
  const int64_t nvox = (int64_t)nx * ny * nz;
  Carve cv(d_ws, ws_bytes);
  uint16_t* tmp = (h > 0 || grid_aniso(g)) ? cv.take<uint16_t>(nvox) : nullptr;
  if (cv.overflow) return fail(SNK_CAPACITY, "workspace too small for preprocess");
  if (grid_aniso(g)) {
    // anisotropic grid sampled without resampling (G28): the physical sigma is
    // sigma / scale_a voxels on axis a — per-axis taps, the vectorised passes
    // (x extent % 8 == 0 is validated) or the generic pass for wide kernels
    uint16_t* t2 = cv.take<uint16_t>(nvox);
    if (cv.overflow || !vec8_ok(g, d_in, d_smooth, tmp)) return fail(SNK_CAPACITY, "workspace too small for preprocess");
    const uint16_t* src = d_in;
    uint16_t* bufs[2] = {tmp, t2};
    for (int a = 0; a < g->dim; ++a) {
      std::vector<int32_t> ta;
      const int ha = q14_taps(p->sigma / grid_scale(g, a), ta);
      Taps tpa{};
      for (size_t i = 0; i < ta.size() && i < (size_t)kMaxTaps; ++i) tpa.w[i] = ta[i];
      uint16_t* dst = a == g->dim - 1 ? d_smooth : bufs[a & 1];
      if (ha <= 8) {
        SNK_TRY(sep_blur(a, ha, tpa, src, dst, nx, ny, nz, st));
      } else {
        const unsigned grid = grid_for((int64_t)((nx + 1) / 2) * ny * nz, 256);
        if (a == 0) blur_pass_kernel<0><<<grid, 256, 0, st>>>(src, dst, nx, ny, nz, ha, tpa);
        else if (a == 1) blur_pass_kernel<1><<<grid, 256, 0, st>>>(src, dst, nx, ny, nz, ha, tpa);
        else blur_pass_kernel<2><<<grid, 256, 0, st>>>(src, dst, nx, ny, nz, ha, tpa);
        SNK_LAUNCH_CHECK("blur_pass_kernel");
      }
      src = dst;
    }
  } else if (h == 0) {
    SNK_CUDA_CHECK(cudaMemcpyAsync(d_smooth, d_in, nvox * sizeof(uint16_t), cudaMemcpyDeviceToDevice, st));
  } else if (SNK_BLUR_TMA && blur_tma_ok(g, h, d_in, d_smooth)) {
    // x, y and z in one TMA-staged pass (stencil.cu): 2 B read + 2 B written per voxel
    SNK_TRY(blur_tma(g, h, taps.data(), d_in, d_smooth, st));
  } else if (h <= 8 && vec8_ok(g, d_in, d_smooth, tmp)) {
    // three (2D: two) streaming separable passes, 8 voxels per thread
    if (g->dim == 3) {
      SNK_TRY(sep_blur(0, h, tp, d_in, d_smooth, nx, ny, nz, st));
      SNK_TRY(sep_blur(1, h, tp, d_smooth, tmp, nx, ny, nz, st));
      SNK_TRY(sep_blur(2, h, tp, tmp, d_smooth, nx, ny, nz, st));
    } else {
      SNK_TRY(sep_blur(0, h, tp, d_in, tmp, nx, ny, nz, st));
      SNK_TRY(sep_blur(1, h, tp, tmp, d_smooth, nx, ny, nz, st));
    }
  } else if (h <= 8) {
    switch (h) {
      case 1: SNK_TRY(launch_fused_blur<1>(g, d_in, d_smooth, tp, st)); break;
      case 2: SNK_TRY(launch_fused_blur<2>(g, d_in, d_smooth, tp, st)); break;
      case 3: SNK_TRY(launch_fused_blur<3>(g, d_in, d_smooth, tp, st)); break;
      case 4: SNK_TRY(launch_fused_blur<4>(g, d_in, d_smooth, tp, st)); break;
      case 5: SNK_TRY(launch_fused_blur<5>(g, d_in, d_smooth, tp, st)); break;
      case 6: SNK_TRY(launch_fused_blur<6>(g, d_in, d_smooth, tp, st)); break;
      case 7: SNK_TRY(launch_fused_blur<7>(g, d_in, d_smooth, tp, st)); break;
      default: SNK_TRY(launch_fused_blur<8>(g, d_in, d_smooth, tp, st)); break;
    }
  } else {
    // wide kernels (sigma > 2): three separable passes through the workspace
    const int64_t pairs = (int64_t)((nx + 1) / 2) * ny * nz;
    const unsigned grid = grid_for(pairs, 256);
    if (g->dim == 3) {
      blur_pass_kernel<0><<<grid, 256, 0, st>>>(d_in, d_smooth, nx, ny, nz, h, tp);
      SNK_LAUNCH_CHECK("blur_pass_kernel<x>");
      blur_pass_kernel<1><<<grid, 256, 0, st>>>(d_smooth, tmp, nx, ny, nz, h, tp);
      SNK_LAUNCH_CHECK("blur_pass_kernel<y>");
      blur_pass_kernel<2><<<grid, 256, 0, st>>>(tmp, d_smooth, nx, ny, nz, h, tp);
      SNK_LAUNCH_CHECK("blur_pass_kernel<z>");
    } else {
      blur_pass_kernel<0><<<grid, 256, 0, st>>>(d_in, tmp, nx, ny, nz, h, tp);
      SNK_LAUNCH_CHECK("blur_pass_kernel<x>");
      blur_pass_kernel<1><<<grid, 256, 0, st>>>(tmp, d_smooth, nx, ny, nz, h, tp);
      SNK_LAUNCH_CHECK("blur_pass_kernel<y>");
    }
  }
  if (d_gradmag && vec8_ok(g, d_smooth, d_gradmag, nullptr)) {
    const unsigned grid = (unsigned)ceil_div(nvox / 8, 256);
    if (g->dim == 3) gradmag8_kernel<3><<<grid, 256, 0, st>>>(d_smooth, d_gradmag, nx, ny, nz);
    else gradmag8_kernel<2><<<grid, 256, 0, st>>>(d_smooth, d_gradmag, nx, ny, nz);
    SNK_LAUNCH_CHECK("gradmag8_kernel");
  } else if (d_gradmag) {
    dim3 grid((unsigned)ceil_div(nx, kBX), (unsigned)ceil_div(ny, kBY),
              g->dim == 3 ? (unsigned)ceil_div(nz, kBZC) : 1u);
    if (g->dim == 3) gradmag_tiled_kernel<3><<<grid, kBThreads, 0, st>>>(d_smooth, d_gradmag, nx, ny, nz);
    else gradmag_tiled_kernel<2><<<grid, kBThreads, 0, st>>>(d_smooth, d_gradmag, nx, ny, nz);
    SNK_LAUNCH_CHECK("gradmag_tiled_kernel");
  }
  return SNK_OK;
}

size_t resample_ws(int32_t dim, const int64_t n_raw[3], const double spacing[3]) {
  int64_t no[3];
  if (snk_resample_dims(dim, n_raw, spacing, no) != SNK_OK) return 0;
  // at most two intermediate volumes (x then y before z)
  int64_t cur[3] = {n_raw[0], n_raw[1], n_raw[2]};
  size_t total = 0;
  int npass = 0;
  for (int a = 0; a < dim; ++a) npass += (no[a] != n_raw[a]);
  int done = 0;
  for (int a = 0; a < dim; ++a) {
    if (no[a] == n_raw[a]) continue;
    cur[a] = no[a];
    ++done;
    if (done < npass) total += (size_t)cur[0] * cur[1] * cur[2] * sizeof(uint16_t) + 256;
  }
  return total;
}

int32_t resample_impl(int32_t dim, const int64_t n_raw[3], const double spacing[3], int64_t zr_lo,
                      int64_t nzr, const uint16_t* d_raw, int64_t z_lo, int64_t nz_out,
                      uint16_t* d_out, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  int64_t no[3];
  SNK_TRY(snk_resample_dims(dim, n_raw, spacing, no));
  double smin = spacing[0];
  for (int a = 1; a < dim; ++a) smin = std::min(smin, spacing[a]);
  if (zr_lo < 0 || nzr < 1 || zr_lo + nzr > n_raw[2] || z_lo < 0 || nz_out < 1 ||
      z_lo + nz_out > no[2])
    return fail(SNK_SHAPE, "resample plane ranges outside the volume");
  const bool rz = no[2] != n_raw[2];
  if (!rz && (zr_lo != z_lo || nzr < nz_out))
    return fail(SNK_SHAPE, "z is not resampled: output planes must equal the raw planes");
  if (rz) {
    // the raw planes the output planes read
    const double ratio = smin / spacing[2];
    auto src_i0 = [&](int64_t k) {
      double s = ((double)k + 0.5) * ratio - 0.5;
      s = std::min(std::max(s, 0.0), (double)(n_raw[2] - 1));
      return std::min((int64_t)std::floor(s), n_raw[2] - 2);
    };
    const int64_t lo = src_i0(z_lo), hi = src_i0(z_lo + nz_out - 1) + 1;
    if (lo < zr_lo || hi > zr_lo + nzr - 1) return fail(SNK_SHAPE, "raw planes missing for resampling");
  }
  int npass = 0;
  for (int a = 0; a < dim; ++a) npass += (no[a] != n_raw[a]);
  // current buffer dims: x, y, planes; z-buffer origin
  int64_t cx = n_raw[0], cy = n_raw[1], cz = rz ? nzr : nz_out, cz0 = rz ? zr_lo : z_lo;
  const uint16_t* cur = d_raw + (rz ? 0 : (z_lo - zr_lo) * n_raw[0] * n_raw[1]);
  if (npass == 0) {
    SNK_CUDA_CHECK(cudaMemcpyAsync(d_out, cur, (size_t)cx * cy * nz_out * sizeof(uint16_t),
                                   cudaMemcpyDeviceToDevice, st));
    return SNK_OK;
  }
  Carve cv(d_ws, ws_bytes);
  int done = 0;
  for (int a = 0; a < dim; ++a) {
    if (no[a] == n_raw[a]) continue;
    ++done;
    int64_t ox = cx, oy = cy, oz = cz, oz0 = cz0;
    if (a == 0) ox = no[0];
    if (a == 1) oy = no[1];
    if (a == 2) { oz = nz_out; oz0 = z_lo; }
    uint16_t* dst = done == npass ? d_out : cv.take<uint16_t>((size_t)ox * oy * oz);
    if (cv.overflow) return fail(SNK_CAPACITY, "workspace too small for resample");
    const double ratio = smin / spacing[a];
    const int64_t total = ox * oy * oz;
    const unsigned grid = grid_for(total, 256);
    if (a == 0)
      resample_kernel<0><<<grid, 256, 0, st>>>(cur, dst, cx, cy, oz, ox, oy, n_raw[0], ratio, cz0, oz0);
    else if (a == 1)
      resample_kernel<1><<<grid, 256, 0, st>>>(cur, dst, cx, cy, oz, ox, oy, n_raw[1], ratio, cz0, oz0);
    else
      resample_kernel<2><<<grid, 256, 0, st>>>(cur, dst, cx, cy, oz, ox, oy, n_raw[2], ratio, cz0, oz0);
    SNK_LAUNCH_CHECK("resample_kernel");
    cur = dst;
    cx = ox; cy = oy; cz = oz; cz0 = oz0;
  }
  return SNK_OK;
}

int32_t ingest_u8_impl(const uint8_t* d_in, uint16_t* d_out, int64_t n, cudaStream_t st) {
  if (n <= 0) return SNK_OK;
  if ((reinterpret_cast<uintptr_t>(d_in) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15)) {
    ingest_u8_scalar_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d_in, d_out, n);   // unaligned buffers
    SNK_LAUNCH_CHECK("ingest_u8_scalar_kernel");
    return SNK_OK;
  }
  const int64_t threads = (n + 15) / 16;
  ingest_u8_kernel<<<(unsigned)ceil_div(threads, 256), 256, 0, st>>>(d_in, d_out, n);
  SNK_LAUNCH_CHECK("ingest_u8_kernel");
  return SNK_OK;
}

}  // namespace snk
