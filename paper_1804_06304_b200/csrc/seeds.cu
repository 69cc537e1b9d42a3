// seeds.cu — a4 seed placement (include/snk.h snk_seeds).
//   LATTICE: the paper's lattice, spacing sqrt(1.5) r0, centred
//            (S:101), positions in IEEE double without contraction then fp32.
//   MAXIMA:  first maxima of the (2w+1)^d box above a threshold (G20):
//            separable box-max (3 u16 passes) -> candidate test B == M, B >= thr
//            -> tie check (no equal value earlier in linear order inside the
//            window, only for candidates) -> order-preserving compaction.
// Integer-exact; bit-identical to the definition.
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "tma.cuh"

namespace snk {

namespace {

constexpr int kChunk = 2048;        // voxels per compaction block
constexpr int kCompactThreads = 256;
constexpr int kPerThread = kChunk / kCompactThreads;   // 8 consecutive voxels per thread

// Box max along AXIS over [p - w, p + w] clipped to [lo, hi] (buffer-local indices).
template <int AXIS>
__global__ void __launch_bounds__(256) boxmax_kernel(const uint16_t* __restrict__ in,
                                                     uint16_t* __restrict__ out, int nx, int ny,
                                                     int nz, int w, int zlo_valid, int zhi_valid) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t plane = (int64_t)nx * ny;
  if (t >= plane * nz) return;
  const int x = (int)(t % nx);
  const int y = (int)((t / nx) % ny);
  const int z = (int)(t / plane);
  int p, lo, hi;
  int64_t stride;
  if (AXIS == 0) { p = x; lo = 0; hi = nx - 1; stride = 1; }
  else if (AXIS == 1) { p = y; lo = 0; hi = ny - 1; stride = nx; }
  else { p = z; lo = zlo_valid; hi = zhi_valid; stride = plane; }
  const int a = max(p - w, lo), b = min(p + w, hi);
  const uint16_t* base = in + t - (int64_t)p * stride;
  uint32_t m = 0;
  for (int q = a; q <= b; ++q) m = max(m, (uint32_t)__ldg(base + (int64_t)q * stride));
  out[t] = (uint16_t)m;
}

struct MaxArgs {
  const uint16_t* B;   // smoothed buffer
  const uint16_t* M;   // box max
  int nx, ny, nz_glob, z_lo;   // z_lo: global plane of buffer plane 0
  int w, dim;
  uint32_t thr;
  int64_t v0, v1;      // buffer-linear voxel range scanned: own planes
  int wx, wy, wz;      // per-axis half-windows (the tie check; = w unless anisotropic, G28)
};

// Seed predicate at buffer-linear index v (3D/2D), §8(c) O4.
__device__ __forceinline__ bool is_seed(const MaxArgs& A, int64_t v, uint16_t b, uint16_t m) {
  if ((uint32_t)b < A.thr || b != m) return false;
  const int64_t plane = (int64_t)A.nx * A.ny;
  const int x = (int)(v % A.nx), y = (int)((v / A.nx) % A.ny);
  const int zb = (int)(v / plane);
  const int z = zb + A.z_lo;
  // earlier equal value in the clipped window?  (linear order: z, then y, then x)
  const int z0 = A.dim == 3 ? max(z - A.w, 0) : z;
  const int y0 = max(y - A.w, 0), y1 = min(y + A.w, A.ny - 1);
  const int x0 = max(x - A.w, 0), x1 = min(x + A.w, A.nx - 1);
  for (int zz = z0; zz <= z; ++zz)
    for (int yy = y0; yy <= (zz == z ? y : y1); ++yy) {
      const uint16_t* row = A.B + ((int64_t)(zz - A.z_lo) * A.ny + yy) * A.nx;
      const int xe = (zz == z && yy == y) ? x - 1 : x1;
      for (int xx = x0; xx <= xe; ++xx)
        if (__ldg(row + xx) == b) return false;
    }
  return true;
}

__device__ __forceinline__ int block_exclusive_scan(int v, int* smem, int* total) {
  // smem: kCompactThreads / 32 ints
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < (kCompactThreads / 32) ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < (kCompactThreads / 32)) smem[lane] = s;
  }
  __syncthreads();
  const int warp_off = warp > 0 ? smem[warp - 1] : 0;
  *total = smem[kCompactThreads / 32 - 1];
  return warp_off + x - v;
}

__device__ __forceinline__ int load8(const MaxArgs& A, int64_t v, uint16_t* b, uint16_t* m) {
  // 8 consecutive voxels starting at v (v % 8 == 0 relative to v0 which is plane-aligned)
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    const int64_t vv = v + k;
    if (vv < A.v1) { b[k] = __ldg(A.B + vv); m[k] = __ldg(A.M + vv); cnt = k + 1; }
    else { b[k] = 0; m[k] = 1; }
  }
  return cnt;
}

__global__ void __launch_bounds__(kCompactThreads) maxima_count_kernel(MaxArgs A, int* counts) {
  __shared__ int sm[kCompactThreads / 32];
  const int64_t v = A.v0 + (int64_t)blockIdx.x * kChunk + (int64_t)threadIdx.x * kPerThread;
  uint16_t b[kPerThread], m[kPerThread];
  load8(A, v, b, m);
  int c = 0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k)
    if (v + k < A.v1 && is_seed(A, v + k, b[k], m[k])) ++c;
  int total;
  block_exclusive_scan(c, sm, &total);
  if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kCompactThreads) maxima_write_kernel(MaxArgs A,
                                                                       const int64_t* offsets,
                                                                       float* seeds, int64_t cap) {
  __shared__ int sm[kCompactThreads / 32];
  const int64_t v = A.v0 + (int64_t)blockIdx.x * kChunk + (int64_t)threadIdx.x * kPerThread;
  uint16_t b[kPerThread], m[kPerThread];
  load8(A, v, b, m);
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k)
    if (v + k < A.v1 && is_seed(A, v + k, b[k], m[k])) mask |= 1u << k;
  int total;
  int64_t o = offsets[blockIdx.x] + block_exclusive_scan(__popc(mask), sm, &total);
  const int64_t plane = (int64_t)A.nx * A.ny;
  for (int k = 0; k < kPerThread; ++k)
    if (mask & (1u << k)) {
      const int64_t vv = v + k;
      if (o < cap) {
        seeds[3 * o + 0] = (float)(vv % A.nx);
        seeds[3 * o + 1] = (float)((vv / A.nx) % A.ny);
        seeds[3 * o + 2] = (float)(vv / plane + A.z_lo);
      }
      ++o;
    }
}

// LATTICE positions: o + i s per axis in double (no FMA), stored as fp32.
__global__ void lattice_kernel(int64_t kx, int64_t ky, int64_t iz0, int64_t nzl, double ox,
                               double oy, double oz, double s, int dim, float* seeds) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kx * ky * nzl) return;
  const int64_t ix = t % kx, iy = (t / kx) % ky, iz = iz0 + t / (kx * ky);
  seeds[3 * t + 0] = __double2float_rn(__dadd_rn(ox, __dmul_rn((double)ix, s)));
  seeds[3 * t + 1] = __double2float_rn(__dadd_rn(oy, __dmul_rn((double)iy, s)));
  seeds[3 * t + 2] = dim == 3 ? __double2float_rn(__dadd_rn(oz, __dmul_rn((double)iz, s))) : 0.0f;
}

// ---------------------------------------------------------------------------
// Fused MAXIMA (3D, w <= 8; 2D any w): one CTA per 64 x 16 output columns and
// a 32-plane z-chunk of the owned planes.  Per input plane the (16+2w) x
// (64+2w) tile is staged in shared memory (voxels outside the volume -> 0,
// the neutral element of max, i.e. the clipped window), the x and y box-max
// run there, and the y-maxima enter a per-thread register ring of 2w+1 planes
// (with the centre values B), from which M = box max of plane z - w follows.
// Candidates B >= thr && B == M get the tie check (an equal value earlier in
// linear order inside the clipped window) from global memory; the result is a
// bitmask (bit x of word (z, y, x/32)), so the compaction below emits seeds in
// linear-index order.
constexpr int kMX = 64, kMY = 16, kMZC = 32, kMThreads = 256;

struct FusedArgs {
  const uint16_t* B;
  uint32_t* bits;          // words per row: ceil(nx/32); rows: own planes x ny
  int nx, ny, nzg, z_lo, own_z0, own_z1, wpr;
  int w;
  uint32_t thr;
  MaxArgs ma;              // for the tie check (is_seed semantics)
};

__device__ __forceinline__ bool tie_free(const MaxArgs& A, int x, int y, int z, uint16_t b) {
  const int z0 = A.dim == 3 ? max(z - A.wz, 0) : z;
  const int y0 = max(y - A.wy, 0), y1 = min(y + A.wy, A.ny - 1);
  const int x0 = max(x - A.wx, 0), x1 = min(x + A.wx, A.nx - 1);
  for (int zz = z0; zz <= z; ++zz)
    for (int yy = y0; yy <= (zz == z ? y : y1); ++yy) {
      const uint16_t* row = A.B + ((int64_t)(zz - A.z_lo) * A.ny + yy) * A.nx;
      const int xe = (zz == z && yy == y) ? x - 1 : x1;
      for (int xx = x0; xx <= xe; ++xx)
        if (__ldg(row + xx) == b) return false;
    }
  return true;
}

// K = 2W+1 z-ring (3D) ; W = 0 selects the 2D kernel with runtime window
template <int D, int W>
__global__ void __launch_bounds__(kMThreads) maxima_fused_kernel(FusedArgs A) {
  constexpr int K = 2 * W + 1;
  extern __shared__ uint16_t sm[];
  const int w = D == 3 ? W : A.w;
  const int RX = kMX + 2 * w, RY = kMY + 2 * w;
  uint16_t* s_in = sm;                   // [RY][RX]
  uint16_t* s_x = sm + RY * RX;          // [RY][kMX]
  const int x0 = blockIdx.x * kMX, y0 = blockIdx.y * kMY;
  const int z0 = A.own_z0 + blockIdx.z * kMZC;
  const int tx = threadIdx.x % kMX, ty = threadIdx.x / kMX;
  const int lane = threadIdx.x & 31;
  const int zend = D == 3 ? min(z0 + kMZC, A.own_z1) : z0 + 1;
  const int nplanes = (zend - z0) + 2 * (D == 3 ? W : 0);
  uint32_t ring[K][4];
  // 3D: the next plane's tile is prefetched into registers while this plane
  // computes (the walk over planes is otherwise latency-bound)
  constexpr int PER3 = ((kMY + 2 * W) * (kMX + 2 * W) + kMThreads - 1) / kMThreads;
  uint16_t pf[D == 3 ? PER3 : 1];
  auto fetch = [&](int zin) {
    const bool valid = zin >= 0 && zin < A.nzg;
    const uint16_t* src = A.B + (int64_t)(zin - A.z_lo) * A.nx * A.ny;
#pragma unroll
    for (int q = 0; q < PER3; ++q) {
      const int e = threadIdx.x + q * kMThreads;
      if (e < RY * RX) {
        const int r = e / RX, c = e % RX;
        const int gy = y0 - w + r, gx = x0 - w + c;
        pf[q] = (valid && gy >= 0 && gy < A.ny && gx >= 0 && gx < A.nx) ? __ldg(src + (int64_t)gy * A.nx + gx) : 0;
      }
    }
  };
  // separable box max of the staged plane: x in shared memory, y per thread
  auto boxmax = [&](uint32_t* ym) {
    __syncthreads();
    for (int e = threadIdx.x; e < RY * kMX; e += kMThreads) {
      const int r = e / kMX, c = e % kMX;
      uint32_t m = 0;
      for (int i = 0; i <= 2 * w; ++i) m = max(m, (uint32_t)s_in[r * RX + c + i]);
      s_x[e] = (uint16_t)m;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t m = 0;
      const int r = ty * 4 + k;
      for (int i = 0; i <= 2 * w; ++i) m = max(m, (uint32_t)s_x[(r + i) * kMX + tx]);
      ym[k] = m;
    }
  };
  auto emit = [&](int zo, const uint32_t* M) {
    const uint16_t* bp = A.B + (int64_t)(zo - A.z_lo) * A.nx * A.ny;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int x = x0 + tx, y = y0 + ty * 4 + k;
      bool seed = false;
      if (x < A.nx && y < A.ny) {
        const uint32_t b = __ldg(bp + (int64_t)y * A.nx + x);
        if (b >= A.thr && b == M[k]) seed = tie_free(A.ma, x, y, zo, (uint16_t)b);
      }
      const unsigned m = __ballot_sync(0xffffffffu, seed);
      if (lane == 0 && y < A.ny && x < A.nx)
        A.bits[((int64_t)(zo - A.own_z0) * A.ny + y) * A.wpr + (x >> 5)] = m;
    }
  };
  if (D == 2) {
    for (int e = threadIdx.x; e < RY * RX; e += kMThreads) {
      const int r = e / RX, c = e % RX;
      const int gy = y0 - w + r, gx = x0 - w + c;
      s_in[e] = (gy >= 0 && gy < A.ny && gx >= 0 && gx < A.nx) ? __ldg(A.B + (int64_t)gy * A.nx + gx) : 0;
    }
    uint32_t ym[4];
    boxmax(ym);
    emit(z0, ym);
    return;
  }
  fetch(z0 - W);
  for (int base = 0; base < nplanes; base += K) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int pi = base + j;
      if (pi >= nplanes) break;
      __syncthreads();   // the previous plane is done with s_in / s_x
#pragma unroll
      for (int q = 0; q < PER3; ++q) {
        const int e = threadIdx.x + q * kMThreads;
        if (e < RY * RX) s_in[e] = pf[q];
      }
      if (pi + 1 < nplanes) fetch(z0 - W + pi + 1);
      boxmax(ring[j]);
      if (pi >= 2 * W) {
        uint32_t M[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t m = 0;
#pragma unroll
          for (int i = 0; i < K; ++i) m = max(m, ring[(j + 1 + i) % K][k]);
          M[k] = m;
        }
        emit(z0 + pi - 2 * W, M);
      }
    }
  }
}

// compaction of the bitmask: words in linear order, 1024 words per block, 4
// consecutive words per thread (256 threads: a quarter of the threads and
// scan of the one-word-per-thread version; the launches were bound by block
// scheduling, not by the 4 B per word they read)
constexpr int kWPT = 4, kBitsThreads = 1024 / kWPT;

__device__ __forceinline__ void load_words(const uint32_t* bits, int64_t nwords, int64_t i0, uint32_t w[kWPT]) {
#pragma unroll
  for (int k = 0; k < kWPT; ++k) w[k] = i0 + k < nwords ? bits[i0 + k] : 0u;
}

__global__ void __launch_bounds__(kBitsThreads) bits_count_kernel(const uint32_t* bits, int64_t nwords, int* counts) {
  uint32_t w[kWPT];
  load_words(bits, nwords, (int64_t)blockIdx.x * 1024 + threadIdx.x * kWPT, w);
  int c = 0;
#pragma unroll
  for (int k = 0; k < kWPT; ++k) c += __popc(w[k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int ws[kBitsThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int v = 0;
#pragma unroll
    for (int k = 0; k < kBitsThreads / 32; ++k) v += ws[k];
    counts[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(kBitsThreads) bits_write_kernel(const uint32_t* bits, int64_t nwords, int wpr,
                                                                  int nx, int ny, int own_z0,
                                                                  const int64_t* offsets, float* seeds,
                                                                  int64_t cap, int linear, double sx = 1.0,
                                                                  double sy = 1.0, double sz = 1.0) {
  constexpr int NWARP = kBitsThreads / 32;
  __shared__ int ws[NWARP];
  const int64_t i0 = (int64_t)blockIdx.x * 1024 + threadIdx.x * kWPT;
  uint32_t w[kWPT];
  load_words(bits, nwords, i0, w);
  int c = 0;
#pragma unroll
  for (int k = 0; k < kWPT; ++k) c += __popc(w[k]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  int before = 0;
#pragma unroll
  for (int k = 0; k < NWARP; ++k) before += k < warp ? ws[k] : 0;
  if (!c) return;
  int64_t o = offsets[blockIdx.x] + before + x - c;
  const int64_t plane = (int64_t)nx * ny;
#pragma unroll 1
  for (int k = 0; k < kWPT; ++k) {
    uint32_t m = w[k];
    if (!m) continue;
    const int64_t i = i0 + k;
    if (linear) {   // bit b of word i = own-region voxel 32 i + b (x fastest)
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const int64_t v = i * 32 + b;
        if (o < cap) {   // physical coordinates (index x scale, G28; exact for scale 1)
          seeds[3 * o + 0] = (float)((double)(v % nx) * sx);
          seeds[3 * o + 1] = (float)((double)((v / nx) % ny) * sy);
          seeds[3 * o + 2] = (float)((double)(v / plane + own_z0) * sz);
        }
        ++o;
      }
      continue;
    }
    const int64_t row = i / wpr;                 // (z - own_z0) * ny + y
    const int xw = (int)(i % wpr) * 32;
    const float fy = (float)(row % ny), fz = (float)(row / ny + own_z0);
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      if (o < cap) {
        seeds[3 * o + 0] = (float)(xw + b);
        seeds[3 * o + 1] = fy;
        seeds[3 * o + 2] = fz;
      }
      ++o;
    }
  }
}

// ---------------------------------------------------------------------------
// Vectorised MAXIMA (w <= 8, nx % 8 == 0): the x and y box-max are two
// streaming sep_pass launches (volume.cu) into XY; this kernel takes one
// 8-voxel group of the owned region per thread, folds the z box-max from the
// 2w+1 XY planes (3D; clipped to the volume), tests B >= thr && B == M, runs
// the tie check for the (rare) candidates, and writes one mask byte (bit k =
// voxel 8 t + k), so the mask words are in linear voxel order.
__device__ __forceinline__ void unpack8s(const uint4 q, uint32_t* v) {
  v[0] = q.x & 0xffffu; v[1] = q.x >> 16; v[2] = q.y & 0xffffu; v[3] = q.y >> 16;
  v[4] = q.z & 0xffffu; v[5] = q.z >> 16; v[6] = q.w & 0xffffu; v[7] = q.w >> 16;
}

// The tie check of one candidate by the whole warp: lane l scans window rows
// l, l + 32, ... (rows in linear order before the candidate's own row, plus the
// part of that row left of it) for a value equal to b.  Same predicate as
// tie_free, 32x shorter serial path (a lone candidate no longer holds its warp
// for the whole (2w+1)^d window).
__device__ __forceinline__ bool tie_free_warp(const MaxArgs& A, int x, int y, int z, uint16_t b, int lane) {
  const int z0 = A.dim == 3 ? max(z - A.wz, 0) : z;
  const int y0 = max(y - A.wy, 0), y1 = min(y + A.wy, A.ny - 1);
  const int x0 = max(x - A.wx, 0), x1 = min(x + A.wx, A.nx - 1);
  const int nyw = y1 - y0 + 1;
  const int rows = (z - z0) * nyw + (y - y0 + 1);
  bool found = false;
  for (int r = lane; r < rows && !found; r += 32) {
    const int zz = z0 + r / nyw, yy = y0 + r % nyw;
    const uint16_t* row = A.B + ((int64_t)(zz - A.z_lo) * A.ny + yy) * A.nx;
    const int xe = (zz == z && yy == y) ? x - 1 : x1;
    for (int xx = x0; xx <= xe; ++xx)
      if (__ldg(row + xx) == b) { found = true; break; }
  }
  return !__any_sync(0xffffffffu, found);
}

template <int D, int W>
// Grid (x groups / 256, y, owned planes): the (x group, y, z) of a thread come
// from the block indices (the 64-bit divisions of a flat index cost ~1/3 of
// the kernel's instructions).
__global__ void __launch_bounds__(256) maxima_pred8_kernel(MaxArgs A, const uint16_t* __restrict__ XY,
                                                           uint8_t* __restrict__ mask, int64_t ngroups,
                                                           int own_z0) {
  (void)ngroups;
  const int lane = threadIdx.x & 31;
  const int nc = A.nx >> 3;
  const int xc0 = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = xc0 < nc;              // every lane stays for the warp-wide tie checks
  const int xc = valid ? xc0 : nc - 1;
  const int y = blockIdx.y;
  const int zo = (int)blockIdx.z + own_z0;   // global plane
  const int64_t t = ((int64_t)blockIdx.z * A.ny + y) * nc + xc;   // the group's index in the owned region
  const int64_t idx = ((int64_t)(zo - A.z_lo) * A.ny + y) * nc + xc;
  const uint4 bq = __ldg(reinterpret_cast<const uint4*>(A.B) + idx);
  uint32_t b[8], m[8];
  unpack8s(bq, b);
  if (D == 3) {
    const int64_t pstride = (int64_t)A.ny * nc;
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = 0;
#pragma unroll
    for (int i = -W; i <= W; ++i) {
      if (zo + i < 0 || zo + i >= A.nz_glob) continue;
      uint32_t v[8];
      unpack8s(__ldg(reinterpret_cast<const uint4*>(XY) + idx + i * pstride), v);
#pragma unroll
      for (int k = 0; k < 8; ++k) m[k] = max(m[k], v[k]);
    }
  } else {
    unpack8s(__ldg(reinterpret_cast<const uint4*>(XY) + idx), m);
  }
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (b[k] >= A.thr && b[k] == m[k]) bits |= 1u << k;
  if (!valid) bits = 0;
  // candidates, one at a time per warp, each checked by all 32 lanes
  uint32_t pending = bits;
  unsigned ballot = __ballot_sync(0xffffffffu, pending != 0u);
  while (ballot) {
    const int src = __ffs(ballot) - 1;
    const uint32_t pb = __shfl_sync(0xffffffffu, pending, src);
    const int k = __ffs(pb) - 1;
    const uint32_t word = (k >> 1) == 0 ? bq.x : (k >> 1) == 1 ? bq.y : (k >> 1) == 2 ? bq.z : bq.w;
    const uint32_t bk = __shfl_sync(0xffffffffu, (k & 1) ? word >> 16 : word & 0xffffu, src);
    const int cx = __shfl_sync(0xffffffffu, xc * 8, src) + k;
    const int cy = __shfl_sync(0xffffffffu, y, src), cz = __shfl_sync(0xffffffffu, zo, src);
    const bool ok = tie_free_warp(A, cx, cy, cz, (uint16_t)bk, lane);
    if (lane == src) {
      if (!ok) bits &= ~(1u << k);
      pending &= ~(1u << k);
    }
    ballot = __ballot_sync(0xffffffffu, pending != 0u);
  }
  if (valid) mask[t] = (uint8_t)bits;
}

// ---------------------------------------------------------------------------
// TMA-staged MAXIMA (3D, isotropic window 1 <= w <= 8, nx % 8 == 0, 16-byte
// aligned B): the whole a4 predicate in ONE pass over B, with the box max
// never leaving the SM.  A CTA owns a 64 x 32 column tile and walks a chunk of
// zc owned planes; every input plane's (64 + 16) x (32 + 2w) box is copied by
// the Tensor Memory Accelerator into a 4-stage mbarrier ring (x start x0 - 8:
// 16-byte aligned, profiles/r2_tma_probe.md).  Box elements outside the volume
// arrive as zeros — the neutral element of max, i.e. the window clipped to the
// volume (O4).  Per plane: the x box max (shared -> shared), the y box max
// (shared -> registers), both on packed u16 pairs (VIMNMX3.U16x2: three-input
// max of two lanes per instruction); the y-maxima enter a per-thread register
// ring of 2w + 1 planes whose max is M of plane z - w.  Candidates B >= thr &&
// B == M (B re-read from L2) get the warp-cooperative tie check; one mask byte
// per 8 voxels, in linear voxel order (bits_count / bits_write compact it).
#ifndef SNK_QTHREADS
#define SNK_QTHREADS 256
#endif
// 256 threads own the 64 x 32 outputs (8 voxels each); the x pass's (32 + 2w) x 8
// tasks run on all kQThreads (a build with 384 threads takes them in one round:
// 1 CTA per SM by registers, C4 seeds 13.4 ms — slower)
constexpr int kQX = 64, kQY = 32, kQNS = 4, kQThreads = SNK_QTHREADS, kQOut = 256;
constexpr int kQBX = kQX + 16;

struct MaxTmaArgs {
  MaxArgs ma;        // B (the buffer), dims, z_lo, windows, thr: the tie check
  uint8_t* mask;     // one byte per 8-voxel group of the own region
  int own_z0, own_z1, zc;
};

__device__ __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }

// Box max over columns c - W .. c + W (lane 0) and c + 1 - W .. c + 1 + W (lane
// 1) of the output word at even column c = 8 + 2j of a row segment whose words
// are E[m] = (cols 2m, 2m + 1) and O[m] = (2m + 1, 2m + 2): W + 1 words of one
// kind and W of the other cover both lanes' windows exactly.
template <int W>
__device__ __forceinline__ uint32_t xwin(const uint32_t* E, const uint32_t* O, int j) {
  uint32_t m;
  if (W & 1) {   // c - W odd: O[(c-W-1)/2 + i], i <= W; E[(c-W+1)/2 + i], i < W
    const int o0 = j + (7 - W) / 2, e0 = j + (9 - W) / 2;
    m = O[o0];
#pragma unroll
    for (int i = 1; i <= W; ++i) m = vmax(m, O[o0 + i]);
#pragma unroll
    for (int i = 0; i < W; ++i) m = vmax(m, E[e0 + i]);
  } else {       // c - W even: E[(c-W)/2 + i], i <= W; O[(c-W)/2 + i], i < W
    const int e0 = j + (8 - W) / 2;
    m = E[e0];
#pragma unroll
    for (int i = 1; i <= W; ++i) m = vmax(m, E[e0 + i]);
#pragma unroll
    for (int i = 0; i < W; ++i) m = vmax(m, O[e0 + i]);
  }
  return m;
}

#ifndef SNK_QMINB
#define SNK_QMINB 2
#endif
template <int W>
__global__ void __launch_bounds__(kQThreads, SNK_QMINB)
    maxima_tma_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ MaxTmaArgs A) {
  constexpr int BY = kQY + 2 * W, K = 2 * W + 1;
  constexpr uint32_t kBoxBytes = kQBX * BY * 2;
  constexpr uint32_t kStage = (kBoxBytes + 127) & ~127u;   // TMA destinations: 128-byte aligned
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem);                 // [NS] x ([BY][QBX] + pad)
  uint16_t* sx = reinterpret_cast<uint16_t*>(smem + kQNS * kStage);   // [BY][QX]
  __shared__ __align__(8) uint64_t full[kQNS];
  const MaxArgs& M = A.ma;
  const int nx = M.nx, ny = M.ny;
  const int x0 = blockIdx.x * kQX, y0 = blockIdx.y * kQY;
  const int zs = A.own_z0 + blockIdx.z * A.zc, ze = min(zs + A.zc, A.own_z1);
  const int nplanes = (ze - zs) + 2 * W;
  const int tid = threadIdx.x, lane = tid & 31;
  auto box_z = [&](int p) { return zs - W + p - M.z_lo; };   // buffer plane (TMA zero-fills outside)
  if (tid == 0) {
    for (int s = 0; s < kQNS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int p = 0; p < kQNS - 1 && p < nplanes; ++p)
      tma_load_box(&map, ring + p * (kStage / 2), &full[p], x0 - 8, y0 - W, box_z(p), kBoxBytes);
  }
  __syncthreads();
  const int q = tid & 7, r = tid >> 3;            // output cols x0 + 8q .. + 7, row y0 + r
  const int xo = x0 + 8 * q, yo = y0 + r;
  const bool outw = tid < kQOut;                  // warp-uniform: this warp owns outputs
  const bool own = outw && xo < nx && yo < ny;
  const uint32_t thr = M.thr;
  const uint32_t thr2 = thr <= 0xffffu ? (thr | (thr << 16)) : 0xffffffffu;
  uint32_t zr[K][4];
  for (int base = 0; base < nplanes; base += K) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int p = base + j;
      if (p >= nplanes) break;
      const int s = p % kQNS;
      const uint16_t* box = ring + s * (kStage / 2);
      mbar_wait(&full[s], (uint32_t)((p / kQNS) & 1));
      __syncthreads();   // box complete; the previous plane's y pass is done with sx
      // x pass: BY rows x 8 groups of 8 outputs; box cols 8g .. 8g + 23 cover x0 + 8g - 8 .. + 15
      for (int it = tid; it < BY * 8; it += kQThreads) {
        const int row = it >> 3, g = it & 7;
        const uint4* src = reinterpret_cast<const uint4*>(box + row * kQBX + 8 * g);
        uint32_t E[12], O[11];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const uint4 a = src[u];
          E[4 * u] = a.x; E[4 * u + 1] = a.y; E[4 * u + 2] = a.z; E[4 * u + 3] = a.w;
        }
#pragma unroll
        for (int m = 0; m < 11; ++m) O[m] = __byte_perm(E[m], E[m + 1], 0x5432);
        uint4 o;
        o.x = xwin<W>(E, O, 0);
        o.y = xwin<W>(E, O, 1);
        o.z = xwin<W>(E, O, 2);
        o.w = xwin<W>(E, O, 3);
        *reinterpret_cast<uint4*>(sx + row * kQX + 8 * g) = o;
      }
      __syncthreads();   // sx complete; every read of this box done
      if (tid == 0 && p + kQNS - 1 < nplanes) {
        const int nq = p + kQNS - 1;
        tma_load_box(&map, ring + (nq % kQNS) * (kStage / 2), &full[nq % kQNS], x0 - 8, y0 - W, box_z(nq), kBoxBytes);
      }
      if (!outw) continue;   // x-pass-only warps (whole warps: the tie check below is warp-collective)
      // y pass: sx rows r .. r + 2W (sx row i = y0 - W + i)
      {
        uint4 a = *reinterpret_cast<const uint4*>(sx + r * kQX + 8 * q);
        uint32_t m0 = a.x, m1 = a.y, m2 = a.z, m3 = a.w;
#pragma unroll
        for (int i = 1; i < K; ++i) {
          a = *reinterpret_cast<const uint4*>(sx + (r + i) * kQX + 8 * q);
          m0 = vmax(m0, a.x); m1 = vmax(m1, a.y); m2 = vmax(m2, a.z); m3 = vmax(m3, a.w);
        }
        zr[j][0] = m0; zr[j][1] = m1; zr[j][2] = m2; zr[j][3] = m3;
      }
      if (p >= 2 * W) {
        // the ring holds the y-maxima of planes zo - W .. zo + W: M = their max
        const int zo = zs + p - 2 * W;
        uint32_t mm[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t m = zr[0][k];
#pragma unroll
          for (int i = 1; i < K; ++i) m = vmax(m, zr[i][k]);
          mm[k] = m;
        }
        uint32_t bits = 0;
        uint4 bq = make_uint4(0, 0, 0, 0);
        if (own) {
          bq = __ldg(reinterpret_cast<const uint4*>(M.B + ((int64_t)(zo - M.z_lo) * ny + yo) * nx + xo));
          const uint32_t bw[4] = {bq.x, bq.y, bq.z, bq.w};
          uint32_t any = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) any |= __vcmpeq2(bw[k], mm[k]) & __vcmpgeu2(bw[k], thr2);
          if (any) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t c = __vcmpeq2(bw[k], mm[k]) & __vcmpgeu2(bw[k], thr2);
              bits |= ((c & 1u) | ((c >> 15) & 2u)) << (2 * k);
            }
          }
        }
        // candidates, one at a time per warp, each checked by all 32 lanes
        uint32_t pending = bits;
        unsigned ballot = __ballot_sync(0xffffffffu, pending != 0u);
        while (ballot) {
          const int src = __ffs(ballot) - 1;
          const uint32_t pb = __shfl_sync(0xffffffffu, pending, src);
          const int k = __ffs(pb) - 1;
          const uint32_t word = (k >> 1) == 0 ? bq.x : (k >> 1) == 1 ? bq.y : (k >> 1) == 2 ? bq.z : bq.w;
          const uint32_t bk = __shfl_sync(0xffffffffu, (k & 1) ? word >> 16 : word & 0xffffu, src);
          const int cx = __shfl_sync(0xffffffffu, xo, src) + k;
          const int cy = __shfl_sync(0xffffffffu, yo, src);
          const bool ok = tie_free_warp(M, cx, cy, zo, (uint16_t)bk, lane);
          if (lane == src) {
            if (!ok) bits &= ~(1u << k);
            pending &= ~(1u << k);
          }
          ballot = __ballot_sync(0xffffffffu, pending != 0u);
        }
        if (own) A.mask[((int64_t)(zo - A.own_z0) * ny + yo) * (nx >> 3) + (xo >> 3)] = (uint8_t)bits;
      }
    }
  }
}

bool maxima_tma_ok(const snk_grid* g, const snk_params* p, const void* B) {
  const int w = p->seed_window;
  return g->dim == 3 && !grid_aniso(g) && w >= 1 && w <= 8 && g->n[0] % 8 == 0 &&
         (reinterpret_cast<uintptr_t>(B) & 15) == 0 && tma_available();
}

template <int W>
int32_t launch_maxima_tma(const MaxTmaArgs& A, int nzb, cudaStream_t st) {
  constexpr int BY = kQY + 2 * W;
  const int smem = kQNS * ((kQBX * BY * 2 + 127) & ~127) + BY * kQX * 2;
  CUtensorMap map;
  SNK_TRY(volume_map(&map, A.ma.B, A.ma.nx, A.ma.ny, nzb, kQBX, BY));
  auto k = maxima_tma_kernel<W>;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] { attr = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  if (attr != cudaSuccess) return cuda_fail(attr, "cudaFuncSetAttribute(maxima_tma_kernel)");
  dim3 grid((unsigned)ceil_div(A.ma.nx, kQX), (unsigned)ceil_div(A.ma.ny, kQY),
            (unsigned)ceil_div(A.own_z1 - A.own_z0, A.zc));
  k<<<grid, kQThreads, smem, st>>>(map, A);
  SNK_LAUNCH_CHECK("maxima_tma_kernel");
  return SNK_OK;
}

int32_t maxima_tma(const MaxTmaArgs& A, int nzb, cudaStream_t st) {
  switch (A.ma.w) {
#define SNK_MT(WW) case WW: return launch_maxima_tma<WW>(A, nzb, st);
    SNK_MT(1) SNK_MT(2) SNK_MT(3) SNK_MT(4) SNK_MT(5) SNK_MT(6) SNK_MT(7) SNK_MT(8)
#undef SNK_MT
  }
  return fail(SNK_INTERNAL, "maxima_tma: window must be 1..8");
}

bool vec_ok(const snk_grid* g, const snk_params* p) {
  return g->n[0] % 8 == 0 && p->seed_window >= 0 && p->seed_window <= 8;
}

size_t vec_ws(const snk_grid* g) {
  const int64_t nvox = g->n[0] * g->n[1] * g->nz_buf;
  const int64_t nown = g->n[0] * g->n[1] * std::max<int64_t>(g->own_z1 - g->own_z0, 0);
  const int64_t nw = ceil_div(std::max<int64_t>(nown, 1), 32);
  const int64_t nb = ceil_div(nw, 1024);
  return 2 * ((size_t)nvox * sizeof(uint16_t) + 256) + (size_t)nw * 4 + 256 + (size_t)nb * sizeof(int) +
         256 + (size_t)(nb + 1) * sizeof(int64_t) + 256 + scan_ws(nb) + 1024;
}

bool fused_ok(const snk_grid* g, const snk_params* p) {
  return (g->dim == 2 && p->seed_window <= 32) || (g->dim == 3 && p->seed_window >= 1 && p->seed_window <= 8);
}

int64_t fused_words(const snk_grid* g) {
  return ceil_div(g->n[0], 32) * g->n[1] * std::max<int64_t>(g->own_z1 - g->own_z0, 0);
}

}  // namespace

size_t seeds_ws(const snk_grid* g, const snk_params* p) {
  if (p->seed_mode != SNK_SEED_MAXIMA) return 0;
  const size_t vws = vec_ok(g, p) ? vec_ws(g) : 0;
  if (fused_ok(g, p)) {
    const int64_t nw = fused_words(g);
    const int64_t nb = ceil_div(std::max<int64_t>(nw, 1), 1024);
    return std::max(vws, (size_t)nw * 4 + 256 + (size_t)nb * sizeof(int) + 256 +
                             (size_t)(nb + 1) * sizeof(int64_t) + 256 + scan_ws(nb) + 1024);
  }
  const int64_t nvox = g->n[0] * g->n[1] * g->nz_buf;
  const int64_t nown = g->n[0] * g->n[1] * (g->own_z1 - g->own_z0);
  const int64_t nb = ceil_div(std::max<int64_t>(nown, 1), kChunk);
  return 2 * ((size_t)nvox * sizeof(uint16_t) + 256) + (size_t)nb * sizeof(int) +
         (size_t)(nb + 1) * sizeof(int64_t) + scan_ws(nb) + 1024;
}

int32_t seeds_impl(const snk_grid* g, const snk_params* p, const uint16_t* d_smooth,
                   float* d_seeds, int64_t cap, int64_t* n_out, int64_t* first_id,
                   void* d_ws, size_t ws_bytes, cudaStream_t st) {
  const int dim = g->dim;
  if (first_id) *first_id = 0;
  if (p->seed_mode == SNK_SEED_LATTICE) {
    // §8(c) O4: m = r0 + dR/2, s = sqrt(1.5) r0, k = floor((L - 2m)/s) + 1,
    // o = m + ((L - 2m) - (k - 1) s)/2 per axis (L = n - 1).
    // (host code is compiled with -ffp-contract=off: every operation rounds as written)
    const double r0 = p->r0;
    const double m = r0 + p->delta_R / 2.0;
    const double s = std::sqrt(1.5) * r0;
    int64_t k[3] = {1, 1, 1};
    double o[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) {
      // physical extent (n - 1) scale (G28; scale 1 unless anisotropic)
      const double span = (double)(g->n[a] - 1) * grid_scale(g, a) - 2.0 * m;
      if (span < 0.0) {
        *n_out = 0;
        return fail(SNK_EMPTY_DOMAIN, "the lattice footprint does not fit the volume");
      }
      k[a] = (int64_t)std::floor(span / s) + 1;
      const double kk = (double)(k[a] - 1) * s;
      o[a] = m + (span - kk) / 2.0;
    }
    // lattice planes whose z lies in [own_z0, own_z1)
    int64_t iz0 = 0, iz1 = k[2];
    if (dim == 3) {
      iz0 = k[2];
      iz1 = 0;
      for (int64_t iz = 0; iz < k[2]; ++iz) {
        const double zpos = (double)(float)(o[2] + (double)iz * s) / grid_scale(g, 2);   // raw plane units
        if (zpos >= (double)g->own_z0 && zpos < (double)g->own_z1) {
          iz0 = std::min(iz0, iz);
          iz1 = std::max(iz1, iz + 1);
        }
      }
      if (iz1 < iz0) iz1 = iz0;
    }
    const int64_t cnt = k[0] * k[1] * (iz1 - iz0);
    *n_out = cnt;
    if (first_id) *first_id = iz0 * k[0] * k[1];
    if (cnt > cap) return fail(SNK_CAPACITY, "seed buffer too small");
    if (cnt > 0) {
      lattice_kernel<<<(unsigned)ceil_div(cnt, 256), 256, 0, st>>>(k[0], k[1], iz0, iz1 - iz0, o[0],
                                                                    o[1], o[2], s, dim, d_seeds);
      SNK_LAUNCH_CHECK("lattice_kernel");
    }
    SNK_CUDA_CHECK(cudaStreamSynchronize(st));
    return SNK_OK;
  }
  // MAXIMA
  const int nx = (int)g->n[0], ny = (int)g->n[1], nzb = (int)g->nz_buf;
  const int w = p->seed_window;
  // per-axis half-windows (anisotropic grids, G28)
  const int wx = axis_window(g, w, 0), wy = axis_window(g, w, 1), wz = dim == 3 ? axis_window(g, w, 2) : 0;
  if (dim == 3) {
    const int64_t need_lo = std::max<int64_t>(g->own_z0 - wz, 0);
    const int64_t need_hi = std::min<int64_t>(g->own_z1 - 1 + wz, g->n[2] - 1);
    if (g->own_z1 > g->own_z0 && (need_lo < g->z_lo || need_hi >= g->z_lo + g->nz_buf))
      return fail(SNK_SHAPE, "slab halo thinner than the seed window");
  }
  const int64_t plane = (int64_t)nx * ny;
  const int64_t nvox = plane * nzb;
  const bool vec = vec_ok(g, p) && ws_bytes >= vec_ws(g) && vec8_ok(g, d_smooth, nullptr, nullptr) &&
                   wx <= 8 && wy <= 8 && wz <= 8;
  if (grid_aniso(g) && !vec)
    return fail(SNK_SHAPE, "anisotropic MAXIMA needs the vectorised path (x % 8 == 0, 16-byte aligned, windows <= 8)");
  if (vec) {
    if (g->own_z1 <= g->own_z0) {
      *n_out = 0;
      return SNK_OK;
    }
    Carve cv(d_ws, ws_bytes);
    uint16_t* ta = cv.take<uint16_t>(nvox);
    uint16_t* tb = cv.take<uint16_t>(nvox);
    const int64_t nown = plane * (g->own_z1 - g->own_z0);
    const int64_t nw = ceil_div(nown, 32);
    const int64_t nbw = ceil_div(nw, 1024);
    uint32_t* bits = cv.take<uint32_t>(nw);
    int* wcounts = cv.take<int>(nbw);
    int64_t* woff = cv.take<int64_t>(nbw + 1);
    void* stmp = cv.take<char>(scan_ws(nbw));
    if (cv.overflow) return fail(SNK_CAPACITY, "workspace too small for seeds");
    // x / y box max only over the planes the z window touches
    const int64_t zb0 = dim == 3 ? std::max<int64_t>(g->own_z0 - wz, 0) - g->z_lo : g->own_z0 - g->z_lo;
    const int64_t zb1 = dim == 3 ? std::min<int64_t>(g->own_z1 - 1 + wz, g->n[2] - 1) - g->z_lo + 1
                                 : g->own_z1 - g->z_lo;
    const int nzp = (int)(zb1 - zb0);
    // x / y / z box-max passes + the predicate; SNK_TMA_MAXIMA=1: the one-pass TMA
    // kernel (isotropic 3D; 4.7 instead of ~25 GB of DRAM traffic on C4, but
    // latency-bound at 28% issue: 7.96 vs 7.69 ms, profiles/r2_volume.md)
    const char* tma_env = getenv("SNK_TMA_MAXIMA");
    const bool tma_pass = maxima_tma_ok(g, p, d_smooth) && tma_env && tma_env[0] == '1';
    if (!tma_pass) {
      SNK_TRY(sep_pass(0, 1, wx, d_smooth + zb0 * plane, ta + zb0 * plane, nx, ny, nzp, 0, nx - 1, st));
      SNK_TRY(sep_pass(1, 1, wy, ta + zb0 * plane, tb + zb0 * plane, nx, ny, nzp, 0, ny - 1, st));
    }
    // 3D: the z box-max as its own column-streamed pass into ta (every plane of
    // the window read ~once from HBM), then the predicate reads B and M once;
    // the flat fold of 2w+1 XY planes re-read them through L2 (43 GB per C4 step)
    const bool zpass = !tma_pass && dim == 3 && wz > 0 && nzp > 32;
    if (zpass) SNK_TRY(sep_pass(2, 1, wz, tb + zb0 * plane, ta + zb0 * plane, nx, ny, nzp, 0, nzp - 1, st));
    SNK_CUDA_CHECK(cudaMemsetAsync(bits + nw - 1, 0, sizeof(uint32_t), st));
    MaxArgs A;
    A.B = d_smooth;
    A.M = tb;
    A.nx = nx;
    A.ny = ny;
    A.nz_glob = (int)g->n[2];
    A.z_lo = (int)g->z_lo;
    A.w = w;
    A.wx = wx;
    A.wy = wy;
    A.wz = wz;
    A.dim = dim;
    A.thr = p->seed_threshold;
    A.v0 = A.v1 = 0;
    const int64_t ng = nown / 8;
    uint8_t* mask = reinterpret_cast<uint8_t*>(bits);
    const dim3 grid((unsigned)ceil_div(nx / 8, 256), (unsigned)ny, (unsigned)(g->own_z1 - g->own_z0));
    const int oz = (int)g->own_z0;
    if (tma_pass) {
      MaxTmaArgs T;
      T.ma = A;
      T.mask = mask;
      T.own_z0 = (int)g->own_z0;
      T.own_z1 = (int)g->own_z1;
      // z chunk: long chunks (less z-halo re-reading) unless the grid would not fill the GPU
      const int64_t cols = ceil_div(nx, kQX) * ceil_div(ny, kQY);
      T.zc = 128;
      while (T.zc > 16 && cols * ceil_div(g->own_z1 - g->own_z0, T.zc) < 1024) T.zc /= 2;
      SNK_TRY(maxima_tma(T, nzb, st));
    } else if (dim == 2) {
      maxima_pred8_kernel<2, 0><<<grid, 256, 0, st>>>(A, tb, mask, ng, oz);
    } else {
      if (zpass) {
        maxima_pred8_kernel<3, 0><<<grid, 256, 0, st>>>(A, ta, mask, ng, oz);   // M = ta
      } else switch (wz) {
#define SNK_PRED_CASE(WW) \
        case WW: maxima_pred8_kernel<3, WW><<<grid, 256, 0, st>>>(A, tb, mask, ng, oz); break;
        SNK_PRED_CASE(0) SNK_PRED_CASE(1) SNK_PRED_CASE(2) SNK_PRED_CASE(3) SNK_PRED_CASE(4)
        SNK_PRED_CASE(5) SNK_PRED_CASE(6) SNK_PRED_CASE(7) SNK_PRED_CASE(8)
#undef SNK_PRED_CASE
      }
    }
    if (!tma_pass) SNK_LAUNCH_CHECK("maxima_pred8_kernel");
    bits_count_kernel<<<(unsigned)nbw, kBitsThreads, 0, st>>>(bits, nw, wcounts);
    SNK_LAUNCH_CHECK("bits_count_kernel");
    SNK_TRY(scan_counts(wcounts, nbw, woff, st, stmp));
    bits_write_kernel<<<(unsigned)nbw, kBitsThreads, 0, st>>>(bits, nw, 0, nx, ny, oz, woff, d_seeds, cap, 1,
                                                      grid_scale(g, 0), grid_scale(g, 1), grid_scale(g, 2));
    SNK_LAUNCH_CHECK("bits_write_kernel");
    int64_t total = 0;
    SNK_TRY(read_back(woff + nbw, &total, sizeof(int64_t), st));
    *n_out = total;
    if (total > cap) return fail(SNK_CAPACITY, "seed buffer too small");
    return SNK_OK;
  }
  Carve cv(d_ws, ws_bytes);
  if (fused_ok(g, p)) {
    if (g->own_z1 <= g->own_z0) {
      *n_out = 0;
      return SNK_OK;
    }
    const int64_t nw = fused_words(g);
    const int64_t nbw = ceil_div(nw, 1024);
    uint32_t* bits = cv.take<uint32_t>(nw);
    int* wcounts = cv.take<int>(nbw);
    int64_t* woff = cv.take<int64_t>(nbw + 1);
    void* stmp = cv.take<char>(scan_ws(nbw));
    if (cv.overflow) return fail(SNK_CAPACITY, "workspace too small for seeds");
    FusedArgs F;
    F.B = d_smooth;
    F.bits = bits;
    F.nx = nx;
    F.ny = ny;
    F.nzg = (int)g->n[2];
    F.z_lo = (int)g->z_lo;
    F.own_z0 = (int)g->own_z0;
    F.own_z1 = (int)g->own_z1;
    F.wpr = (int)ceil_div(nx, 32);
    F.w = w;
    F.thr = p->seed_threshold;
    F.ma.B = d_smooth;
    F.ma.M = nullptr;
    F.ma.nx = nx;
    F.ma.ny = ny;
    F.ma.nz_glob = (int)g->n[2];
    F.ma.z_lo = (int)g->z_lo;
    F.ma.w = F.ma.wx = F.ma.wy = F.ma.wz = w;
    F.ma.dim = dim;
    F.ma.thr = p->seed_threshold;
    const int RX = kMX + 2 * w, RY = kMY + 2 * w;
    const size_t smem = (size_t)(RY * RX + RY * kMX) * sizeof(uint16_t);
    dim3 grid((unsigned)ceil_div(nx, kMX), (unsigned)ceil_div(ny, kMY),
              dim == 3 ? (unsigned)ceil_div(g->own_z1 - g->own_z0, kMZC) : 1u);
    if (dim == 2) {
      maxima_fused_kernel<2, 0><<<grid, kMThreads, smem, st>>>(F);
    } else {
      switch (w) {
        case 1: maxima_fused_kernel<3, 1><<<grid, kMThreads, smem, st>>>(F); break;
        case 2: maxima_fused_kernel<3, 2><<<grid, kMThreads, smem, st>>>(F); break;
        case 3: maxima_fused_kernel<3, 3><<<grid, kMThreads, smem, st>>>(F); break;
        case 4: maxima_fused_kernel<3, 4><<<grid, kMThreads, smem, st>>>(F); break;
        case 5: maxima_fused_kernel<3, 5><<<grid, kMThreads, smem, st>>>(F); break;
        case 6: maxima_fused_kernel<3, 6><<<grid, kMThreads, smem, st>>>(F); break;
        case 7: maxima_fused_kernel<3, 7><<<grid, kMThreads, smem, st>>>(F); break;
        default: maxima_fused_kernel<3, 8><<<grid, kMThreads, smem, st>>>(F); break;
      }
    }
    SNK_LAUNCH_CHECK("maxima_fused_kernel");
    bits_count_kernel<<<(unsigned)nbw, kBitsThreads, 0, st>>>(bits, nw, wcounts);
    SNK_LAUNCH_CHECK("bits_count_kernel");
    SNK_TRY(scan_counts(wcounts, nbw, woff, st, stmp));
    bits_write_kernel<<<(unsigned)nbw, kBitsThreads, 0, st>>>(bits, nw, F.wpr, nx, ny, F.own_z0, woff, d_seeds, cap, 0);
    SNK_LAUNCH_CHECK("bits_write_kernel");
    int64_t total = 0;
    SNK_TRY(read_back(woff + nbw, &total, sizeof(int64_t), st));
    *n_out = total;
    if (total > cap) return fail(SNK_CAPACITY, "seed buffer too small");
    return SNK_OK;
  }
  uint16_t* ta = cv.take<uint16_t>(nvox);
  uint16_t* tb = cv.take<uint16_t>(nvox);
  const int64_t v0 = (g->own_z0 - g->z_lo) * plane, v1 = (g->own_z1 - g->z_lo) * plane;
  const int64_t nb = ceil_div(std::max<int64_t>(v1 - v0, 1), kChunk);
  int* counts = cv.take<int>(nb);
  int64_t* offsets = cv.take<int64_t>(nb + 1);
  void* stmp = cv.take<char>(scan_ws(nb));
  if (cv.overflow) return fail(SNK_CAPACITY, "workspace too small for seeds");
  const unsigned grid = (unsigned)ceil_div(nvox, 256);
  // window clipped to the volume; z additionally to the buffer (only own planes are used)
  const int zlo_valid = 0, zhi_valid = nzb - 1;
  boxmax_kernel<0><<<grid, 256, 0, st>>>(d_smooth, ta, nx, ny, nzb, w, zlo_valid, zhi_valid);
  SNK_LAUNCH_CHECK("boxmax_kernel<x>");
  const uint16_t* M = ta;
  boxmax_kernel<1><<<grid, 256, 0, st>>>(ta, tb, nx, ny, nzb, w, zlo_valid, zhi_valid);
  SNK_LAUNCH_CHECK("boxmax_kernel<y>");
  M = tb;
  if (dim == 3) {
    boxmax_kernel<2><<<grid, 256, 0, st>>>(tb, ta, nx, ny, nzb, w, zlo_valid, zhi_valid);
    SNK_LAUNCH_CHECK("boxmax_kernel<z>");
    M = ta;
  }
  MaxArgs A;
  A.B = d_smooth;
  A.M = M;
  A.nx = nx;
  A.ny = ny;
  A.nz_glob = (int)g->n[2];
  A.z_lo = (int)g->z_lo;
  A.w = A.wx = A.wy = A.wz = w;
  A.dim = dim;
  A.thr = p->seed_threshold;
  A.v0 = v0;
  A.v1 = v1;
  if (v1 <= v0) {
    *n_out = 0;
    return SNK_OK;
  }
  maxima_count_kernel<<<(unsigned)nb, kCompactThreads, 0, st>>>(A, counts);
  SNK_LAUNCH_CHECK("maxima_count_kernel");
  SNK_TRY(scan_counts(counts, nb, offsets, st, stmp));
  maxima_write_kernel<<<(unsigned)nb, kCompactThreads, 0, st>>>(A, offsets, d_seeds, cap);
  SNK_LAUNCH_CHECK("maxima_write_kernel");
  int64_t total = 0;
  SNK_TRY(read_back(offsets + nb, &total, sizeof(int64_t), st));
  *n_out = total;
  if (total > cap) return fail(SNK_CAPACITY, "seed buffer too small");
  return SNK_OK;
}

}  // namespace snk
