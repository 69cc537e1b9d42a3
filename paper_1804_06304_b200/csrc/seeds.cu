// seeds.cu — a4 seed placement (include/snk.h snk_seeds).
//   LATTICE: the paper's lattice, spacing sqrt(1.5) r0, centred
//            (S:101), positions in IEEE double without contraction then fp32.
//   MAXIMA:  first maxima of the (2w+1)^d box above a threshold (G20):
//            separable box-max (3 u16 passes) -> candidate test B == M, B >= thr
//            -> tie check (no equal value earlier in linear order inside the
//            window, only for candidates) -> order-preserving compaction.
// Integer-exact; bit-identical to the definition.
#include <cmath>

#include "common.cuh"

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

}  // namespace

size_t seeds_ws(const snk_grid* g, const snk_params* p) {
  if (p->seed_mode != SNK_SEED_MAXIMA) return 0;
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
      const double span = (double)(g->n[a] - 1) - 2.0 * m;
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
        const double zpos = (double)(float)(o[2] + (double)iz * s);
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
  if (dim == 3) {
    const int64_t need_lo = std::max<int64_t>(g->own_z0 - w, 0);
    const int64_t need_hi = std::min<int64_t>(g->own_z1 - 1 + w, g->n[2] - 1);
    if (g->own_z1 > g->own_z0 && (need_lo < g->z_lo || need_hi >= g->z_lo + g->nz_buf))
      return fail(SNK_SHAPE, "slab halo thinner than the seed window");
  }
  const int64_t plane = (int64_t)nx * ny;
  const int64_t nvox = plane * nzb;
  Carve cv(d_ws, ws_bytes);
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
  A.w = w;
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
  SNK_CUDA_CHECK(cudaMemcpyAsync(&total, offsets + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SNK_CUDA_CHECK(cudaStreamSynchronize(st));
  *n_out = total;
  if (total > cap) return fail(SNK_CAPACITY, "seed buffer too small");
  return SNK_OK;
}

}  // namespace snk
