// label.cu — a8: the voxel label map (north_star "voxel label map out";
// reading G19).  Voxel x gets 1 + the index of the detection whose inner ball
// (radius rho R, the nucleus at the Eq. 3 optimum) contains it with
// the smallest normalised key d2/thr, ties to the smaller index; 0 if none.
// The decisions are those of IEEE fp64 with explicit _rn intrinsics (no
// contraction): an fp32 filter with a proven margin settles membership, fp64
// the rest, so the map is bit-identical to the definition.
//
// Mapping: detections are binned onto 32x8x8-voxel tiles (2D: 32x32) by the
// bounding box of their inner ball; one CTA (256 threads) per tile stages the
// tile's list in shared memory; thread (x, y) walks the tile's 8 z-planes,
// re-using dx^2 + dy^2 across planes.  Each warp stores 32 consecutive int32
// (128 B) per plane: the output is streamed once (4 B/voxel, HBM-bound).
#include <cmath>

#include "common.cuh"

namespace snk {

namespace {

constexpr int kTX = 32, kTY = 8, kTY2 = 32, kThreads = 256;
#ifndef SNK_LABEL_TZ
#define SNK_LABEL_TZ 8
#endif
constexpr int kTZ3 = SNK_LABEL_TZ;   // tile depth: voxels per thread (3D)
constexpr int kStage = 256;

struct TileGrid {
  int tx, ty, tz;      // tile dims (voxels)
  int nt[3];           // tiles per axis over the owned region
  int nx, ny;
  int z0, z1;          // owned planes [z0, z1)
  double rho2;         // rho^2 (G19)
  double rho;          // bbox radius factor
  double sc[3];        // physical voxel size per axis (G28; 1 isotropic)
  float scf[3];        // the same in fp32 (the fp32 filter)
  double band;         // relative half-width of the fp32 filter's uncertain band
};

__device__ __forceinline__ bool tile_range(const snk_cell& d, const TileGrid& G, int lo[3], int hi[3]) {
  const float c[3] = {d.c[0], d.c[1], d.c[2]};
  // inner-ball radius with a small safety margin for the fp32 bbox
  const double r = G.rho * (double)d.R * 1.000001 + 1e-4;
  const int n[3] = {G.nx, G.ny, G.z1};
  const int base[3] = {0, 0, G.z0};
  const int tdim[3] = {G.tx, G.ty, G.tz};
  for (int a = 0; a < 3; ++a) {
    // raw voxel range of the ball (physical c and r divided by the voxel size, G28)
    const int vlo = max((int)ceil(((double)c[a] - r) / G.sc[a]), base[a]);
    const int vhi = min((int)floor(((double)c[a] + r) / G.sc[a]), n[a] - 1);
    if (vlo > vhi) return false;
    lo[a] = (vlo - base[a]) / tdim[a];
    hi[a] = (vhi - base[a]) / tdim[a];
  }
  return true;
}

__global__ void tile_count_kernel(const snk_cell* __restrict__ dets, int64_t n, TileGrid G, int* counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo[3], hi[3];
  if (!tile_range(dets[i], G, lo, hi)) return;
  for (int z = lo[2]; z <= hi[2]; ++z)
    for (int y = lo[1]; y <= hi[1]; ++y)
      for (int x = lo[0]; x <= hi[0]; ++x)
        atomicAdd(&counts[((int64_t)z * G.nt[1] + y) * G.nt[0] + x], 1);
}

__global__ void tile_fill_kernel(const snk_cell* __restrict__ dets, int64_t n, TileGrid G,
                                 const int64_t* offsets, int* cursor, int* entries) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo[3], hi[3];
  if (!tile_range(dets[i], G, lo, hi)) return;
  for (int z = lo[2]; z <= hi[2]; ++z)
    for (int y = lo[1]; y <= hi[1]; ++y)
      for (int x = lo[0]; x <= hi[0]; ++x) {
        const int64_t t = ((int64_t)z * G.nt[1] + y) * G.nt[0] + x;
        entries[offsets[t] + atomicAdd(&cursor[t], 1)] = (int)i;
      }
}

// The exact O7 quantities of voxel (px, py, pz) against detection i (fp64, no
// contraction, the oracle's order): d2 = (dx^2 + dy^2) + dz^2 and key = d2 / thr.
__device__ __forceinline__ double exact_d2(double px, double py, double pz, const snk_cell& d) {
  const double dx = __dsub_rn(px, (double)d.c[0]), dy = __dsub_rn(py, (double)d.c[1]);
  const double dz = __dsub_rn(pz, (double)d.c[2]);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}
__device__ __forceinline__ double exact_thr(const snk_cell& d, double rho2) {
  return __dmul_rn(__dmul_rn((double)d.R, (double)d.R), rho2);
}

// One tile's staged detection data (shared memory), filled from registers.
struct Stage {
  float c[3][kStage];
  float lo[kStage], hi[kStage];
  int idx[kStage];
};

// Registers of thread k's share of a tile list (k < count): loaded one tile
// ahead, so the dependent loads (entries -> records) overlap the current tile.
struct Prefetch {
  int cnt;
  int i;
  float c[3], lo, hi;
};

__device__ __forceinline__ void prefetch_tile(Prefetch& f, const snk_cell* __restrict__ dets, const TileGrid& G,
                                              const int64_t* __restrict__ offsets, const int* __restrict__ entries,
                                              int64_t tile) {
  const int64_t e0 = offsets[tile], e1 = offsets[tile + 1];
  f.cnt = (int)(e1 - e0);
  if ((int)threadIdx.x < min(f.cnt, kStage)) {
    f.i = entries[e0 + threadIdx.x];
    const snk_cell d = dets[f.i];
    f.c[0] = d.c[0];
    f.c[1] = d.c[1];
    f.c[2] = d.c[2];
    const double thr = exact_thr(d, G.rho2);
    f.lo = (float)__dmul_rn(thr, 1.0 - G.band);
    f.hi = (float)__dmul_rn(thr, 1.0 + G.band);
  }
}

// The exact O7 rules for one (voxel, candidate) pair the fp32 filter could not
// settle (near a ball's boundary, or a second ball containing the voxel): rare,
// and called from one site.  Returns the new best index (the current best's key
// is recomputed rather than cached: second balls are rare).
__device__ __forceinline__ int label_exact(const snk_cell* __restrict__ dets, double px, double py, double pz,
                                          double rho2, int i, int best, float d2f, float lo) {
  if (!(d2f < lo)) {
    const snk_cell d = dets[i];
    if (!(exact_d2(px, py, pz, d) <= exact_thr(d, rho2))) return best;
  }
  if (best < 0) return i;
  const snk_cell b = dets[best];
  const double kb = __ddiv_rn(exact_d2(px, py, pz, b), exact_thr(b, rho2));
  const snk_cell d = dets[i];
  const double k = __ddiv_rn(exact_d2(px, py, pz, d), exact_thr(d, rho2));
  return (k < kb || (k == kb && i < best)) ? i : best;
}

// D = 3: tile 32 x 8 x kTZ3, thread (x, y) walks the tile's kTZ3 planes; a CTA
// takes kZT tiles along z (the next tile's list is prefetched into registers
// while the current one is evaluated).  D = 2: tile 32 x 32, a thread takes 4
// rows (y, y + 8, y + 16, y + 24).
//
// Membership d2 <= thr is decided in fp32 outside a relative band of 1e-5
// (anisotropic grids: 1e-3) around thr: d2f (fp32, FFMA) is within 1e-6
// (relative) of the exact d2 and thr_lo / thr_hi bracket thr by the band, so
// d2f > thr_hi implies d2 > thr and d2f < thr_lo implies d2 < thr; only pairs
// inside the band take the exact fp64 test (one call site, planes looped with
// the running bests in shared memory).  The key d2 / thr (fp64 division)
// is evaluated only when a voxel lies inside two or more inner balls — a lone
// candidate wins whatever its key — so the map equals the all-fp64 definition
// bit for bit.  The common case (every plane of the column certain, and first)
// is a branch-free select on bit masks.
constexpr int kZT = 4;

template <int D>
__global__ void __launch_bounds__(kThreads) label_kernel(const snk_cell* __restrict__ dets, TileGrid G,
                                                         const int64_t* __restrict__ offsets,
                                                         const int* __restrict__ entries,
                                                         int32_t* __restrict__ labels) {
  constexpr int NV = D == 3 ? kTZ3 : kTY2 / kTY;   // voxels per thread
  __shared__ Stage S[2];
  __shared__ int sbest[NV][kThreads];              // the exact path's running bests
  const int ntz = D == 3 ? G.nt[2] : 1;
  const int zgroups = D == 3 ? (ntz + kZT - 1) / kZT : 1;
  const int64_t col = blockIdx.x / zgroups;        // (tx, ty)
  const int tz0 = D == 3 ? (int)(blockIdx.x % zgroups) * kZT : 0;
  const int tz1 = D == 3 ? min(tz0 + kZT, ntz) : 1;
  const int tx = (int)(col % G.nt[0]), ty = (int)(col / G.nt[0]);
  const int lx = threadIdx.x % kTX, ly = threadIdx.x / kTX;
  const int x = tx * G.tx + lx;
  const int y0 = ty * G.ty + ly;                   // 3D: the thread's row; 2D: its first row
  const float pxf = __fmul_rn((float)x, G.scf[0]);
  const float pyf0 = __fmul_rn((float)y0, G.scf[1]);
  const int64_t plane = (int64_t)G.ny * G.nx;
  const int64_t vstep = D == 3 ? plane : (int64_t)kTY * G.nx;   // between a thread's voxels
  // the store stride in bytes, held in a register: left to itself the compiler
  // re-derives ny * nx for every plane's address (IMAD.WIDE + LEA + LEA.HI.X)
  int64_t vstep_b = vstep * (int64_t)sizeof(int32_t);
  asm("" : "+l"(vstep_b));
  auto tile_id = [&](int tz) { return ((int64_t)tz * G.nt[1] + ty) * G.nt[0] + tx; };
  Prefetch f;
  prefetch_tile(f, dets, G, offsets, entries, tile_id(tz0));
  for (int tz = tz0; tz < tz1; ++tz) {
    Stage& st = S[tz & 1];
    const int cnt = f.cnt;
    if ((int)threadIdx.x < min(cnt, kStage)) {
      st.c[0][threadIdx.x] = f.c[0];
      st.c[1][threadIdx.x] = f.c[1];
      st.c[2][threadIdx.x] = f.c[2];
      st.lo[threadIdx.x] = f.lo;
      st.hi[threadIdx.x] = f.hi;
      st.idx[threadIdx.x] = f.i;
    }
    __syncthreads();   // stage complete (the other stage was last read before this barrier's predecessor)
    if (tz + 1 < tz1) prefetch_tile(f, dets, G, offsets, entries, tile_id(tz + 1));
    const int zt = D == 3 ? G.z0 + tz * G.tz : G.z0;   // the tile's first plane (3D)
    float pvf[NV];   // per voxel: 3D its plane's z, 2D its row's y (the filter's fp32 positions)
#pragma unroll
    for (int v = 0; v < NV; ++v)
      pvf[v] = D == 3 ? __fmul_rn((float)(zt + v), G.scf[2]) : __fmul_rn((float)(y0 + v * kTY), G.scf[1]);
    int best[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) best[v] = -1;
    uint32_t has = 0;   // planes with a best
    for (int s0 = 0; s0 < cnt; s0 += kStage) {
      // lists longer than one stage (never on the throughput configs): re-stage synchronously
      const Stage* sp = &st;
      if (s0 > 0) {
        __syncthreads();
        const int64_t e0 = offsets[tile_id(tz)] + s0;
        const int m = cnt - s0 < kStage ? cnt - s0 : kStage;
        Stage& o = S[(tz + 1) & 1];   // free: its next use is the next tile (after a barrier)
        if ((int)threadIdx.x < m) {
          const int i = entries[e0 + threadIdx.x];
          const snk_cell d = dets[i];
          const double thr = exact_thr(d, G.rho2);
          o.c[0][threadIdx.x] = d.c[0];
          o.c[1][threadIdx.x] = d.c[1];
          o.c[2][threadIdx.x] = d.c[2];
          o.lo[threadIdx.x] = (float)__dmul_rn(thr, 1.0 - G.band);
          o.hi[threadIdx.x] = (float)__dmul_rn(thr, 1.0 + G.band);
          o.idx[threadIdx.x] = i;
        }
        __syncthreads();
        sp = &o;
      }
      const int m = cnt - s0 < kStage ? cnt - s0 : kStage;
      for (int k = 0; k < m; ++k) {
        const float hi = sp->hi[k], lo = sp->lo[k];
        const float dxf = __fsub_rn(pxf, sp->c[0][k]);
        float d2f[NV];
        if (D == 3) {
          const float dyf = __fsub_rn(pyf0, sp->c[1][k]);
          const float dxy = __fmaf_rn(dxf, dxf, __fmul_rn(dyf, dyf));
          if (dxy > hi) continue;   // dz^2 >= 0: no plane of this column can qualify
          const float cz = sp->c[2][k];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const float dzf = __fsub_rn(pvf[v], cz);
            d2f[v] = __fmaf_rn(dzf, dzf, dxy);
          }
        } else {
          const float cy = sp->c[1][k];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const float dyf = __fsub_rn(pvf[v], cy);
            d2f[v] = __fmaf_rn(dxf, dxf, __fmul_rn(dyf, dyf));
          }
        }
        uint32_t mhi = 0, mlo = 0;   // planes with d2f <= hi (maybe inside), d2f < lo (certainly inside)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          mhi |= (uint32_t)(d2f[v] <= hi) << v;
          mlo |= (uint32_t)(d2f[v] < lo) << v;
        }
        const int i = sp->idx[k];
        if (!(mhi & (has | ~mlo))) {   // every maybe-inside plane is certain and first
#pragma unroll
          for (int v = 0; v < NV; ++v) best[v] = (mlo >> v) & 1u ? i : best[v];
          has |= mlo;
        } else {
#pragma unroll
          for (int v = 0; v < NV; ++v) sbest[v][threadIdx.x] = best[v];
          const double px = __dmul_rn((double)x, G.sc[0]);
#pragma unroll 1
          for (int v = 0; v < NV; ++v) {
            if (!((mhi >> v) & 1u)) continue;
            float dv = d2f[0];
#pragma unroll
            for (int u = 1; u < NV; ++u) dv = u == v ? d2f[u] : dv;
            const double py = D == 3 ? __dmul_rn((double)y0, G.sc[1]) : __dmul_rn((double)(y0 + v * kTY), G.sc[1]);
            const double pz = D == 3 ? __dmul_rn((double)(zt + v), G.sc[2]) : 0.0;
            sbest[v][threadIdx.x] = label_exact(dets, px, py, pz, G.rho2, i, sbest[v][threadIdx.x], dv, lo);
          }
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            best[v] = sbest[v][threadIdx.x];
            has |= (uint32_t)(best[v] >= 0) << v;
          }
        }
      }
    }
    if (cnt > kStage) __syncthreads();   // the re-staged buffer is the next tile's stage
    if (x < G.nx) {
      char* dst = reinterpret_cast<char*>(labels + ((int64_t)(zt - G.z0) * G.ny + y0) * G.nx + x);
      const int nv = D == 3 ? min(NV, G.z1 - zt) : min(NV, (G.ny - y0 + kTY - 1) / kTY);
      if (D == 3 && y0 >= G.ny) continue;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (v < nv) *reinterpret_cast<int32_t*>(dst) = best[v] + 1;
        dst += vstep_b;
      }
    }
  }
}

TileGrid make_grid(const snk_grid* g) {
  TileGrid G;
  if (g->dim == 3) { G.tx = kTX; G.ty = kTY; G.tz = kTZ3; }
  else { G.tx = kTX; G.ty = kTY2; G.tz = 1; }
  G.nx = (int)g->n[0];
  G.ny = (int)g->n[1];
  G.z0 = (int)g->own_z0;
  G.z1 = (int)g->own_z1;
  G.nt[0] = (int)ceil_div(G.nx, G.tx);
  G.nt[1] = (int)ceil_div(G.ny, G.ty);
  G.nt[2] = (int)ceil_div(std::max(G.z1 - G.z0, 0), G.tz);
  G.rho2 = g->dim == 3 ? kRhoSq3 : kRhoSq2;
  G.rho = rho_of(g->dim);
  for (int a = 0; a < 3; ++a) {
    G.sc[a] = grid_scale(g, a);
    G.scf[a] = (float)G.sc[a];
  }
  // isotropic: fp32 positions are exact integers and d2f is within 1e-6 of d2;
  // physical positions x * scale round in fp32 (1e-4 voxel at x ~ 1000)
  G.band = grid_aniso(g) ? 1e-3 : 1e-5;
  return G;
}

size_t tiles_per_det_bound(const snk_grid* g, const snk_params* p, const TileGrid& G) {
  const double r = G.rho * std::max(p->r_max, p->r0) * 1.000001 + 1e-4;
  size_t b = 1;
  const int td[3] = {G.tx, G.ty, G.tz};
  for (int a = 0; a < g->dim; ++a) b *= (size_t)(std::floor(2 * r / (td[a] * grid_scale(g, a))) + 2);
  return b;
}

}  // namespace

size_t label_ws(const snk_grid* g, const snk_params* p, int64_t max_cells) {
  const TileGrid G = make_grid(g);
  const size_t ntiles = (size_t)G.nt[0] * G.nt[1] * std::max(G.nt[2], 1);
  const size_t ent = (size_t)std::max<int64_t>(max_cells, 1) * tiles_per_det_bound(g, p, G);
  return ntiles * (2 * sizeof(int) + sizeof(int64_t)) + sizeof(int64_t) + ent * sizeof(int) +
         scan_ws((int64_t)ntiles) + 4096;
}

int32_t label_impl(const snk_grid* g, const snk_params* p, const snk_cell* d_dets, int64_t n,
                   int32_t* d_labels, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  const TileGrid G = make_grid(g);
  if (G.z1 <= G.z0) return SNK_OK;
  const int64_t ntiles = (int64_t)G.nt[0] * G.nt[1] * G.nt[2];
  Carve cv(d_ws, ws_bytes);
  int* counts = cv.take<int>(ntiles);
  int* cursor = cv.take<int>(ntiles);
  int64_t* offsets = cv.take<int64_t>(ntiles + 1);
  void* stmp = cv.take<char>(scan_ws(ntiles));
  const size_t ent_cap = (size_t)std::max<int64_t>(n, 1) * tiles_per_det_bound(g, p, G);
  int* entries = cv.take<int>(ent_cap);
  if (cv.overflow || !d_ws) return fail(SNK_CAPACITY, "workspace too small for label");
  SNK_CUDA_CHECK(cudaMemsetAsync(counts, 0, ntiles * sizeof(int), st));
  SNK_CUDA_CHECK(cudaMemsetAsync(cursor, 0, ntiles * sizeof(int), st));
  if (n > 0) {
    tile_count_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d_dets, n, G, counts);
    SNK_LAUNCH_CHECK("tile_count_kernel");
  }
  SNK_TRY(scan_counts(counts, ntiles, offsets, st, stmp));
  int64_t total = 0;
  SNK_TRY(read_back(offsets + ntiles, &total, sizeof total, st));
  if ((size_t)total > ent_cap) return fail(SNK_CAPACITY, "detection radii exceed r_max: tile lists overflow");
  if (n > 0) {
    tile_fill_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d_dets, n, G, offsets, cursor, entries);
    SNK_LAUNCH_CHECK("tile_fill_kernel");
  }
  // 3D: one CTA per column of kZT tiles along z
  const int64_t nblk = g->dim == 3 ? (int64_t)G.nt[0] * G.nt[1] * ceil_div(G.nt[2], kZT) : ntiles;
  if (g->dim == 3) label_kernel<3><<<(unsigned)nblk, kThreads, 0, st>>>(d_dets, G, offsets, entries, d_labels);
  else label_kernel<2><<<(unsigned)nblk, kThreads, 0, st>>>(d_dets, G, offsets, entries, d_labels);
  SNK_LAUNCH_CHECK("label_kernel");
  return SNK_OK;
}

}  // namespace snk
