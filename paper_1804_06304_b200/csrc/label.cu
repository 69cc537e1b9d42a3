// label.cu — a8: the voxel label map (north_star "voxel label map out";
// reading G19).  Voxel x gets 1 + the index of the detection whose inner ball
// (radius rho R, the nucleus at the Eq. 3 optimum) contains it with
// the smallest normalised key d2/thr, ties to the smaller index; 0 if none.
// Arithmetic is IEEE fp64 with explicit _rn intrinsics (no contraction), so the
// map is bit-identical to the definition.
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

constexpr int kTX = 32, kTY = 8, kTZ3 = 8, kTY2 = 32, kThreads = 256;
constexpr int kStage = 256;

struct TileGrid {
  int tx, ty, tz;      // tile dims (voxels)
  int nt[3];           // tiles per axis over the owned region
  int nx, ny;
  int z0, z1;          // owned planes [z0, z1)
  double rho2;         // rho^2 (G19)
  double rho;          // bbox radius factor
  double sc[3];        // physical voxel size per axis (G28; 1 isotropic)
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

// D = 3: tile 32x8x8, thread (x, y) walks 8 planes.  D = 2: tile 32x32x1, thread
// handles 4 rows (y, y+8, y+16, y+24).
template <int D>
__global__ void __launch_bounds__(kThreads) label_kernel(const snk_cell* __restrict__ dets, TileGrid G,
                                                         const int64_t* __restrict__ offsets,
                                                         const int* __restrict__ entries,
                                                         int32_t* __restrict__ labels) {
  constexpr int NV = D == 3 ? kTZ3 : kTY2 / kTY;   // voxels per thread
  __shared__ double s_c[3][kStage];
  __shared__ double s_thr[kStage];
  __shared__ int s_idx[kStage];
  const int64_t tile = blockIdx.x;
  const int tx = (int)(tile % G.nt[0]), ty = (int)((tile / G.nt[0]) % G.nt[1]),
            tz = (int)(tile / ((int64_t)G.nt[0] * G.nt[1]));
  const int lx = threadIdx.x % kTX, ly = threadIdx.x / kTX;
  const int x = tx * G.tx + lx;
  int yv[NV], zv[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    yv[k] = D == 3 ? ty * G.ty + ly : ty * G.ty + ly + k * kTY;
    zv[k] = D == 3 ? G.z0 + tz * G.tz + k : G.z0;
  }
  int best[NV];
  double best_key[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) { best[k] = -1; best_key[k] = 0.0; }
  const double px = __dmul_rn((double)x, G.sc[0]);   // physical voxel position (G28; exact for scale 1)
  const int64_t e0 = offsets[tile], e1 = offsets[tile + 1];
  for (int64_t s = e0; s < e1; s += kStage) {
    const int cnt = (int)(e1 - s < kStage ? e1 - s : kStage);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
      const int i = entries[s + k];
      const snk_cell d = dets[i];
      s_c[0][k] = (double)d.c[0];
      s_c[1][k] = (double)d.c[1];
      s_c[2][k] = (double)d.c[2];
      s_thr[k] = __dmul_rn(__dmul_rn((double)d.R, (double)d.R), G.rho2);
      s_idx[k] = i;
    }
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      const double thr = s_thr[k];
      const int i = s_idx[k];
      const double dx = __dsub_rn(px, s_c[0][k]);
      const double dx2 = __dmul_rn(dx, dx);
      if (D == 3) {
        const double dy = __dsub_rn(__dmul_rn((double)yv[0], G.sc[1]), s_c[1][k]);
        const double dxy = __dadd_rn(dx2, __dmul_rn(dy, dy));   // d2 = (dx^2 + dy^2) + dz^2
        if (!(dxy <= thr)) continue;                             // dz^2 >= 0: no plane can qualify
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double dz = __dsub_rn(__dmul_rn((double)zv[v], G.sc[2]), s_c[2][k]);
          const double d2 = __dadd_rn(dxy, __dmul_rn(dz, dz));
          if (d2 <= thr) {
            const double key = __ddiv_rn(d2, thr);
            if (best[v] < 0 || key < best_key[v] || (key == best_key[v] && i < best[v])) {
              best[v] = i;
              best_key[v] = key;
            }
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double dy = __dsub_rn(__dmul_rn((double)yv[v], G.sc[1]), s_c[1][k]);
          const double d2 = __dadd_rn(dx2, __dmul_rn(dy, dy));
          if (d2 <= thr) {
            const double key = __ddiv_rn(d2, thr);
            if (best[v] < 0 || key < best_key[v] || (key == best_key[v] && i < best[v])) {
              best[v] = i;
              best_key[v] = key;
            }
          }
        }
      }
    }
  }
  if (x >= G.nx) return;
#pragma unroll
  for (int v = 0; v < NV; ++v)
    if (yv[v] < G.ny && zv[v] < G.z1)
      labels[((int64_t)(zv[v] - G.z0) * G.ny + yv[v]) * G.nx + x] = best[v] + 1;
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
  for (int a = 0; a < 3; ++a) G.sc[a] = grid_scale(g, a);
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
  if (g->dim == 3) label_kernel<3><<<(unsigned)ntiles, kThreads, 0, st>>>(d_dets, G, offsets, entries, d_labels);
  else label_kernel<2><<<(unsigned)ntiles, kThreads, 0, st>>>(d_dets, G, offsets, entries, d_labels);
  SNK_LAUNCH_CHECK("label_kernel");
  return SNK_OK;
}

}  // namespace snk
