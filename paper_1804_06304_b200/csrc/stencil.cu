// stencil.cu — the TMA-staged volume passes (BASELINE.json north_star
// subsystem (1): "TMA-staged separable 3D convolution in shared memory"):
//
//   blur_tma_kernel<D, H>   a2: the whole separable Q14 Gaussian (reading
//                           G18) in ONE pass over the volume: x, y and z passes
//                           each rounding (sum w_i v_i + 8192) >> 14 exactly as
//                           the three-pass definition (O2).
//
// Tiling.  A CTA owns a TX x TY column tile of the volume and walks a chunk of
// ZC planes.  Every input plane's (TX + 16) x (TY + 2H) box is copied by the
// Tensor Memory Accelerator (cp.async.bulk.tensor, one elected thread,
// completion on an mbarrier) into an NS-stage ring in shared memory, NS - 1
// planes ahead of the compute.  The box starts at x0 - 8: on this pool's GPUs
// a tensor load whose innermost start coordinate is not 16-byte aligned faults
// (profiles/r2_tma_probe.md).  Out-of-volume box elements arrive zero-filled;
// clamp-to-edge is restored in shared memory for tiles on the volume
// boundary, and z is clamped by choosing which plane to load.  The x pass
// (shared -> shared, u32), the y pass (shared -> a per-thread register ring of
// 2H + 1 planes) and the z pass (ring -> HBM, 16-byte stores) run per plane.
// Taps are symmetric (w_-i = w_i): H + 1 multiplies and H adds per output.
#include <cuda.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace snk {

namespace {

constexpr int kTX = 64, kTY = 32, kZC = 64, kNS = 4, kThreads = 256;
constexpr int kBX = kTX + 16;   // box row: x0 - 8 .. x0 + TX + 7 (16-byte aligned start, H <= 8)

struct StencilTaps {
  uint32_t w[9];   // w[0] = centre, w[i] = w_(+-i), i <= 8
};

__device__ __forceinline__ void unpack8(const uint4 q, uint32_t* v) {
  v[0] = q.x & 0xffffu; v[1] = q.x >> 16; v[2] = q.y & 0xffffu; v[3] = q.y >> 16;
  v[4] = q.z & 0xffffu; v[5] = q.z >> 16; v[6] = q.w & 0xffffu; v[7] = q.w >> 16;
}

// (w_0 v_0 + sum_i w_i (v_-i + v_i) + 8192) >> 14 for v = c[-H .. H]
template <int H>
__device__ __forceinline__ uint32_t q14(const StencilTaps& T, const uint32_t* c) {
  uint32_t acc = 8192u + T.w[0] * c[0];
#pragma unroll
  for (int i = 1; i <= H; ++i) acc += T.w[i] * (c[-i] + c[i]);
  return acc >> 14;
}

// Restore clamp-to-edge in a box whose rows/columns fall outside the volume
// (TMA filled them with zeros).  x first (every row), then whole rows in y.
template <int BY>
__device__ __forceinline__ void fix_edges(uint16_t* box, int x0, int y0, int H, int nx, int ny) {
  const int xb = x0 - 8, yb = y0 - H;
  const int cl = max(0, -xb), cr = min(kBX, nx - xb);   // columns [cl, cr) are inside
  if (cl > 0 || cr < kBX) {
    for (int e = threadIdx.x; e < BY * kBX; e += kThreads) {
      const int r = e / kBX, c = e % kBX;
      if (c < cl) box[r * kBX + c] = box[r * kBX + cl];
      else if (c >= cr) box[r * kBX + c] = box[r * kBX + cr - 1];
    }
    __syncthreads();
  }
  const int rl = max(0, -yb), rr = min(BY, ny - yb);
  if (rl > 0 || rr < BY) {
    for (int e = threadIdx.x; e < BY * kBX; e += kThreads) {
      const int r = e / kBX, c = e % kBX;
      if (r < rl) box[r * kBX + c] = box[rl * kBX + c];
      else if (r >= rr) box[r * kBX + c] = box[(rr - 1) * kBX + c];
    }
  }
}

template <int D, int H>
__global__ void __launch_bounds__(kThreads, H <= 5 ? 2 : 1) blur_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                                           uint16_t* __restrict__ out, int nx, int ny,
                                                                           int nz, const __grid_constant__ StencilTaps T) {
  constexpr int BY = kTY + 2 * H, K = 2 * H + 1;
  constexpr uint32_t kBoxBytes = kBX * BY * 2;
  constexpr uint32_t kStage = (kBoxBytes + 127) & ~127u;   // TMA destinations: 128-byte aligned
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem);                // [NS] x ([BY][BX] + pad): the TMA boxes
  uint32_t* sx = reinterpret_cast<uint32_t*>(smem + kNS * kStage);   // [BY][TX]: x-passed rows (u32: no unpacking)
  __shared__ __align__(8) uint64_t full[kNS];
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const int z0 = D == 3 ? blockIdx.z * kZC : 0;
  const int zend = D == 3 ? min(z0 + kZC, nz) : 1;
  const int nplanes = D == 3 ? (zend - z0) + 2 * H : 1;
  const bool edge = x0 == 0 || x0 + kTX + 8 > nx || y0 - H < 0 || y0 + kTY + H > ny;
  const int tid = threadIdx.x;
  auto plane_z = [&](int p) { return D == 3 ? min(max(z0 - H + p, 0), nz - 1) : 0; };
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int p = 0; p < kNS - 1 && p < nplanes; ++p)
      tma_load_box(&map, ring + p * (kStage / 2), &full[p], x0 - 8, y0 - H, plane_z(p), kBoxBytes);
  }
  __syncthreads();
  // this thread's outputs: rows 2 rb, 2 rb + 1 of the tile, x 4 q .. 4 q + 3
  const int q = tid & 15, rb = tid >> 4;
  const int xo = x0 + 4 * q, yo = y0 + 2 * rb;
  const bool xok = xo < nx;
  uint32_t zr[D == 3 ? K : 1][2][4];
  for (int base = 0; base < nplanes; base += (D == 3 ? K : 1)) {
#pragma unroll
    for (int j = 0; j < (D == 3 ? K : 1); ++j) {
      const int p = base + j;
      if (p >= nplanes) break;
      const int s = p % kNS;
      uint16_t* box = ring + s * (kStage / 2);
      mbar_wait(&full[s], (uint32_t)((p / kNS) & 1));
      if (edge) fix_edges<BY>(box, x0, y0, H, nx, ny);
      __syncthreads();   // box complete; the previous plane's y pass is done with sx
      // x pass: BY rows x 16 quads of 4 outputs (2 x 16-byte loads cover x - 8 .. x + 7 + 4)
      for (int it = tid; it < BY * 16; it += kThreads) {
        const int row = it >> 4, qq = it & 15;
        const uint16_t* src = box + row * kBX + 4 * qq;   // box col 4 qq = x0 - 8 + 4 qq
        constexpr int NV = (12 + H + 3) / 4 * 4;   // box cols 4 qq .. 4 qq + NV - 1 (outputs need 8 - H .. 11 + H)
        uint32_t v[NV];
#pragma unroll
        for (int u = 0; u < NV / 4; ++u) {
          const uint2 a = *reinterpret_cast<const uint2*>(src + 4 * u);
          v[4 * u] = a.x & 0xffffu; v[4 * u + 1] = a.x >> 16; v[4 * u + 2] = a.y & 0xffffu; v[4 * u + 3] = a.y >> 16;
        }
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = q14<H>(T, v + 8 + k);   // output x0 + 4 qq + k = box col 8 + 4 qq + k
        *reinterpret_cast<uint4*>(sx + row * kTX + 4 * qq) = make_uint4(o[0], o[1], o[2], o[3]);
      }
      __syncthreads();   // sx complete; every read of this box done
      if (tid == 0 && p + kNS - 1 < nplanes) {
        const int nq = p + kNS - 1;
        tma_load_box(&map, ring + (nq % kNS) * (kStage / 2), &full[nq % kNS], x0 - 8, y0 - H, plane_z(nq), kBoxBytes);
      }
      // y pass, two output rows per thread: sx rows 2 rb .. 2 rb + 2H + 1 (row i + H is output row i)
      uint32_t yv[2][4];
      {
        uint32_t col[K + 1][4];
#pragma unroll
        for (int i = 0; i <= K; ++i) {
          const uint4 w4 = *reinterpret_cast<const uint4*>(sx + (2 * rb + i) * kTX + 4 * q);
          col[i][0] = w4.x; col[i][1] = w4.y; col[i][2] = w4.z; col[i][3] = w4.w;
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t acc = 8192u + T.w[0] * col[rr + H][k];
#pragma unroll
            for (int i = 1; i <= H; ++i) acc += T.w[i] * (col[rr + H - i][k] + col[rr + H + i][k]);
            yv[rr][k] = acc >> 14;
          }
      }
      if (D == 2) {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
          if (xok && yo + rr < ny)
            *reinterpret_cast<uint2*>(out + (int64_t)(yo + rr) * nx + xo) =
                make_uint2(yv[rr][0] | (yv[rr][1] << 16), yv[rr][2] | (yv[rr][3] << 16));
      } else {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
          for (int k = 0; k < 4; ++k) zr[j][rr][k] = yv[rr][k];
        if (p >= 2 * H) {
          // z pass: ring slots j + 1 .. j + K (mod K) hold planes p - 2H .. p
          const int zo = z0 + p - 2 * H;
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint32_t acc = 8192u + T.w[0] * zr[(j + 1 + H) % K][rr][k];
#pragma unroll
              for (int i = 1; i <= H; ++i)
                acc += T.w[i] * (zr[(j + 1 + H - i) % K][rr][k] + zr[(j + 1 + H + i) % K][rr][k]);
              o[k] = acc >> 14;
            }
            if (xok && yo + rr < ny)
              *reinterpret_cast<uint2*>(out + ((int64_t)zo * ny + yo + rr) * nx + xo) =
                  make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
          }
        }
      }
    }
  }
}

template <int D, int H>
int32_t launch_blur_tma(const uint16_t* in, uint16_t* out, int nx, int ny, int nz, const StencilTaps& T,
                        cudaStream_t st) {
  constexpr int BY = kTY + 2 * H;
  const int smem = kNS * ((kBX * BY * 2 + 127) & ~127) + BY * kTX * 4;
  CUtensorMap map;
  SNK_TRY(volume_map(&map, in, nx, ny, nz, kBX, BY));
  auto k = blur_tma_kernel<D, H>;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] { attr = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  if (attr != cudaSuccess) return cuda_fail(attr, "cudaFuncSetAttribute(blur_tma_kernel)");
  dim3 grid((unsigned)ceil_div(nx, kTX), (unsigned)ceil_div(ny, kTY), D == 3 ? (unsigned)ceil_div(nz, kZC) : 1u);
  k<<<grid, kThreads, smem, st>>>(map, out, nx, ny, nz, T);
  SNK_LAUNCH_CHECK("blur_tma_kernel");
  return SNK_OK;
}

}  // namespace

// ------------------------------------------------------------------ host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static std::once_flag once;
  static EncodeTiledFn fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int32_t volume_map(CUtensorMap* map, const uint16_t* base, int nx, int ny, int nz, int bx, int by) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(SNK_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)nx * 2, (cuuint64_t)nx * ny * 2};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<uint16_t*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SNK_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return SNK_OK;
}

bool tma_available() { return encode_fn() != nullptr; }

bool blur_tma_ok(const snk_grid* g, int h, const void* in, const void* out) {
  return h >= 1 && h <= 8 && !grid_aniso(g) && g->n[0] % 8 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(out) & 15) == 0 && tma_available();
}

int32_t blur_tma(const snk_grid* g, int h, const int32_t* taps, const uint16_t* in, uint16_t* out,
                 cudaStream_t st) {
  StencilTaps T{};
  for (int i = 0; i <= h; ++i) T.w[i] = (uint32_t)taps[h + i];
  const int nx = (int)g->n[0], ny = (int)g->n[1], nz = (int)g->nz_buf;
  if (g->dim == 3) {
    switch (h) {
#define SNK_BT(HH) case HH: return launch_blur_tma<3, HH>(in, out, nx, ny, nz, T, st);
      SNK_BT(1) SNK_BT(2) SNK_BT(3) SNK_BT(4) SNK_BT(5) SNK_BT(6) SNK_BT(7) SNK_BT(8)
#undef SNK_BT
    }
  } else {
    switch (h) {
#define SNK_BT(HH) case HH: return launch_blur_tma<2, HH>(in, out, nx, ny, 1, T, st);
      SNK_BT(1) SNK_BT(2) SNK_BT(3) SNK_BT(4) SNK_BT(5) SNK_BT(6) SNK_BT(7) SNK_BT(8)
#undef SNK_BT
    }
  }
  return fail(SNK_INTERNAL, "blur_tma: radius must be 1..8");
}

}  // namespace snk
