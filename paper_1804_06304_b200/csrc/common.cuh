// common.cuh — shared host/device helpers of libsnk (the CUDA path).
// Nothing here is shared with oracle/ (the test oracle).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "../../include/snk.h"

namespace snk {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
void clear_error();
int32_t fail(int32_t status, const std::string& msg);
int32_t cuda_fail(cudaError_t e, const char* where);
void count_launch(int64_t k = 1);

#define SNK_CUDA_CHECK(expr)                                  \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::snk::cuda_fail(_e, #expr); \
  } while (0)

#define SNK_LAUNCH_CHECK(name)                                     \
  do {                                                             \
    ::snk::count_launch();                                         \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return ::snk::cuda_fail(_e, name);      \
  } while (0)

#define SNK_TRY(expr)                   \
  do {                                  \
    int32_t _s = (expr);                \
    if (_s != SNK_OK) return _s;        \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- constants
// rho = 2^(-1/d), as correctly rounded doubles; rho^2 for labels.
constexpr double kRho3 = 0.7937005259840998;
constexpr double kRho2 = 0.7071067811865476;
constexpr double kRhoSq3 = 0.6299605249474366;
constexpr double kRhoSq2 = 0.5;
inline double rho_of(int dim) { return dim == 3 ? kRho3 : kRho2; }

// physical voxel size of axis a (G28); 0 means 1
inline double grid_scale(const snk_grid* g, int a) { return g->scale[a] > 0.0 ? g->scale[a] : 1.0; }
inline bool grid_aniso(const snk_grid* g) {
  for (int a = 0; a < g->dim; ++a)
    if (grid_scale(g, a) != 1.0) return true;
  return false;
}
// the MAXIMA half-window of axis a: floor(w / scale_a + 0.5) voxels (G28)
inline int axis_window(const snk_grid* g, int w, int a) {
  return (int)std::floor((double)w / grid_scale(g, a) + 0.5);
}

// ---------------------------------------------------------------- workspace
// A bump allocator over the caller's workspace; 256-byte aligned slices.
struct Carve {
  char* base;
  size_t cap;
  size_t off = 0;
  bool overflow = false;
  Carve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    if (off > cap) overflow = true;
    return p;
  }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- sizes
size_t preprocess_ws(const snk_grid* g, const snk_params* p);
size_t seeds_ws(const snk_grid* g, const snk_params* p);
size_t evolve_ws(const snk_grid* g, const snk_params* p, int64_t max_cells);
size_t cull_ws(const snk_grid* g, const snk_params* p, int64_t max_cells);
size_t label_ws(const snk_grid* g, const snk_params* p, int64_t max_cells);
size_t resample_ws(int32_t dim, const int64_t n_raw[3], const double spacing[3]);

// ---------------------------------------------------------------- entry points per file
int32_t preprocess_impl(const snk_grid* g, const snk_params* p, const uint16_t* d_in,
                        uint16_t* d_smooth, uint16_t* d_gradmag, void* d_ws, size_t ws_bytes,
                        cudaStream_t st);
// a0: u8 -> u16 (x257, exact), volume.cu
int32_t ingest_u8_impl(const uint8_t* d_in, uint16_t* d_out, int64_t n, cudaStream_t st);
int32_t resample_impl(int32_t dim, const int64_t n_raw[3], const double spacing[3], int64_t zr_lo,
                      int64_t nzr, const uint16_t* d_raw, int64_t z_lo, int64_t nz_out,
                      uint16_t* d_out, void* d_ws, size_t ws_bytes, cudaStream_t st);
int32_t seeds_impl(const snk_grid* g, const snk_params* p, const uint16_t* d_smooth,
                   float* d_seeds, int64_t cap, int64_t* n_out, int64_t* first_id, void* d_ws,
                   size_t ws_bytes, cudaStream_t st);
int32_t evolve_impl(const snk_grid* g, const snk_params* p, const uint16_t* d_image,
                    const float* d_seeds, const int64_t* d_ids, int64_t id_base, int64_t n,
                    snk_cell* d_cells, void* d_ws, size_t ws_bytes, cudaStream_t st, int it0 = 0,
                    int it1 = 0, bool resume = false);
int32_t cells_init_impl(const snk_params* p, const float* d_seeds, const int64_t* d_ids,
                        int64_t id_base, int64_t n, snk_cell* d_cells, cudaStream_t st);
// the periodic-culling segments of G25: ends k, 2k, ... (< T), then T + 1
int32_t compact_impl(const snk_params* p, const snk_cell* d_cells, int64_t n, snk_cell* d_out,
                     int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes, cudaStream_t st);
int32_t select_ids_impl(const snk_cell* d_cells, int64_t n, int64_t id_lo, int64_t id_hi,
                        snk_cell* d_out, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                        cudaStream_t st);
int32_t cull_impl(const snk_grid* g, const snk_params* p, const snk_cell* d_cells, int64_t n,
                  snk_cell* d_dets, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                  cudaStream_t st);
int32_t label_impl(const snk_grid* g, const snk_params* p, const snk_cell* d_dets, int64_t n,
                   int32_t* d_labels, void* d_ws, size_t ws_bytes, cudaStream_t st);

// Small device -> host readback (counts; <= 256 bytes), then synchronises st.
// A one-thread kernel stores into mapped pinned host memory, so the readback
// never queues behind a bulk copy on the copy engines (snk_run_batch downloads
// a label map while the next volume's kernels need their counts).
int32_t read_back(const void* d_src, void* h_dst, size_t bytes, cudaStream_t st);

int evolve_warps_per_cell(const snk_params* p, int64_t n_cells);
int32_t evolve_stats(int64_t out[4], bool reset);

// vectorised separable pass (volume.cu): op must be 1 = box max clipped to
// [lo, hi] on the pass axis (the blur passes are internal to preprocess);
// radius h <= 8; needs nx % 8 == 0 and 16-byte aligned buffers (vec8_ok)
bool vec8_ok(const snk_grid* g, const void* a, const void* b, const void* c);
int32_t sep_pass(int axis, int op, int h, const uint16_t* in, uint16_t* out, int nx, int ny, int nz,
                 int lo, int hi, cudaStream_t st);

// a2 as one TMA-staged pass (stencil.cu): isotropic grids, radius 1..8, x extent
// % 8 == 0, 16-byte aligned buffers; taps = the 2h + 1 Q14 taps
bool blur_tma_ok(const snk_grid* g, int h, const void* in, const void* out);
int32_t blur_tma(const snk_grid* g, int h, const int32_t* taps, const uint16_t* in, uint16_t* out,
                 cudaStream_t st);

// exclusive scan of n int counts into n + 1 int64 offsets (offsets[n] = total);
// tmp: scan_ws(n) bytes of scratch (nullptr: single-block scan)
size_t scan_ws(int64_t n);
int32_t scan_counts(const int* counts, int64_t n, int64_t* offsets, cudaStream_t st, void* tmp);

}  // namespace snk
