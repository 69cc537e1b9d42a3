// abi.cu — the extern "C" boundary of libsnk.so (include/snk.h): validation,
// workspace sizing, status/error reporting and the single-GPU snk_run chain.
// All device work is in the kernels of volume.cu, seeds.cu, evolve.cu,
// cull.cu and label.cu.
#include <cmath>
#include <cstring>
#include <string>

#include "common.cuh"

namespace snk {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
void clear_error() { g_err.clear(); }
int32_t fail(int32_t status, const std::string& msg) {
  g_err = msg;
  return status;
}
int32_t cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e);
  return SNK_CUDA;
}
void count_launch(int64_t k) { g_launches += k; }

namespace {
__global__ void read_back_kernel(const unsigned char* src, unsigned char* dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

int32_t read_back(const void* d_src, void* h_dst, size_t bytes, cudaStream_t st) {
  constexpr size_t kCap = 256;
  static thread_local unsigned char* host = nullptr;   // mapped pinned host memory (per thread)
  static thread_local unsigned char* dev = nullptr;
  if (bytes > kCap) return fail(SNK_INTERNAL, "read_back: more than 256 bytes");
  if (!host) {
    SNK_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&host), kCap, cudaHostAllocMapped));
    SNK_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
  }
  read_back_kernel<<<1, 32, 0, st>>>(static_cast<const unsigned char*>(d_src), dev, (int)bytes);
  SNK_LAUNCH_CHECK("read_back_kernel");
  SNK_CUDA_CHECK(cudaStreamSynchronize(st));
  std::memcpy(h_dst, host, bytes);
  return SNK_OK;
}

static bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

static int32_t validate_grid(const snk_grid* g) {
  if (!g) return fail(SNK_CONFIG, "grid is null");
  if (g->dim != 2 && g->dim != 3) return fail(SNK_SHAPE, "dim must be 2 or 3");
  for (int a = 0; a < g->dim; ++a)
    if (g->n[a] < 2) return fail(SNK_SHAPE, "every used axis needs at least 2 voxels");
  if (g->dim == 2 && g->n[2] != 1) return fail(SNK_SHAPE, "2D images need n[2] == 1");
  if (g->n[0] > (1 << 30) || g->n[1] > (1 << 30) || g->n[2] > (1 << 30))
    return fail(SNK_SHAPE, "axis too long");
  if (g->z_lo < 0 || g->nz_buf < 1 || g->z_lo + g->nz_buf > g->n[2])
    return fail(SNK_SHAPE, "buffer planes [z_lo, z_lo+nz_buf) must lie inside the volume");
  if (g->dim == 3 && g->nz_buf < 2) return fail(SNK_SHAPE, "3D buffers need at least 2 planes");
  if (g->own_z0 < g->z_lo || g->own_z1 > g->z_lo + g->nz_buf || g->own_z0 > g->own_z1)
    return fail(SNK_SHAPE, "owned planes must lie inside the buffer");
  for (int a = 0; a < 3; ++a)
    if (!(g->scale[a] >= 0.0) || g->scale[a] > 1e6) return fail(SNK_SHAPE, "scale must be >= 0 (0 = 1)");
  const double nvox = (double)g->n[0] * (double)g->n[1] * (double)g->nz_buf;
  if (nvox >= 4294967296.0) return fail(SNK_SHAPE, "buffer exceeds 2^32 voxels; use z-slabs");
  return SNK_OK;
}

static int32_t validate_params(const snk_params* p, int dim) {
  if (!p) return fail(SNK_CONFIG, "params is null");
  if (!(p->r0 > 0) || !(p->delta_R > 0) || !(p->eps0 > 0) || !(p->max_step > 0))
    return fail(SNK_CONFIG, "r0, delta_R, eps0 and max_step must be > 0");
  if (!(p->e0 <= 0)) return fail(SNK_CONFIG, "e0 must be <= 0 (S:262)");
  if (!(p->r_min > 0) || !(p->r0 > p->r_min) || !(p->r_max >= p->r0))
    return fail(SNK_CONFIG, "need 0 < r_min < r0 <= r_max");
  if (!(p->leash >= 0) || !(p->conv_tol >= 0) || !(p->intensity_scale > 0))
    return fail(SNK_CONFIG, "leash, conv_tol >= 0 and intensity_scale > 0");
  if (!(p->sigma >= 0) || std::ceil(4.0 * p->sigma) > 32)
    return fail(SNK_CONFIG, "sigma must be in [0, 8]");
  if (p->max_iters < 1 || p->max_iters > (1 << 24)) return fail(SNK_CONFIG, "max_iters in [1, 2^24]");
  if (!is_pow2(p->n_samples) || p->n_samples < 32 || p->n_samples > (1 << 20))
    return fail(SNK_CONFIG, "n_samples must be a power of two in [32, 2^20]");
  if (p->cta_warps != 0 && !(is_pow2(p->cta_warps) && p->cta_warps <= 8))
    return fail(SNK_CONFIG, "cta_warps must be 0 (auto), 1, 2, 4 or 8");
  if (p->cta_warps > 0 && p->n_samples < 32 * p->cta_warps)
    return fail(SNK_CONFIG, "n_samples must be >= 32 * cta_warps");
  if (p->seed_mode < 0 || p->seed_mode > 2) return fail(SNK_CONFIG, "bad seed_mode");
  if (p->seed_mode == SNK_SEED_MAXIMA && (p->seed_window < 0 || p->seed_window > 64))
    return fail(SNK_CONFIG, "seed_window must be in [0, 64]");
  if (p->image_term != SNK_IMAGE_INTENSITY && p->image_term != SNK_IMAGE_GRADMAG)
    return fail(SNK_CONFIG, "bad image_term");
  if (p->kernel_variant > 3) return fail(SNK_CONFIG, "kernel_variant must be 0, 1, 2 or 3");
  if (p->estimator < SNK_EST_MC || p->estimator > SNK_EST_RAY)
    return fail(SNK_CONFIG, "estimator must be SNK_EST_MC, _GRID, _MC_CV or _RAY");
  if (p->cull_every < 0) return fail(SNK_CONFIG, "cull_every must be >= 0");
  if (p->estimator != SNK_EST_MC && (p->kernel_variant == 1 || p->kernel_variant == 3))
    return fail(SNK_CONFIG, "the grid / CV / ray estimators run in the brick kernel only (kernel_variant 0 or 2)");
  (void)dim;
  return SNK_OK;
}

static int32_t validate(const snk_grid* g, const snk_params* p) {
  SNK_TRY(validate_grid(g));
  SNK_TRY(validate_params(p, g->dim));
  if (grid_aniso(g)) {
    if (g->n[0] % 8 != 0) return fail(SNK_SHAPE, "anisotropic grids need an x extent divisible by 8");
    if (p->estimator == SNK_EST_GRID) return fail(SNK_CONFIG, "the grid estimator is isotropic only");
    if (p->image_term == SNK_IMAGE_GRADMAG) return fail(SNK_CONFIG, "the gradient-magnitude term is isotropic only");
  }
  return SNK_OK;
}

static int32_t check_ws(size_t need, void* d_ws, size_t ws_bytes) {
  if (need > 0 && (d_ws == nullptr || ws_bytes < need))
    return fail(SNK_CAPACITY, "workspace too small: need " + std::to_string(need) + " bytes");
  return SNK_OK;
}

}  // namespace snk

using namespace snk;

extern "C" {

int32_t snk_abi_version(void) { return SNK_ABI_VERSION; }

const char* snk_last_error(void) { return g_err.c_str(); }

const char* snk_status_string(int32_t s) {
  switch (s) {
    case SNK_OK: return "ok";
    case SNK_EMPTY_DOMAIN: return "empty domain";
    case SNK_CONFIG: return "invalid configuration";
    case SNK_SHAPE: return "invalid shape";
    case SNK_INTERNAL: return "internal error";
    case SNK_CUDA: return "CUDA error";
    case SNK_CAPACITY: return "capacity exceeded";
    default: return "unknown status";
  }
}

int64_t snk_launch_count(void) { return g_launches; }

int32_t snk_evolve_stats(int64_t* out4, int32_t reset) {
  clear_error();
  if (!out4) return fail(SNK_CONFIG, "out4 is null");
  return evolve_stats(out4, reset != 0);
}

int32_t snk_validate(const snk_grid* g, const snk_params* p) {
  clear_error();
  return validate(g, p);
}

int32_t snk_workspace_bytes(const snk_grid* g, const snk_params* p, int64_t max_cells,
                            size_t* bytes) {
  clear_error();
  SNK_TRY(validate(g, p));
  if (!bytes || max_cells < 0) return fail(SNK_CONFIG, "bytes is null or max_cells < 0");
  size_t b = preprocess_ws(g, p);
  b = std::max(b, seeds_ws(g, p));
  b = std::max(b, evolve_ws(g, p, max_cells));
  b = std::max(b, cull_ws(g, p, max_cells));
  b = std::max(b, label_ws(g, p, max_cells));
  *bytes = b;
  return SNK_OK;
}

int32_t snk_resample_dims(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                          int64_t n_out[3]) {
  clear_error();
  if ((dim != 2 && dim != 3) || !n_raw || !spacing || !n_out) return fail(SNK_CONFIG, "bad args");
  double smin = spacing[0];
  for (int a = 0; a < dim; ++a) {
    if (!(spacing[a] > 0)) return fail(SNK_CONFIG, "spacing must be > 0");
    smin = std::min(smin, spacing[a]);
  }
  for (int a = 0; a < 3; ++a) {
    n_out[a] = n_raw[a];
    if (a < dim && spacing[a] > smin) n_out[a] = (int64_t)std::llround((double)n_raw[a] * spacing[a] / smin);
  }
  return SNK_OK;
}

int32_t snk_resample(int32_t dim, const int64_t n_raw[3], const double spacing[3], int64_t zr_lo,
                     int64_t nzr, const uint16_t* d_raw, int64_t z_lo, int64_t nz_out,
                     uint16_t* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  clear_error();
  if (!d_raw || !d_out) return fail(SNK_CONFIG, "null buffer");
  SNK_TRY(check_ws(resample_ws(dim, n_raw, spacing), d_ws, ws_bytes));
  return resample_impl(dim, n_raw, spacing, zr_lo, nzr, d_raw, z_lo, nz_out, d_out, d_ws,
                       ws_bytes, as_stream(stream));
}

int32_t snk_preprocess(const snk_grid* g, const snk_params* p, const uint16_t* d_in,
                       uint16_t* d_smooth, uint16_t* d_gradmag, void* d_ws, size_t ws_bytes,
                       void* stream) {
  clear_error();
  SNK_TRY(validate(g, p));
  if (!d_in || !d_smooth) return fail(SNK_CONFIG, "null buffer");
  SNK_TRY(check_ws(preprocess_ws(g, p), d_ws, ws_bytes));
  return preprocess_impl(g, p, d_in, d_smooth, d_gradmag, d_ws, ws_bytes, as_stream(stream));
}

int32_t snk_seeds(const snk_grid* g, const snk_params* p, const uint16_t* d_smooth,
                  float* d_seeds, int64_t cap, int64_t* n_out, int64_t* first_id_out,
                  void* d_ws, size_t ws_bytes, void* stream) {
  clear_error();
  SNK_TRY(validate(g, p));
  if (!n_out || cap < 0 || (cap > 0 && !d_seeds)) return fail(SNK_CONFIG, "bad output buffer");
  if (p->seed_mode == SNK_SEED_GIVEN) return fail(SNK_CONFIG, "seed_mode GIVEN: seeds come from the caller");
  if (p->seed_mode == SNK_SEED_MAXIMA && !d_smooth) return fail(SNK_CONFIG, "null volume");
  SNK_TRY(check_ws(seeds_ws(g, p), d_ws, ws_bytes));
  return seeds_impl(g, p, d_smooth, d_seeds, cap, n_out, first_id_out, d_ws, ws_bytes,
                    as_stream(stream));
}

int32_t snk_evolve(const snk_grid* g, const snk_params* p, const uint16_t* d_image,
                   const float* d_seeds, const int64_t* d_ids, int64_t id_base, int64_t n,
                   snk_cell* d_cells, void* d_ws, size_t ws_bytes, void* stream) {
  clear_error();
  SNK_TRY(validate(g, p));
  if (n < 0) return fail(SNK_CONFIG, "n < 0");
  if (n == 0) return SNK_OK;
  if (!d_image || !d_seeds || !d_cells) return fail(SNK_CONFIG, "null buffer");
  SNK_TRY(check_ws(evolve_ws(g, p, n), d_ws, ws_bytes));
  return evolve_impl(g, p, d_image, d_seeds, d_ids, id_base, n, d_cells, d_ws, ws_bytes,
                     as_stream(stream));
}

int32_t snk_cells_init(const snk_params* p, const float* d_seeds, const int64_t* d_ids,
                       int64_t id_base, int64_t n, snk_cell* d_cells, void* stream) {
  clear_error();
  if (!p || n < 0) return fail(SNK_CONFIG, "bad args");
  if (n > 0 && (!d_seeds || !d_cells)) return fail(SNK_CONFIG, "null buffer");
  return cells_init_impl(p, d_seeds, d_ids, id_base, n, d_cells, as_stream(stream));
}

int32_t snk_evolve_range(const snk_grid* g, const snk_params* p, const uint16_t* d_image,
                         snk_cell* d_cells, int64_t n, int32_t it0, int32_t it1, void* d_ws,
                         size_t ws_bytes, void* stream) {
  clear_error();
  SNK_TRY(validate(g, p));
  if (n < 0) return fail(SNK_CONFIG, "n < 0");
  if (it0 < 1 || it1 < it0 || it1 > p->max_iters + 1) return fail(SNK_CONFIG, "need 1 <= it0 <= it1 <= T + 1");
  if (n == 0) return SNK_OK;
  if (!d_image || !d_cells) return fail(SNK_CONFIG, "null buffer");
  SNK_TRY(check_ws(evolve_ws(g, p, n), d_ws, ws_bytes));
  return evolve_impl(g, p, d_image, nullptr, nullptr, 0, n, d_cells, d_ws, ws_bytes,
                     as_stream(stream), it0, it1, true);
}

int32_t snk_compact_candidates(const snk_params* p, const snk_cell* d_cells, int64_t n,
                               snk_cell* d_out, int64_t cap, int64_t* n_out, void* d_ws,
                               size_t ws_bytes, void* stream) {
  clear_error();
  if (!p || !n_out || n < 0 || cap < 0) return fail(SNK_CONFIG, "bad args");
  if (n > 0 && (!d_cells || (cap > 0 && !d_out))) return fail(SNK_CONFIG, "null buffer");
  return compact_impl(p, d_cells, n, d_out, cap, n_out, d_ws, ws_bytes, as_stream(stream));
}

int32_t snk_select_ids(const snk_cell* d_cells, int64_t n, int64_t id_lo, int64_t id_hi,
                       snk_cell* d_out, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                       void* stream) {
  clear_error();
  if (!n_out || n < 0 || cap < 0) return fail(SNK_CONFIG, "bad args");
  if (n > 0 && (!d_cells || (cap > 0 && !d_out))) return fail(SNK_CONFIG, "null buffer");
  return select_ids_impl(d_cells, n, id_lo, id_hi, d_out, cap, n_out, d_ws, ws_bytes, as_stream(stream));
}

int32_t snk_cull(const snk_grid* g, const snk_params* p, const snk_cell* d_cells, int64_t n,
                 snk_cell* d_dets, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                 void* stream) {
  clear_error();
  SNK_TRY(validate(g, p));
  if (!n_out || n < 0 || cap < 0) return fail(SNK_CONFIG, "bad args");
  if (n > 0 && (!d_cells || (cap > 0 && !d_dets))) return fail(SNK_CONFIG, "null buffer");
  if (n >= ((int64_t)1 << 31)) return fail(SNK_SHAPE, "too many cells");
  SNK_TRY(check_ws(cull_ws(g, p, n), d_ws, ws_bytes));
  return cull_impl(g, p, d_cells, n, d_dets, cap, n_out, d_ws, ws_bytes, as_stream(stream));
}

int32_t snk_label(const snk_grid* g, const snk_params* p, const snk_cell* d_dets, int64_t n,
                  int32_t* d_labels, void* d_ws, size_t ws_bytes, void* stream) {
  clear_error();
  SNK_TRY(validate(g, p));
  if (!d_labels || n < 0 || (n > 0 && !d_dets)) return fail(SNK_CONFIG, "bad args");
  SNK_TRY(check_ws(label_ws(g, p, n), d_ws, ws_bytes));
  return label_impl(g, p, d_dets, n, d_labels, d_ws, ws_bytes, as_stream(stream));
}

// --------------------------------------------------------------------------
// snk_run: the single-GPU end-to-end call from host buffers.
// Workspace layout: [raw | (resampled) | smooth | gradmag? | seeds | cells |
//                    dets | labels | scratch]
struct RunLayout {
  snk_grid g;
  int64_t n_iso[3];
  bool resample;
  size_t off_raw, off_iso, off_smooth, off_grad, off_seeds, off_cells, off_dets, off_labels,
      off_scratch, scratch_bytes, total;
};

static int32_t run_layout(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                          const snk_params* p, int64_t max_cells, RunLayout* L) {
  SNK_TRY(snk_resample_dims(dim, n_raw, spacing, L->n_iso));
  L->resample = false;
  for (int a = 0; a < 3; ++a) L->resample |= (L->n_iso[a] != n_raw[a]);
  snk_grid& g = L->g;
  std::memset(&g, 0, sizeof g);
  g.dim = dim;
  for (int a = 0; a < 3; ++a) g.n[a] = L->n_iso[a];
  g.z_lo = 0;
  g.nz_buf = L->n_iso[2];
  g.own_z0 = 0;
  g.own_z1 = L->n_iso[2];
  SNK_TRY(validate(&g, p));
  const size_t nraw = (size_t)n_raw[0] * n_raw[1] * n_raw[2];
  const size_t niso = (size_t)g.n[0] * g.n[1] * g.n[2];
  Carve c(nullptr, ~size_t(0));
  L->off_raw = 0; c.take<uint16_t>(nraw);
  c.off = (c.off + 255) & ~size_t(255); L->off_iso = c.off; if (L->resample) c.take<uint16_t>(niso);
  c.off = (c.off + 255) & ~size_t(255); L->off_smooth = c.off; c.take<uint16_t>(niso);
  c.off = (c.off + 255) & ~size_t(255); L->off_grad = c.off;
  if (p->image_term == SNK_IMAGE_GRADMAG) c.take<uint16_t>(niso);
  c.off = (c.off + 255) & ~size_t(255); L->off_seeds = c.off; c.take<float>(3 * (size_t)max_cells);
  c.off = (c.off + 255) & ~size_t(255); L->off_cells = c.off; c.take<snk_cell>(max_cells);
  c.off = (c.off + 255) & ~size_t(255); L->off_dets = c.off; c.take<snk_cell>(max_cells);
  c.off = (c.off + 255) & ~size_t(255); L->off_labels = c.off; c.take<int32_t>(niso);
  c.off = (c.off + 255) & ~size_t(255); L->off_scratch = c.off;
  size_t s = 0;
  SNK_TRY(snk_workspace_bytes(&g, p, max_cells, &s));
  s = std::max(s, resample_ws(dim, n_raw, spacing));
  L->scratch_bytes = s;
  L->total = L->off_scratch + s;
  return SNK_OK;
}

int32_t snk_run_workspace_bytes(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                                const snk_params* p, int64_t max_cells, size_t* bytes) {
  clear_error();
  if (!bytes || !n_raw || !spacing || max_cells < 1) return fail(SNK_CONFIG, "bad args");
  RunLayout L;
  SNK_TRY(run_layout(dim, n_raw, spacing, p, max_cells, &L));
  *bytes = L.total;
  return SNK_OK;
}

// The device part of one end-to-end step: raw volume (device) -> detections
// (d_dets) and, if d_labels, the label map.  raw_free (nullable) is recorded on
// st once the raw buffer has been consumed (after a1/a2), so a batch can
// upload the next volume into it.
static int32_t run_compute(const RunLayout& L, int32_t dim, const int64_t n_raw[3], const double spacing[3],
                           const snk_params* p, const uint16_t* d_raw, snk_cell* d_dets, int32_t* d_labels,
                           int64_t max_cells, char* base, cudaStream_t st, cudaEvent_t raw_free,
                           int64_t* nd_out) {
  uint16_t* d_iso = L.resample ? reinterpret_cast<uint16_t*>(base + L.off_iso) : const_cast<uint16_t*>(d_raw);
  uint16_t* d_smooth = reinterpret_cast<uint16_t*>(base + L.off_smooth);
  uint16_t* d_grad = p->image_term == SNK_IMAGE_GRADMAG ? reinterpret_cast<uint16_t*>(base + L.off_grad) : nullptr;
  float* d_seeds = reinterpret_cast<float*>(base + L.off_seeds);
  snk_cell* d_cells = reinterpret_cast<snk_cell*>(base + L.off_cells);
  void* scratch = base + L.off_scratch;
  const size_t sb = L.scratch_bytes;
  if (L.resample)
    SNK_TRY(resample_impl(dim, n_raw, spacing, 0, n_raw[2], d_raw, 0, L.g.n[2], d_iso, scratch, sb, st));
  SNK_TRY(preprocess_impl(&L.g, p, d_iso, d_smooth, d_grad, scratch, sb, st));
  if (raw_free) SNK_CUDA_CHECK(cudaEventRecord(raw_free, st));
  int64_t ns = 0, first = 0;
  SNK_TRY(seeds_impl(&L.g, p, d_smooth, d_seeds, max_cells, &ns, &first, scratch, sb, st));
  const uint16_t* d_img = d_grad ? d_grad : d_smooth;
  int64_t nd = 0;
  if (p->cull_every > 0 && p->cull_every < p->max_iters) {
    // periodic culling (G25): segments [1, k], [k+1, 2k], ... (checkpoints
    // after iterations k, 2k, ... < T), the last one ending at T + 1; the a7
    // cull after each but the last.  Bounds computed on the fly (any T, k).
    snk_cell* cur = d_cells;
    snk_cell* nxt = d_dets;
    int64_t live = ns;
    SNK_TRY(cells_init_impl(p, d_seeds, nullptr, first, ns, cur, st));
    const int T = p->max_iters, kc = p->cull_every;
    for (int a = 1; a <= T + 1;) {
      const int e = (a + kc - 1 < T) ? a + kc - 1 : T + 1;
      SNK_TRY(evolve_impl(&L.g, p, d_img, nullptr, nullptr, 0, live, cur, scratch, sb, st, a, e, true));
      if (e <= T) {
        SNK_TRY(cull_impl(&L.g, p, cur, live, nxt, max_cells, &live, scratch, sb, st));
        std::swap(cur, nxt);
      }
      a = e + 1;
    }
    SNK_TRY(cull_impl(&L.g, p, cur, live, nxt, max_cells, &nd, scratch, sb, st));
    if (nxt != d_dets)
      SNK_CUDA_CHECK(cudaMemcpyAsync(d_dets, nxt, nd * sizeof(snk_cell), cudaMemcpyDeviceToDevice, st));
  } else {
    if (ns > 0)
      SNK_TRY(evolve_impl(&L.g, p, d_img, d_seeds, nullptr, first, ns, d_cells, scratch, sb, st));
    SNK_TRY(cull_impl(&L.g, p, d_cells, ns, d_dets, max_cells, &nd, scratch, sb, st));
  }
  if (d_labels) SNK_TRY(label_impl(&L.g, p, d_dets, nd, d_labels, scratch, sb, st));
  *nd_out = nd;
  return SNK_OK;
}

// snk_run / snk_run_u8: h_raw holds u16 (bpv 2) or u8 (bpv 1) voxels
static int32_t run_host(int32_t dim, const int64_t n_raw[3], const double spacing[3], const snk_params* p,
                        const void* h_raw, int bpv, snk_cell* h_dets, int64_t det_cap, int64_t* n_dets,
                        int32_t* h_labels, int64_t max_cells, void* d_ws, size_t ws_bytes, void* stream) {
  clear_error();
  if (!h_raw || !n_dets || det_cap < 0 || (det_cap > 0 && !h_dets) || max_cells < 1)
    return fail(SNK_CONFIG, "bad args");
  RunLayout L;
  SNK_TRY(run_layout(dim, n_raw, spacing, p, max_cells, &L));
  SNK_TRY(check_ws(L.total, d_ws, ws_bytes));
  cudaStream_t st = as_stream(stream);
  char* base = static_cast<char*>(d_ws);
  uint16_t* d_raw = reinterpret_cast<uint16_t*>(base + L.off_raw);
  snk_cell* d_dets = reinterpret_cast<snk_cell*>(base + L.off_dets);
  int32_t* d_labels = reinterpret_cast<int32_t*>(base + L.off_labels);
  const size_t nraw = (size_t)n_raw[0] * n_raw[1] * n_raw[2];
  const size_t niso = (size_t)L.g.n[0] * L.g.n[1] * L.g.n[2];
  if (bpv == 2) {
    SNK_CUDA_CHECK(cudaMemcpyAsync(d_raw, h_raw, nraw * sizeof(uint16_t), cudaMemcpyHostToDevice, st));
  } else {
    // a0: the bytes land in the label region (>= 4 niso >= nraw bytes, written
    // only by a8), then promote into the raw u16 buffer
    uint8_t* d_u8 = reinterpret_cast<uint8_t*>(base + L.off_labels);
    SNK_CUDA_CHECK(cudaMemcpyAsync(d_u8, h_raw, nraw, cudaMemcpyHostToDevice, st));
    SNK_TRY(ingest_u8_impl(d_u8, d_raw, (int64_t)nraw, st));
  }
  int64_t nd = 0;
  SNK_TRY(run_compute(L, dim, n_raw, spacing, p, d_raw, d_dets, h_labels ? d_labels : nullptr, max_cells, base,
                      st, nullptr, &nd));
  *n_dets = nd;
  const int64_t ncopy = std::min(nd, det_cap);
  if (ncopy > 0)
    SNK_CUDA_CHECK(cudaMemcpyAsync(h_dets, d_dets, ncopy * sizeof(snk_cell), cudaMemcpyDeviceToHost, st));
  if (h_labels)
    SNK_CUDA_CHECK(cudaMemcpyAsync(h_labels, d_labels, niso * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SNK_CUDA_CHECK(cudaStreamSynchronize(st));
  if (nd > det_cap) return fail(SNK_CAPACITY, "detection buffer too small");
  return SNK_OK;
}

int32_t snk_run(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                const snk_params* p, const uint16_t* h_raw, snk_cell* h_dets, int64_t det_cap,
                int64_t* n_dets, int32_t* h_labels, int64_t max_cells, void* d_ws,
                size_t ws_bytes, void* stream) {
  return run_host(dim, n_raw, spacing, p, h_raw, 2, h_dets, det_cap, n_dets, h_labels, max_cells, d_ws, ws_bytes,
                  stream);
}

int32_t snk_run_u8(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                   const snk_params* p, const uint8_t* h_raw, snk_cell* h_dets, int64_t det_cap,
                   int64_t* n_dets, int32_t* h_labels, int64_t max_cells, void* d_ws,
                   size_t ws_bytes, void* stream) {
  return run_host(dim, n_raw, spacing, p, h_raw, 1, h_dets, det_cap, n_dets, h_labels, max_cells, d_ws, ws_bytes,
                  stream);
}

int32_t snk_ingest_u8(const uint8_t* d_in, uint16_t* d_out, int64_t n, void* stream) {
  clear_error();
  if (n < 0 || (n > 0 && (!d_in || !d_out))) return fail(SNK_CONFIG, "bad args");
  return ingest_u8_impl(d_in, d_out, n, as_stream(stream));
}

// snk_run over a sequence of volumes: the next volume's upload and the previous
// results' download run on two internal streams while the current volume's
// kernels run on `stream` (double-buffered raw volume, detections and label map).
static size_t batch_extra(const RunLayout& L, const int64_t n_raw[3], int64_t max_cells) {
  const size_t nraw = (size_t)n_raw[0] * n_raw[1] * n_raw[2];
  const size_t niso = (size_t)L.g.n[0] * L.g.n[1] * L.g.n[2];
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return al(nraw * sizeof(uint16_t)) + al(niso * sizeof(int32_t)) + al((size_t)max_cells * sizeof(snk_cell));
}

int32_t snk_run_batch_workspace_bytes(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                                      const snk_params* p, int64_t max_cells, size_t* bytes) {
  clear_error();
  if (!bytes || !n_raw || !spacing || max_cells < 1) return fail(SNK_CONFIG, "bad args");
  RunLayout L;
  SNK_TRY(run_layout(dim, n_raw, spacing, p, max_cells, &L));
  *bytes = ((L.total + 255) & ~size_t(255)) + batch_extra(L, n_raw, max_cells);
  return SNK_OK;
}

int32_t snk_run_batch(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                      const snk_params* p, int64_t nvol, const uint16_t* const* h_raw,
                      snk_cell* const* h_dets, int64_t det_cap, int64_t* n_dets,
                      int32_t* const* h_labels, int64_t max_cells, void* d_ws, size_t ws_bytes,
                      void* stream) {
  clear_error();
  if (nvol < 0 || (nvol > 0 && (!h_raw || !n_dets || !h_dets)) || det_cap < 0 || max_cells < 1)
    return fail(SNK_CONFIG, "bad args");
  RunLayout L;
  SNK_TRY(run_layout(dim, n_raw, spacing, p, max_cells, &L));
  const size_t off2 = (L.total + 255) & ~size_t(255);
  SNK_TRY(check_ws(off2 + batch_extra(L, n_raw, max_cells), d_ws, ws_bytes));
  for (int64_t i = 0; i < nvol; ++i)
    if (!h_raw[i] || (det_cap > 0 && !h_dets[i])) return fail(SNK_CONFIG, "null host buffer");
  if (nvol == 0) return SNK_OK;
  cudaStream_t st = as_stream(stream);
  char* base = static_cast<char*>(d_ws);
  const size_t nraw = (size_t)n_raw[0] * n_raw[1] * n_raw[2];
  const size_t niso = (size_t)L.g.n[0] * L.g.n[1] * L.g.n[2];
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  uint16_t* raw[2] = {reinterpret_cast<uint16_t*>(base + L.off_raw), reinterpret_cast<uint16_t*>(base + off2)};
  int32_t* lab[2] = {reinterpret_cast<int32_t*>(base + L.off_labels),
                     reinterpret_cast<int32_t*>(base + off2 + al(nraw * 2))};
  snk_cell* dets[2] = {reinterpret_cast<snk_cell*>(base + L.off_dets),
                       reinterpret_cast<snk_cell*>(base + off2 + al(nraw * 2) + al(niso * 4))};
  const bool want_labels = h_labels != nullptr;
  cudaStream_t su = nullptr, sd = nullptr;
  cudaEvent_t up[2] = {}, raw_free[2] = {}, done[2] = {}, out_free[2] = {};
  int32_t status = SNK_OK;
  auto ck = [&](cudaError_t e, const char* w) {
    if (e != cudaSuccess && status == SNK_OK) status = cuda_fail(e, w);
    return status == SNK_OK;
  };
  bool ok = ck(cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking), "cudaStreamCreate") &&
            ck(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking), "cudaStreamCreate");
  for (int k = 0; k < 2 && ok; ++k)
    ok = ck(cudaEventCreateWithFlags(&up[k], cudaEventDisableTiming), "cudaEventCreate") &&
         ck(cudaEventCreateWithFlags(&raw_free[k], cudaEventDisableTiming), "cudaEventCreate") &&
         ck(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming), "cudaEventCreate") &&
         ck(cudaEventCreateWithFlags(&out_free[k], cudaEventDisableTiming), "cudaEventCreate");
  if (ok) ok = ck(cudaMemcpyAsync(raw[0], h_raw[0], nraw * 2, cudaMemcpyHostToDevice, su), "upload") &&
               ck(cudaEventRecord(up[0], su), "cudaEventRecord");
  for (int64_t i = 0; i < nvol && ok; ++i) {
    const int s = (int)(i & 1), s1 = 1 - s;
    if (i + 1 < nvol) {   // upload the next volume once its buffer has been consumed
      if (i >= 1) ok = ck(cudaStreamWaitEvent(su, raw_free[s1], 0), "wait");
      ok = ok && ck(cudaMemcpyAsync(raw[s1], h_raw[i + 1], nraw * 2, cudaMemcpyHostToDevice, su), "upload") &&
           ck(cudaEventRecord(up[s1], su), "cudaEventRecord");
    }
    ok = ok && ck(cudaStreamWaitEvent(st, up[s], 0), "wait");
    if (i >= 2) ok = ok && ck(cudaStreamWaitEvent(st, out_free[s], 0), "wait");   // results i-2 downloaded
    if (!ok) break;
    int64_t nd = 0;
    const int32_t rs = run_compute(L, dim, n_raw, spacing, p, raw[s], dets[s], want_labels ? lab[s] : nullptr,
                                   max_cells, base, st, raw_free[s], &nd);
    if (rs != SNK_OK) { status = rs; break; }
    n_dets[i] = nd;
    ok = ck(cudaEventRecord(done[s], st), "cudaEventRecord") && ck(cudaStreamWaitEvent(sd, done[s], 0), "wait");
    const int64_t ncopy = std::min(nd, det_cap);
    if (ok && ncopy > 0)
      ok = ck(cudaMemcpyAsync(h_dets[i], dets[s], ncopy * sizeof(snk_cell), cudaMemcpyDeviceToHost, sd), "download");
    if (ok && want_labels && h_labels[i])
      ok = ck(cudaMemcpyAsync(h_labels[i], lab[s], niso * sizeof(int32_t), cudaMemcpyDeviceToHost, sd), "download");
    ok = ok && ck(cudaEventRecord(out_free[s], sd), "cudaEventRecord");
    if (nd > det_cap && status == SNK_OK) status = fail(SNK_CAPACITY, "detection buffer too small");
  }
  // drain and release (also on failure)
  if (su) { cudaStreamSynchronize(su); }
  if (sd) { cudaStreamSynchronize(sd); }
  cudaStreamSynchronize(st);
  for (int k = 0; k < 2; ++k) {
    if (up[k]) cudaEventDestroy(up[k]);
    if (raw_free[k]) cudaEventDestroy(raw_free[k]);
    if (done[k]) cudaEventDestroy(done[k]);
    if (out_free[k]) cudaEventDestroy(out_free[k]);
  }
  if (su) cudaStreamDestroy(su);
  if (sd) cudaStreamDestroy(sd);
  return status;
}

}  // extern "C"

static_assert(sizeof(snk_grid) == 88, "snk_grid layout is part of the ABI");
static_assert(sizeof(snk_params) == 136, "snk_params layout is part of the ABI");
static_assert(sizeof(snk_cell) == 64, "snk_cell layout is part of the ABI");
