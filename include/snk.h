/*
 * snk.h — C ABI of libsnk.so, the B200 (sm_100a) hot path of arXiv 1804.06304
 * ("Three-Dimensional GPU-Accelerated Active Contours for Automated
 * Localization of Cells in Large Images"): batched Monte-Carlo evolution of
 * independent 3D snakuscules plus the volume passes around it.
 *
 * Citation keys: P:n = PAPER.md line n (section / equation), S:n = SPEC.md
 * line n, Gk = reading k of the paper in DESIGN.md §3.
 *
 * Problem statement (north_star): volume + seeds + parameters in,
 * per-cell (centre, radius, energy) records and a voxel label map out.
 *
 * Conventions (every function)
 *   - Volumes are u16, x fastest: idx = ((z - z_lo) * ny + y) * nx + x.
 *   - Device pointers (d_*) are CALLER-OWNED and borrowed for the call; the
 *     library never allocates device memory.  Scratch memory is the caller's
 *     workspace d_ws of at least snk_workspace_bytes() bytes.  Host pointers
 *     (h_*) are plain host memory (pinned memory makes the copies async).
 *   - Every call that launches work takes a cudaStream_t (as void*) and is
 *     asynchronous on it, EXCEPT the calls that return a count to the host
 *     (snk_seeds, snk_compact_candidates, snk_cull, snk_run): those
 *     synchronise the stream before returning.
 *   - Every function returns an snk_status; no C++ exception crosses the ABI.
 *     On failure snk_last_error() (thread-local) describes the cause; CUDA
 *     errors keep the CUDA error string.  Per-cell problems are flags, never
 *     errors.  An empty result is SNK_OK with a count of 0.
 */
#ifndef SNK_H
#define SNK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNK_ABI_VERSION 5

/* Status codes — mirror SPEC's exit scheme plus CUDA / capacity. */
typedef enum {
  SNK_OK = 0,
  SNK_EMPTY_DOMAIN = 1, /* no seed can be placed */
  SNK_CONFIG = 2,       /* a parameter invariant is violated */
  SNK_SHAPE = 3,        /* size mismatch, unsupported dims, halo too thin */
  SNK_INTERNAL = 4,
  SNK_CUDA = 5,         /* a CUDA call failed; the CUDA error text is kept */
  SNK_CAPACITY = 6      /* output buffer too small; the required count is still written */
} snk_status;

/* Per-cell flags (snk_cell.flags) — SURVEY §8(b). */
enum {
  SNK_F_CONVERGED = 1u,       /* state moved < conv_tol in iteration T (G9) */
  SNK_F_COLLAPSED = 2u,       /* R reached r_min (trivial contour) */
  SNK_F_RMAX = 4u,            /* R reached r_max (runaway) */
  SNK_F_DOMAIN = 8u,          /* domain clamp active in iteration T */
  SNK_F_LEASHED = 16u,        /* leash clamp active in iteration T */
  SNK_F_CULLED_E0 = 32u,      /* reserved: E > E0 */
  SNK_F_CULLED_OVERLAP = 64u, /* reserved: lost an overlap competition */
  SNK_F_HALO = 128u           /* a gather fell outside the slab buffer (halo too thin) */
};

enum { SNK_SEED_LATTICE = 0, SNK_SEED_MAXIMA = 1, SNK_SEED_GIVEN = 2 };
enum { SNK_IMAGE_INTENSITY = 0, SNK_IMAGE_GRADMAG = 1 };
/* How the energy integral of Eq. 5 is evaluated each iteration:
 *   SNK_EST_MC   N Monte-Carlo samples uniform in the ball — the path;
 *   SNK_EST_GRID the paper's original uniform integration, Eq. 5 summed over the
 *                voxels k with |k - c| < R + dR/2 (unit voxel volume, I(k) read
 *                at the voxel, the radial term 0 at r = 0) — deterministic,
 *                no samples (n_samples is ignored); the baseline MC replaced
 *                ("~4X gain");
 *   SNK_EST_MC_CV MC with the control variate I(c) subtracted from every sample
 *                (reading G21): unbiased for the same integrals, exactly zero on a
 *                uniform image;
 *   SNK_EST_RAY  stratified ray march (reading G27): N/8 rays per cell-iteration,
 *                ray j's direction from words 0, 1 of Philox blocks 3j..3j+2 and
 *                8 steps t = rho_s (m + u_m)/8 (words 2..9), each weighted
 *                |S^(d-1)| rho_s t^(d-1) / N.
 *   MC_CV and RAY run in the brick kernel with 8 samples per thread:
 *   n_samples = 256 * warps per cell (cta_warps 0 or 4: N = 1024; 8: N = 2048). */
enum { SNK_EST_MC = 0, SNK_EST_GRID = 1, SNK_EST_MC_CV = 2, SNK_EST_RAY = 3 };

/* Geometry of the (isotropic) volume and of this rank's slab (§8(e)).
 *   n[3]        global dims (x, y, z); 2D images have dim = 2 and n[2] = 1.
 *   z_lo,nz_buf the device volume buffers hold global planes [z_lo, z_lo+nz_buf).
 *   own_z0/1    planes this rank owns: seeds are detected, and labels written,
 *               only for z in [own_z0, own_z1).  Single GPU: z_lo = own_z0 = 0,
 *               nz_buf = own_z1 = n[2].
 *   scale[3]    physical size of a voxel along each axis, in the contour's units
 *               (reading G28): {1, 1, 1} (or zeros) = isotropic.  An
 *               anisotropic raw volume is then used WITHOUT resampling: centres,
 *               radii, seeds and detections are physical; a lookup at physical k
 *               reads the grid at k_a / scale_a; the blur sigma of axis a is
 *               sigma / scale_a voxels, the MAXIMA half-window floor(w / scale_a +
 *               0.5) voxels; labels are decided at the voxels' physical positions.
 *               Needs x extent % 8 == 0 (vectorised volume passes) and the brick
 *               evolve kernel with 8 samples per thread (N = 256 x warps); the
 *               grid estimator and the gradient-magnitude image term are isotropic
 *               only. */
typedef struct snk_grid {
  int32_t dim;
  int32_t _pad0;
  int64_t n[3];
  int64_t z_lo, nz_buf;
  int64_t own_z0, own_z1;
  double scale[3];
} snk_grid;

/* Parameters (S:259-263 SwarmConfig; defaults in DESIGN.md §3):
 *   r0        initial radius R0 (15 px)         delta_R  ramp width dR (G2, fixed voxels)
 *   eps0      step scale, eps_n = eps0/sqrt(n) e0       energy threshold E0 (-3)
 *   sigma     Gaussian low-pass sigma (G18)      intensity_scale  u16 -> image units (G6)
 *   max_step, r_min, r_max, leash  safeguards (G8)       conv_tol CONVERGED tolerance (G9)
 *   max_iters T (400)                            n_samples N per cell-iteration, a power of 2
 *   seed_mode LATTICE | MAXIMA | GIVEN                  seed_window w, seed_threshold thr (G20)
 *   image_term INTENSITY | GRADMAG                      cta_warps warps per cell: 0 auto, 1, 2, 4, 8
 *   kernel_variant  0 auto (N < 128: group kernel; else brick kernel when nx is even),
 *             1 warp kernel, 2 brick kernel, 3 group kernel (N / 8 lanes per cell, 4..16)
 *   estimator SNK_EST_MC | SNK_EST_GRID | SNK_EST_MC_CV | SNK_EST_RAY (not MC: brick
 *             kernel only, even nx)
 *   cull_every  periodic culling ("dynamic culling", reading G25): 0 = off
 *             (the paper's end-of-run cull only); k > 0 = after iterations k, 2k, ...
 *             (< T) the live cells go through the a7 cull (E0, then the overlap
 *             competition, on their state after that iteration and its energy) and
 *             only the survivors evolve on.  Used by snk_run and the drivers; the
 *             building blocks are snk_cells_init / snk_evolve_range / snk_cull.
 *   seed      Philox key (G11) */
typedef struct snk_params {
  double r0, delta_R, eps0, e0, sigma, intensity_scale, max_step, r_min, r_max, leash, conv_tol;
  int32_t max_iters, n_samples, seed_mode, seed_window, image_term, cta_warps;
  uint32_t seed_threshold;
  uint32_t kernel_variant; /* evolve kernel: 0 auto, 1 warp (global gathers), 2 brick (shared memory), 3 group */
  int32_t estimator;       /* SNK_EST_MC (default), _GRID, _MC_CV or _RAY */
  int32_t cull_every;      /* 0 off, else periodic culling every cull_every iterations (G25) */
  uint64_t seed;
} snk_params;

/* One contour (64 bytes): the per-cell "radius field" (a sphere: r(omega) = R),
 * centre, seed, final energy E_final (G13), flags, iterations run, global id.
 * disp = c - seed is the evolved state itself: the kernels step the
 * displacement from the seed (fp32 resolution ~2e-6 voxel at |disp| < 32)
 * rather than the absolute centre (resolution 1.2e-4 voxel at x ~ 2000, which
 * let the fp32 trajectory drift ~1e-3 voxel from the fp64 oracle's on C4);
 * c = seed + disp rounded to fp32.  snk_evolve_range resumes from disp, so a
 * segmented run is bit-identical to an uninterrupted one. */
typedef struct snk_cell {
  float c[3];
  float R;
  float seed[3];
  float energy;
  uint32_t flags;
  int32_t iters;
  int64_t id;
  float disp[3];
  uint32_t reserved; /* 0 */
} snk_cell;

int32_t snk_abi_version(void);
const char* snk_last_error(void);
const char* snk_status_string(int32_t status);

/* Check grid/params invariants (e0 <= 0, max_iters >= 1, r0 > r_min;
 * n_samples a power of two >= 32 * warps-per-cell; dims >= 2 on every used
 * axis; planes inside the volume).  No device work. */
int32_t snk_validate(const snk_grid* g, const snk_params* p);

/* Bytes of device workspace any single call below needs for cells up to
 * max_cells (the calls run in stream order and may share one workspace). */
int32_t snk_workspace_bytes(const snk_grid* g, const snk_params* p, int64_t max_cells,
                            size_t* bytes);

/* a1 — isotropic resampling ("re-sampled to obtain a uniform pixel size";
 * S:358-366; G16).  Target spacing s_min = min spacing; axis a with s_a > s_min
 * gets round(n_a s_a / s_min) samples; output k reads source (k + 0.5) s_min/s_a
 * - 0.5 (clamped), i0 = min(floor, n-2), w1 = round(16384 frac) and writes
 * (v[i0](16384 - w1) + v[i0+1] w1 + 8192) >> 14; axes x, y, z in order.
 * snk_resample_dims computes the output dims (host only).
 * Output planes [z_lo, z_lo + nz_out) are produced from raw planes
 * [zr_lo, zr_lo + nzr) (z-slabs); SHAPE if the needed raw planes are missing.
 * Needs workspace when more than one axis is resampled. */
int32_t snk_resample_dims(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                          int64_t n_out[3]);
int32_t snk_resample(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                     int64_t zr_lo, int64_t nzr, const uint16_t* d_raw, int64_t z_lo,
                     int64_t nz_out, uint16_t* d_out, void* d_ws, size_t ws_bytes,
                     void* stream);

/* a2 + a3 — the low-pass filter of P:202 (G18): separable Gaussian,
 * truncated at 4 sigma, Q14 integer taps summing to 16384, passes x, y, z each
 * (sum w_i v[clamp(x+i)] + 8192) >> 14 (clamp-to-edge at the buffer's planes).
 * Optional gradient magnitude (north_star; O3): G = (isqrt(gx^2+gy^2+gz^2)+1)>>1
 * with clamped central differences.  d_in, d_smooth, d_gradmag (nullable) each
 * hold nz_buf planes. */
int32_t snk_preprocess(const snk_grid* g, const snk_params* p, const uint16_t* d_in,
                       uint16_t* d_smooth, uint16_t* d_gradmag, void* d_ws, size_t ws_bytes,
                       void* stream);

/* a0 — ingest of an 8-bit volume (SPEC S:348-356, S:402 dtype "u8"; SURVEY
 * 8(c) O0): d_out[i] = 257 * d_in[i], the exact u16 image of the 8-bit value
 * (0 -> 0, 255 -> 65535), for n voxels (x-fastest layout unchanged).  Device
 * buffers are the caller's; any alignment (16-byte aligned buffers take the
 * vectorised kernel).  Asynchronous on `stream`. */
int32_t snk_ingest_u8(const uint8_t* d_in, uint16_t* d_out, int64_t n, void* stream);

/* a4 — seeds (P:169 lattice "located at a distance sqrt(1.5) R apart", P:238;
 * north_star seed detection, G20).  LATTICE: centred cubic lattice spaced
 * sqrt(1.5) r0, footprint m = r0 + dR/2 inside (EMPTY_DOMAIN if it does not fit),
 * ids z-major x fastest.  MAXIMA: x with B(x) >= thr that is the first (lowest
 * linear index) maximum of its (2w+1)^d box clipped to the volume; listed in
 * linear-index order.  Writes fp32 xyz triples for z in [own_z0, own_z1) to
 * d_seeds (capacity cap) and the count to *n_out (host).  LATTICE with slabs
 * also writes *first_id_out (host; nullable) = the global lattice index of the
 * first seed.  Synchronises the stream. */
int32_t snk_seeds(const snk_grid* g, const snk_params* p, const uint16_t* d_smooth,
                  float* d_seeds, int64_t cap, int64_t* n_out, int64_t* first_id_out,
                  void* d_ws, size_t ws_bytes, void* stream);

/* a5 + a6 — contour evolution (Eqs. 11-14 with eps0/sqrt(n); MC
 * integration P:191-207; gradients Eqs. 7-10 in (c, R) form, G3/G4).  For each
 * cell i (global id = d_ids ? d_ids[i] : id_base + i) from c = seed, R = r0: for
 * n = 1..T, N Philox4x32-10 samples keyed {j, n, id_lo, id_hi}/{seed} give a
 * direction omega and distance t uniform in the ball of radius R + dR/2; the
 * image (d_image: smoothed intensity or gradient magnitude) is sampled
 * trilinearly at c + t omega; the weights S, dS/dr, dS/dR (G1) give E and its
 * gradient; (c, R) takes a clipped step of eps_n/2 (G8) with the R, leash and
 * domain clamps.  Iteration T+1 only computes E_final (G13).  Writes n records
 * to d_cells.  Reductions use a fixed pairwise tree: results are bit-identical
 * for every cta_warps setting and every rank decomposition. */
int32_t snk_evolve(const snk_grid* g, const snk_params* p, const uint16_t* d_image,
                   const float* d_seeds, const int64_t* d_ids, int64_t id_base, int64_t n,
                   snk_cell* d_cells, void* d_ws, size_t ws_bytes, void* stream);

/* Periodic culling (G25) — evolution in segments.  snk_cells_init writes
 * the records of cells at the start of evolution (c = seed = d_seeds[i], R = r0,
 * E = 0, flags = 0, id = d_ids ? d_ids[i] : id_base + i).  snk_evolve_range
 * continues the n records of d_cells IN PLACE (their c, R, E, seed = leash
 * centre, flags and id are the whole state) through iterations it0..it1
 * (1 <= it0 <= it1 <= T + 1, the step schedule eps0/sqrt(n) and every rule of
 * snk_evolve unchanged); afterwards E is the energy of iteration it1 (E_final if
 * it1 = T + 1) and COLLAPSED / RMAX reflect the radius after it1.  Evolving
 * 1..k, then k+1..T+1 gives records bit-identical to snk_evolve.  Between
 * segments, snk_cull(d_cells -> survivors) is the checkpoint cull; the
 * survivors (any order) are the next segment's records.  Asynchronous. */
int32_t snk_cells_init(const snk_params* p, const float* d_seeds, const int64_t* d_ids,
                       int64_t id_base, int64_t n, snk_cell* d_cells, void* stream);
int32_t snk_evolve_range(const snk_grid* g, const snk_params* p, const uint16_t* d_image,
                         snk_cell* d_cells, int64_t n, int32_t it0, int32_t it1, void* d_ws,
                         size_t ws_bytes, void* stream);

/* a7, first half — the energy cull ("energy greater than a threshold
 * (E0) are also removed", G14): copies cells with E <= e0 that are neither
 * COLLAPSED nor RMAX to d_out, preserving order; count to *n_out (host).
 * Used before exchanging candidates between ranks.  Synchronises. */
int32_t snk_compact_candidates(const snk_params* p, const snk_cell* d_cells, int64_t n,
                               snk_cell* d_out, int64_t cap, int64_t* n_out, void* d_ws,
                               size_t ws_bytes, void* stream);

/* Multi-GPU periodic culling (§8(e), G25): after a checkpoint cull of the
 * all-gathered candidates, each rank keeps the survivors it owns, i.e. the
 * records with id_lo <= id < id_hi (its exclusive prefix of seed counts).
 * Order-preserving copy of those records of d_cells to d_out; count to *n_out
 * (host).  Workspace: as snk_compact_candidates.  Synchronises. */
int32_t snk_select_ids(const snk_cell* d_cells, int64_t n, int64_t id_lo, int64_t id_hi,
                       snk_cell* d_out, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                       void* stream);

/* a7 — culling: E0 filter as above, then the overlap competition
 * |c' - c''| < max(R', R'')/2^(1/d) -> the lower energy survives, resolved as
 * the greedy in (E asc, id asc) order (G15), i.e. keep i iff for every
 * kept a: dx^2+dy^2+dz^2 >= (rho max(R_i, R_a))^2 in fp64 from the fp32 values.
 * Writes the detections to d_dets in (E, id) order; count to *n_out (host).
 * Synchronises. */
int32_t snk_cull(const snk_grid* g, const snk_params* p, const snk_cell* d_cells, int64_t n,
                 snk_cell* d_dets, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                 void* stream);

/* a8 — voxel label map (north_star; G19): voxel x gets 1 + the index i of the
 * detection whose inner ball (radius rho R_i, the nucleus at the Eq. 3 optimum,
 * P:96-100) contains it with the smallest key d2/thr (d2 = sum (x_a - c_a)^2,
 * thr = (R_i R_i) rho^2, IEEE fp64, ties to the smaller index), else 0.  Writes
 * int32 planes [own_z0, own_z1) to d_labels. */
int32_t snk_label(const snk_grid* g, const snk_params* p, const snk_cell* d_dets, int64_t n,
                  int32_t* d_labels, void* d_ws, size_t ws_bytes, void* stream);

/* Whole path on one GPU from HOST buffers (the end-to-end call): copies the
 * raw volume h_raw (dims n_raw, spacing) to the device, runs a1 (if
 * anisotropic) .. a8, and copies the detections (and labels if h_labels is
 * non-null; dims of the isotropic volume) back.  Device memory: the caller's
 * d_ws of snk_run_workspace_bytes().  Synchronises. */
int32_t snk_run_workspace_bytes(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                                const snk_params* p, int64_t max_cells, size_t* bytes);
int32_t snk_run(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                const snk_params* p, const uint16_t* h_raw, snk_cell* h_dets, int64_t det_cap,
                int64_t* n_dets, int32_t* h_labels, int64_t max_cells, void* d_ws,
                size_t ws_bytes, void* stream);

/* snk_run for an 8-bit raw volume: h_raw holds n_raw voxels of
 * u8; they are uploaded as bytes (half the host->device traffic of u16) and
 * promoted on the device by snk_ingest_u8, then the path runs exactly as
 * snk_run on the u16 volume 257 * h_raw (bit-identical results).  Same
 * workspace (snk_run_workspace_bytes).  Synchronises. */
int32_t snk_run_u8(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                   const snk_params* p, const uint8_t* h_raw, snk_cell* h_dets, int64_t det_cap,
                   int64_t* n_dets, int32_t* h_labels, int64_t max_cells, void* d_ws,
                   size_t ws_bytes, void* stream);

/* snk_run over nvol volumes of the same shape (the end-to-end call for a
 * stream of volumes): volume i is read from h_raw[i], its detections written to
 * h_dets[i] (capacity det_cap each, count n_dets[i]) and, if h_labels is
 * non-null and h_labels[i] non-null, its label map to h_labels[i].  The upload
 * of volume i+1 and the download of volume i-1's results run on two internal
 * streams while volume i's kernels run on `stream` (double-buffered device
 * volume, detections and labels in the caller's workspace of
 * snk_run_batch_workspace_bytes() bytes), so host<->device copies overlap the
 * kernels.  Pinned host buffers are needed for the overlap.  Results are those
 * of nvol snk_run calls.  Synchronises. */
int32_t snk_run_batch_workspace_bytes(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                                      const snk_params* p, int64_t max_cells, size_t* bytes);
int32_t snk_run_batch(int32_t dim, const int64_t n_raw[3], const double spacing[3],
                      const snk_params* p, int64_t nvol, const uint16_t* const* h_raw,
                      snk_cell* const* h_dets, int64_t det_cap, int64_t* n_dets,
                      int32_t* const* h_labels, int64_t max_cells, void* d_ws, size_t ws_bytes,
                      void* stream);

/* Diagnostics: number of kernel launches issued by this thread since load. */
int64_t snk_launch_count(void);

/* Diagnostics of the evolve brick kernel on the current device since the last
 * reset: out4[0] = brick (re)loads, out4[1] = cell-iterations that gathered
 * from global memory (sampled ball larger than the brick), out4[2..3] = 0.
 * reset != 0 zeroes the counters.  Synchronous. */
int32_t snk_evolve_stats(int64_t* out4, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* SNK_H */
