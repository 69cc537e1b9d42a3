// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct fp64 CPU implementation of what the hot path
// of arXiv 1804.06304 ("Three-Dimensional GPU-Accelerated Active Contours for
// Automated Localization of Cells in Large Images") computes.  It exists to
// check the CUDA path; it is NOT part of the product.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it.  It shares no code, header, table or constant generator with
// paper_1804_06304_b200/ (the CUDA path); neither side includes the other.
//
// Citation keys: P:n = /root/reference/PAPER.md line n (section / equation),
// S:n = SPEC.md line n, §8(c) Ok = SURVEY.md §8(c) oracle item Ok, Gk = the
// gap reading Gk listed in DESIGN.md §3.
//
// Conventions
//   * volumes are x-fastest: idx = (z*ny + y)*nx + x;
//   * floating point is IEEE double, compiled with -ffp-contract=off so every
//     expression rounds exactly as written (no FMA contraction);
//   * integer volume passes use int64 accumulation (exact).
//
// Parity status of every function is listed in DESIGN.md §4; every function
// here is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---------------------------------------------------------------------------
// Status codes and cell flags — SURVEY §8(b) (mirrors SPEC's exit scheme S:524).
enum { ORA_OK = 0, ORA_EMPTY = 1, ORA_CONFIG = 2, ORA_SHAPE = 3, ORA_CAPACITY = 6 };
enum : uint32_t {
  F_CONVERGED = 1u, F_COLLAPSED = 2u, F_RMAX = 4u, F_DOMAIN = 8u,
  F_LEASHED = 16u, F_CULLED_E0 = 32u, F_CULLED_OVERLAP = 64u, F_HALO = 128u
};

const double PI = 3.14159265358979323846;
// rho = 2^(-1/d): P:93 (3D, "rho = 1/cbrt(2)") and P:68 (2D, "rho = 1/sqrt(2)").
// Written as the correctly rounded doubles; tests/test_oracle_constants.py pins
// them against high-precision evaluations.
const double RHO_3D = 0.7937005259840998;   // 2^(-1/3)
const double RHO_2D = 0.7071067811865476;   // 2^(-1/2)
// rho^2 for the label map's inner ball (G19): 2^(-2/3) and 1/2.
const double RHO2_3D = 0.6299605249474366;
const double RHO2_2D = 0.5;

inline double rho_of(int dim) { return dim == 3 ? RHO_3D : RHO_2D; }
inline double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., Random123) — the counter-based generator the
// north_star names; stream key per SPEC S:186/S:238 and G11:
//   ctr = {block b, iteration n, id_lo, id_hi}, key = {seed_lo, seed_hi}
// (the samples' words are laid out over the blocks by stream_word below).
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;   // Philox multipliers
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;   // Weyl key increments
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += W0; k1 += W1; }              // bump key between rounds
    const uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    const uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Uniform in [0,1) from 32 random bits: u = (x >> 9) * 2^-23 (G11).  Exact in
// both fp32 and fp64.
inline double uniform01(uint32_t x) { return (double)(x >> 9) * 0x1p-23; }

// ---------------------------------------------------------------------------
// §8(c) O5 steps 1-3 — one Monte-Carlo sample: a direction omega and a
// distance t, uniform in the ball (3D, "uniform sampling is done within a
// sphere with radius (R + dR/2)") or disk (2D, x = sqrt(r) cos(theta)).
//   3D direction by Archimedes' hat-box theorem (G10): z = 1 - 2u0, phi = 2 pi u1;
//   3D radius t = rho_s * cbrt(u2) (volume-uniform radial law);
//   2D radius t = rho_s * sqrt(u2).
// Word w of the stream of one cell-iteration (G11): word w is output w mod 4 of
// Philox4x32-10 at ctr = {floor(w / 4), n, id_lo, id_hi}, key = seed.  A 3D
// sample j takes words 3j, 3j+1, 3j+2 (u0, u1, u2); a 2D sample j takes words
// 2j, 2j+1 (u1, u2): every generated word is used exactly once.
uint32_t stream_word(uint64_t w, uint32_t iter, int64_t id, uint64_t seed) {
  const uint32_t ctr[4] = {(uint32_t)(w >> 2), iter, (uint32_t)((uint64_t)id & 0xffffffffu),
                           (uint32_t)((uint64_t)id >> 32)};
  const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  uint32_t x[4];
  philox4x32_10(ctr, key, x);
  return x[w & 3];
}

void mc_sample(int dim, uint32_t j, uint32_t iter, int64_t id, uint64_t seed,
               double rho_s, double omega[3], double* t) {
  double u0 = 0.0, u1, u2;
  if (dim == 3) {
    u0 = uniform01(stream_word(3ull * j, iter, id, seed));
    u1 = uniform01(stream_word(3ull * j + 1, iter, id, seed));
    u2 = uniform01(stream_word(3ull * j + 2, iter, id, seed));
  } else {
    u1 = uniform01(stream_word(2ull * j, iter, id, seed));
    u2 = uniform01(stream_word(2ull * j + 1, iter, id, seed));
  }
  const double phi = 2.0 * PI * u1;
  if (dim == 3) {
    const double z = 1.0 - 2.0 * u0;
    const double st = 2.0 * std::sqrt(u0 * (1.0 - u0));
    omega[0] = st * std::cos(phi);
    omega[1] = st * std::sin(phi);
    omega[2] = z;
    *t = rho_s * std::cbrt(u2);
  } else {
    omega[0] = std::cos(phi);
    omega[1] = std::sin(phi);
    omega[2] = 0.0;
    *t = rho_s * std::sqrt(u2);
  }
}

// ---------------------------------------------------------------------------
// §8(c) O5 step 6 — the weight S(r) of Eq. 5 (Fig. 4c/d) and its
// partial derivatives.  Reading G1: S = B(r; R, dR) - 2 B(r; rho R, rho dR)
// where B(r; a, w) = 1 - s3((r - (a - w/2)) / w) is a C^1 smoothstep ramp from
// 1 to 0 of width w centred at a; s3(u) = 3u^2 - 2u^3 on clamp(u, 0, 1).
// Inner ramp width rho*dR = dR / cbrt(2) = dr ("Delta r = Delta R/cbrt 2").
// Plateaus: -1 inside rho R, +1 in the annulus, 0 beyond R + dR/2 (Fig. 4d).
inline double s3(double u) { u = clampd(u, 0.0, 1.0); return u * u * (3.0 - 2.0 * u); }
inline double ds3(double u) { return (u <= 0.0 || u >= 1.0) ? 0.0 : 6.0 * u * (1.0 - u); }

void weight(double r, double R, double dR, double rho, double* S, double* S_r, double* S_R) {
  const double tau_o = (r - (R - dR / 2.0)) / dR;
  const double tau_i = (r - rho * (R - dR / 2.0)) / (rho * dR);
  *S = (1.0 - s3(tau_o)) - 2.0 * (1.0 - s3(tau_i));
  *S_r = -ds3(tau_o) / dR + 2.0 * ds3(tau_i) / (rho * dR);   // dS/dr
  *S_R = ds3(tau_o) / dR - 2.0 * ds3(tau_i) / dR;             // dS/dR
}

// ---------------------------------------------------------------------------
// The image I(x) of Eq. 2 at a non-integer point: d-linear interpolation of the
// u16 smoothed volume (G17), clamp-to-edge, scaled by iscale
// (G6: u16 -> 8-bit units, 1/257).  The volume buffer may hold only a box of a
// volume of global size n: voxels org + [0, nb) (z-slabs, §8(e), or a crop
// used by the full-size tests); a lookup outside the box is clamped into it
// and reported via *halo.
struct Image {
  const uint16_t* v;
  int64_t n[3];
  int64_t org[3], nb[3];
  int dim;
  double iscale;
  double scale[3];   // physical voxel size per axis (G28); the lookup point is k / scale

  double voxel(int64_t x, int64_t y, int64_t z, bool* halo) const {
    int64_t p[3] = {x - org[0], y - org[1], z - org[2]};
    for (int a = 0; a < 3; ++a)
      if (p[a] < 0 || p[a] >= nb[a]) { *halo = true; p[a] = clampi(p[a], 0, nb[a] - 1); }
    return (double)v[(p[2] * nb[1] + p[1]) * nb[0] + p[0]];
  }

  // trilinear (bilinear in 2D): clamp k to [0, n-1], i0 = min(floor(k), n-2),
  // f = k - i0, interpolate in x, then y, then z (§8(c) O5 step 4).
  double interp(const double kp[3], bool* halo) const {
    int64_t i0[3] = {0, 0, 0};
    double f[3] = {0.0, 0.0, 0.0};
    const double k[3] = {kp[0] / scale[0], kp[1] / scale[1], kp[2] / scale[2]};
    for (int a = 0; a < dim; ++a) {
      const double kc = clampd(k[a], 0.0, (double)(n[a] - 1));
      if (n[a] == 1) { i0[a] = 0; f[a] = 0.0; continue; }
      i0[a] = std::min((int64_t)std::floor(kc), n[a] - 2);
      f[a] = kc - (double)i0[a];
    }
    auto lerp = [](double a, double b, double t) { return a + t * (b - a); };
    const int64_t x = i0[0], y = i0[1], z = i0[2];
    const double c00 = lerp(voxel(x, y, z, halo), voxel(x + 1, y, z, halo), f[0]);
    const double c10 = lerp(voxel(x, y + 1, z, halo), voxel(x + 1, y + 1, z, halo), f[0]);
    const double c0 = lerp(c00, c10, f[1]);
    if (dim == 2) return iscale * c0;
    const double c01 = lerp(voxel(x, y, z + 1, halo), voxel(x + 1, y, z + 1, halo), f[0]);
    const double c11 = lerp(voxel(x, y + 1, z + 1, halo), voxel(x + 1, y + 1, z + 1, halo), f[0]);
    const double c1 = lerp(c01, c11, f[1]);
    return iscale * lerp(c0, c1, f[2]);
  }
};

}  // namespace

// ===========================================================================
// Public C ABI of the oracle (loaded by oracle/__init__.py through ctypes).
// ===========================================================================
extern "C" {

struct ora_params {
  double r0, delta_R, eps0, e0, iscale, max_step, r_min, r_max, leash, conv_tol;
  int32_t max_iters, n_samples, dim, mode;   // mode 0 MC, 1 grid (Eq. 5), 2 MC + control variate, 3 ray march
  uint64_t seed;
  // physical size of a voxel along each axis in the contour's units (SURVEY
  // §8(f) 4, reading G28): 1 = isotropic; an anisotropic volume is sampled at
  // raw coordinate k_a / scale_a without resampling (MC modes only)
  double scale[3];
};

struct ora_cell {
  double c[3];
  double R;
  double E;
  double seed[3];
  uint32_t flags;
  int32_t iters;
  int64_t id;
};

int ora_abi_version(void) { return 1; }

// rho_3D, rho_2D, rho^2_3D, rho^2_2D — pinned against high precision in tests.
void ora_constants(double* out4) { out4[0] = RHO_3D; out4[1] = RHO_2D; out4[2] = RHO2_3D; out4[3] = RHO2_2D; }

void ora_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox4x32_10(ctr, key, out);
}

void ora_sample(int dim, uint32_t j, uint32_t iter, int64_t id, uint64_t seed, double rho_s,
                double* omega3, double* t) {
  mc_sample(dim, j, iter, id, seed, rho_s, omega3, t);
}

void ora_weight(double r, double R, double dR, int dim, double* out3) {
  weight(r, R, dR, rho_of(dim), &out3[0], &out3[1], &out3[2]);
}

// ---------------------------------------------------------------------------
// §8(c) O1 — isotropic resampling ("the images were re-sampled to obtain
// a uniform pixel size"; G16).  Target spacing s_min = min spacing;
// an axis with s_a > s_min gets n' = round(n s_a / s_min) samples; output k maps
// to src = (k + 0.5) * (s_min / s_a) - 0.5 (centre-aligned), clamped to
// [0, n-1]; i0 = min(floor(src), n-2); w1 = round(16384 (src - i0)); the value
// is (v[i0] (16384 - w1) + v[i0+1] w1 + 8192) >> 14.  Axes are processed in
// the order x, y, z, each pass rounding to u16.
void ora_resample_dims(const int64_t n[3], const double spacing[3], int dim, int64_t nout[3]) {
  double smin = spacing[0];
  for (int a = 1; a < dim; ++a) smin = std::min(smin, spacing[a]);
  for (int a = 0; a < 3; ++a) {
    nout[a] = n[a];
    if (a < dim && spacing[a] > smin) nout[a] = (int64_t)std::llround((double)n[a] * spacing[a] / smin);
  }
}

int ora_resample(const uint16_t* in, const int64_t n[3], const double spacing[3], int dim,
                 uint16_t* out) {
  double smin = spacing[0];
  for (int a = 1; a < dim; ++a) smin = std::min(smin, spacing[a]);
  std::vector<uint16_t> cur(in, in + n[0] * n[1] * n[2]);
  int64_t cn[3] = {n[0], n[1], n[2]};
  for (int a = 0; a < dim; ++a) {
    if (!(spacing[a] > smin)) continue;
    const int64_t na = cn[a];
    const int64_t nn = (int64_t)std::llround((double)na * spacing[a] / smin);
    const double ratio = smin / spacing[a];
    std::vector<int64_t> i0(nn), w1(nn);
    for (int64_t k = 0; k < nn; ++k) {
      double src = ((double)k + 0.5) * ratio - 0.5;
      src = clampd(src, 0.0, (double)(na - 1));
      if (na == 1) { i0[k] = 0; w1[k] = 0; continue; }
      i0[k] = std::min((int64_t)std::floor(src), na - 2);
      w1[k] = (int64_t)std::floor(16384.0 * (src - (double)i0[k]) + 0.5);
    }
    int64_t on[3] = {cn[0], cn[1], cn[2]};
    on[a] = nn;
    std::vector<uint16_t> nxt(on[0] * on[1] * on[2]);
    const int64_t stride_in[3] = {1, cn[0], cn[0] * cn[1]};
    const int64_t stride_out[3] = {1, on[0], on[0] * on[1]};
    for (int64_t z = 0; z < on[2]; ++z)
      for (int64_t y = 0; y < on[1]; ++y)
        for (int64_t x = 0; x < on[0]; ++x) {
          int64_t p[3] = {x, y, z};
          const int64_t k = p[a];
          p[a] = i0[k];
          const int64_t base = p[0] * stride_in[0] + p[1] * stride_in[1] + p[2] * stride_in[2];
          const int64_t v0 = cur[base];
          const int64_t v1 = (na == 1) ? v0 : cur[base + stride_in[a]];
          const int64_t v = (v0 * (16384 - w1[k]) + v1 * w1[k] + 8192) >> 14;
          nxt[x * stride_out[0] + y * stride_out[1] + z * stride_out[2]] = (uint16_t)v;
        }
    cur.swap(nxt);
    cn[a] = nn;
  }
  std::memcpy(out, cur.data(), cur.size() * sizeof(uint16_t));
  return ORA_OK;
}

// ---------------------------------------------------------------------------
// §8(c) O2 — the low-pass filter of P:202 ("it can be mathematically enforced
// using a low-pass filter"), read as a separable Gaussian truncated at 4 sigma
// and renormalised, with integer Q14 taps (G18):
//   h = ceil(4 sigma), g_i = exp(-i^2 / (2 sigma^2)), w_i = round(16384 g_i / sum g),
//   centre tap adjusted so that sum w = 16384; sigma = 0 is the identity.
int ora_q14_taps(double sigma, int32_t* taps, int cap) {
  if (!(sigma > 0.0)) {
    if (cap < 1) return -1;
    taps[0] = 16384;
    return 0;
  }
  const int h = (int)std::ceil(4.0 * sigma);
  if (2 * h + 1 > cap) return -1;
  std::vector<double> g(2 * h + 1);
  double sum = 0.0;
  for (int i = -h; i <= h; ++i) { g[i + h] = std::exp(-(double)(i * i) / (2.0 * sigma * sigma)); sum += g[i + h]; }
  int64_t tot = 0;
  for (int i = 0; i <= 2 * h; ++i) { taps[i] = (int32_t)std::floor(16384.0 * g[i] / sum + 0.5); tot += taps[i]; }
  taps[h] += (int32_t)(16384 - tot);
  return h;
}

// Passes x, then y, then z (3D only): out = (sum_i w_i in[clamp(x + i)] + 8192) >> 14.
// ora_blur3: a sigma per axis (in voxels of that axis) — on an anisotropic grid
// sampled without resampling the physical sigma becomes sigma / scale_a (G28).
int ora_blur3(const uint16_t* in, const int64_t n[3], int dim, const double sigma[3], uint16_t* out) {
  int32_t taps[3][257];
  int h[3];
  for (int a = 0; a < 3; ++a) {
    h[a] = ora_q14_taps(sigma[a], taps[a], 257);
    if (h[a] < 0) return ORA_CONFIG;
  }
  const int64_t N = n[0] * n[1] * n[2];
  std::vector<uint16_t> cur(in, in + N), nxt(N);
  const int64_t stride[3] = {1, n[0], n[0] * n[1]};
  for (int a = 0; a < dim; ++a) {
    const int ha = h[a];
    const int32_t* ta = taps[a];
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < n[2]; ++z)
      for (int64_t y = 0; y < n[1]; ++y)
        for (int64_t x = 0; x < n[0]; ++x) {
          const int64_t p[3] = {x, y, z};
          const int64_t base = x + y * stride[1] + z * stride[2] - p[a] * stride[a];
          int64_t acc = 0;
          for (int i = -ha; i <= ha; ++i) {
            const int64_t q = clampi(p[a] + i, 0, n[a] - 1);
            acc += (int64_t)ta[i + ha] * (int64_t)cur[base + q * stride[a]];
          }
          nxt[x + y * stride[1] + z * stride[2]] = (uint16_t)((acc + 8192) >> 14);
        }
    cur.swap(nxt);
  }
  std::memcpy(out, cur.data(), N * sizeof(uint16_t));
  return ORA_OK;
}

int ora_blur(const uint16_t* in, const int64_t n[3], int dim, double sigma, uint16_t* out) {
  const double s3[3] = {sigma, sigma, sigma};
  return ora_blur3(in, n, dim, s3, out);
}

// ---------------------------------------------------------------------------
// §8(c) O3 — gradient magnitude (north_star "trilinear samples of gradient
// magnitude"; reading in SURVEY §0.3): central differences in index space with
// clamp-to-edge, g_a = B[x + e_a] - B[x - e_a]; G = (isqrt(gx^2 + gy^2 + gz^2) + 1) >> 1.
static uint64_t isqrt_u64(uint64_t v) {
  uint64_t r = (uint64_t)std::sqrt((double)v);
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return r;
}

int ora_gradmag(const uint16_t* B, const int64_t n[3], int dim, uint16_t* out) {
  const int64_t stride[3] = {1, n[0], n[0] * n[1]};
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < n[2]; ++z)
    for (int64_t y = 0; y < n[1]; ++y)
      for (int64_t x = 0; x < n[0]; ++x) {
        const int64_t p[3] = {x, y, z};
        const int64_t idx = x + y * stride[1] + z * stride[2];
        uint64_t s = 0;
        for (int a = 0; a < dim; ++a) {
          const int64_t up = clampi(p[a] + 1, 0, n[a] - 1), dn = clampi(p[a] - 1, 0, n[a] - 1);
          const int64_t g = (int64_t)B[idx + (up - p[a]) * stride[a]] - (int64_t)B[idx + (dn - p[a]) * stride[a]];
          s += (uint64_t)(g * g);
        }
        out[idx] = (uint16_t)((isqrt_u64(s) + 1) >> 1);
      }
  return ORA_OK;
}

// ---------------------------------------------------------------------------
// §8(c) O4 LATTICE — initial contours on a lattice spaced sqrt(1.5) R0 apart
// (Fig. 1b caption, Fig. 4b caption), every footprint
// (radius m = R0 + dR/2) inside the domain.  Cubic lattice,
// centred in each axis: with L = n - 1, k = floor((L - 2m)/s) + 1 and offset
// o = m + ((L - 2m) - (k - 1) s)/2.  Ids z-major, x fastest.  Status EMPTY if
// any lattice axis has L - 2m < 0 ("reported as a distinct condition").
// ora_seeds_lattice3: on an anisotropic grid (G28) the lattice lives in
// physical units: axis extent L = (n - 1) scale, output in physical coordinates.
int ora_seeds_lattice3(const int64_t n[3], int dim, double r0, double dR, const double scale[3],
                       float* out_xyz, int64_t cap, int64_t* count) {
  const double m = r0 + dR / 2.0;
  const double s = std::sqrt(1.5) * r0;
  int64_t k[3] = {1, 1, 1};
  double o[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < dim; ++a) {
    const double span = (double)(n[a] - 1) * scale[a] - 2.0 * m;
    if (span < 0.0) { *count = 0; return ORA_EMPTY; }
    k[a] = (int64_t)std::floor(span / s) + 1;
    o[a] = m + (span - (double)(k[a] - 1) * s) / 2.0;
  }
  const int64_t total = k[0] * k[1] * k[2];
  *count = total;
  if (total > cap) return ORA_CAPACITY;
  int64_t id = 0;
  for (int64_t iz = 0; iz < k[2]; ++iz)
    for (int64_t iy = 0; iy < k[1]; ++iy)
      for (int64_t ix = 0; ix < k[0]; ++ix, ++id) {
        out_xyz[3 * id + 0] = (float)(o[0] + (double)ix * s);
        out_xyz[3 * id + 1] = (float)(o[1] + (double)iy * s);
        out_xyz[3 * id + 2] = dim == 3 ? (float)(o[2] + (double)iz * s) : 0.0f;
      }
  return ORA_OK;
}

int ora_seeds_lattice(const int64_t n[3], int dim, double r0, double dR, float* out_xyz,
                      int64_t cap, int64_t* count) {
  const double one[3] = {1.0, 1.0, 1.0};
  return ora_seeds_lattice3(n, dim, r0, dR, one, out_xyz, cap, count);
}

// §8(c) O4 MAXIMA — seed detection (north_star; reading G20, "any method
// that reliably places initial contours").  x is a seed iff B(x) >= thr and no
// y in the (2w+1)^d box W(x) (clipped to the volume) has B(y) > B(x), or
// B(y) = B(x) with lin(y) < lin(x).  Seeds are listed in linear-index order.
// The buffer holds the box org + [0, nb) of a global volume n; the box
// lo..hi (inclusive, global coordinates) is scanned.  Every scanned window
// must lie inside the buffer (the slab driver and the crop tests size their
// margins for that); returns SHAPE otherwise.
struct Box {
  const uint16_t* B;
  int64_t n[3], org[3], nb[3];
  uint16_t at(int64_t x, int64_t y, int64_t z) const {
    return B[((z - org[2]) * nb[1] + (y - org[1])) * nb[0] + (x - org[0])];
  }
};

// per-axis half-widths w[a] (an anisotropic grid: w / scale_a voxels, G28)
static bool is_maxima_seed(const Box& b, int dim, const int w[3], uint32_t thr, int64_t x, int64_t y,
                           int64_t z) {
  const int64_t nx = b.n[0], ny = b.n[1];
  const uint16_t v = b.at(x, y, z);
  if ((uint32_t)v < thr) return false;
  const int64_t lin = (z * ny + y) * nx + x;
  const int64_t z0 = dim == 3 ? std::max<int64_t>(z - w[2], 0) : z;
  const int64_t z1 = dim == 3 ? std::min<int64_t>(z + w[2], b.n[2] - 1) : z;
  for (int64_t zz = z0; zz <= z1; ++zz)
    for (int64_t yy = std::max<int64_t>(y - w[1], 0); yy <= std::min<int64_t>(y + w[1], ny - 1); ++yy)
      for (int64_t xx = std::max<int64_t>(x - w[0], 0); xx <= std::min<int64_t>(x + w[0], nx - 1); ++xx) {
        const uint16_t u = b.at(xx, yy, zz);
        if (u > v) return false;
        if (u == v && (zz * ny + yy) * nx + xx < lin) return false;
      }
  return true;
}

static bool window_inside(const Box& b, int dim, const int w[3], const int64_t lo[3], const int64_t hi[3]) {
  for (int a = 0; a < dim; ++a) {
    const int64_t wl = std::max<int64_t>(lo[a] - w[a], 0), wh = std::min<int64_t>(hi[a] + w[a], b.n[a] - 1);
    if (wl < b.org[a] || wh >= b.org[a] + b.nb[a]) return false;
  }
  return true;
}

int ora_is_maxima_seed(const uint16_t* B, const int64_t n[3], const int64_t org[3],
                       const int64_t nb[3], int dim, int w, uint32_t thr, int64_t x, int64_t y,
                       int64_t z) {
  Box b{B, {n[0], n[1], n[2]}, {org[0], org[1], org[2]}, {nb[0], nb[1], nb[2]}};
  const int64_t p[3] = {x, y, z};
  const int w3[3] = {w, w, w};
  if (!window_inside(b, dim, w3, p, p)) return -1;
  return is_maxima_seed(b, dim, w3, thr, x, y, z) ? 1 : 0;
}

// ora_seeds_maxima3: per-axis half-widths w3 and output in physical
// coordinates (voxel index x scale, G28); ora_seeds_maxima: w3 = (w, w, w), scale 1.
int ora_seeds_maxima3(const uint16_t* B, const int64_t n[3], const int64_t org[3],
                      const int64_t nb[3], const int64_t lo[3], const int64_t hi[3], int dim,
                      const int w3[3], const double scale[3], uint32_t thr, float* out_xyz,
                      int64_t cap, int64_t* count) {
  const int* w = w3;
  Box b{B, {n[0], n[1], n[2]}, {org[0], org[1], org[2]}, {nb[0], nb[1], nb[2]}};
  if (!window_inside(b, dim, w, lo, hi)) return ORA_SHAPE;
  const int64_t nplanes = hi[2] - lo[2] + 1;
  std::vector<std::vector<int64_t>> per_plane(nplanes > 0 ? nplanes : 0);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t zi = 0; zi < nplanes; ++zi) {
    const int64_t z = lo[2] + zi;
    for (int64_t y = lo[1]; y <= hi[1]; ++y)
      for (int64_t x = lo[0]; x <= hi[0]; ++x)
        if (is_maxima_seed(b, dim, w, thr, x, y, z))
          per_plane[zi].push_back((z * n[1] + y) * n[0] + x);
  }
  int64_t total = 0;
  for (auto& v : per_plane) total += (int64_t)v.size();
  *count = total;
  if (total > cap) return ORA_CAPACITY;
  int64_t i = 0;
  for (auto& v : per_plane)
    for (int64_t lin : v) {
      out_xyz[3 * i + 0] = (float)((double)(lin % n[0]) * scale[0]);
      out_xyz[3 * i + 1] = (float)((double)((lin / n[0]) % n[1]) * scale[1]);
      out_xyz[3 * i + 2] = (float)((double)(lin / (n[0] * n[1])) * scale[2]);
      ++i;
    }
  return ORA_OK;
}

int ora_seeds_maxima(const uint16_t* B, const int64_t n[3], const int64_t org[3],
                     const int64_t nb[3], const int64_t lo[3], const int64_t hi[3], int dim, int w,
                     uint32_t thr, float* out_xyz, int64_t cap, int64_t* count) {
  const int w3[3] = {w, w, w};
  const double one[3] = {1.0, 1.0, 1.0};
  return ora_seeds_maxima3(B, n, org, nb, lo, hi, dim, w3, one, thr, out_xyz, cap, count);
}

// ---------------------------------------------------------------------------
// Energies of one contour (c, R).  All return out[0] = E, out[1..3] = dE/dc,
// out[4] = dE/dR, plus out[5] = 1 if a lookup left the slab buffer.
//
// Normalisation (G3): gamma = 1/(q_x - p_x)^d = (2R)^-d  (Eq. 6),
// alpha = d.  Gradients (G4): Eqs. 7-10 rewritten
// for (c, R) = ((p+q)/2, (q_x - p_x)/2):
//   dE/dc = gamma * sum S_r(r) I(k) dr/dc = -gamma * sum S_r I omega,
//   dE/dR = gamma * (sum S_R I - (d/R) sum S I).
struct EnergyOut { double E, gc[3], gR; bool halo; };

// Monte-Carlo estimate: N samples uniform in the ball of radius
// rho_s = R + dR/2, each of weight V/N, V = ball volume.  r := t and the
// unit vector := omega (never recomputed from k - c; §8(c) O5 step 5).
// Control variate (mode 2, reading G21 / SURVEY §8(f) 4): I(k) is replaced by
// I(k) - I(c).  Unbiased for the same integrals because the ball integrals of
// S, S_R and S_r omega are all zero (the zero moment of G1, its R-derivative
// with S(rho_s) = 0, and the symmetry of omega); on a uniform image every sum
// is then exactly zero ("the energy is zero ... uniform intensity").
static EnergyOut energy_mc(const Image& img, const ora_params& p, const double c[3], double R,
                           uint32_t iter, int64_t id) {
  const int d = p.dim;
  const double rho = rho_of(d);
  const double rho_s = R + p.delta_R / 2.0;
  double A0 = 0.0, Ac[3] = {0.0, 0.0, 0.0}, AR = 0.0;
  bool halo = false;
  const double Ic = (p.mode == 2) ? img.interp(c, &halo) : 0.0;
  for (int32_t j = 0; j < p.n_samples; ++j) {
    double om[3], t;
    mc_sample(d, (uint32_t)j, iter, id, p.seed, rho_s, om, &t);
    const double k[3] = {c[0] + t * om[0], c[1] + t * om[1], c[2] + t * om[2]};
    const double I = img.interp(k, &halo) - Ic;
    double S, S_r, S_R;
    weight(t, R, p.delta_R, rho, &S, &S_r, &S_R);
    A0 += S * I;
    for (int a = 0; a < 3; ++a) Ac[a] += S_r * I * om[a];
    AR += S_R * I;
  }
  const double V = (d == 3) ? (4.0 / 3.0) * PI * rho_s * rho_s * rho_s / (double)p.n_samples
                            : PI * rho_s * rho_s / (double)p.n_samples;
  A0 *= V; AR *= V;
  for (int a = 0; a < 3; ++a) Ac[a] *= V;
  const double gamma = std::pow(2.0 * R, -(double)d);
  EnergyOut o;
  o.E = gamma * A0;
  for (int a = 0; a < 3; ++a) o.gc[a] = -gamma * Ac[a];
  o.gR = gamma * (AR - ((double)d / R) * A0);
  o.halo = halo;
  return o;
}

// Stratified ray-march estimate (mode 3: the north_star's
// "marches a ray"; reading G27).  The ball integral in polar form,
//   int_ball f dV = int_{S^{d-1}} int_0^{rho_s} f(t omega) t^{d-1} dt d omega,
// estimated with N/M rays of M = 8 stratified steps: ray j has direction
// omega_j (the MC direction law of G10 from words 0, 1) and steps
// t_jm = rho_s (m + u_jm) / M, m = 0..M-1, u_jm uniform (words 2 + m); its
// Philox words are the 12 words of blocks 3j, 3j+1, 3j+2 of the cell-iteration
// stream (words 10, 11 unused).  Each step weighs |S^{d-1}| rho_s t^{d-1} / N
// (|S^2| = 4 pi, |S^1| = 2 pi): unbiased for every stratum and direction.
static const int RAY_M = 8;
static EnergyOut energy_ray(const Image& img, const ora_params& p, const double c[3], double R,
                            uint32_t iter, int64_t id) {
  const int d = p.dim;
  const double rho = rho_of(d);
  const double rho_s = R + p.delta_R / 2.0;
  double A0 = 0.0, Ac[3] = {0.0, 0.0, 0.0}, AR = 0.0;
  bool halo = false;
  const int32_t rays = p.n_samples / RAY_M;
  for (int32_t j = 0; j < rays; ++j) {
    uint32_t x[12];
    for (int w = 0; w < 12; ++w) x[w] = stream_word(12ull * (uint64_t)j + (uint64_t)w, iter, id, p.seed);
    const double u0 = uniform01(x[0]), u1 = uniform01(x[1]);
    const double phi = 2.0 * PI * u1;
    double om[3];
    if (d == 3) {
      const double z = 1.0 - 2.0 * u0;
      const double st = 2.0 * std::sqrt(u0 * (1.0 - u0));
      om[0] = st * std::cos(phi); om[1] = st * std::sin(phi); om[2] = z;
    } else {
      om[0] = std::cos(phi); om[1] = std::sin(phi); om[2] = 0.0;
    }
    for (int m = 0; m < RAY_M; ++m) {
      const double t = rho_s * ((double)m + uniform01(x[2 + m])) / (double)RAY_M;
      const double k[3] = {c[0] + t * om[0], c[1] + t * om[1], c[2] + t * om[2]};
      const double Iw = img.interp(k, &halo) * (d == 3 ? t * t : t);
      double S, S_r, S_R;
      weight(t, R, p.delta_R, rho, &S, &S_r, &S_R);
      A0 += S * Iw;
      for (int a = 0; a < 3; ++a) Ac[a] += S_r * Iw * om[a];
      AR += S_R * Iw;
    }
  }
  const double V = (d == 3 ? 4.0 * PI : 2.0 * PI) * rho_s / (double)(rays * RAY_M);
  A0 *= V; AR *= V;
  for (int a = 0; a < 3; ++a) Ac[a] *= V;
  const double gamma = std::pow(2.0 * R, -(double)d);
  EnergyOut o;
  o.E = gamma * A0;
  for (int a = 0; a < 3; ++a) o.gc[a] = -gamma * Ac[a];
  o.gR = gamma * (AR - ((double)d / R) * A0);
  o.halo = halo;
  return o;
}

// Uniform-grid estimate, Eq. 5: sum over the voxels k with
// |k - c| < R + dR/2 of S(|k - c|) I(k), unit voxel volume.  At r = 0 the
// radial term is 0.  Oracle-only (grid mode, O8).
static EnergyOut energy_grid(const Image& img, const ora_params& p, const double c[3], double R) {
  const int d = p.dim;
  const double rho = rho_of(d);
  const double rho_s = R + p.delta_R / 2.0;
  double A0 = 0.0, Ac[3] = {0.0, 0.0, 0.0}, AR = 0.0;
  bool halo = false;
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    lo[a] = std::max<int64_t>((int64_t)std::floor(c[a] - rho_s), 0);
    hi[a] = std::min<int64_t>((int64_t)std::ceil(c[a] + rho_s), img.n[a] - 1);
  }
  for (int64_t z = lo[2]; z <= hi[2]; ++z)
    for (int64_t y = lo[1]; y <= hi[1]; ++y)
      for (int64_t x = lo[0]; x <= hi[0]; ++x) {
        const double dx = (double)x - c[0], dy = (double)y - c[1], dz = d == 3 ? (double)z - c[2] : 0.0;
        const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
        if (!(r < rho_s)) continue;
        const double I = img.iscale * img.voxel(x, y, z, &halo);
        double S, S_r, S_R;
        weight(r, R, p.delta_R, rho, &S, &S_r, &S_R);
        A0 += S * I;
        if (r > 0.0) { Ac[0] += S_r * I * dx / r; Ac[1] += S_r * I * dy / r; Ac[2] += S_r * I * dz / r; }
        AR += S_R * I;
      }
  const double gamma = std::pow(2.0 * R, -(double)d);
  EnergyOut o;
  o.E = gamma * A0;
  for (int a = 0; a < 3; ++a) o.gc[a] = -gamma * Ac[a];
  o.gR = gamma * (AR - ((double)d / R) * A0);
  o.halo = halo;
  return o;
}

static Image make_image(const uint16_t* v, const int64_t n[3], const int64_t org[3],
                        const int64_t nb[3], const ora_params* p) {
  Image img;
  img.v = v;
  for (int a = 0; a < 3; ++a) {
    img.n[a] = n[a];
    img.org[a] = org ? org[a] : 0;
    img.nb[a] = nb ? nb[a] : n[a];
  }
  img.dim = p->dim;
  img.iscale = p->iscale;
  for (int a = 0; a < 3; ++a) img.scale[a] = p->scale[a] > 0.0 ? p->scale[a] : 1.0;
  return img;
}

void ora_energy_mc(const uint16_t* v, const int64_t n[3], const int64_t org[3], const int64_t nb[3],
                   const ora_params* p, const double c[3], double R, uint32_t iter, int64_t id,
                   double* out6) {
  const Image img = make_image(v, n, org, nb, p);
  const EnergyOut o = p->mode == 3 ? energy_ray(img, *p, c, R, iter, id) : energy_mc(img, *p, c, R, iter, id);
  out6[0] = o.E; out6[1] = o.gc[0]; out6[2] = o.gc[1]; out6[3] = o.gc[2]; out6[4] = o.gR;
  out6[5] = o.halo ? 1.0 : 0.0;
}

// The d-linear lookup itself (§8(c) O5 step 4, G17), exposed so that tests pin
// it directly: out[i] = iscale * I(k_i) at the physical points k_i (xyz).
void ora_interp(const uint16_t* v, const int64_t n[3], const int64_t org[3], const int64_t nb[3],
                const ora_params* p, const double* k_xyz, int64_t npts, double* out, int32_t* halo_out) {
  const Image img = make_image(v, n, org, nb, p);
  for (int64_t i = 0; i < npts; ++i) {
    bool halo = false;
    out[i] = img.interp(&k_xyz[3 * i], &halo);
    if (halo_out) halo_out[i] = halo ? 1 : 0;
  }
}

void ora_energy_grid(const uint16_t* v, const int64_t n[3], const int64_t org[3], const int64_t nb[3],
                     const ora_params* p, const double c[3], double R, double* out6) {
  const Image img = make_image(v, n, org, nb, p);
  const EnergyOut o = energy_grid(img, *p, c, R);
  out6[0] = o.E; out6[1] = o.gc[0]; out6[2] = o.gc[1]; out6[3] = o.gc[2]; out6[4] = o.gR;
  out6[5] = o.halo ? 1.0 : 0.0;
}

// E_ss (O8): supersampled quadrature of the d-linear interpolant, q^d midpoints
// per voxel, i.e. the continuous integral the MC estimator is unbiased for.
double ora_energy_ss(const uint16_t* v, const int64_t n[3], const ora_params* p, const double c[3],
                     double R, int q) {
  const Image img = make_image(v, n, nullptr, nullptr, p);
  const int d = p->dim;
  const double rho = rho_of(d);
  const double rho_s = R + p->delta_R / 2.0;
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    lo[a] = (int64_t)std::floor(c[a] - rho_s) - 1;
    hi[a] = (int64_t)std::ceil(c[a] + rho_s) + 1;
  }
  double A0 = 0.0;
  const int qz = d == 3 ? q : 1;
#pragma omp parallel for reduction(+ : A0) schedule(static)
  for (int64_t z = lo[2]; z <= hi[2]; ++z) {
    bool halo = false;
    for (int64_t y = lo[1]; y <= hi[1]; ++y)
      for (int64_t x = lo[0]; x <= hi[0]; ++x)
        for (int az = 0; az < qz; ++az)
          for (int ay = 0; ay < q; ++ay)
            for (int ax = 0; ax < q; ++ax) {
              const double k[3] = {(double)x + (ax + 0.5) / q, (double)y + (ay + 0.5) / q,
                                   d == 3 ? (double)z + (az + 0.5) / q : 0.0};
              const double dx = k[0] - c[0], dy = k[1] - c[1], dz = d == 3 ? k[2] - c[2] : 0.0;
              const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
              if (!(r < rho_s)) continue;
              double S, S_r, S_R;
              weight(r, R, p->delta_R, rho, &S, &S_r, &S_R);
              A0 += S * img.interp(k, &halo);
            }
  }
  A0 /= std::pow((double)q, (double)d);
  return std::pow(2.0 * R, -(double)d) * A0;
}

// ---------------------------------------------------------------------------
// §8(c) O5 — contour evolution (Eqs. 11-14): for n = 1..T,
// (p, q) <- (p, q) - eps_n grad E with eps_n = eps0 / sqrt(n), which in
// (c, R) is a step of eps_n / 2 (c = (p+q)/2, R = (q_x - p_x)/2).  Safeguards
// (G8): each component of the step clipped to +-max_step; R clamped to
// [r_min, r_max]; leash c_a in [s_a - leash, s_a + leash]; domain c_a in
// [m, n_a - 1 - m], m = R + dR/2, or (n_a - 1)/2 if the axis is
// shorter than 2m.  Iteration T+1 only evaluates E_final (G13).  CONVERGED if the
// state moved by less than conv_tol (max norm) in iteration T (G9);
// cells are never frozen.  Stops at T = max_iters.
// One contour from its current state through iterations it0..it1 (1 <= it0,
// it1 <= T + 1); the state is the record itself: c, R, E, seed (the leash
// centre), flags (accumulated), id (the Philox stream key).
static void evolve_cell(const Image& img, const ora_params* p, const int64_t n[3], int it0, int it1,
                        ora_cell& cell) {
  const int d = p->dim;
  const int T = p->max_iters;
  const double* s = cell.seed;
  double c[3] = {cell.c[0], cell.c[1], cell.c[2]};
  double R = cell.R;
  uint32_t flags = cell.flags;
  double E = cell.E;
  for (int it = it0; it <= it1; ++it) {
    const EnergyOut eo = (p->mode == 1)   ? energy_grid(img, *p, c, R)
                         : (p->mode == 3) ? energy_ray(img, *p, c, R, (uint32_t)it, cell.id)
                                          : energy_mc(img, *p, c, R, (uint32_t)it, cell.id);
    if (eo.halo) flags |= F_HALO;
    E = eo.E;
    if (it == T + 1) break;
    const double eps = p->eps0 / std::sqrt((double)it);
    const double c_old[3] = {c[0], c[1], c[2]};
    const double R_old = R;
    for (int a = 0; a < 3; ++a) c[a] += clampd(-(eps / 2.0) * eo.gc[a], -p->max_step, p->max_step);
    R = clampd(R + clampd(-(eps / 2.0) * eo.gR, -p->max_step, p->max_step), p->r_min, p->r_max);
    bool leashed = false, domained = false;
    for (int a = 0; a < 3; ++a) {
      const double cl = clampd(c[a], s[a] - p->leash, s[a] + p->leash);
      if (cl != c[a]) leashed = true;
      c[a] = cl;
    }
    const double m = R + p->delta_R / 2.0;
    for (int a = 0; a < 3; ++a) {
      // the domain in physical units: [0, (n_a - 1) scale_a] (G28)
      const double L = (double)(n[a] - 1) * img.scale[a];
      double cd;
      if (L < 2.0 * m) cd = L / 2.0;
      else cd = clampd(c[a], m, L - m);
      if (cd != c[a] && a < d) domained = true;
      c[a] = cd;
    }
    if (it == T) {
      double mv = std::fabs(R - R_old);
      for (int a = 0; a < 3; ++a) mv = std::max(mv, std::fabs(c[a] - c_old[a]));
      if (mv < p->conv_tol) flags |= F_CONVERGED;
      if (leashed) flags |= F_LEASHED;
      if (domained) flags |= F_DOMAIN;
    }
  }
  // trivial contours as of the last iteration run
  flags &= ~(uint32_t)(F_COLLAPSED | F_RMAX);
  if (R <= p->r_min) flags |= F_COLLAPSED;
  if (R >= p->r_max) flags |= F_RMAX;
  for (int a = 0; a < 3; ++a) cell.c[a] = c[a];
  cell.R = R;
  cell.E = E;
  cell.flags = flags;
  cell.iters = std::min(it1, T);
}

void ora_evolve(const uint16_t* v, const int64_t n[3], const int64_t org[3], const int64_t nb[3],
                const ora_params* p, const float* seeds_xyz, const int64_t* ids, int64_t ncell,
                ora_cell* out) {
  const Image img = make_image(v, n, org, nb, p);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < ncell; ++i) {
    ora_cell& o = out[i];
    for (int a = 0; a < 3; ++a) o.c[a] = o.seed[a] = (double)seeds_xyz[3 * i + a];
    o.R = p->r0;
    o.E = 0.0;
    o.flags = 0;
    o.iters = 0;
    o.id = ids[i];
    evolve_cell(img, p, n, 1, p->max_iters + 1, o);
  }
}

// Periodic culling ("dynamic culling"; reading G25 in
// DESIGN.md): evolution in segments.  Continues every record of cells[] from
// its state through iterations it0..it1; E is the MC (grid) energy of
// iteration it1 (E_final when it1 = T + 1), COLLAPSED / RMAX reflect the
// radius after it1.  ora_evolve = one segment 1..T+1.
void ora_evolve_range(const uint16_t* v, const int64_t n[3], const int64_t org[3],
                      const int64_t nb[3], const ora_params* p, ora_cell* cells, int64_t ncell,
                      int32_t it0, int32_t it1) {
  const Image img = make_image(v, n, org, nb, p);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < ncell; ++i) evolve_cell(img, p, n, it0, it1, cells[i]);
}

// ---------------------------------------------------------------------------
// §8(c) O6 — culling: contours with E > E0 are removed, then
// overlapping contours, |c' - c''| < max(R', R'')/2^(1/d), compete and the lower
// energy survives.  Readings G14 (E0 first), G15 (greedy in (E asc, id asc)
// order = lexicographically-first maximal independent set).  COLLAPSED
// and RMAX cells are trivial contours and never candidates.  Inputs are the fp32
// cell values; comparisons are in fp64 without contraction: keep i iff for every
// kept a, dx^2 + dy^2 + dz^2 >= (rho * max(R_i, R_a))^2.
// Writes the survivors' input indices in (E, id) order to keep_idx.
int ora_cull(const float* c_xyz, const float* R, const float* E, const uint32_t* flags,
             const int64_t* ids, int64_t n, int dim, double e0, int64_t* keep_idx, int64_t* n_keep) {
  const double rho = rho_of(dim);
  std::vector<int64_t> cand;
  for (int64_t i = 0; i < n; ++i)
    if ((double)E[i] <= e0 && !(flags[i] & (F_COLLAPSED | F_RMAX))) cand.push_back(i);
  std::sort(cand.begin(), cand.end(), [&](int64_t a, int64_t b) {
    if (E[a] != E[b]) return E[a] < E[b];
    return ids[a] < ids[b];
  });
  // the kept cells' values (exact fp32 -> fp64 conversions) in kept order
  std::vector<int64_t> kept;
  std::vector<double> kx, ky, kz, kR;
  for (int64_t i : cand) {
    const double cx = (double)c_xyz[3 * i], cy = (double)c_xyz[3 * i + 1], cz = (double)c_xyz[3 * i + 2];
    const double Ri = (double)R[i];
    // "for every kept a: d2 >= t^2" — an AND over the kept set (order-free;
    // OpenMP splits the set when it is large)
    const int64_t nk = (int64_t)kept.size();
    int ok = 1;
#pragma omp parallel for reduction(&& : ok) schedule(static) if (nk > 8192)
    for (int64_t a = 0; a < nk; ++a) {
      const double dx = cx - kx[a];
      const double dy = cy - ky[a];
      const double dz = cz - kz[a];
      const double d2 = dx * dx + dy * dy + dz * dz;
      const double t = rho * std::max(Ri, kR[a]);
      ok = ok && (d2 >= t * t);
    }
    if (ok) {
      kept.push_back(i);
      kx.push_back(cx); ky.push_back(cy); kz.push_back(cz); kR.push_back(Ri);
    }
  }
  *n_keep = (int64_t)kept.size();
  for (size_t k = 0; k < kept.size(); ++k) keep_idx[k] = kept[k];
  return ORA_OK;
}

// ---------------------------------------------------------------------------
// §8(c) O7 — voxel label map (north_star "voxel label map out"; reading G19):
// voxel x belongs to detection i iff it lies in i's inner ball, radius rho R_i
// (at the Eq. 3 optimum R* = cbrt(2) r0 the inner ball is the nucleus,
// P:96-100).  d2 = sum_a (x_a - c_a)^2 (double, left to right, no FMA),
// thr = (R_i R_i) rho^2, key = d2 / thr; the winner is the minimum key among
// detections with d2 <= thr, ties to the smaller index; label = index + 1, or 0.
static int32_t label_of(int dim, double x, double y, double z, const float* c_xyz, const float* R,
                        int64_t k) {
  const double rho2 = dim == 3 ? RHO2_3D : RHO2_2D;
  int64_t best = -1;
  double best_key = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    const double dx = x - (double)c_xyz[3 * i];
    const double dy = y - (double)c_xyz[3 * i + 1];
    double d2 = dx * dx + dy * dy;
    if (dim == 3) { const double dz = z - (double)c_xyz[3 * i + 2]; d2 = d2 + dz * dz; }
    const double thr = ((double)R[i] * (double)R[i]) * rho2;
    if (d2 <= thr) {
      const double key = d2 / thr;
      if (best < 0 || key < best_key) { best = i; best_key = key; }
    }
  }
  return (int32_t)(best + 1);
}

// ora_label3: voxel (x, y, z) sits at the physical point (x sx, y sy, z sz) (G28).
int ora_label3(const int64_t n[3], int dim, int64_t z0, int64_t nz, const double scale[3],
               const float* c_xyz, const float* R, int64_t k, int32_t* labels) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t zi = 0; zi < nz; ++zi)
    for (int64_t y = 0; y < n[1]; ++y)
      for (int64_t x = 0; x < n[0]; ++x)
        labels[(zi * n[1] + y) * n[0] + x] =
            label_of(dim, (double)x * scale[0], (double)y * scale[1], (double)(z0 + zi) * scale[2],
                     c_xyz, R, k);
  return ORA_OK;
}

int ora_label(const int64_t n[3], int dim, int64_t z0, int64_t nz, const float* c_xyz,
              const float* R, int64_t k, int32_t* labels) {
  const double one[3] = {1.0, 1.0, 1.0};
  return ora_label3(n, dim, z0, nz, one, c_xyz, R, k, labels);
}

int ora_label_points(int dim, const int64_t* pts_xyz, int64_t npts, const float* c_xyz,
                     const float* R, int64_t k, int32_t* labels) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npts; ++i)
    labels[i] = label_of(dim, (double)pts_xyz[3 * i], (double)pts_xyz[3 * i + 1],
                         (double)pts_xyz[3 * i + 2], c_xyz, R, k);
  return ORA_OK;
}

int ora_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ora_set_num_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

}  // extern "C"
