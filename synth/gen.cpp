// synth/gen.cpp — seeded synthetic input generator (SURVEY §8(d) "Synthetic
// inputs").  Serves both the oracle tests and the CUDA path; it holds none of
// the method's arithmetic (no Philox, no blur, no energy): DAPI-like bright
// ellipsoidal nuclei on a dark, slowly modulated background with additive
// Gaussian noise, as in the paper's data, written as u16.
//
// Every voxel is a pure function of (spec, voxel index): nuclei parameters come
// from a splitmix64 hash keyed by the nucleus' lattice index, noise from a hash
// keyed by the voxel's linear index, so any z-range can be generated on its own
// (z-slabs, §8(e)).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return splitmix64(splitmix64(seed ^ splitmix64(a)) ^ (b * 0xD1B54A32D192ED03ull));
}
// uniform in (0, 1): 53 random bits, never exactly 0
inline double unif(uint64_t h) { return ((double)(h >> 11) + 0.5) * 0x1p-53; }
inline double normal(uint64_t h1, uint64_t h2) {
  const double u1 = unif(h1), u2 = unif(h2);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

}  // namespace

extern "C" {

struct synth_spec {
  int32_t dim;            // 2 or 3
  int32_t _pad;
  int64_t n[3];           // raw voxel dims (x, y, z); z = 1 in 2D
  double spacing[3];      // raw voxel spacing; nuclei live in isotropic units of min spacing
  int64_t count[3];       // nuclei per axis on the lattice
  double pitch[3];        // lattice pitch (isotropic units)
  double origin[3];       // centre of lattice cell 0 (isotropic units)
  double jitter;          // centre jitter U(-jitter, +jitter) per axis (isotropic units)
  double rbar_lo, rbar_hi;// mean radius U(rbar_lo, rbar_hi)
  double axis_var;        // semi-axis = rbar (1 + U(-axis_var, axis_var))
  double amp, amp_cv;     // amplitude A = amp (1 + amp_cv N(0,1)), 8-bit units
  double edge;            // sigmoid edge width (voxels)
  double bg, bg_mod, bg_wavelength;  // background bg + bg_mod * modulation
  double noise;           // additive N(0, noise), 8-bit units
  uint64_t seed;
};

struct synth_nucleus {
  double c[3];
  double axes[3];
  double rot[9];   // row-major rotation: body = rot * (p - c)
  double amp;
  double rbar;
};

static void nucleus_params(const synth_spec* s, int64_t idx, synth_nucleus* nu) {
  const int64_t ix = idx % s->count[0];
  const int64_t iy = (idx / s->count[0]) % s->count[1];
  const int64_t iz = idx / (s->count[0] * s->count[1]);
  const int64_t ii[3] = {ix, iy, iz};
  for (int a = 0; a < 3; ++a) {
    const double j = a < s->dim ? (2.0 * unif(hash3(s->seed, idx, 10 + a)) - 1.0) * s->jitter : 0.0;
    nu->c[a] = a < s->dim ? s->origin[a] + (double)ii[a] * s->pitch[a] + j : 0.0;
  }
  nu->rbar = s->rbar_lo + (s->rbar_hi - s->rbar_lo) * unif(hash3(s->seed, idx, 20));
  for (int a = 0; a < 3; ++a)
    nu->axes[a] = nu->rbar * (1.0 + s->axis_var * (2.0 * unif(hash3(s->seed, idx, 30 + a)) - 1.0));
  nu->amp = s->amp * (1.0 + s->amp_cv * normal(hash3(s->seed, idx, 40), hash3(s->seed, idx, 41)));
  if (s->dim == 3) {
    // uniform random rotation from a normalised Gaussian quaternion
    double q[4];
    double nrm = 0.0;
    for (int k = 0; k < 4; ++k) {
      q[k] = normal(hash3(s->seed, idx, 50 + 2 * k), hash3(s->seed, idx, 51 + 2 * k));
      nrm += q[k] * q[k];
    }
    nrm = std::sqrt(nrm);
    const double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
    const double r[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                         2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                         2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)};
    std::memcpy(nu->rot, r, sizeof r);
  } else {
    const double th = 6.283185307179586 * unif(hash3(s->seed, idx, 60));
    const double r[9] = {std::cos(th), std::sin(th), 0, -std::sin(th), std::cos(th), 0, 0, 0, 1};
    std::memcpy(nu->rot, r, sizeof r);
  }
}

int64_t synth_num_nuclei(const synth_spec* s) { return s->count[0] * s->count[1] * s->count[2]; }

void synth_nuclei(const synth_spec* s, synth_nucleus* out) {
  const int64_t k = synth_num_nuclei(s);
  for (int64_t i = 0; i < k; ++i) nucleus_params(s, i, &out[i]);
}

// Isotropic position of raw voxel index i along axis a (centre-aligned).
static inline double iso_coord(const synth_spec* s, int a, double smin, int64_t i) {
  return ((double)i + 0.5) * (s->spacing[a] / smin) - 0.5;
}

// Generate raw planes [z0, z1) into out ((z1 - z0) * ny * nx u16, x fastest).
int synth_generate(const synth_spec* s, int64_t z0, int64_t z1, uint16_t* out) {
  const int d = s->dim;
  double smin = s->spacing[0];
  for (int a = 1; a < d; ++a) smin = std::min(smin, s->spacing[a]);
  const int64_t K = synth_num_nuclei(s);
  std::vector<synth_nucleus> nuc(K);
  for (int64_t i = 0; i < K; ++i) nucleus_params(s, i, &nuc[i]);
  const double cut = 8.0;    // sigmoid argument beyond which a nucleus contributes 0
  std::vector<double> ext(K);
  for (int64_t i = 0; i < K; ++i) {
    const double amax = std::max(nuc[i].axes[0], std::max(nuc[i].axes[1], nuc[i].axes[2]));
    ext[i] = amax * (1.0 + cut * s->edge / nuc[i].rbar) + 1.0;
  }
  const int64_t nx = s->n[0], ny = s->n[1];
  const double kz = (s->spacing[2] / smin);
  // bucket nuclei by the raw planes they touch
  const int64_t nzr = z1 - z0;
  std::vector<std::vector<int32_t>> plane_list(nzr);
  for (int64_t i = 0; i < K; ++i) {
    int64_t lo = 0, hi = 0;
    if (d == 3) {
      // raw index i maps to iso (i + 0.5) kz - 0.5
      lo = (int64_t)std::floor((nuc[i].c[2] - ext[i] + 0.5) / kz - 0.5) - 1;
      hi = (int64_t)std::ceil((nuc[i].c[2] + ext[i] + 0.5) / kz - 0.5) + 1;
    }
    lo = std::max(lo, z0);
    hi = std::min(hi, z1 - 1);
    for (int64_t z = lo; z <= hi; ++z) plane_list[z - z0].push_back((int32_t)i);
  }
#pragma omp parallel
  {
    std::vector<float> fg(nx * ny);
    std::vector<double> bx(nx);
#pragma omp for schedule(dynamic, 1)
    for (int64_t zi = 0; zi < nzr; ++zi) {
      const int64_t z = z0 + zi;
      std::fill(fg.begin(), fg.end(), 0.0f);
      const double pz = d == 3 ? iso_coord(s, 2, smin, z) : 0.0;
      for (int32_t i : plane_list[zi]) {
        const synth_nucleus& nu = nuc[i];
        const double e = ext[i];
        const double dz = pz - nu.c[2];
        if (d == 3 && std::fabs(dz) > e) continue;
        const double kx = s->spacing[0] / smin, ky = s->spacing[1] / smin;
        const double ec = std::sqrt(std::max(0.0, e * e - dz * dz)) + 1.0;   // bounding-sphere section
        const int64_t xlo = std::max<int64_t>(0, (int64_t)std::floor((nu.c[0] - ec + 0.5) / kx - 0.5));
        const int64_t xhi = std::min<int64_t>(nx - 1, (int64_t)std::ceil((nu.c[0] + ec + 0.5) / kx - 0.5));
        const int64_t ylo = std::max<int64_t>(0, (int64_t)std::floor((nu.c[1] - ec + 0.5) / ky - 0.5));
        const int64_t yhi = std::min<int64_t>(ny - 1, (int64_t)std::ceil((nu.c[1] + ec + 0.5) / ky - 0.5));
        const double rin = 1.0 - cut * s->edge / nu.rbar, rout = 1.0 + cut * s->edge / nu.rbar;
        const double ia0 = 1.0 / nu.axes[0], ia1 = 1.0 / nu.axes[1], ia2 = 1.0 / nu.axes[2];
        for (int64_t y = ylo; y <= yhi; ++y) {
          const double dy = iso_coord(s, 1, smin, y) - nu.c[1];
          for (int64_t x = xlo; x <= xhi; ++x) {
            const double dx = iso_coord(s, 0, smin, x) - nu.c[0];
            const double b0 = (nu.rot[0] * dx + nu.rot[1] * dy + nu.rot[2] * dz) * ia0;
            const double b1 = (nu.rot[3] * dx + nu.rot[4] * dy + nu.rot[5] * dz) * ia1;
            const double b2 = d == 3 ? (nu.rot[6] * dx + nu.rot[7] * dy + nu.rot[8] * dz) * ia2 : 0.0;
            const double rr = b0 * b0 + b1 * b1 + b2 * b2;
            if (rr >= rout * rout) continue;
            double v;
            if (rr <= rin * rin) v = nu.amp;
            else {
              const double arg = (1.0 - std::sqrt(rr)) * nu.rbar / s->edge;
              v = nu.amp / (1.0 + std::exp(-arg));
            }
            float& f = fg[y * nx + x];
            if ((float)v > f) f = (float)v;
          }
        }
      }
      // background modulation (separable) + noise: one hash per voxel pair,
      // Box-Muller gives the two normals of the pair.
      const double tw = 6.283185307179586 / s->bg_wavelength;
      const double mz = d == 3 ? std::sin(tw * pz + 2.0) : 1.0;
      for (int64_t x = 0; x < nx; ++x) bx[x] = std::sin(tw * iso_coord(s, 0, smin, x) + 0.3);
      for (int64_t y = 0; y < ny; ++y) {
        const double my = std::sin(tw * iso_coord(s, 1, smin, y) + 1.1) * mz;
        const uint64_t row = (uint64_t)((z * ny + y) * nx);
        for (int64_t x = 0; x < nx; x += 2) {
          const uint64_t h = splitmix64(s->seed ^ 0xA5A5A5A5A5A5A5A5ull ^ ((row + (uint64_t)x) * 0x9E3779B97F4A7C15ull));
          const double u1 = ((double)(h >> 40) + 0.5) * 0x1p-24, u2 = ((double)((h >> 16) & 0xFFFFFF) + 0.5) * 0x1p-24;
          const double rad = s->noise * std::sqrt(-2.0 * std::log(u1));
          const double ang = 6.283185307179586 * u2;
          const double nzs[2] = {rad * std::cos(ang), rad * std::sin(ang)};
          for (int k = 0; k < 2 && x + k < nx; ++k) {
            const double val = (s->bg + s->bg_mod * bx[x + k] * my + (double)fg[y * nx + x + k] + nzs[k]) * 257.0;
            const double r = std::floor(val + 0.5);
            out[(zi * ny + y) * nx + x + k] = (uint16_t)(r < 0.0 ? 0.0 : (r > 65535.0 ? 65535.0 : r));
          }
        }
      }
    }
  }
  return 0;
}

int synth_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
