// cull.cu — a7: the energy cull and the overlap competition, and the
// order-preserving candidate compaction used before a multi-GPU exchange.
//
// The paper's competition ("overlapping snakes ... undergo a competition with
// the lower energy snake surviving") is read as the greedy in (E asc, id asc)
// order (G15), i.e. the lexicographically-first maximal independent set of the
// overlap graph.  On the GPU: sort candidates by a 64-bit (E, id) key (bitonic
// sort), bin them on a uniform grid of pitch >= rho R_max, then decide in
// rounds: a cell is IN once every higher-priority overlapping cell is OUT, and
// OUT as soon as one is IN.  Decisions are final when made, so the fixed point
// equals the sequential greedy.  Overlap tests use IEEE fp64 without FMA on the
// fp32 cell values, exactly as the definition.
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace snk {

namespace {

constexpr uint32_t kCandMask = SNK_F_COLLAPSED | SNK_F_RMAX;
constexpr int kSortBlock = 1024;   // threads; 2 * kSortBlock keys per shared-memory tile

__device__ __forceinline__ bool is_candidate(const snk_cell& c, float e0) {
  return c.energy <= e0 && !(c.flags & kCandMask);
}

__device__ __forceinline__ uint32_t ord_float(float f) {
  uint32_t b = __float_as_uint(f == 0.0f ? 0.0f : f);   // canonical +0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void keys_kernel(const snk_cell* __restrict__ cells, int64_t n, int64_t npow2, float e0,
                            uint64_t* keys, int* vals, unsigned long long* ncand, int* bad_id) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npow2) return;
  uint64_t k = ~0ull;
  if (i < n) {
    const snk_cell c = cells[i];
    if (is_candidate(c, e0)) {
      if (c.id < 0 || c.id > 0xffffffffll) atomicExch(bad_id, 1);
      k = ((uint64_t)ord_float(c.energy) << 32) | (uint64_t)(uint32_t)c.id;
      atomicAdd(ncand, 1ull);
    }
  }
  keys[i] = k;
  vals[i] = (int)i;
}

__global__ void bitonic_global_kernel(uint64_t* keys, int* vals, int64_t j, int64_t k) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = i ^ j;
  if (p <= i) return;
  const bool asc = (i & k) == 0;
  const uint64_t a = keys[i], b = keys[p];
  if ((a > b) == asc) {
    keys[i] = b;
    keys[p] = a;
    const int t = vals[i];
    vals[i] = vals[p];
    vals[p] = t;
  }
}

// all steps j = jmax .. 1 of stage k inside 2 * kSortBlock-key tiles
__global__ void __launch_bounds__(kSortBlock) bitonic_shared_kernel(uint64_t* keys, int* vals,
                                                                    int64_t k, int64_t jmax) {
  __shared__ uint64_t sk[2 * kSortBlock];
  __shared__ int sv[2 * kSortBlock];
  const int64_t base = (int64_t)blockIdx.x * 2 * kSortBlock;
  const int t = threadIdx.x;
  sk[t] = keys[base + t];
  sv[t] = vals[base + t];
  sk[t + kSortBlock] = keys[base + t + kSortBlock];
  sv[t + kSortBlock] = vals[base + t + kSortBlock];
  __syncthreads();
  for (int64_t j = jmax; j >= 1; j >>= 1) {
    // thread t handles the pair (i, i ^ j) with i having bit j clear
    const int64_t lo = ((t / j) * 2 * j) + (t % j);
    const int64_t hi = lo + j;
    const int64_t gi = base + lo;
    const bool asc = (gi & k) == 0;
    const uint64_t a = sk[lo], b = sk[hi];
    if ((a > b) == asc) {
      sk[lo] = b;
      sk[hi] = a;
      const int v = sv[lo];
      sv[lo] = sv[hi];
      sv[hi] = v;
    }
    __syncthreads();
  }
  keys[base + t] = sk[t];
  vals[base + t] = sv[t];
  keys[base + t + kSortBlock] = sk[t + kSortBlock];
  vals[base + t + kSortBlock] = sv[t + kSortBlock];
}

struct SortedCells {
  float* cx;
  float* cy;
  float* cz;
  float* R;
};

__global__ void gather_sorted_kernel(const snk_cell* __restrict__ cells, const int* __restrict__ vals,
                                     int64_t nc, SortedCells S, unsigned int* rmax_bits) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nc) return;
  const snk_cell c = cells[vals[p]];
  S.cx[p] = c.c[0];
  S.cy[p] = c.c[1];
  S.cz[p] = c.c[2];
  S.R[p] = c.R;
  atomicMax(rmax_bits, __float_as_uint(fmaxf(c.R, 0.0f)));
}

struct BinGrid {
  int nb[3];
  float inv_h;
};

__device__ __forceinline__ int bin_of(float v, float inv_h, int nb) {
  return min(max((int)floorf(v * inv_h), 0), nb - 1);
}

__global__ void bin_count_kernel(SortedCells S, int64_t nc, BinGrid G, int* counts) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nc) return;
  const int bx = bin_of(S.cx[p], G.inv_h, G.nb[0]), by = bin_of(S.cy[p], G.inv_h, G.nb[1]),
            bz = bin_of(S.cz[p], G.inv_h, G.nb[2]);
  atomicAdd(&counts[((int64_t)bz * G.nb[1] + by) * G.nb[0] + bx], 1);
}

__global__ void bin_fill_kernel(SortedCells S, int64_t nc, BinGrid G, const int64_t* offsets,
                                int* cursor, int* entries) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nc) return;
  const int bx = bin_of(S.cx[p], G.inv_h, G.nb[0]), by = bin_of(S.cy[p], G.inv_h, G.nb[1]),
            bz = bin_of(S.cz[p], G.inv_h, G.nb[2]);
  const int64_t b = ((int64_t)bz * G.nb[1] + by) * G.nb[0] + bx;
  entries[offsets[b] + atomicAdd(&cursor[b], 1)] = (int)p;
}

// fp64 overlap test of §8(c) O6: !(dx^2 + dy^2 + dz^2 >= (rho max(R_i, R_j))^2)
__device__ __forceinline__ bool overlaps(const SortedCells& S, int i, int j, double rho) {
  const double dx = __dsub_rn((double)S.cx[i], (double)S.cx[j]);
  const double dy = __dsub_rn((double)S.cy[i], (double)S.cy[j]);
  const double dz = __dsub_rn((double)S.cz[i], (double)S.cz[j]);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double t = __dmul_rn(rho, (double)fmaxf(S.R[i], S.R[j]));
  return !(d2 >= __dmul_rn(t, t));
}

enum : int { UNDECIDED = 0, IN = 1, OUT = 2 };

__global__ void mis_round_kernel(SortedCells S, int64_t nc, BinGrid G, const int64_t* offsets,
                                 const int* entries, int* status, double rho,
                                 unsigned long long* undecided) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nc) return;
  volatile int* vs = status;
  if (vs[p] != UNDECIDED) return;
  const int bx = bin_of(S.cx[p], G.inv_h, G.nb[0]), by = bin_of(S.cy[p], G.inv_h, G.nb[1]),
            bz = bin_of(S.cz[p], G.inv_h, G.nb[2]);
  bool pending = false;
  for (int z = max(bz - 1, 0); z <= min(bz + 1, G.nb[2] - 1); ++z)
    for (int y = max(by - 1, 0); y <= min(by + 1, G.nb[1] - 1); ++y)
      for (int x = max(bx - 1, 0); x <= min(bx + 1, G.nb[0] - 1); ++x) {
        const int64_t b = ((int64_t)z * G.nb[1] + y) * G.nb[0] + x;
        for (int64_t e = offsets[b]; e < offsets[b + 1]; ++e) {
          const int q = entries[e];
          if (q >= p) continue;   // only higher priority (earlier in (E, id) order)
          if (!overlaps(S, (int)p, q, rho)) continue;
          const int sq = vs[q];
          if (sq == IN) {
            vs[p] = OUT;
            return;
          }
          if (sq == UNDECIDED) pending = true;
        }
      }
  if (!pending) vs[p] = IN;
  else atomicAdd(undecided, 1ull);
}

// exclusive scan of counts -> int64 offsets (+ total at [n]); one block
template <typename T>
__global__ void __launch_bounds__(1024) scan_any_kernel(const T* counts, int64_t n, int64_t* offsets) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = t * per, e = min(n, b + per);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += counts[i];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t y = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += y;
    __syncthreads();
  }
  int64_t run = t > 0 ? part[t - 1] : 0;
  for (int64_t i = b; i < e; ++i) {
    offsets[i] = run;
    run += counts[i];
  }
  if (t == 1023) offsets[n] = part[1023];
}
#define scan_kernel scan_any_kernel<int>
#define scan_i64_kernel scan_any_kernel<int64_t>

// order-preserving compaction, 1024 elements per block
template <typename Pred>
__global__ void __launch_bounds__(1024) flag_count_kernel(int64_t n, Pred pred, int* counts) {
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int c = __syncthreads_count(i < n && pred(i));
  if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

template <typename Pred, typename Emit>
__global__ void __launch_bounds__(1024) flag_write_kernel(int64_t n, Pred pred, Emit emit,
                                                          const int64_t* offsets, int64_t cap) {
  __shared__ int wsum[32];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const bool f = i < n && pred(i);
  const unsigned m = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = __popc(m);
  __syncthreads();
  if (warp == 0) {
    int v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v - wsum[lane];   // exclusive
  }
  __syncthreads();
  if (f) {
    const int64_t o = offsets[blockIdx.x] + wsum[warp] + __popc(m & ((1u << lane) - 1u));
    if (o < cap) emit(i, o);
  }
}

struct CandPred {
  const snk_cell* cells;
  float e0;
  __device__ bool operator()(int64_t i) const { return is_candidate(cells[i], e0); }
};
struct CandEmit {
  const snk_cell* cells;
  snk_cell* out;
  __device__ void operator()(int64_t i, int64_t o) const { out[o] = cells[i]; }
};
struct IdPred {
  const snk_cell* cells;
  int64_t lo, hi;
  __device__ bool operator()(int64_t i) const { return cells[i].id >= lo && cells[i].id < hi; }
};
struct InPred {
  const int* status;
  __device__ bool operator()(int64_t p) const { return status[p] == IN; }
};
struct InEmit {
  const snk_cell* cells;
  const int* vals;
  snk_cell* out;
  __device__ void operator()(int64_t p, int64_t o) const { out[o] = cells[vals[p]]; }
};

int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <typename Pred, typename Emit>
int32_t compact(int64_t n, Pred pred, Emit emit, int64_t cap, int* counts, int64_t* offsets,
                int64_t* n_out, cudaStream_t st) {
  const int64_t nb = ceil_div(std::max<int64_t>(n, 1), 1024);
  flag_count_kernel<<<(unsigned)nb, 1024, 0, st>>>(n, pred, counts);
  SNK_LAUNCH_CHECK("flag_count_kernel");
  scan_kernel<<<1, 1024, 0, st>>>(counts, nb, offsets);
  SNK_LAUNCH_CHECK("scan_kernel");
  flag_write_kernel<<<(unsigned)nb, 1024, 0, st>>>(n, pred, emit, offsets, cap);
  SNK_LAUNCH_CHECK("flag_write_kernel");
  SNK_TRY(read_back(offsets + nb, n_out, sizeof(int64_t), st));
  return SNK_OK;
}

size_t bins_cap(int64_t max_cells) { return (size_t)(4 * std::max<int64_t>(max_cells, 1) + 4096); }

}  // namespace

namespace {

constexpr int kScanThreads = 1024, kScanPer = 4, kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ int64_t block_scan_excl(int64_t v, int64_t* total) {
  __shared__ int64_t wsum[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t s = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  *total = wsum[31];
  return (warp > 0 ? wsum[warp - 1] : 0) + x - v;
}

__global__ void __launch_bounds__(kScanThreads) tile_sum_kernel(const int* counts, int64_t n, int64_t* sums) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k)
    if (base + k < n) s += counts[base + k];
  int64_t total;
  block_scan_excl(s, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) tile_scan_kernel(const int* counts, int64_t n,
                                                                 const int64_t* tile_off, int64_t* offsets) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  int c[kScanPer];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    c[k] = base + k < n ? counts[base + k] : 0;
    s += c[k];
  }
  int64_t total;
  int64_t run = tile_off[blockIdx.x] + block_scan_excl(s, &total);
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    if (base + k < n) offsets[base + k] = run;
    run += c[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) offsets[n] = tile_off[blockIdx.x] + total;
}

}  // namespace

size_t scan_ws(int64_t n) { return (size_t)(ceil_div(std::max<int64_t>(n, 1), kScanTile) + 1) * sizeof(int64_t) * 2 + 512; }

// Exclusive scan of int counts.  Small n: one block.  Large n: per-tile sums ->
// one-block scan of the tile sums (into `tmp`, scan_ws(n) bytes) -> per-tile scans.
int32_t scan_counts(const int* counts, int64_t n, int64_t* offsets, cudaStream_t st, void* tmp) {
  if (n <= 4 * kScanTile || tmp == nullptr) {
    scan_kernel<<<1, 1024, 0, st>>>(counts, n, offsets);
    SNK_LAUNCH_CHECK("scan_kernel");
    return SNK_OK;
  }
  const int64_t nt = ceil_div(n, kScanTile);
  int64_t* sums = static_cast<int64_t*>(tmp);
  int64_t* toff = sums + nt + 1;
  tile_sum_kernel<<<(unsigned)nt, kScanThreads, 0, st>>>(counts, n, sums);
  SNK_LAUNCH_CHECK("tile_sum_kernel");
  scan_i64_kernel<<<1, 1024, 0, st>>>(sums, nt, toff);
  SNK_LAUNCH_CHECK("scan_i64_kernel");
  tile_scan_kernel<<<(unsigned)nt, kScanThreads, 0, st>>>(counts, n, toff, offsets);
  SNK_LAUNCH_CHECK("tile_scan_kernel");
  return SNK_OK;
}

size_t cull_ws(const snk_grid* g, const snk_params* p, int64_t max_cells) {
  (void)g; (void)p;
  const int64_t n = std::max<int64_t>(max_cells, 1);
  const int64_t np2 = std::max<int64_t>(next_pow2(n), 2 * kSortBlock);
  const size_t nbins = bins_cap(n);
  size_t b = 0;
  b += np2 * (sizeof(uint64_t) + sizeof(int)) + 512;
  b += 4 * (size_t)n * sizeof(float) + 1024;
  b += (size_t)n * sizeof(int) * 2 + 512;          // status, entries
  b += nbins * (sizeof(int) * 2 + sizeof(int64_t)) + sizeof(int64_t) + 1024;   // counts, cursor, offsets
  b += scan_ws((int64_t)nbins) + 256;
  b += (size_t)(ceil_div(n, 1024) + 1) * (sizeof(int) + sizeof(int64_t)) + 512;
  b += 4096;
  return b;
}

int32_t compact_impl(const snk_params* p, const snk_cell* d_cells, int64_t n, snk_cell* d_out,
                     int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  if (n == 0) {
    *n_out = 0;
    return SNK_OK;
  }
  Carve cv(d_ws, ws_bytes);
  const int64_t nb = ceil_div(n, 1024);
  int* counts = cv.take<int>(nb);
  int64_t* offsets = cv.take<int64_t>(nb + 1);
  if (cv.overflow || !d_ws) return fail(SNK_CAPACITY, "workspace too small for compaction");
  SNK_TRY(compact(n, CandPred{d_cells, (float)p->e0}, CandEmit{d_cells, d_out}, cap, counts, offsets,
                  n_out, st));
  if (*n_out > cap) return fail(SNK_CAPACITY, "candidate buffer too small");
  return SNK_OK;
}

int32_t select_ids_impl(const snk_cell* d_cells, int64_t n, int64_t id_lo, int64_t id_hi,
                        snk_cell* d_out, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                        cudaStream_t st) {
  if (n == 0) {
    *n_out = 0;
    return SNK_OK;
  }
  Carve cv(d_ws, ws_bytes);
  const int64_t nb = ceil_div(n, 1024);
  int* counts = cv.take<int>(nb);
  int64_t* offsets = cv.take<int64_t>(nb + 1);
  if (cv.overflow || !d_ws) return fail(SNK_CAPACITY, "workspace too small for compaction");
  SNK_TRY(compact(n, IdPred{d_cells, id_lo, id_hi}, CandEmit{d_cells, d_out}, cap, counts, offsets,
                  n_out, st));
  if (*n_out > cap) return fail(SNK_CAPACITY, "output buffer too small");
  return SNK_OK;
}

int32_t cull_impl(const snk_grid* g, const snk_params* p, const snk_cell* d_cells, int64_t n,
                  snk_cell* d_dets, int64_t cap, int64_t* n_out, void* d_ws, size_t ws_bytes,
                  cudaStream_t st) {
  *n_out = 0;
  if (n == 0) return SNK_OK;
  const int64_t np2 = std::max<int64_t>(next_pow2(n), 2 * kSortBlock);
  Carve cv(d_ws, ws_bytes);
  uint64_t* keys = cv.take<uint64_t>(np2);
  int* vals = cv.take<int>(np2);
  SortedCells S;
  S.cx = cv.take<float>(n);
  S.cy = cv.take<float>(n);
  S.cz = cv.take<float>(n);
  S.R = cv.take<float>(n);
  int* status = cv.take<int>(n);
  int* entries = cv.take<int>(n);
  const size_t nbins_cap = bins_cap(n);
  int* bcount = cv.take<int>(nbins_cap);
  int* bcursor = cv.take<int>(nbins_cap);
  int64_t* boff = cv.take<int64_t>(nbins_cap + 1);
  void* bscan = cv.take<char>(scan_ws(nbins_cap));
  const int64_t nblk = ceil_div(n, 1024);
  int* ccounts = cv.take<int>(nblk);
  int64_t* coffsets = cv.take<int64_t>(nblk + 1);
  struct Scalars {
    unsigned long long ncand;
    unsigned long long undecided;
    unsigned int rmax_bits;
    int bad_id;
  };
  Scalars* sc = cv.take<Scalars>(1);
  if (cv.overflow || !d_ws) return fail(SNK_CAPACITY, "workspace too small for cull");

  SNK_CUDA_CHECK(cudaMemsetAsync(sc, 0, sizeof(Scalars), st));
  keys_kernel<<<(unsigned)ceil_div(np2, 256), 256, 0, st>>>(d_cells, n, np2, (float)p->e0, keys, vals,
                                                           &sc->ncand, &sc->bad_id);
  SNK_LAUNCH_CHECK("keys_kernel");
  // bitonic sort of (E, id) keys
  for (int64_t k = 2; k <= np2; k <<= 1) {
    int64_t j = k >> 1;
    for (; j >= 2 * kSortBlock; j >>= 1) {
      bitonic_global_kernel<<<(unsigned)ceil_div(np2, 256), 256, 0, st>>>(keys, vals, j, k);
      SNK_LAUNCH_CHECK("bitonic_global_kernel");
    }
    bitonic_shared_kernel<<<(unsigned)(np2 / (2 * kSortBlock)), kSortBlock, 0, st>>>(keys, vals, k, j);
    SNK_LAUNCH_CHECK("bitonic_shared_kernel");
  }
  Scalars h{};
  SNK_TRY(read_back(sc, &h, sizeof(Scalars), st));
  if (h.bad_id) return fail(SNK_SHAPE, "cull needs cell ids in [0, 2^32)");
  const int64_t nc = (int64_t)h.ncand;
  if (nc == 0) return SNK_OK;
  gather_sorted_kernel<<<(unsigned)ceil_div(nc, 256), 256, 0, st>>>(d_cells, vals, nc, S, &sc->rmax_bits);
  SNK_LAUNCH_CHECK("gather_sorted_kernel");
  SNK_TRY(read_back(sc, &h, sizeof(Scalars), st));
  const double rho = rho_of(g->dim);
  float rmax = 0.0f;
  std::memcpy(&rmax, &h.rmax_bits, sizeof rmax);
  // bin pitch >= rho R_max (so overlapping cells are in adjacent bins), and large
  // enough that the bin count stays within the workspace
  // (1% + 0.01 margin covers the fp32 rounding of v * inv_h for v < 2^24)
  double hb = std::max(rho * (double)rmax * 1.01 + 0.01, 0.01);
  BinGrid G;
  for (;;) {
    int64_t tot = 1;
    for (int a = 0; a < 3; ++a) {
      G.nb[a] = a < g->dim ? (int)std::floor((double)(g->n[a] - 1) / hb) + 1 : 1;
      tot *= G.nb[a];
    }
    if (tot <= (int64_t)nbins_cap) break;
    hb *= 1.25;
  }
  G.inv_h = (float)(1.0 / hb);
  // the float bin index must never split a pair closer than rho R_max: inv_h is
  // rounded down enough that floor(v * inv_h) differs by at most 1 across d < hb
  G.inv_h = std::nextafter(G.inv_h, 0.0f);
  const int64_t nbins = (int64_t)G.nb[0] * G.nb[1] * G.nb[2];
  SNK_CUDA_CHECK(cudaMemsetAsync(bcount, 0, nbins * sizeof(int), st));
  SNK_CUDA_CHECK(cudaMemsetAsync(bcursor, 0, nbins * sizeof(int), st));
  SNK_CUDA_CHECK(cudaMemsetAsync(status, 0, nc * sizeof(int), st));
  bin_count_kernel<<<(unsigned)ceil_div(nc, 256), 256, 0, st>>>(S, nc, G, bcount);
  SNK_LAUNCH_CHECK("bin_count_kernel");
  SNK_TRY(scan_counts(bcount, nbins, boff, st, bscan));
  bin_fill_kernel<<<(unsigned)ceil_div(nc, 256), 256, 0, st>>>(S, nc, G, boff, bcursor, entries);
  SNK_LAUNCH_CHECK("bin_fill_kernel");
  for (int round = 0;; ++round) {
    SNK_CUDA_CHECK(cudaMemsetAsync(&sc->undecided, 0, sizeof(unsigned long long), st));
    mis_round_kernel<<<(unsigned)ceil_div(nc, 256), 256, 0, st>>>(S, nc, G, boff, entries, status, rho,
                                                                  &sc->undecided);
    SNK_LAUNCH_CHECK("mis_round_kernel");
    unsigned long long und = 0;
    SNK_TRY(read_back(&sc->undecided, &und, sizeof und, st));
    if (und == 0) break;
    if (round > nc + 2) return fail(SNK_INTERNAL, "overlap competition did not converge");
  }
  int64_t nd = 0;
  SNK_TRY(compact(nc, InPred{status}, InEmit{d_cells, vals, d_dets}, cap, ccounts, coffsets, &nd, st));
  *n_out = nd;
  if (nd > cap) return fail(SNK_CAPACITY, "detection buffer too small");
  return SNK_OK;
}

}  // namespace snk
