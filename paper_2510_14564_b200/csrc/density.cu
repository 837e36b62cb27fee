// density.cu -- NEXT-1: the paper's T1 statistical density thresholding on the GPU.
//
// PAPER.md §III-C1 (l.181-186): "For each point p, the local density rho is determined as
// the number of neighboring points within a fixed radius r"; rho_low = mu_rho - alpha
// sigma_rho, rho_high = mu_rho + beta sigma_rho over all local densities.  SPEC.md l.221:
// exact, via a uniform spatial grid (results identical to brute force).
//
// Grid: cell size r * (1 + 1e-4) >= r, so every q within r of p lies in one of p's 27
// neighbour cells.  Cells are hashed into M >= 2n buckets; points are stable-sorted by
// bucket with the onesweep pass (radix.cu), bucket ranges are marked, and each point scans
// its 27 neighbour buckets (distinct ones only: a hash collision must not count a bucket
// twice), testing ((dx*dx + dy*dy) + dz*dz) <= r*r in float -- the oracle's expression, so
// the integer counts are bit-exact.  The statistics reduce the counts in 64-bit integers
// (exact), then mu and sigma (population) in double.
#include "common.cuh"

namespace bgs {

constexpr int kDensBins = 256;

struct DensityWs {
  uint32_t *key[2], *val[2], *start, *end, *status, *hist, *counters;
  unsigned long long* sums;
  uint32_t M, bits;
  int64_t status_tiles;
};

static size_t dens_align(size_t x) { return (x + 255) & ~(size_t)255; }

static bool dens_layout(int64_t n, char* base, DensityWs* w, size_t* total) {
  if (n < 1 || n >= ((int64_t)1 << 30)) return false;
  uint32_t M = 1024, bits = 10;
  while ((int64_t)M < 2 * n) {
    M <<= 1;
    ++bits;
  }
  const int64_t tiles = (n + 4095) / 4096;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o = dens_align(o + b);
    return at;
  };
  const size_t k0 = take(4 * (size_t)n), k1 = take(4 * (size_t)n), v0 = take(4 * (size_t)n),
               v1 = take(4 * (size_t)n), st = take(4 * (size_t)M), en = take(4 * (size_t)M),
               ss = take(4 * 256 * (size_t)tiles), hi = take(4 * 4 * kDensBins), co = take(4 * 32), su = take(8 * 4);
  if (total) *total = o;
  if (w && base) {
    w->key[0] = (uint32_t*)(base + k0);
    w->key[1] = (uint32_t*)(base + k1);
    w->val[0] = (uint32_t*)(base + v0);
    w->val[1] = (uint32_t*)(base + v1);
    w->start = (uint32_t*)(base + st);
    w->end = (uint32_t*)(base + en);
    w->status = (uint32_t*)(base + ss);
    w->hist = (uint32_t*)(base + hi);
    w->counters = (uint32_t*)(base + co);
    w->sums = (unsigned long long*)(base + su);
    w->M = M;
    w->bits = bits;
    w->status_tiles = tiles;
  }
  return true;
}

__device__ __forceinline__ void cell_of(const float* means, int64_t i, float inv_cs, int& cx, int& cy, int& cz) {
  cx = (int)floorf(means[3 * i] * inv_cs);
  cy = (int)floorf(means[3 * i + 1] * inv_cs);
  cz = (int)floorf(means[3 * i + 2] * inv_cs);
}

__device__ __forceinline__ uint32_t cell_hash(int cx, int cy, int cz, uint32_t mask) {
  return (((uint32_t)cx * 73856093u) ^ ((uint32_t)cy * 19349663u) ^ ((uint32_t)cz * 83492791u)) & mask;
}

__global__ void __launch_bounds__(256) k_cell_keys(int64_t n, const float* __restrict__ means, float inv_cs,
                                                   uint32_t mask, uint32_t* key, uint32_t* val, uint32_t* hist) {
  __shared__ uint32_t s_h[4][kDensBins];
  for (int k = threadIdx.x; k < 4 * kDensBins; k += blockDim.x) (&s_h[0][0])[k] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int cx, cy, cz;
    cell_of(means, i, inv_cs, cx, cy, cz);
    const uint32_t h = cell_hash(cx, cy, cz, mask);
    key[i] = h;
    val[i] = (uint32_t)i;
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&s_h[p][(h >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 4 * kDensBins; k += blockDim.x)
    if ((&s_h[0][0])[k]) atomicAdd(&hist[k], (&s_h[0][0])[k]);
}

__global__ void __launch_bounds__(256) k_bucket_ranges(int64_t n, const uint32_t* __restrict__ key, uint32_t* start,
                                                       uint32_t* end) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = key[i];
    if (i == 0 || key[i - 1] != h) start[h] = (uint32_t)i;
    if (i == n - 1 || key[i + 1] != h) end[h] = (uint32_t)(i + 1);
  }
}

__global__ void __launch_bounds__(256) k_local_density(int64_t n, const float* __restrict__ means, float inv_cs,
                                                       float r2, uint32_t mask, const uint32_t* __restrict__ sval,
                                                       const uint32_t* __restrict__ start,
                                                       const uint32_t* __restrict__ end, uint32_t* counts,
                                                       unsigned long long* sums) {
  unsigned long long s1 = 0, s2 = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int cx, cy, cz;
    cell_of(means, i, inv_cs, cx, cy, cz);
    const float px = means[3 * i], py = means[3 * i + 1], pz = means[3 * i + 2];
    uint32_t seen[27];
    int nseen = 0;
    uint32_t c = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const uint32_t h = cell_hash(cx + dx, cy + dy, cz + dz, mask);
          bool dup = false;
          for (int t = 0; t < nseen; ++t) dup |= seen[t] == h;
          if (dup) continue;
          seen[nseen++] = h;
          const uint32_t e = end[h];
          for (uint32_t j = start[h]; j < e; ++j) {
            const uint32_t q = sval[j];
            if (q == (uint32_t)i) continue;
            const float ddx = means[3 * (int64_t)q] - px;
            const float ddy = means[3 * (int64_t)q + 1] - py;
            const float ddz = means[3 * (int64_t)q + 2] - pz;
            if ((ddx * ddx + ddy * ddy) + ddz * ddz <= r2) ++c;
          }
        }
    counts[i] = c;
    s1 += c;
    s2 += (unsigned long long)c * c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&sums[0], s1);
    atomicAdd(&sums[1], s2);
  }
}

__global__ void k_density_finish(int64_t n, const unsigned long long* sums, float alpha, float beta, double* out) {
  const double S = (double)sums[0], S2 = (double)sums[1], N = (double)n;
  const double mu = S / N;
  const double var = fmax(0.0, (N * S2 - S * S) / (N * N));
  const double sd = sqrt(var);
  out[0] = mu;
  out[1] = sd;
  out[2] = mu - (double)alpha * sd;
  out[3] = mu + (double)beta * sd;
}

}  // namespace bgs

using namespace bgs;

extern "C" {

size_t bgs_density_workspace_bytes(int64_t n) {
  size_t total = 0;
  return dens_layout(n, nullptr, nullptr, &total) ? total : 0;
}

bgs_status bgs_local_density(const float* means, int64_t n, float r, float alpha, float beta, uint32_t* counts,
                             double* stats, void* workspace, size_t bytes, void* stream) {
  DensityWs w;
  size_t total = 0;
  if (!means || !counts || !stats || !workspace || !(r > 0.0f) || !dens_layout(n, (char*)workspace, &w, &total) ||
      bytes < total || ((uintptr_t)workspace & 255u))
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const float cs = r * 1.0001f;  // >= r: every neighbour within r is in the 27 cells
  const float inv_cs = 1.0f / cs;
  const uint32_t mask = w.M - 1;
  if (cudaMemsetAsync(w.hist, 0, 4 * 4 * kDensBins, s) != cudaSuccess ||
      cudaMemsetAsync(w.counters, 0, 4 * 32, s) != cudaSuccess || cudaMemsetAsync(w.sums, 0, 32, s) != cudaSuccess ||
      cudaMemsetAsync(w.start, 0, 4 * (size_t)w.M, s) != cudaSuccess ||
      cudaMemsetAsync(w.end, 0, 4 * (size_t)w.M, s) != cudaSuccess)
    return check_launch("density memset");
  const int grid = 4 * num_sms();
  k_cell_keys<<<grid, 256, 0, s>>>(n, means, inv_cs, mask, w.key[0], w.val[0], w.hist);
  note_launch();
  bgs_status st = check_launch("k_cell_keys");
  if (st != BGS_OK) return st;
  const int passes = (int)((w.bits + 7) / 8);
  for (int p = 0; p < passes; ++p) {
    if (cudaMemsetAsync(w.status, 0, 4 * 256 * (size_t)w.status_tiles, s) != cudaSuccess)
      return check_launch("density status memset");
    const int a = p & 1, b = (p + 1) & 1;
    st = launch_sort_pass32(w.key[a], w.val[a], w.key[b], w.val[b], w.hist + p * kDensBins, w.status,
                            w.counters + 1 + p, w.counters + 8, 8 * p, n, s);
    if (st != BGS_OK) return st;
  }
  const int fb = passes & 1;
  k_bucket_ranges<<<grid, 256, 0, s>>>(n, w.key[fb], w.start, w.end);
  note_launch();
  if ((st = check_launch("k_bucket_ranges")) != BGS_OK) return st;
  k_local_density<<<grid, 256, 0, s>>>(n, means, inv_cs, r * r, mask, w.val[fb], w.start, w.end, counts, w.sums);
  note_launch();
  if ((st = check_launch("k_local_density")) != BGS_OK) return st;
  k_density_finish<<<1, 1, 0, s>>>(n, w.sums, alpha, beta, stats);
  note_launch();
  return check_launch("k_density_finish");
}

}  // extern "C"
