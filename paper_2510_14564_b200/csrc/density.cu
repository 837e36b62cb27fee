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


// ============================================================================ density step
// NEXT-1, the rest of T1 (§III-C2-C4 l.188-228; readings R31-R36 in DESIGN.md §3):
// per point rho (as above) and its k nearest neighbours within 3 r (rings of grid cells are
// added until the k-th candidate lies within the searched radius, at most 3 rings; distances
// beyond 3 r count as 3 r, R32),
// the pooled neighbour-distance statistics and d_merge, mutual-nearest dense pairs within
// d_merge, the densification deficit of sparse points, and the compaction of the new
// theta / Adam moments.  Distances for kNN and merging are squared in double from the float
// coordinates ((dx^2 + dy^2) + dz^2, dx exact), with ties by the lower index -- the oracle's
// (oracle/density.py) decisions.
constexpr int kKnnMax = 16, kMaxRing = 3, kStepThreads = 256;

struct StepWs {
  DensityWs g;                  // the hashed grid (cell size r * 1.0001)
  uint32_t* rho;                // [n]
  double* dbar;                 // [n] mean distance to the k nearest
  int32_t* nn;                  // [n] nearest dense neighbour within d_merge, or -1
  unsigned long long* packed;   // [n] (keep << 32 | children), then its exclusive scan
  unsigned long long* blk;      // [scan blocks] block totals
  double* part;                 // [stat blocks][4] {sum rho, sum rho^2, sum d, sum d^2}
  uint32_t* flags;              // [4] {points with < k neighbours within 3 r, ...}
  bgs_density_report* rep;      // device copy of the report
  float4* spts;                 // [n] {x, y, z, index bits} in grid (bucket) order
  uint32_t* srho;               // [n] rho in grid order
  uint32_t* occ;                // [M / 32] bucket occupancy bits (L2-resident: empty cells skip start/end)
  int64_t stat_blocks, scan_blocks;
};

static bool step_layout(int64_t n, char* base, StepWs* w, size_t* total) {
  size_t gtotal = 0;
  if (!dens_layout(n, nullptr, nullptr, &gtotal)) return false;
  const int64_t stat_blocks = 4 * 148, scan_blocks = (n + 1023) / 1024;
  size_t o = dens_align(gtotal);
  auto take = [&](size_t b) {
    size_t at = o;
    o = dens_align(o + b);
    return at;
  };
  const size_t a_rho = take(4 * (size_t)n), a_dbar = take(8 * (size_t)n), a_nn = take(4 * (size_t)n),
               a_pk = take(8 * (size_t)n), a_blk = take(8 * (size_t)(scan_blocks + 1)),
               a_part = take(32 * (size_t)stat_blocks), a_fl = take(16), a_rep = take(sizeof(bgs_density_report)),
               a_sp = take(16 * (size_t)n), a_sr = take(4 * (size_t)n);
  uint32_t Mb = 1024;  // the grid's bucket count, as dens_layout picks it
  while ((int64_t)Mb < 2 * n) Mb <<= 1;
  const size_t a_occ = take(4 * (size_t)(Mb / 32));
  if (total) *total = o;
  if (w && base) {
    dens_layout(n, base, &w->g, nullptr);
    w->rho = (uint32_t*)(base + a_rho);
    w->dbar = (double*)(base + a_dbar);
    w->nn = (int32_t*)(base + a_nn);
    w->packed = (unsigned long long*)(base + a_pk);
    w->blk = (unsigned long long*)(base + a_blk);
    w->part = (double*)(base + a_part);
    w->flags = (uint32_t*)(base + a_fl);
    w->rep = (bgs_density_report*)(base + a_rep);
    w->spts = (float4*)(base + a_sp);
    w->srho = (uint32_t*)(base + a_sr);
    w->occ = (uint32_t*)(base + a_occ);
    w->stat_blocks = stat_blocks;
    w->scan_blocks = scan_blocks;
  }
  return true;
}

__device__ __forceinline__ double sqd(const float* means, int64_t p, int64_t q) {
  const double dx = (double)means[3 * q] - (double)means[3 * p];
  const double dy = (double)means[3 * q + 1] - (double)means[3 * p + 1];
  const double dz = (double)means[3 * q + 2] - (double)means[3 * p + 2];
  return (dx * dx + dy * dy) + dz * dz;
}

// the points in grid order: neighbour scans read a bucket's points as consecutive float4s
// (no index -> coordinate gather per candidate)
__global__ void __launch_bounds__(256) k_sorted_pts(int64_t n, const float* __restrict__ means,
                                                   const uint32_t* __restrict__ sval, float4* spts) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t q = sval[j];
    spts[j] = make_float4(means[3 * (int64_t)q], means[3 * (int64_t)q + 1], means[3 * (int64_t)q + 2],
                          __uint_as_float(q));
  }
}

__device__ __forceinline__ bool occupied(const uint32_t* occ, uint32_t h) { return (occ[h >> 5] >> (h & 31)) & 1u; }

__device__ __forceinline__ double sqd_f(float px, float py, float pz, const float4 q) {
  const double dx = (double)q.x - (double)px, dy = (double)q.y - (double)py, dz = (double)q.z - (double)pz;
  return (dx * dx + dy * dy) + dz * dz;
}

// rho (27 cells, float decision) + the k nearest (double) per point, one thread per point in
// grid order (a warp's points share their neighbour buckets); rings 0-1 serve both, rings
// 2..3 only the kNN of points whose k-th neighbour is farther than one cell.  Per-block
// partial sums of rho, rho^2, the k distances and their squares.
__global__ void __launch_bounds__(kStepThreads) k_rho_knn(int64_t n, const float4* __restrict__ spts, float inv_cs,
                                                          float cs, float r2, float r_param, uint32_t mask, int k,
                                                          const uint32_t* __restrict__ start,
                                                          const uint32_t* __restrict__ end,
                                                          const uint32_t* __restrict__ occ, uint32_t* rho_out,
                                                          double* dbar, double* part, uint32_t* flags) {
  double s_r = 0, s_r2 = 0, s_d = 0, s_d2 = 0;
  const int kk = (int)((int64_t)k < n - 1 ? (int64_t)k : n - 1);
  for (int64_t jp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jp < n; jp += (int64_t)gridDim.x * blockDim.x) {
    const float4 me = spts[jp];
    const uint32_t i = __float_as_uint(me.w);
    const float px = me.x, py = me.y, pz = me.z;
    const int cx = (int)floorf(px * inv_cs), cy = (int)floorf(py * inv_cs), cz = (int)floorf(pz * inv_cs);
    double bd[kKnnMax];
    uint32_t bq[kKnnMax];
    int nb = 0;
    // the current k-th best (d2, q) in registers: the common case -- a candidate farther
    // than it -- is rejected without touching the (local-memory) sorted list
    double wd = 1.0e300;
    uint32_t wq = 0xffffffffu;
    auto insert = [&](double d2, uint32_t q) {
      if (d2 > wd || (d2 == wd && q >= wq)) return;
      for (int t = 0; t < nb; ++t)
        if (bq[t] == q) return;  // reached again through a colliding cell
      int pos = nb < kk ? nb++ : kk - 1;
      while (pos > 0 && (bd[pos - 1] > d2 || (bd[pos - 1] == d2 && bq[pos - 1] > q))) {
        bd[pos] = bd[pos - 1];
        bq[pos] = bq[pos - 1];
        --pos;
      }
      bd[pos] = d2;
      bq[pos] = q;
      if (nb == kk) {
        wd = bd[kk - 1];
        wq = bq[kk - 1];
      }
    };
    // rings 0-1: the 27 buckets (each distinct one once) for rho and the kNN
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
          if (!occupied(occ, h)) continue;
          const uint32_t e = end[h];
          for (uint32_t j = start[h]; j < e; ++j) {
            const float4 qp = spts[j];
            const uint32_t q = __float_as_uint(qp.w);
            if (q == i) continue;
            const float ddx = qp.x - px, ddy = qp.y - py, ddz = qp.z - pz;
            if ((ddx * ddx + ddy * ddy) + ddz * ddz <= r2) ++c;
            if (kk > 0) insert(sqd_f(px, py, pz, qp), q);
          }
        }
    rho_out[i] = c;
    s_r += (double)c;
    s_r2 += (double)c * (double)c;
    // every point within R cs has been seen after ring R; rings 2..kMaxRing when needed
    bool exact = kk == 0 || (nb == kk && bd[kk - 1] <= (double)cs * (double)cs);
    for (int R = 2; R <= kMaxRing && !exact; ++R) {
      for (int dz = -R; dz <= R; ++dz)
        for (int dy = -R; dy <= R; ++dy)
          for (int dx = -R; dx <= R; ++dx) {
            if (max(abs(dx), max(abs(dy), abs(dz))) != R) continue;  // the shell of ring R
            const uint32_t h = cell_hash(cx + dx, cy + dy, cz + dz, mask);
            if (!occupied(occ, h)) continue;
            const uint32_t e = end[h];
            for (uint32_t j = start[h]; j < e; ++j) {
              const float4 qp = spts[j];
              const uint32_t q = __float_as_uint(qp.w);
              if (q != i) insert(sqd_f(px, py, pz, qp), q);
            }
          }
      const double reach = (double)R * (double)cs;
      exact = nb == kk && bd[kk - 1] <= reach * reach;
    }
    // R32: distances truncated at the 3 r neighbourhood (every point within 3 r <= 3 cs was
    // seen); a neighbour beyond it, or a missing one, counts as 3 r
    const double cap = (double)kMaxRing * (double)r_param;
    int short_k = 0;
    double sum = 0.0;
    for (int t = 0; t < kk; ++t) {
      double d = cap;
      if (t < nb && bd[t] <= cap * cap) d = sqrt(bd[t]);
      else ++short_k;
      sum += d;
      s_d += d;
      s_d2 += d * d;
    }
    if (short_k) atomicAdd(&flags[0], 1u);
    dbar[i] = kk ? sum / (double)kk : 0.0;
  }
  __shared__ double s_p[4][kStepThreads / 32];
  double v[4] = {s_r, s_r2, s_d, s_d2};
#pragma unroll
  for (int a = 0; a < 4; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[a] += __shfl_xor_sync(0xffffffffu, v[a], o);
    if ((threadIdx.x & 31) == 0) s_p[a][threadIdx.x >> 5] = v[a];
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0;
    for (int w = 0; w < kStepThreads / 32; ++w) t += s_p[threadIdx.x][w];
    part[4 * blockIdx.x + threadIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) k_bucket_occ(int64_t n, const uint32_t* __restrict__ key, uint32_t* occ) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = key[i];
    if (i == 0 || key[i - 1] != h) atomicOr(&occ[h >> 5], 1u << (h & 31));
  }
}

__global__ void __launch_bounds__(256) k_sorted_rho(int64_t n, const float4* __restrict__ spts,
                                                   const uint32_t* __restrict__ rho, uint32_t* srho) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    srho[j] = rho[__float_as_uint(spts[j].w)];
}

// The statistics (R31-R32) into the device report: population sigma of rho and of the
// pooled k-distances, the thresholds and d_merge.
__global__ void k_step_stats(int64_t n, int k, int blocks, const double* part, bgs_density_params prm,
                             bgs_density_report* rep) {
  if (threadIdx.x != 0) return;
  double S[4] = {0, 0, 0, 0};
  for (int b = 0; b < blocks; ++b)
    for (int a = 0; a < 4; ++a) S[a] += part[4 * b + a];
  const double N = (double)n, M = (double)n * (double)(k < n - 1 ? k : n - 1);
  rep->n_in = n;
  rep->mu_rho = S[0] / N;
  rep->sigma_rho = sqrt(fmax(0.0, S[1] / N - rep->mu_rho * rep->mu_rho));
  rep->rho_low = rep->mu_rho - (double)prm.alpha * rep->sigma_rho;
  rep->rho_high = rep->mu_rho + (double)prm.beta * rep->sigma_rho;
  rep->mu_d = M > 0 ? S[2] / M : 0.0;
  rep->sigma_d = M > 0 ? sqrt(fmax(0.0, S[3] / M - rep->mu_d * rep->mu_d)) : 0.0;
  rep->d_merge = rep->mu_d + (double)prm.gamma * rep->sigma_d;
}

// R33: each dense point's nearest other dense point within d_merge (ties: lower index); one
// thread per point in grid order, candidates read as consecutive float4s with their rho.
__global__ void __launch_bounds__(kStepThreads) k_merge_nn(int64_t n, const float4* __restrict__ spts,
                                                           const uint32_t* __restrict__ srho, float inv_cs,
                                                           float cs, uint32_t mask,
                                                           const uint32_t* __restrict__ start,
                                                           const uint32_t* __restrict__ end,
                                                           const uint32_t* __restrict__ occ,
                                                           const bgs_density_report* rep, int32_t* nn) {
  const double hi = rep->rho_high, dm = rep->d_merge, lim = dm * dm;
  const int R = (int)ceil(dm / (double)cs);
  for (int64_t jp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jp < n; jp += (int64_t)gridDim.x * blockDim.x) {
    const float4 me = spts[jp];
    const uint32_t i = __float_as_uint(me.w);
    int best = -1;
    if ((double)srho[jp] > hi) {
      const int cx = (int)floorf(me.x * inv_cs), cy = (int)floorf(me.y * inv_cs), cz = (int)floorf(me.z * inv_cs);
      double bd = 0.0;
      // rings of cells outwards; after ring R every point within R cs has been seen, so the
      // search stops once the best candidate lies within that reach (or at d_merge's ring)
      for (int Rg = 0; Rg <= R; ++Rg) {
        for (int dz = -Rg; dz <= Rg; ++dz)
          for (int dy = -Rg; dy <= Rg; ++dy)
            for (int dx = -Rg; dx <= Rg; ++dx) {
              if (max(abs(dx), max(abs(dy), abs(dz))) != Rg) continue;
              const uint32_t h = cell_hash(cx + dx, cy + dy, cz + dz, mask);
              if (!occupied(occ, h)) continue;
              const uint32_t e = end[h];
              for (uint32_t j = start[h]; j < e; ++j) {
                const float4 qp = spts[j];
                const uint32_t q = __float_as_uint(qp.w);
                if (q == i || !((double)srho[j] > hi)) continue;
                const double d2 = sqd_f(me.x, me.y, me.z, qp);
                if (d2 > lim) continue;
                if (best < 0 || d2 < bd || (d2 == bd && (int)q < best)) {
                  bd = d2;
                  best = (int)q;
                }
              }
            }
        const double reach = (double)Rg * (double)cs;
        if (best >= 0 && bd <= reach * reach) break;
      }
    }
    nn[i] = best;
  }
}

// R33/R35: keep flag (not the higher member of a mutual pair) and children per point,
// packed as keep << 32 | children for one scan.
__global__ void __launch_bounds__(kStepThreads) k_step_flags(int64_t n, const int32_t* __restrict__ nn,
                                                             const uint32_t* __restrict__ rho,
                                                             bgs_density_report* rep, int max_new,
                                                             unsigned long long* packed) {
  const double lo = rep->rho_low;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = nn[i];
    const bool removed = q >= 0 && q < i && nn[q] == (int32_t)i;
    uint32_t c = 0;
    if (lo > 0.0 && (double)rho[i] < lo) {
      c = (uint32_t)min((double)max_new, ceil(lo - (double)rho[i]));
      atomicAdd(reinterpret_cast<unsigned long long*>(&rep->n_sparse), 1ull);
    }
    packed[i] = ((unsigned long long)(removed ? 0u : 1u) << 32) | c;
  }
}

// exclusive scan of packed (two 32-bit lanes, no carry between them): per-block scan,
// one block scans the block totals, then the block offsets are added.
__global__ void __launch_bounds__(1024) k_scan64_blocks(int64_t n, unsigned long long* v, unsigned long long* blk) {
  __shared__ unsigned long long s_w[32];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const unsigned long long x = i < n ? v[i] : 0ull;
  unsigned long long inc = x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned long long t = s_w[lane], ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    s_w[lane] = ti - t;
    if (lane == 31) blk[blockIdx.x] = ti;
  }
  __syncthreads();
  if (i < n) v[i] = inc - x + s_w[w];
}

__global__ void k_scan64_top(int64_t nb, unsigned long long* blk, int64_t n, bgs_density_report* rep) {
  if (threadIdx.x != 0) return;
  unsigned long long run = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const unsigned long long t = blk[b];
    blk[b] = run;
    run += t;
  }
  const int64_t keep = (int64_t)(run >> 32), kids = (int64_t)(run & 0xffffffffull);
  rep->n_pairs = n - keep;
  rep->n_children = kids;
  rep->n_out = keep + kids;
}

__global__ void __launch_bounds__(1024) k_scan64_add(int64_t n, unsigned long long* v, const unsigned long long* blk) {
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  if (i < n) v[i] += blk[blockIdx.x];
}

struct ThetaView {  // theta's segments for a given count
  const float *means, *ls, *q, *op, *sh;
};
__device__ __forceinline__ ThetaView tview(const float* t, int64_t n) {
  return {t, t + 3 * n, t + 6 * n, t + 10 * n, t + 11 * n};
}

// R34-R36: the new theta / m / v (n_out Gaussians) in theta's segment layout.
__global__ void __launch_bounds__(kStepThreads) k_step_emit(int64_t n, int64_t n_out, const float* __restrict__ th,
                                                            const float* __restrict__ m, const float* __restrict__ v,
                                                            const int32_t* __restrict__ nn,
                                                            const unsigned long long* __restrict__ off,
                                                            const double* __restrict__ dbar,
                                                            const bgs_density_report* rep, const float* normals,
                                                            const float* uniforms, bgs_density_params prm,
                                                            float* th_o, float* m_o, float* v_o) {
  const int64_t n_keep = n_out - rep->n_children;
  const ThetaView I = tview(th, n), Mi = tview(m, n), Vi = tview(v, n);
  float* const seg_o[3] = {th_o, m_o, v_o};
  auto put = [&](int which, int64_t o, const float* mean, const float* ls, const float* q, float op, const float* sh) {
    float* b = seg_o[which];
    for (int a = 0; a < 3; ++a) b[3 * o + a] = mean[a];
    for (int a = 0; a < 3; ++a) b[3 * n_out + 3 * o + a] = ls[a];
    for (int a = 0; a < 4; ++a) b[6 * n_out + 4 * o + a] = q[a];
    b[10 * n_out + o] = op;
    for (int a = 0; a < 48; ++a) b[11 * n_out + 48 * o + a] = sh[a];
  };
  const float zero[48] = {};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long pk = off[i];
    const int64_t o = (int64_t)(pk >> 32);
    const uint32_t c0 = (uint32_t)(pk & 0xffffffffull);
    const unsigned long long nx = i + 1 < n ? off[i + 1] : ((unsigned long long)n_keep << 32) | (unsigned long long)rep->n_children;
    const bool keep = (nx >> 32) != (pk >> 32);
    const uint32_t nc = (uint32_t)(nx & 0xffffffffull) - c0;
    const int32_t q = nn[i];
    if (keep) {
      if (q > i && nn[q] == (int32_t)i) {  // the merged pair (i, q), kept at i (R34)
        const double op = 1.0 / (1.0 + exp(-(double)I.op[i])), oq = 1.0 / (1.0 + exp(-(double)I.op[q]));
        const double w = op + oq;
        float mean[3], ls[3], sh[48];
        for (int a = 0; a < 3; ++a) {
          mean[a] = (float)((op * (double)I.means[3 * i + a] + oq * (double)I.means[3 * (int64_t)q + a]) / w);
          ls[a] = (float)log(0.5 * (exp((double)I.ls[3 * i + a]) + exp((double)I.ls[3 * (int64_t)q + a])));
        }
        const float* quat = op >= oq ? I.q + 4 * i : I.q + 4 * (int64_t)q;
        const double oo = fmin(0.999, w);
        for (int a = 0; a < 48; ++a)
          sh[a] = (float)((op * (double)I.sh[48 * i + a] + oq * (double)I.sh[48 * (int64_t)q + a]) / w);
        put(0, o, mean, ls, quat, (float)log(oo / (1.0 - oo)), sh);
        put(1, o, zero, zero, zero, 0.f, zero);
        put(2, o, zero, zero, zero, 0.f, zero);
      } else {
        put(0, o, I.means + 3 * i, I.ls + 3 * i, I.q + 4 * i, I.op[i], I.sh + 48 * i);
        put(1, o, Mi.means + 3 * i, Mi.ls + 3 * i, Mi.q + 4 * i, Mi.op[i], Mi.sh + 48 * i);
        put(2, o, Vi.means + 3 * i, Vi.ls + 3 * i, Vi.q + 4 * i, Vi.op[i], Vi.sh + 48 * i);
      }
    }
    // R35: children of a sparse point, numbered in (parent, j) order
    const double sig = (double)prm.alpha_sigma * dbar[i];
    for (uint32_t j = 0; j < nc; ++j) {
      const int64_t ci = (int64_t)c0 + j;
      float mean[3];
      for (int a = 0; a < 3; ++a)
        mean[a] = (float)((double)I.means[3 * i + a] + sig * (double)normals[3 * ci + a] +
                          (double)prm.delta * (double)uniforms[3 * ci + a]);
      const int64_t oc = n_keep + ci;
      put(0, oc, mean, I.ls + 3 * i, I.q + 4 * i, I.op[i], I.sh + 48 * i);
      put(1, oc, zero, zero, zero, 0.f, zero);
      put(2, oc, zero, zero, zero, 0.f, zero);
    }
  }
}

// ---------------------------------------------------------------- R35': further rounds
// exclusive scan of u32 values in place (1024-value blocks, block totals scanned by one
// thread, then added); total to *total
__global__ void __launch_bounds__(1024) k_u32_scan_blocks(int64_t n, uint32_t* v, uint32_t* blk) {
  __shared__ uint32_t s_w[32];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const uint32_t x = i < n ? v[i] : 0u;
  uint32_t inc = x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t t = s_w[lane], ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    s_w[lane] = ti - t;
    if (lane == 31) blk[blockIdx.x] = ti;
  }
  __syncthreads();
  if (i < n) v[i] = inc - x + s_w[w];
}

__global__ void k_u32_scan_top(int64_t nb, uint32_t* blk, uint32_t* total) {
  if (threadIdx.x != 0) return;
  uint32_t run = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const uint32_t t = blk[b];
    blk[b] = run;
    run += t;
  }
  *total = run;
}

__global__ void __launch_bounds__(1024) k_u32_scan_add(int64_t n, uint32_t* v, const uint32_t* blk) {
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  if (i < n) v[i] += blk[blockIdx.x];
}

static bgs_status u32_scan(uint32_t* v, int64_t n, uint32_t* blk, uint32_t* total, cudaStream_t s) {
  const int64_t nb = (n + 1023) / 1024;
  if (nb > 0) {
    k_u32_scan_blocks<<<(int)nb, 1024, 0, s>>>(n, v, blk);
    note_launch();
  }
  k_u32_scan_top<<<1, 32, 0, s>>>(nb, blk, total);
  note_launch();
  if (nb > 0) {
    k_u32_scan_add<<<(int)nb, 1024, 0, s>>>(n, v, blk);
    note_launch();
  }
  return check_launch("density u32 scan");
}

// the sparse points of the plan, in index order: their apply-output index (the keep scan)
// and sigma_p = alpha_sigma d_bar_p; slot = the sparse flags' exclusive scan
__global__ void __launch_bounds__(256) k_sparse_flags(int64_t n, const uint32_t* __restrict__ rho,
                                                      const bgs_density_report* rep, uint32_t* flag) {
  const double lo = rep->rho_low;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (lo > 0.0 && (double)rho[i] < lo) ? 1u : 0u;
}

__global__ void __launch_bounds__(256) k_sparse_emit(int64_t n, const uint32_t* __restrict__ rho,
                                                     const bgs_density_report* rep,
                                                     const uint32_t* __restrict__ slot,
                                                     const unsigned long long* __restrict__ packed,
                                                     const double* __restrict__ dbar, float alpha_sigma,
                                                     uint32_t* parents, double* sigma) {
  const double lo = rep->rho_low;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (lo > 0.0 && (double)rho[i] < lo) {
      parents[slot[i]] = (uint32_t)(packed[i] >> 32);  // survivors before i = its output index
      sigma[slot[i]] = (double)alpha_sigma * dbar[i];  // k_step_emit's spread
    }
}

__global__ void __launch_bounds__(256) k_round_counts(int64_t np, const uint32_t* __restrict__ parents,
                                                      const uint32_t* __restrict__ rho, double lo, int max_new,
                                                      uint32_t* cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = (double)rho[parents[i]];
    cnt[i] = r < lo ? (uint32_t)min((double)max_new, ceil(lo - r)) : 0u;
  }
}

// the n_t points copied into the n_out layout (moments kept), then each parent's children
__global__ void __launch_bounds__(256) k_round_emit(int64_t n_t, int64_t n_out, const float* __restrict__ th,
                                                    const float* __restrict__ m, const float* __restrict__ v,
                                                    int64_t np, const uint32_t* __restrict__ parents,
                                                    const double* __restrict__ sigma,
                                                    const uint32_t* __restrict__ off, const uint32_t* total,
                                                    float delta, const float* normals, const float* uniforms,
                                                    float* th_o, float* m_o, float* v_o) {
  const float* src[3] = {th, m, v};
  float* dst[3] = {th_o, m_o, v_o};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // segment s of a buffer: [s_off(n) .. + width n); widths 3, 3, 4, 1, 48
  const int wid[5] = {3, 3, 4, 1, 48}, at[5] = {0, 3, 6, 10, 11};
  for (int b = 0; b < 3; ++b)
    for (int sg = 0; sg < 5; ++sg)
      for (int64_t e = t0; e < wid[sg] * n_t; e += stride) dst[b][at[sg] * n_out + e] = src[b][at[sg] * n_t + e];
  const uint32_t nc = *total;
  for (int64_t i = t0; i < np; i += stride) {
    const uint32_t c0 = off[i], c1 = i + 1 < np ? off[i + 1] : nc;
    const int64_t p = parents[i];
    for (uint32_t c = c0; c < c1; ++c) {
      const int64_t o = n_t + c;
      for (int a = 0; a < 3; ++a)
        th_o[3 * o + a] = (float)((double)th[3 * p + a] + sigma[i] * (double)normals[3 * (int64_t)c + a] +
                                  (double)delta * (double)uniforms[3 * (int64_t)c + a]);
      for (int a = 0; a < 3; ++a) th_o[3 * n_out + 3 * o + a] = th[3 * n_t + 3 * p + a];
      for (int a = 0; a < 4; ++a) th_o[6 * n_out + 4 * o + a] = th[6 * n_t + 4 * p + a];
      th_o[10 * n_out + o] = th[10 * n_t + p];
      for (int a = 0; a < 48; ++a) th_o[11 * n_out + 48 * o + a] = th[11 * n_t + 48 * p + a];
      for (int b = 1; b < 3; ++b)
        for (int sg = 0; sg < 5; ++sg)
          for (int a = 0; a < wid[sg]; ++a) dst[b][at[sg] * n_out + wid[sg] * o + a] = 0.0f;
    }
  }
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


size_t bgs_density_step_workspace_bytes(int64_t n) {
  size_t total = 0;
  return step_layout(n, nullptr, nullptr, &total) ? total : 0;
}

static bool params_ok(const bgs_density_params* p) {
  return p && p->r > 0.0f && p->alpha >= 0.0f && p->beta >= 0.0f && p->gamma >= 0.0f && p->alpha_sigma > 0.0f &&
         p->delta >= 0.0f && p->k >= 1 && p->k <= kKnnMax && p->max_new >= 0 && p->max_new <= 64;
}

bgs_status bgs_density_plan(const float* theta, int64_t n, const bgs_density_params* p, void* workspace, size_t bytes,
                            void* stream) {
  StepWs w;
  size_t total = 0;
  if (!theta || !workspace || !params_ok(p) || ((uintptr_t)workspace & 255u) ||
      !step_layout(n, (char*)workspace, &w, &total) || bytes < total)
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const float* means = theta;  // theta's first segment
  const float cs = p->r * 1.0001f, inv_cs = 1.0f / cs;
  const uint32_t mask = w.g.M - 1;
  if (cudaMemsetAsync(w.g.hist, 0, 4 * 4 * kDensBins, s) != cudaSuccess ||
      cudaMemsetAsync(w.g.counters, 0, 4 * 32, s) != cudaSuccess ||
      cudaMemsetAsync(w.g.start, 0, 4 * (size_t)w.g.M, s) != cudaSuccess ||
      cudaMemsetAsync(w.g.end, 0, 4 * (size_t)w.g.M, s) != cudaSuccess ||
      cudaMemsetAsync(w.flags, 0, 16, s) != cudaSuccess ||
      cudaMemsetAsync(w.rep, 0, sizeof(bgs_density_report), s) != cudaSuccess)
    return check_launch("density step memset");
  const int grid = 4 * num_sms();
  k_cell_keys<<<grid, 256, 0, s>>>(n, means, inv_cs, mask, w.g.key[0], w.g.val[0], w.g.hist);
  note_launch();
  bgs_status st = check_launch("k_cell_keys");
  if (st != BGS_OK) return st;
  const int passes = (int)((w.g.bits + 7) / 8);
  for (int q = 0; q < passes; ++q) {
    if (cudaMemsetAsync(w.g.status, 0, 4 * 256 * (size_t)w.g.status_tiles, s) != cudaSuccess)
      return check_launch("density status memset");
    const int a = q & 1, b = (q + 1) & 1;
    st = launch_sort_pass32(w.g.key[a], w.g.val[a], w.g.key[b], w.g.val[b], w.g.hist + q * kDensBins, w.g.status,
                            w.g.counters + 1 + q, w.g.counters + 8, 8 * q, n, s);
    if (st != BGS_OK) return st;
  }
  const int fb = passes & 1;
  k_bucket_ranges<<<grid, 256, 0, s>>>(n, w.g.key[fb], w.g.start, w.g.end);
  note_launch();
  if ((st = check_launch("k_bucket_ranges")) != BGS_OK) return st;
  k_sorted_pts<<<grid, 256, 0, s>>>(n, means, w.g.val[fb], w.spts);
  note_launch();
  if (cudaMemsetAsync(w.occ, 0, 4 * (size_t)(w.g.M / 32), s) != cudaSuccess) return check_launch("occ memset");
  k_bucket_occ<<<grid, 256, 0, s>>>(n, w.g.key[fb], w.occ);
  note_launch();
  k_rho_knn<<<(int)w.stat_blocks, kStepThreads, 0, s>>>(n, w.spts, inv_cs, cs, p->r * p->r, p->r, mask, p->k,
                                                        w.g.start, w.g.end, w.occ, w.rho, w.dbar, w.part, w.flags);
  note_launch();
  if ((st = check_launch("k_rho_knn")) != BGS_OK) return st;
  k_sorted_rho<<<grid, 256, 0, s>>>(n, w.spts, w.rho, w.srho);
  note_launch();
  k_step_stats<<<1, 32, 0, s>>>(n, p->k, (int)w.stat_blocks, w.part, *p, w.rep);
  note_launch();
  if ((st = check_launch("k_step_stats")) != BGS_OK) return st;
  k_merge_nn<<<grid, kStepThreads, 0, s>>>(n, w.spts, w.srho, inv_cs, cs, mask, w.g.start, w.g.end, w.occ, w.rep,
                                          w.nn);
  note_launch();
  if ((st = check_launch("k_merge_nn")) != BGS_OK) return st;
  k_step_flags<<<grid, kStepThreads, 0, s>>>(n, w.nn, w.rho, w.rep, p->max_new, w.packed);
  note_launch();
  if ((st = check_launch("k_step_flags")) != BGS_OK) return st;
  k_scan64_blocks<<<(int)w.scan_blocks, 1024, 0, s>>>(n, w.packed, w.blk);
  note_launch();
  k_scan64_top<<<1, 32, 0, s>>>(w.scan_blocks, w.blk, n, w.rep);
  note_launch();
  k_scan64_add<<<(int)w.scan_blocks, 1024, 0, s>>>(n, w.packed, w.blk);
  note_launch();
  return check_launch("density step scan");
}

bgs_status bgs_density_result(const void* workspace, int64_t n, bgs_density_report* out, uint32_t* short_knn) {
  StepWs w;
  if (!workspace || !out || !step_layout(n, (char*)workspace, &w, nullptr)) return BGS_ERR_INVALID;
  if (cudaMemcpy(out, w.rep, sizeof(bgs_density_report), cudaMemcpyDeviceToHost) != cudaSuccess)
    return check_launch("bgs_density_result");
  if (short_knn && cudaMemcpy(short_knn, w.flags, 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return check_launch("bgs_density_result");
  return BGS_OK;
}

bgs_status bgs_density_apply(const float* theta, const float* exp_avg, const float* exp_avg_sq, int64_t n,
                             const void* workspace, const bgs_density_params* p, const float* normals,
                             const float* uniforms, int64_t n_children, float* theta_out, float* exp_avg_out,
                             float* exp_avg_sq_out, int64_t n_out, void* stream) {
  StepWs w;
  if (!theta || !exp_avg || !exp_avg_sq || !workspace || !params_ok(p) || !theta_out || !exp_avg_out ||
      !exp_avg_sq_out || n_out < 1 || n_children < 0 || (n_children > 0 && (!normals || !uniforms)) ||
      !step_layout(n, (char*)workspace, &w, nullptr))
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  k_step_emit<<<4 * num_sms(), kStepThreads, 0, s>>>(n, n_out, theta, exp_avg, exp_avg_sq, w.nn, w.packed, w.dbar,
                                                     w.rep, normals, uniforms, *p, theta_out, exp_avg_out,
                                                     exp_avg_sq_out);
  note_launch();
  return check_launch("k_step_emit");
}

bgs_status bgs_density_parents(const void* workspace, int64_t n, const bgs_density_params* p, uint32_t* parents,
                               double* sigma, void* stream) {
  StepWs w;
  if (!workspace || !params_ok(p) || !parents || !sigma || !step_layout(n, (char*)workspace, &w, nullptr))
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  // the grid's key buffers are free after the plan: flags / slots and the block totals
  uint32_t* slot = w.g.key[0];
  uint32_t* blk = w.g.key[1];
  const int grid = 4 * num_sms();
  k_sparse_flags<<<grid, 256, 0, s>>>(n, w.rho, w.rep, slot);
  note_launch();
  bgs_status st = u32_scan(slot, n, blk, blk + (n + 1023) / 1024 + 1, s);
  if (st != BGS_OK) return st;
  k_sparse_emit<<<grid, 256, 0, s>>>(n, w.rho, w.rep, slot, w.packed, w.dbar, p->alpha_sigma, parents, sigma);
  note_launch();
  return check_launch("k_sparse_emit");
}

// round workspace: counts / offsets [np], block totals [np / 1024 + 1], total [1]
static size_t round_bytes(int64_t np) { return dens_align(4 * (size_t)np) + dens_align(4 * (size_t)(np / 1024 + 2)); }

size_t bgs_density_round_workspace_bytes(int64_t n_parents) { return n_parents < 0 ? 0 : round_bytes(n_parents); }

bgs_status bgs_density_round_plan(const uint32_t* rho, int64_t n_t, const uint32_t* parents, int64_t n_parents,
                                  double rho_low, int32_t max_new, void* workspace, size_t bytes, void* stream) {
  if (!rho || n_t < 1 || n_parents < 0 || (n_parents > 0 && !parents) || !workspace ||
      ((uintptr_t)workspace & 255u) || bytes < round_bytes(n_parents) || max_new < 0 || max_new > 64)
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* cnt = (uint32_t*)workspace;
  uint32_t* blk = (uint32_t*)((char*)workspace + dens_align(4 * (size_t)n_parents));
  if (n_parents > 0) {
    k_round_counts<<<4 * num_sms(), 256, 0, s>>>(n_parents, parents, rho, rho_low, max_new, cnt);
    note_launch();
  }
  return u32_scan(cnt, n_parents, blk, blk + n_parents / 1024 + 1, s);
}

bgs_status bgs_density_round_result(const void* workspace, int64_t n_parents, int64_t* n_children) {
  if (!workspace || n_parents < 0 || !n_children) return BGS_ERR_INVALID;
  const uint32_t* blk = (const uint32_t*)((const char*)workspace + dens_align(4 * (size_t)n_parents));
  uint32_t t = 0;
  if (cudaMemcpy(&t, blk + n_parents / 1024 + 1, 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return check_launch("bgs_density_round_result");
  *n_children = t;
  return BGS_OK;
}

bgs_status bgs_density_round_apply(const float* theta, const float* exp_avg, const float* exp_avg_sq, int64_t n_t,
                                   const uint32_t* parents, const double* sigma, int64_t n_parents,
                                   const void* workspace, float delta, const float* normals, const float* uniforms,
                                   int64_t n_children, float* theta_out, float* exp_avg_out, float* exp_avg_sq_out,
                                   void* stream) {
  if (!theta || !exp_avg || !exp_avg_sq || n_t < 1 || n_parents < 0 || (n_parents > 0 && (!parents || !sigma)) ||
      !workspace || !(delta >= 0.0f) || n_children < 0 || (n_children > 0 && (!normals || !uniforms)) ||
      !theta_out || !exp_avg_out || !exp_avg_sq_out)
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t* off = (const uint32_t*)workspace;
  const uint32_t* total = (const uint32_t*)((const char*)workspace + dens_align(4 * (size_t)n_parents)) +
                          n_parents / 1024 + 1;
  k_round_emit<<<4 * num_sms(), 256, 0, s>>>(n_t, n_t + n_children, theta, exp_avg, exp_avg_sq, n_parents, parents,
                                             sigma, off, total, delta, normals, uniforms, theta_out, exp_avg_out,
                                             exp_avg_sq_out);
  note_launch();
  return check_launch("k_round_emit");
}

}  // extern "C"
