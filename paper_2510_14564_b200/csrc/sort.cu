// sort.cu -- a4-a6: (tile | depth) key duplication (K9), the radix passes (K10, radix.cu)
// and tile ranges (K11).
//
// "N denotes the set of Gaussians contributing to the pixel, sorted by depth" (PAPER.md
// l.149, §II-A); per 16x16 tile; ties by Gaussian index.
// Reading R13: key = (ty*tiles_x + tx) << 32 | float_bits(t_z), value = Gaussian index,
// produced in index order with each rect ty-major; a stable ascending sort on bits
// [0, 32 + bit_width(tiles-1)) then yields the lexicographic (tile, depth bits, index).
//
// K9 is load balanced: a warp takes 32 consecutive Gaussians, scans their tiles_touched,
// and emits the chunk's keys 32 at a time -- lane k finds its Gaussian by a shuffle binary
// search over the inclusive scan -- so a 4000-tile background Gaussian does not
// serialise one thread, and the 32 writes of a round are consecutive (coalesced).  The
// same kernel accumulates, in shared memory, the pass histograms of the depth digits
// (one atomic per Gaussian, weighted by its key count) and the key count of every tile.
// K11 then needs no pass over the sorted keys: one CTA scans the tile counts into the
// ranges, derives the tile-digit pass histograms from them, and orders the tiles heavy
// first for the blend kernels.
#include "common.cuh"

namespace bgs {

constexpr int kRadixBins = 256;
constexpr int kDupThreads = 256;
constexpr int kSmemTiles = 8192;  // tile counts kept in shared memory up to this many tiles

// ---------------------------------------------------------------- K9 duplicate
__global__ void __launch_bounds__(kDupThreads) k_duplicate(int64_t n, const float4* __restrict__ record,
                                                           const int32_t* __restrict__ radius,
                                                           const float* __restrict__ depth,
                                                           const uint32_t* __restrict__ offsets,
                                                           const uint32_t* __restrict__ tiles_touched,
                                                           int32_t tiles_x, int32_t tiles_y, int32_t num_tiles,
                                                           const uint32_t* counters, uint64_t* keys, uint32_t* vals,
                                                           uint32_t* tile_count, uint32_t* hist) {
  __shared__ uint32_t s_tc[kSmemTiles];
  __shared__ uint32_t s_h[4][kRadixBins];
  if (counters[C_OVERFLOW]) return;
  const bool smem_tiles = num_tiles <= kSmemTiles;
  for (int k = threadIdx.x; k < 4 * kRadixBins; k += kDupThreads) (&s_h[0][0])[k] = 0;
  if (smem_tiles)
    for (int k = threadIdx.x; k < num_tiles; k += kDupThreads) s_tc[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int warps = kDupThreads / 32;
  const float ftx = (float)tiles_x, fty = (float)tiles_y;
  for (int64_t base = ((int64_t)blockIdx.x * warps + warp) * 32; base < n; base += (int64_t)gridDim.x * warps * 32) {
    const int64_t i = base + lane;
    uint32_t t = 0, off = 0, dbits = 0;
    int rx0 = 0, ry0 = 0, w = 1;
    if (i < n) {
      off = offsets[i];
      t = tiles_touched[i];
      if (t) {
        const float4 r0 = record[3 * i];
        const int rad = radius[i];
        // the preprocess's canonical rect expression (R11)
        rx0 = (int)fminf(ftx, fmaxf(0.0f, floorf((r0.x - (float)rad) * 0.0625f)));
        ry0 = (int)fminf(fty, fmaxf(0.0f, floorf((r0.y - (float)rad) * 0.0625f)));
        const int rx1 = (int)fminf(ftx, fmaxf(0.0f, floorf((r0.x + (float)(rad + 15)) * 0.0625f)));
        w = rx1 - rx0;
        dbits = __float_as_uint(depth[i]);
#pragma unroll
        for (int p = 0; p < 4; ++p) atomicAdd(&s_h[p][(dbits >> (8 * p)) & 0xff], t);
      }
    }
    uint32_t incl = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t base_off = __shfl_sync(0xffffffffu, off, 0);
    for (uint32_t kb = 0; kb < total; kb += 32) {
      const uint32_t k = kb + lane;
      const bool valid = k < total;
      const uint32_t kk = valid ? k : total - 1;
      int lo = 0, hi = 31;  // smallest lane g with incl_g > kk
#pragma unroll
      for (int it = 0; it < 5; ++it) {
        const int mid = (lo + hi) >> 1;
        const uint32_t v = __shfl_sync(0xffffffffu, incl, mid);
        if (v > kk) hi = mid; else lo = mid + 1;
      }
      const int g = lo;
      const uint32_t g_incl = __shfl_sync(0xffffffffu, incl, g);
      const uint32_t g_t = __shfl_sync(0xffffffffu, t, g);
      const int g_w = __shfl_sync(0xffffffffu, w, g);
      const int g_x0 = __shfl_sync(0xffffffffu, rx0, g);
      const int g_y0 = __shfl_sync(0xffffffffu, ry0, g);
      const uint32_t g_d = __shfl_sync(0xffffffffu, dbits, g);
      if (valid) {
        const uint32_t local = kk - (g_incl - g_t);
        const uint32_t row = local / (uint32_t)g_w;
        const uint32_t tile = (uint32_t)(g_y0 + (int)row) * (uint32_t)tiles_x + (uint32_t)g_x0 +
                              (local - row * (uint32_t)g_w);
        const uint32_t pos = base_off + kk;
        keys[pos] = ((uint64_t)tile << 32) | g_d;
        vals[pos] = (uint32_t)(base + g);
        if (smem_tiles) atomicAdd(&s_tc[tile], 1u);
        else atomicAdd(&tile_count[tile], 1u);
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 4 * kRadixBins; k += kDupThreads) {
    const uint32_t v = (&s_h[0][0])[k];
    if (v) atomicAdd(&hist[k], v);
  }
  if (smem_tiles)
    for (int k = threadIdx.x; k < num_tiles; k += kDupThreads)
      if (s_tc[k]) atomicAdd(&tile_count[k], s_tc[k]);
}

// ---------------------------------------------------------------- heavy-first tile order
// One CTA: bucket the tiles by cost (4 buckets per octave, heaviest bucket first) and
// scatter them.  Only the CTA scheduling order depends on it, never a result.
constexpr int kOrderThreads = 1024, kOrderBuckets = 128;

__device__ void order_tiles(const uint32_t* cost, int32_t nt, uint32_t* order, uint32_t* s_b) {
  for (int k = threadIdx.x; k < kOrderBuckets; k += blockDim.x) s_b[k] = 0;
  __syncthreads();
  auto bucket = [](uint32_t c) {
    const float l = log2f((float)c + 1.0f) * 4.0f;
    const int b = (int)l;
    return kOrderBuckets - 1 - (b < kOrderBuckets - 1 ? b : kOrderBuckets - 1);
  };
  for (int t = threadIdx.x; t < nt; t += blockDim.x) atomicAdd(&s_b[bucket(cost[t])], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int b = 0; b < kOrderBuckets; ++b) {
      const uint32_t c = s_b[b];
      s_b[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nt; t += blockDim.x) order[atomicAdd(&s_b[bucket(cost[t])], 1u)] = (uint32_t)t;
}

__global__ void __launch_bounds__(kOrderThreads) k_tile_order(const uint32_t* cost, int32_t nt,
                                                               const uint32_t* counters, uint32_t* order) {
  __shared__ uint32_t s_b[kOrderBuckets];
  if (counters[C_OVERFLOW]) {
    for (int t = threadIdx.x; t < nt; t += blockDim.x) order[t] = (uint32_t)t;
    return;
  }
  order_tiles(cost, nt, order, s_b);
}

bgs_status launch_tile_order(const uint32_t* cost, int32_t num_tiles, const uint32_t* counters, uint32_t* order,
                             cudaStream_t s) {
  k_tile_order<<<1, kOrderThreads, 0, s>>>(cost, num_tiles, counters, order);
  note_launch();
  return check_launch("k_tile_order");
}

// ---------------------------------------------------------------- K11: tile counts -> ranges
__global__ void __launch_bounds__(kOrderThreads) k_tile_scan(const uint32_t* __restrict__ tile_count, int32_t nt,
                                                              const uint32_t* counters, uint2* ranges, uint32_t* hist,
                                                              int passes, uint32_t* order) {
  __shared__ uint32_t s_warp[kOrderThreads / 32];
  __shared__ uint32_t s_h[4][kRadixBins];
  __shared__ uint32_t s_b[kOrderBuckets];
  if (counters[C_OVERFLOW]) {
    for (int t = threadIdx.x; t < nt; t += blockDim.x) order[t] = (uint32_t)t;
    return;
  }
  for (int k = threadIdx.x; k < 4 * kRadixBins; k += blockDim.x) (&s_h[0][0])[k] = 0;
  const int chunk = (nt + kOrderThreads - 1) / kOrderThreads;
  const int t0 = threadIdx.x * chunk, t1 = min(nt, t0 + chunk);
  uint32_t sum = 0;
  for (int t = t0; t < t1; ++t) sum += tile_count[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t run = incl - sum;
  for (int w = 0; w < warp; ++w) run += s_warp[w];
  for (int t = t0; t < t1; ++t) {
    const uint32_t c = tile_count[t];
    ranges[t] = c ? make_uint2(run, run + c) : make_uint2(0u, 0u);
    run += c;
    if (c)
      for (int p = 4; p < passes; ++p) atomicAdd(&s_h[p - 4][((uint32_t)t >> (8 * (p - 4))) & 0xff], c);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < (passes - 4) * kRadixBins; k += blockDim.x)
    hist[4 * kRadixBins + k] = (&s_h[0][0])[k];
  order_tiles(tile_count, nt, order, s_b);
}

bgs_status launch_sort(Frame* F, cudaStream_t s) {
  if (cudaMemsetAsync(F->ranges, 0, 8 * (size_t)F->num_tiles, s) != cudaSuccess ||
      cudaMemsetAsync(F->tile_count, 0, 4 * (size_t)F->num_tiles, s) != cudaSuccess ||
      cudaMemsetAsync(F->sort_hist, 0, 4 * 8 * kRadixBins, s) != cudaSuccess ||
      cudaMemsetAsync(F->counters + C_SORT_TICKET, 0, 4 * 8, s) != cudaSuccess)
    return check_launch("sort memset");
  if (F->n == 0) {
    // empty scene: identity tile order, no keys
    return launch_tile_order(F->tile_count, F->num_tiles, F->counters, F->tile_order, s);
  }
  const int grid = 4 * num_sms();
  k_duplicate<<<grid, kDupThreads, 0, s>>>(F->n, F->record, F->radius, F->depth, F->offsets, F->tiles_touched,
                                           F->tiles_x, F->tiles_y, F->num_tiles, F->counters, F->keys[0], F->vals[0],
                                           F->tile_count, F->sort_hist);
  note_launch();
  bgs_status st = check_launch("k_duplicate");
  if (st != BGS_OK) return st;
  const int P = F->sort_passes;
  k_tile_scan<<<1, kOrderThreads, 0, s>>>(F->tile_count, F->num_tiles, F->counters, F->ranges, F->sort_hist, P,
                                          F->tile_order);
  note_launch();
  if ((st = check_launch("k_tile_scan")) != BGS_OK || (F->debug_flags & BGS_DEBUG_SKIP_SORT)) return st;
  for (int p = 0; p < P; ++p) {
    if (cudaMemsetAsync(F->sort_status, 0, 4 * kRadixBins * (size_t)F->sort_tiles_max, s) != cudaSuccess)
      return check_launch("sort status memset");
    const int a = p & 1, b = (p + 1) & 1;
    st = launch_sort_pass(F->keys[a], F->vals[a], F->keys[b], F->vals[b], F->sort_hist + p * kRadixBins,
                          F->sort_status, F->counters + C_SORT_TICKET + p, F->counters, 8 * p, s);
    if (st != BGS_OK) return st;
  }
  return BGS_OK;
}

}  // namespace bgs
