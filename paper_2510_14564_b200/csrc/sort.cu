// sort.cu -- a4-a6: tile/depth ordering of the (tile, Gaussian) pairs (K9-K11).
//
// "N denotes the set of Gaussians contributing to the pixel, sorted by depth" (PAPER.md
// l.149, §II-A); per 16x16 tile; ties by Gaussian index.
// Reading R13 defines the order as that of a stable ascending sort of the 64-bit keys
// (ty*tiles_x + tx) << 32 | float_bits(t_z) produced in Gaussian-index order (each rect
// ty-major): lexicographic (tile, depth bits, index).  Two paths produce it:
//
//  * reference (BGS_DEBUG_SORT_ONESWEEP64): the 64-bit keys are materialised by a
//    load-balanced duplication (K9) and LSD-sorted on bits [0, 32 + bit_width(tiles-1))
//    with the onesweep pass of radix.cu (K10): ~8 + 24 p bytes per key (p = 6 passes).
//  * default, depth first (SURVEY.md §8(a) a5 alternative): (1) stable LSD sort of the N
//    Gaussians by depth bits (4 passes of 32-bit keys, not K; the first pass over N drops
//    the culled Gaussians, the other three see the V visible ones); (2) scan of their tile counts in that order;
//    (3) emission of (tile, Gaussian) items in depth order; (4) a stable split of the
//    items by tile id (ceil(bits/8) 32-bit passes).  A stable split of a depth-ordered
//    (stable in index) sequence by tile is exactly the (tile, depth, index) order, so the
//    values and ranges are bit-identical to the reference (tests/test_gpu_parity.py), at
//    ~40 bytes per key instead of ~152.
//
// Both paths count the keys of every tile while emitting them; one CTA (K11) turns the
// counts into the ranges and the tile-digit pass histograms, and orders the tiles heavy
// first for the blend kernels -- no pass over the sorted keys is needed.
#include "common.cuh"

namespace bgs {

constexpr int kRadixBins = 256;
constexpr int kDupThreads = 256;
constexpr int kSmemTiles = 8192;  // tile counts kept in shared memory up to this many tiles

// ---------------------------------------------------------------- K9: item emission
// A warp takes 32 consecutive Gaussians (index order) or 32 consecutive depth ranks, scans
// their tiles_touched and emits their items 32 at a time: lane k finds its Gaussian by a
// shuffle binary search over the inclusive scan, so a 4000-tile background Gaussian does
// not serialise one thread and the 32 writes of a round are consecutive.
template <bool kByRank>
__global__ void __launch_bounds__(kDupThreads) k_emit(int64_t n, const uint2* __restrict__ rect,
                                                      const float* __restrict__ depth,
                                                      const uint32_t* __restrict__ offsets,  // index or rank order
                                                      const uint32_t* __restrict__ sigma,    // rank -> Gaussian
                                                      const uint32_t* __restrict__ tiles_touched, int32_t tiles_x,
                                                      int32_t tiles_y, int32_t num_tiles, const uint32_t* counters,
                                                      void* keys_out, uint32_t* vals, uint32_t* tile_count,
                                                      uint32_t* hist) {
  __shared__ uint32_t s_tc[kSmemTiles];
  __shared__ uint32_t s_h[4][kRadixBins];
  if (counters[C_OVERFLOW]) return;
  const bool smem_tiles = num_tiles <= kSmemTiles;
  if (!kByRank)
    for (int k = threadIdx.x; k < 4 * kRadixBins; k += kDupThreads) (&s_h[0][0])[k] = 0;
  if (smem_tiles)
    for (int k = threadIdx.x; k < num_tiles; k += kDupThreads) s_tc[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int warps = kDupThreads / 32;
  for (int64_t base = ((int64_t)blockIdx.x * warps + warp) * 32; base < n; base += (int64_t)gridDim.x * warps * 32) {
    const int64_t r = base + lane;
    uint32_t t = 0, off = 0, dbits = 0, gid = 0;
    int rx0 = 0, ry0 = 0, w = 1;
    if (r < n) {
      gid = kByRank ? sigma[r] : (uint32_t)r;
      off = offsets[r];
      t = tiles_touched[gid];
      if (t) {
        // the preprocess's rect (R11' or R11), packed {x0 | y0 << 16, w | h << 16}
        const uint2 q = rect[gid];
        rx0 = (int)(q.x & 0xffffu);
        ry0 = (int)(q.x >> 16);
        w = (int)(q.y & 0xffffu);
        if (!kByRank) {
          dbits = __float_as_uint(depth[gid]);
#pragma unroll
          for (int p = 0; p < 4; ++p) atomicAdd(&s_h[p][(dbits >> (8 * p)) & 0xff], t);
        }
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
      const uint32_t g_id = __shfl_sync(0xffffffffu, gid, g);
      if (valid) {
        const uint32_t local = kk - (g_incl - g_t);
        const uint32_t row = local / (uint32_t)g_w;
        const uint32_t tile = (uint32_t)(g_y0 + (int)row) * (uint32_t)tiles_x + (uint32_t)g_x0 +
                              (local - row * (uint32_t)g_w);
        const uint32_t pos = base_off + kk;
        if (kByRank) reinterpret_cast<uint32_t*>(keys_out)[pos] = tile;
        else reinterpret_cast<uint64_t*>(keys_out)[pos] = ((uint64_t)tile << 32) | g_d;
        vals[pos] = g_id;
        if (smem_tiles) atomicAdd(&s_tc[tile], 1u);
        else atomicAdd(&tile_count[tile], 1u);
      }
    }
  }
  __syncthreads();
  if (!kByRank)
    for (int k = threadIdx.x; k < 4 * kRadixBins; k += kDupThreads) {
      const uint32_t v = (&s_h[0][0])[k];
      if (v) atomicAdd(&hist[k], v);
    }
  if (smem_tiles)
    for (int k = threadIdx.x; k < num_tiles; k += kDupThreads)
      if (s_tc[k]) atomicAdd(&tile_count[k], s_tc[k]);
}

// ---------------------------------------------------------------- depth-first path, step 1
#ifdef BGS_NO_COMPACT  // A/B experiment: every pass over N, culled keys sorted last
constexpr bool kNoCompact = true;
#else
constexpr bool kNoCompact = false;
#endif
// The 4 pass histograms of the VISIBLE Gaussians' 32-bit depth keys and their count V
// (counters[C_VISIBLE]).  The first pass generates its (key, index) pairs from the depths
// and tiles_touched itself (culled: key 0xffffffff, dropped), so the other three run over
// [0, V), and the ranks [V, N) own no tiles.
// It also zeroes, for the later kernels of the sort, the look-back status words of the
// four passes (one region each) and the tile ranges and counts (z0 / z1 / z2, 4-byte words;
// one launch instead of six memsets).
__device__ __forceinline__ void zero_words(uint32_t* p, int64_t words) {
  if (!p) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t w4 = words >> 2;  // 16-byte stores (the frame's buffers are 256-byte aligned)
  for (int64_t i = t0; i < w4; i += stride) reinterpret_cast<uint4*>(p)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int64_t i = 4 * w4 + t0; i < words; i += stride) p[i] = 0u;
}

__global__ void __launch_bounds__(256) k_depth_keys(int64_t n, const float* __restrict__ depth,
                                                    const uint32_t* __restrict__ tiles_touched,
                                                    uint32_t* counters, uint32_t* hist, uint32_t* z0, int64_t z0_words,
                                                    uint32_t* z1, int64_t z1_words, uint32_t* z2, int64_t z2_words) {
  __shared__ uint32_t s_h[8][4][kRadixBins];  // one copy per warp: conflicts stay inside a warp
  __shared__ uint32_t s_vis;
  zero_words(z0, z0_words);
  zero_words(z1, z1_words);
  zero_words(z2, z2_words);
  if (counters[C_OVERFLOW]) return;
  for (int k = threadIdx.x; k < 8 * 4 * kRadixBins; k += blockDim.x) (&s_h[0][0][0])[k] = 0;
  if (threadIdx.x == 0) s_vis = 0;
  __syncthreads();
  uint32_t(*h)[kRadixBins] = s_h[threadIdx.x >> 5];
  uint32_t vis = 0;
  auto add = [&](uint32_t tt, float d) {
    const bool visible = tt != 0;
    if (visible || kNoCompact) {
      const uint32_t key = visible ? __float_as_uint(d) : 0xffffffffu;
      ++vis;
#pragma unroll
      for (int p = 0; p < 4; ++p) atomicAdd(&h[p][(key >> (8 * p)) & 0xff], 1u);
    }
  };
  // four Gaussians per thread and iteration by 16-byte loads (the frame's arrays are
  // 256-byte aligned), the n % 4 tail by scalar loads
  const int64_t n4 = n >> 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 t4 = __ldg(reinterpret_cast<const uint4*>(tiles_touched) + i);
    const float4 d4 = __ldg(reinterpret_cast<const float4*>(depth) + i);
    add(t4.x, d4.x);
    add(t4.y, d4.y);
    add(t4.z, d4.z);
    add(t4.w, d4.w);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    add(tiles_touched[i], depth[i]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) vis += __shfl_xor_sync(0xffffffffu, vis, d);
  if ((threadIdx.x & 31) == 0 && vis) atomicAdd(&s_vis, vis);
  __syncthreads();
  if (threadIdx.x == 0 && s_vis && !kNoCompact) atomicAdd(&counters[C_VISIBLE], s_vis);
  for (int k = threadIdx.x; k < 4 * kRadixBins; k += blockDim.x) {
    uint32_t v = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += (&s_h[w][0][0])[k];
    if (v) atomicAdd(&hist[k], v);
  }
}

// step 2: per depth rank, the Gaussian's tile count and rect, packed as {x0 | y0 << 16, w}
// so the emission reads contiguous data instead of dependent random gathers -- written by
// the depth sort's last pass as it places each rank (radix.cu)

// step 3: emission of the (tile, Gaussian) items in depth order, from the packed rank info.
// Balanced by items, not ranks: warp w emits the item positions [w L, (w + 1) L) (the nearest
// Gaussians cover thousands of tiles each, so equal rank ranges would leave a few warps with
// most of the work).  A warp finds the rank holding its first item with a 32-ary search of
// item_off, then walks 32-rank windows; each 32-item batch finds its items' ranks with a
// 5-step shuffle search of the window's inclusive ends.
__global__ void __launch_bounds__(kDupThreads) k_emit_ranked(int64_t n, const uint32_t* __restrict__ item_off,
                                                             const uint32_t* __restrict__ sigma,
                                                             const uint32_t* __restrict__ rank_cnt,
                                                             const uint2* __restrict__ rank_rect, int32_t tiles_x,
                                                             int32_t num_tiles, const uint32_t* counters,
                                                             uint32_t* keys_out, uint32_t* vals,
                                                             uint32_t* tile_count) {
  __shared__ uint32_t s_tc[kSmemTiles];
  if (counters[C_OVERFLOW]) return;
  const bool smem_tiles = num_tiles <= kSmemTiles;
  if (smem_tiles)
    for (int k = threadIdx.x; k < num_tiles; k += kDupThreads) s_tc[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t K = counters[C_SCAN_TOTAL];  // sum of rank_cnt (= the key count)
  const uint32_t n_warps = gridDim.x * (kDupThreads / 32);
  const uint32_t gw = blockIdx.x * (kDupThreads / 32) + (threadIdx.x >> 5);
  const uint32_t L = ((K + n_warps - 1) / n_warps + 31) & ~31u;
  const uint64_t a64 = (uint64_t)gw * L;
  if (a64 < K) {
    const uint32_t a = (uint32_t)a64, b = (uint32_t)(a64 + L < K ? a64 + L : K);
    // largest rank r with item_off[r] <= a (a rank with zero items shares its offset with
    // the next, so the largest such rank is the one holding item a)
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const int64_t step = (hi - lo + 31) / 32;
      const int64_t p = lo + lane * step;
      const bool ok = p < hi && item_off[p] <= a;
      const int j = 31 - __clz(__ballot_sync(0xffffffffu, ok));  // lane 0 always ok
      lo += j * step;
      hi = min(hi, lo + step);
    }
    int64_t rb = lo;
    uint32_t pos = a;
    while (pos < b) {
      const int64_t r = rb + lane;
      uint32_t t = 0, off = K, gid = 0;
      uint2 rc = make_uint2(0u, 1u);
      if (r < n) {
        t = rank_cnt[r];
        off = item_off[r];
        gid = sigma[r];
        if (t) rc = rank_rect[r];
      }
      const uint32_t incl = off + t;
      const float inv_w = 1.0f / (float)rc.y;  // once per Gaussian, not per item
      const uint32_t end = min(b, __shfl_sync(0xffffffffu, incl, 31));
      for (uint32_t kb = pos; kb < end; kb += 32) {
        const uint32_t k = kb + lane;
        const bool valid = k < end;
        const uint32_t kk = valid ? k : end - 1;
        int l = 0, h = 31;  // smallest lane g with incl_g > kk
#pragma unroll
        for (int it = 0; it < 5; ++it) {
          const int mid = (l + h) >> 1;
          const uint32_t v = __shfl_sync(0xffffffffu, incl, mid);
          if (v > kk) h = mid; else l = mid + 1;
        }
        const int g = l;
        const uint32_t g_off = __shfl_sync(0xffffffffu, off, g);
        const uint32_t g_xy = __shfl_sync(0xffffffffu, rc.x, g);
        const uint32_t g_w = __shfl_sync(0xffffffffu, rc.y, g);
        const float g_iw = __shfl_sync(0xffffffffu, inv_w, g);
        const uint32_t g_id = __shfl_sync(0xffffffffu, gid, g);
        if (valid) {
          const uint32_t local = kk - g_off;
          // exact: (local + 0.5) / w is >= 1/(2w) away from an integer and its float error is
          // <= row * 2^-23 < 2^-13 for rows <= 1024 tiles, so truncation gives local / w
          const uint32_t row = (uint32_t)(((float)local + 0.5f) * g_iw);
          const uint32_t tile = ((g_xy >> 16) + row) * (uint32_t)tiles_x + (g_xy & 0xffffu) + (local - row * g_w);
          keys_out[kk] = tile;
          vals[kk] = g_id;
          if (smem_tiles) atomicAdd(&s_tc[tile], 1u);
          else atomicAdd(&tile_count[tile], 1u);
        }
      }
      pos = end;
      rb += 32;
    }
  }
  __syncthreads();
  if (smem_tiles)
    for (int k = threadIdx.x; k < num_tiles; k += kDupThreads)
      if (s_tc[k]) atomicAdd(&tile_count[k], s_tc[k]);
}

// ---------------------------------------------------------------- direct tile split
// Replaces (3)-(4) of the depth-first path when the tile grid is small enough for
// per-warp shared-memory tile counters: the depth-ordered item sequence is cut into
// chunks of chunk_items_of(K) items (common.cuh); (a) each chunk counts its items per tile (its ranks'
// rects, clipped to the chunk, added as 2D difference rectangles and prefix-summed);
// (b) a column scan over chunks gives each (chunk, tile) its offset inside the tile's
// list; (c) each chunk emits its items in depth order straight to their final positions,
// a running per-tile counter in shared memory numbering the items of a tile in order (in
// a 32-item batch, equal tiles are ranked by match_any).  The order is the stable split
// of the depth-ordered sequence by tile -- the same (tile, depth, index) order -- with no
// keys materialised and no radix passes over K.
constexpr int kChunkWarps = 4;

// largest rank r with item_off[r] <= a (a rank with zero items shares its offset with the
// next one, so the largest such rank holds item a); 32-ary search by one warp
__device__ __forceinline__ int64_t rank_of_item(const uint32_t* __restrict__ item_off, int64_t n, uint32_t a,
                                                int lane) {
  int64_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const bool ok = p < hi && item_off[p] <= a;
    const int j = 31 - __clz(__ballot_sync(0xffffffffu, ok));  // lane 0 always ok
    lo += j * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// (a) per-(chunk, tile) item counts.  Grid cells: (tiles_y + 1) x (tiles_x + 1) ints per
// chunk; the kChunkWarps warps of a CTA share one chunk's grid (a warp per chunk held 17 KB
// of shared memory per warp: 12 warps per SM, latency-bound at 86 us per garden view).
__global__ void __launch_bounds__(kChunkWarps * 32) k_chunk_hist(int64_t n, const uint32_t* __restrict__ item_off,
                                                                 const uint32_t* __restrict__ rank_cnt,
                                                                 const uint2* __restrict__ rank_rect, int32_t tiles_x,
                                                                 int32_t tiles_y, const uint32_t* counters,
                                                                 uint32_t* chunk_cnt) {
  extern __shared__ int32_t s_grid[];
  if (counters[C_OVERFLOW]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  constexpr int T = kChunkWarps * 32;
  const int gw = tiles_x + 1, cells = gw * (tiles_y + 1), nt = tiles_x * tiles_y;
  int32_t* G = s_grid;
  const uint32_t K = counters[C_SCAN_TOTAL];
  const uint32_t CI = chunk_items_of(K), n_chunks = (K + CI - 1) / CI;
  const uint32_t c = blockIdx.x;
  if (c >= n_chunks) return;
  for (int k = tid; k < cells; k += T) G[k] = 0;
  __syncthreads();
  const uint32_t a = c * CI, b = min(K, a + CI);
  auto add_rect = [&](int x0, int y0, int x1, int y1) {  // [x0, x1) x [y0, y1), non-empty
    atomicAdd(&G[y0 * gw + x0], 1);
    atomicAdd(&G[y0 * gw + x1], -1);
    atomicAdd(&G[y1 * gw + x0], -1);
    atomicAdd(&G[y1 * gw + x1], 1);
  };
  // the chunk's ranks [r0, r1] (each warp searches; the loads hit L1/L2): per warp and
  // round, 4 windows of 32 ranks, their loads independent
  const int64_t r0 = rank_of_item(item_off, n, a, lane), r1 = rank_of_item(item_off, n, b - 1, lane);
  for (int64_t rb = r0 + 128 * warp; rb <= r1; rb += 128 * kChunkWarps) {
    uint32_t o[4], t[4];
    uint2 rc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t r = rb + 32 * q + lane;
      o[q] = 0;
      t[q] = 0;
      rc[q] = make_uint2(0u, 1u);
      if (r <= r1) {
        o[q] = item_off[r];
        t[q] = rank_cnt[r];
        rc[q] = rank_rect[r];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t s0 = max(a, o[q]), e0 = min(b, o[q] + t[q]);
      if (t[q] && s0 < e0) {
        const int w = (int)rc[q].y, x0 = (int)(rc[q].x & 0xffffu), y0 = (int)(rc[q].x >> 16);
        const int ls = (int)(s0 - o[q]), le = (int)(e0 - o[q]) - 1;  // inclusive local item range
        // rows by the exact float split of k_emit_ranked (no integer divisions)
        const float iw = 1.0f / (float)w;
        const int q1 = (int)(((float)ls + 0.5f) * iw), c1 = ls - q1 * w;
        const int q2 = (int)(((float)le + 0.5f) * iw), c2 = le - q2 * w;
        if (q1 == q2) {
          add_rect(x0 + c1, y0 + q1, x0 + c2 + 1, y0 + q1 + 1);
        } else {
          add_rect(x0 + c1, y0 + q1, x0 + w, y0 + q1 + 1);
          if (q2 > q1 + 1) add_rect(x0, y0 + q1 + 1, x0 + w, y0 + q2);
          add_rect(x0, y0 + q2, x0 + c2 + 1, y0 + q2 + 1);
        }
      }
    }
  }
  __syncthreads();
  for (int y = tid; y <= tiles_y; y += T) {  // prefix along rows
    int32_t run = 0;
#pragma unroll 8
    for (int x = 0; x <= tiles_x; ++x) run = (G[y * gw + x] += run);
  }
  __syncthreads();
  for (int x = tid; x <= tiles_x; x += T) {  // then along columns
    int32_t run = 0;
#pragma unroll 8
    for (int y = 0; y <= tiles_y; ++y) run = (G[y * gw + x] += run);
  }
  __syncthreads();
  uint32_t* row = chunk_cnt + (size_t)c * nt;
  for (int y = warp; y < tiles_y; y += kChunkWarps)
    for (int x = lane; x < tiles_x; x += 32) row[y * tiles_x + x] = (uint32_t)G[y * gw + x];
}

// (b) exclusive prefix over chunks of each tile's column (in place) and the tile totals.
// Block = 32 tiles x 32 chunk ranges.
__global__ void __launch_bounds__(1024) k_chunk_scan(uint32_t* chunk_cnt, int32_t nt, const uint32_t* counters,
                                                     uint32_t* tile_count) {
  __shared__ uint32_t s[32][33];
  if (counters[C_OVERFLOW]) return;
  const uint32_t K = counters[C_SCAN_TOTAL];
  const uint32_t CI = chunk_items_of(K);
  const int n_chunks = (int)((K + CI - 1) / CI);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + tx;
  const int per = (n_chunks + 31) / 32;
  const int c0 = ty * per, c1 = min(n_chunks, c0 + per);
  uint32_t sum = 0;
  if (t < nt) {
#pragma unroll 8
    for (int c = c0; c < c1; ++c) sum += chunk_cnt[(size_t)c * nt + t];  // loads in flight together
  }
  s[ty][tx] = sum;
  __syncthreads();
  if (ty == 0) {
    uint32_t run = 0;
    for (int k = 0; k < 32; ++k) {
      const uint32_t v = s[k][tx];
      s[k][tx] = run;
      run += v;
    }
    if (t < nt) tile_count[t] = run;
  }
  __syncthreads();
  if (t < nt) {
    uint32_t run = s[ty][tx];
    int c = c0;
    for (; c + 8 <= c1; c += 8) {  // 8 loads in flight, then the 8 stores
      uint32_t v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = chunk_cnt[(size_t)(c + q) * nt + t];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        chunk_cnt[(size_t)(c + q) * nt + t] = run;
        run += v[q];
      }
    }
    for (; c < c1; ++c) {
      uint32_t* p = chunk_cnt + (size_t)c * nt + t;
      const uint32_t v = *p;
      *p = run;
      run += v;
    }
  }
}

// (c) items of each chunk, in depth order, to their final positions.  Per warp: the next
// final position of each tile's items (u32) and a per-tile item count (u8) that detects
// two items of a 32-item batch falling into the same tile.
constexpr int kEmitWarps = 2;
#ifndef BGS_EMIT_PEER_LOOP
#define BGS_EMIT_PEER_LOOP 4
#endif

__global__ void __launch_bounds__(kEmitWarps * 32) k_emit_direct(int64_t n, const uint32_t* __restrict__ item_off,
                                                                 const uint32_t* __restrict__ sigma,
                                                                 const uint32_t* __restrict__ rank_cnt,
                                                                 const uint2* __restrict__ rank_rect,
                                                                 int32_t tiles_x, int32_t nt,
                                                                 const uint32_t* counters,
                                                                 const uint32_t* __restrict__ chunk_cnt,
                                                                 const uint2* __restrict__ ranges, uint32_t* vals) {
  extern __shared__ uint32_t s_dyn[];
  if (counters[C_OVERFLOW]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t K = counters[C_SCAN_TOTAL];
  const uint32_t CI = chunk_items_of(K), n_chunks = (K + CI - 1) / CI;
  const uint32_t c = blockIdx.x * kEmitWarps + warp;
  if (c >= n_chunks) return;
  const int nt_pad = (nt + 3) & ~3;
  uint32_t* nxt = s_dyn + warp * (nt_pad + nt_pad / 4);  // the next position of each tile's items
  uint32_t* cnt8 = nxt + nt_pad;                          // a batch's items per tile, one byte each
  const uint32_t* row = chunk_cnt + (size_t)c * nt;
#pragma unroll 8
  for (int t = lane; t < nt; t += 32) nxt[t] = ranges[t].x + row[t];
  for (int t = lane; t < nt_pad / 4; t += 32) cnt8[t] = 0u;
  __syncwarp();
  const uint32_t a = c * CI, b = min(K, a + CI);
  int64_t rb = rank_of_item(item_off, n, a, lane);
  auto load_win = [&](int64_t base, uint32_t& t, uint32_t& off, uint32_t& gid, uint2& rc) {
    const int64_t r = base + lane;
    t = 0;
    off = K;
    gid = 0;
    rc = make_uint2(0u, 1u);
    if (r < n) {
      t = rank_cnt[r];
      off = item_off[r];
      gid = sigma[r];
      rc = rank_rect[r];
    }
  };
  uint32_t t, off, gid, t_n, off_n, gid_n;
  uint2 rc, rc_n;
  load_win(rb, t, off, gid, rc);
  uint32_t pos = a;
  while (pos < b) {
    load_win(rb + 32, t_n, off_n, gid_n, rc_n);  // next window, in flight during this one
    if (!t) rc = make_uint2(0u, 1u);
    const uint32_t incl = off + t;
    const float inv_w = 1.0f / (float)rc.y;
    const uint32_t end = min(b, __shfl_sync(0xffffffffu, incl, 31));
    // item kb + lane -> (owning lane g of the window, tile, Gaussian): the owner of item kb + j
    // is the owner of item kb - 1 plus the ranks of the window starting in [kb, kb + j] (one
    // OR-reduction of their start bits; the 5-step shuffle search it replaces was a quarter
    // of the kernel's instructions)
    const uint32_t le = lanemask_lt() | (1u << lane);
    int g_prev = __shfl_sync(0xffffffffu, off, 0) == pos ? -1 : 0;  // owner of item pos - 1
    auto locate = [&](uint32_t kb, int& g, uint32_t& tile, uint32_t& g_id) {
      const uint32_t rel = off - kb;
      const uint32_t heads = __reduce_or_sync(0xffffffffu, (t && rel < 32u) ? 1u << rel : 0u);
      g = g_prev + __popc(heads & le);
      g_prev += __popc(heads);
      const uint32_t g_off = __shfl_sync(0xffffffffu, off, g);
      const uint32_t g_xy = __shfl_sync(0xffffffffu, rc.x, g);
      const uint32_t g_w = __shfl_sync(0xffffffffu, rc.y, g);
      const float g_iw = __shfl_sync(0xffffffffu, inv_w, g);
      g_id = __shfl_sync(0xffffffffu, gid, g);
      const uint32_t local = kb + (uint32_t)lane - g_off;
      // exact row split: see k_emit_ranked
      const uint32_t rowi = (uint32_t)(((float)local + 0.5f) * g_iw);
      tile = ((g_xy >> 16) + rowi) * (uint32_t)tiles_x + (g_xy & 0xffffu) + (local - rowi * g_w);
    };
    // commit one 32-item batch in order: items of tiles no other item of the batch shares
    // take their positions at once; a Gaussian's items have distinct tiles, so the items of
    // contended tiles take theirs one Gaussian at a time, in depth order (lanes of a Gaussian
    // are contiguous).  The batch's items per tile are counted in a byte per tile with shared
    // atomics (4 tiles per word), and the counts are taken back after the commit: no two
    // lanes store to one shared-memory word in the same instruction (racecheck-clean,
    // tests/test_gpu_sanitizer.py; MATCH.ANY peer sets instead: 0.58 -> 0.65 ms per view).
    auto commit = [&](bool valid, int g, uint32_t tile, uint32_t g_id) {
      const uint32_t one = 1u << (8u * (tile & 3u));
      if (valid) atomicAdd(&cnt8[tile >> 2], one);
      __syncwarp();
      const bool contended = valid && ((cnt8[tile >> 2] >> (8u * (tile & 3u))) & 0xffu) > 1u;
      if (valid && !contended) {
        const uint32_t p = nxt[tile];
        nxt[tile] = p + 1u;
        vals[p] = g_id;
      }
      if (__any_sync(0xffffffffu, contended)) {
        // the items of a contended tile belong to distinct Gaussians, so lane order is their
        // depth order: each takes the tile's next position plus its rank among the tile's
        // lanes (one MATCH.ANY), and the tile's last lane advances the counter
        __syncwarp();
#if BGS_EMIT_PEER_LOOP
        // few contended lanes (<= BGS_EMIT_PEER_LOOP: at most half as many tiles): their peer
        // sets by one ballot per contended tile instead of the long-latency MATCH.ANY
        const uint32_t cm = __ballot_sync(0xffffffffu, contended);
        uint32_t peers = 0;
        if (__popc(cm) <= BGS_EMIT_PEER_LOOP) {
          uint32_t todo = cm;
          while (todo) {
            const uint32_t lt_tile = __shfl_sync(0xffffffffu, tile, __ffs(todo) - 1);
            const uint32_t mine = __ballot_sync(0xffffffffu, contended && tile == lt_tile);
            if (contended && tile == lt_tile) peers = mine;
            todo &= ~mine;
          }
        } else {
          peers = __match_any_sync(0xffffffffu, contended ? tile : 0x80000000u | (uint32_t)lane);
        }
#else
        const uint32_t peers = __match_any_sync(0xffffffffu, contended ? tile : 0x80000000u | (uint32_t)lane);
#endif
        uint32_t p = 0;
        if (contended) p = nxt[tile] + (uint32_t)__popc(peers & lanemask_lt());
        __syncwarp();
        if (contended) {
          if ((peers >> lane) == 1u) nxt[tile] = p + 1u;
          vals[p] = g_id;
        }
      }
      __syncwarp();
      if (valid) atomicSub(&cnt8[tile >> 2], one);
    };
    // two batches per round: their lookups are independent (ILP), commits stay in order
    for (uint32_t kb = pos; kb < end; kb += 64) {
      const uint32_t k0 = kb + lane, k1 = kb + 32 + lane;
      const bool v0 = k0 < end, v1 = k1 < end;
      int g0, g1;
      uint32_t t0, t1, id0, id1;
      locate(kb, g0, t0, id0);
      locate(kb + 32, g1, t1, id1);
      commit(v0, g0, t0, id0);
      if (__any_sync(0xffffffffu, v1)) commit(v1, g1, t1, id1);
    }
    pos = end;
    rb += 32;
    t = t_n;
    off = off_n;
    gid = gid_n;
    rc = rc_n;
  }
}

// ---------------------------------------------------------------- K11: tile counts -> ranges
constexpr int kOrderThreads = 1024;

// Also writes the tile-digit pass histograms hist[4 .. passes) (digit p-4 of the tile id)
// and the heavy-first forward tile order.
__global__ void __launch_bounds__(kOrderThreads) k_tile_scan(const uint32_t* __restrict__ tile_count, int32_t nt,
                                                              const uint32_t* counters, uint2* ranges, uint32_t* hist,
                                                              int passes) {
  __shared__ uint32_t s_warp[kOrderThreads / 32];
  __shared__ uint32_t s_h[4][kRadixBins];
  if (counters[C_OVERFLOW]) return;
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
}

bgs_status launch_tile_scan(Frame* F, cudaStream_t s) {
  k_tile_scan<<<1, kOrderThreads, 0, s>>>(F->tile_count, F->num_tiles, F->counters, F->ranges, F->sort_hist, 4);
  note_launch();
  return check_launch("k_tile_scan");
}

// look-back status words of a pass over at most `count` keys
static bgs_status memset_status(Frame* F, cudaStream_t s, int64_t count = -1) {
  const int64_t tiles = count < 0 ? F->sort_tiles_max : (count + kSortTileKeys - 1) / kSortTileKeys;
  if (cudaMemsetAsync(F->sort_status, 0, 4 * kRadixBins * (size_t)tiles, s) != cudaSuccess)
    return check_launch("sort status memset");
  return BGS_OK;
}

bgs_status launch_sort(Frame* F, cudaStream_t s) {
  const bool ref64 = (F->debug_flags & (BGS_DEBUG_SORT_ONESWEEP64 | BGS_DEBUG_SKIP_SORT)) != 0;
  // depth-first path: k_depth_keys zeroes the ranges, tile counts and the four passes' status
  // regions when the status buffer holds four regions of the N-key pass
  const int64_t region = (int64_t)kRadixBins * ((F->n + kSortTileKeys - 1) / kSortTileKeys);
  const bool fused_zero = !ref64 && F->n > 0 && 4 * region <= (int64_t)kRadixBins * F->sort_tiles_max;
  if ((!fused_zero && (cudaMemsetAsync(F->ranges, 0, 8 * (size_t)F->num_tiles, s) != cudaSuccess ||
                       cudaMemsetAsync(F->tile_count, 0, 4 * (size_t)F->num_tiles, s) != cudaSuccess)) ||
      cudaMemsetAsync(F->sort_hist, 0, 4 * 8 * kRadixBins, s) != cudaSuccess ||
      cudaMemsetAsync(F->counters + C_SORT_TICKET, 0, 4 * 8, s) != cudaSuccess ||
      cudaMemsetAsync(F->counters + C_SORT32_TICKET, 0, 4 * 8, s) != cudaSuccess ||
      cudaMemsetAsync(F->counters + C_VISIBLE, 0, 4, s) != cudaSuccess)
    return check_launch("sort memset");
  const int P = F->sort_passes;
  F->sort_mode = ref64 ? 1 : 0;
  F->final_buf = ref64 ? (P & 1) : ((P - 4) & 1);
  if (F->n == 0) return BGS_OK;
  const int grid = 4 * num_sms();
  bgs_status st;
  if (ref64) {
    if ((st = launch_scan(F->tiles_touched, F->offsets, F->n, F, true, s)) != BGS_OK) return st;  // a3, K
    k_emit<false><<<grid, kDupThreads, 0, s>>>(F->n, F->rect, F->depth, F->offsets, nullptr,
                                               F->tiles_touched, F->tiles_x, F->tiles_y, F->num_tiles, F->counters,
                                               F->keys[0], F->vals[0], F->tile_count, F->sort_hist);
    note_launch();
    if ((st = check_launch("k_emit<index>")) != BGS_OK) return st;
    k_tile_scan<<<1, kOrderThreads, 0, s>>>(F->tile_count, F->num_tiles, F->counters, F->ranges, F->sort_hist, P);
    note_launch();
    if ((st = check_launch("k_tile_scan")) != BGS_OK || (F->debug_flags & BGS_DEBUG_SKIP_SORT)) return st;
    for (int p = 0; p < P; ++p) {
      if ((st = memset_status(F, s)) != BGS_OK) return st;
      const int a = p & 1, b = (p + 1) & 1;
      st = launch_sort_pass(F->keys[a], F->vals[a], F->keys[b], F->vals[b], F->sort_hist + p * kRadixBins,
                            F->sort_status, F->counters + C_SORT_TICKET + p, F->counters, 8 * p, s);
      if (st != BGS_OK) return st;
    }
    return BGS_OK;
  }
  // ---- depth first: (1) stable sort of the Gaussians by depth bits
  k_depth_keys<<<grid, 256, 0, s>>>(F->n, F->depth, F->tiles_touched, F->counters, F->sort_hist,
                                    fused_zero ? F->sort_status : nullptr, 4 * region,
                                    fused_zero ? reinterpret_cast<uint32_t*>(F->ranges) : nullptr,
                                    2 * (int64_t)F->num_tiles, fused_zero ? F->tile_count : nullptr,
                                    (int64_t)F->num_tiles);
  note_launch();
  if ((st = check_launch("k_depth_keys")) != BGS_OK) return st;
  for (int p = 0; p < 4; ++p) {
    if (!fused_zero && (st = memset_status(F, s, F->n)) != BGS_OK) return st;
    const int a = p & 1, b = (p + 1) & 1;
    // the first pass compacts the visible Gaussians; (2) the last pass also writes the
    // per-rank tile counts and packed rects (zero past V)
    const bool last = p == 3;
    // the first pass reads the depths and visibility directly (keys and values generated)
    const uint32_t* kin = p ? F->dkey[a] : reinterpret_cast<const uint32_t*>(F->depth);
    st = launch_sort_pass32(kin, p ? F->dval[a] : nullptr, F->dkey[b], F->dval[b], F->sort_hist + p * kRadixBins,
                            F->sort_status + (fused_zero ? p * region : 0), F->counters + C_SORT32_TICKET + p, F->counters, 8 * p, (p && !kNoCompact) ? -2 : F->n, s,
                            last ? F->rect : nullptr, last ? F->rank_cnt : nullptr, last ? F->rank_rect : nullptr,
                            last ? F->rank_h : nullptr, p == 0 && !kNoCompact, last ? F->n : 0,
                            p ? nullptr : F->tiles_touched);
    if (st != BGS_OK) return st;
  }
  // K (published with the capacity check) = the total of the depth-order scan
  if ((st = launch_scan(F->rank_cnt, F->item_off, F->n, F, true, s)) != BGS_OK) return st;
  const bool rowsplit_ok = F->tiles_x <= kRsMaxTiles && F->tiles_y <= kRsMaxTiles;
  if (rowsplit_ok && (F->debug_flags & BGS_DEBUG_SORT_ROWSPLIT)) {
    // (3'') row split (rowsplit.cu, measured slower than the direct split: DESIGN.md §6):
    // the ranks' heights scanned for the entry count
    F->final_buf = 0;
    if ((st = launch_scan(F->rank_h, F->offsets, F->n, F, false, s)) != BGS_OK) return st;
    return launch_rowsplit(F, s);
  }
  if (F->chunk_cnt && !(F->debug_flags & BGS_DEBUG_SORT_RADIX_SPLIT)) {
    // (3') direct tile split: per-(chunk, tile) counts, column scan, ranges, emission
    F->final_buf = 0;
    const int gw = F->tiles_x + 1, cells = gw * (F->tiles_y + 1), nt = F->num_tiles;
    const int64_t max_chunks = (F->max_keys + kChunkItemsMin - 1) / kChunkItemsMin;  // device picks the size
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_chunk_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_emit_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    k_chunk_hist<<<(int)max_chunks, kChunkWarps * 32, (size_t)cells * 4, s>>>(
        F->n, F->item_off, F->rank_cnt, F->rank_rect, F->tiles_x, F->tiles_y, F->counters, F->chunk_cnt);
    note_launch();
    if ((st = check_launch("k_chunk_hist")) != BGS_OK) return st;
    k_chunk_scan<<<(nt + 31) / 32, 1024, 0, s>>>(F->chunk_cnt, nt, F->counters, F->tile_count);
    note_launch();
    if ((st = check_launch("k_chunk_scan")) != BGS_OK) return st;
    k_tile_scan<<<1, kOrderThreads, 0, s>>>(F->tile_count, nt, F->counters, F->ranges, F->sort_hist, 4);
    note_launch();
    if ((st = check_launch("k_tile_scan")) != BGS_OK) return st;
    const int nt_pad = (nt + 3) & ~3;
    k_emit_direct<<<(int)((max_chunks + kEmitWarps - 1) / kEmitWarps), kEmitWarps * 32,
                    (size_t)kEmitWarps * 5 * nt_pad, s>>>(
        F->n, F->item_off, F->dval[0], F->rank_cnt, F->rank_rect, F->tiles_x, nt, F->counters, F->chunk_cnt,
        F->ranges, F->vals[0]);
    note_launch();
    return check_launch("k_emit_direct");
  }
  // (3) (tile, Gaussian) items in depth order + per-tile counts
  uint32_t* tkey[2] = {reinterpret_cast<uint32_t*>(F->keys[0]), reinterpret_cast<uint32_t*>(F->keys[1])};
  k_emit_ranked<<<grid, kDupThreads, 0, s>>>(F->n, F->item_off, F->dval[0], F->rank_cnt, F->rank_rect, F->tiles_x,
                                             F->num_tiles, F->counters, tkey[0], F->vals[0], F->tile_count);
  note_launch();
  if ((st = check_launch("k_emit_ranked")) != BGS_OK) return st;
  k_tile_scan<<<1, kOrderThreads, 0, s>>>(F->tile_count, F->num_tiles, F->counters, F->ranges, F->sort_hist, P);
  note_launch();
  if ((st = check_launch("k_tile_scan")) != BGS_OK) return st;
  // (4) stable split by tile id
  for (int p = 0; p < P - 4; ++p) {
    if ((st = memset_status(F, s)) != BGS_OK) return st;
    const int a = p & 1, b = (p + 1) & 1;
    st = launch_sort_pass32(tkey[a], F->vals[a], tkey[b], F->vals[b], F->sort_hist + (4 + p) * kRadixBins,
                            F->sort_status, F->counters + C_SORT32_TICKET + 4 + p, F->counters, 8 * p, -1, s);
    if (st != BGS_OK) return st;
  }
  return BGS_OK;
}

}  // namespace bgs
