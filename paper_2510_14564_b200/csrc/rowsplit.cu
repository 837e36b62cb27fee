// rowsplit.cu -- a4-a6, default path: the depth-ordered (tile, Gaussian) items split by
// tile in two small-alphabet stable splits, tile rows first, then the tiles of each row.
//
// "N denotes the set of Gaussians contributing to the pixel, sorted by depth" (PAPER.md
// l.149, §II-A), per 16x16 tile, ties by Gaussian index:
// reading R13's order (tile, depth bits, index).  The depth sort (sort.cu, radix.cu) gives
// the visible Gaussians in that (depth, index) order as ranks r, each with its tile rect
// [x0, x0 + w) x [y0, y0 + h).  A stable split of the rank-ordered sequence of (tile, r)
// items by tile id is the list order; this file computes it as two stable splits:
//
//  A. entries: the (row y, rank r) pairs, r-major, stably split by y (tiles_y bins): each
//     row's entry list = the ranks whose rect spans the row, in depth order, each entry
//     {x0 | w << 16, Gaussian};
//  B. items: each row's entries expanded to their w items (tiles x0 .. x0 + w - 1 of the
//     row), stably split by x (tiles_x bins).  Tile t = y * tiles_x + x, so the row-major
//     concatenation of B's per-tile lists is the tile-major list order.
//
// Both splits are chunked (A: fixed pair ranges; B: item ranges inside one row): a count
// table per (chunk, bin) from 1-D difference arrays over each chunk's sources, an
// exclusive scan of each bin's column over the chunks, then the emission -- one warp per
// chunk, a position counter per bin in shared memory (tiles_y or tiles_x words, not one
// per tile of the image), each 32-item batch ranked at once by MATCH.ANY on the bin.  A
// chunk of B writes runs of ~chunk / tiles_x consecutive items per tile (full sectors),
// instead of the scattered 4-byte stores of a one-pass split over all tiles.
#include "common.cuh"

namespace bgs {

constexpr int kRsWarps = 4, kRsThreads = kRsWarps * 32;
constexpr int kRsCtasPerSm = 16;
extern __shared__ __align__(16) uint32_t s_rs_dyn[];  // per-warp counters, rings, difference arrays

// largest s in [lo, hi) with off[s] <= a (off non-decreasing, off[lo] <= a); one warp
__device__ __forceinline__ int64_t rs_search(const uint32_t* __restrict__ off, int64_t lo, int64_t hi, uint32_t a,
                                             int lane) {
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const bool ok = p < hi && off[p] <= a;
    const int j = 31 - __clz(__ballot_sync(0xffffffffu, ok));  // lane 0 always ok
    lo += j * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// warp-cooperative difference array -> counts: d[0..nb] in, counts out[0..nb) (inclusive
// prefix of d), lane-parallel by blocks of 32 bins
__device__ __forceinline__ void rs_prefix_out(int32_t* d, int nb, uint32_t* out, int lane) {
  __syncwarp();
  int32_t carry = 0;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    int32_t v = b < nb ? d[b] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    v += carry;
    if (b < nb) out[b] = (uint32_t)v;
    carry = __shfl_sync(0xffffffffu, v, 31);
  }
}

// ---------------------------------------------------------------- A1: per-(chunk, row) entry counts
// chunk c = pairs [c CA, (c + 1) CA) of the r-major pair sequence (pair_off = exclusive scan
// of the ranks' heights)
__global__ void __launch_bounds__(kRsThreads) k_rs_pair_hist(int64_t n, const uint32_t* __restrict__ pair_off,
                                                             const uint32_t* __restrict__ rank_h,
                                                             const uint2* __restrict__ rank_rect, int32_t tiles_y,
                                                             const uint32_t* counters, uint32_t* tabA,
                                                             uint32_t* chunk_r0) {
  if (counters[C_OVERFLOW]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* D = reinterpret_cast<int32_t*>(s_rs_dyn) + warp * (tiles_y + 1);
  const uint32_t P = counters[C_PAIRS];
  const uint32_t n_chunks = (P + kRsPairChunk - 1) / kRsPairChunk;
  for (uint32_t c = blockIdx.x * kRsWarps + warp; c < n_chunks; c += gridDim.x * kRsWarps) {
    for (int k = lane; k <= tiles_y; k += 32) D[k] = 0;
    __syncwarp();
    const uint32_t a = c * kRsPairChunk, b = min(P, a + kRsPairChunk);
    const int64_t r0 = rs_search(pair_off, 0, n, a, lane);
    if (lane == 0) chunk_r0[c] = (uint32_t)r0;
    for (int64_t rb = r0;; rb += 32) {
      const int64_t r = rb + lane;
      uint32_t off = P, h = 0, y0 = 0;
      if (r < n) {
        off = pair_off[r];
        h = rank_h[r];
        y0 = rank_rect[r].x >> 16;
      }
      const uint32_t s0 = max(a, off), e0 = min(b, off + h);
      if (h && s0 < e0) {
        atomicAdd(&D[y0 + (s0 - off)], 1);
        atomicAdd(&D[y0 + (e0 - off)], -1);
      }
      if (__shfl_sync(0xffffffffu, off + h, 31) >= b || rb + 32 >= n) break;
    }
    rs_prefix_out(D, tiles_y, tabA + (size_t)c * tiles_y, lane);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- column scans
// Exclusive prefix over the rows [lo, hi) of each column of tab (ncols wide), in place;
// column totals to tot.  A: one segment (rows = the pair chunks), grid.y = 1; B: one
// segment per tile row y = blockIdx.y (rows = the row's units, [seg[y], seg[y + 1])),
// totals to tot[y * ncols + col].  Block: 32 columns x 32 row ranges.
__global__ void __launch_bounds__(1024) k_rs_colscan(uint32_t* tab, int32_t ncols, const uint32_t* counters,
                                                     const uint32_t* __restrict__ seg, uint32_t* tot) {
  __shared__ uint32_t s[32][33];
  if (counters[C_OVERFLOW]) return;
  int lo = 0, hi;
  if (seg) {
    lo = (int)seg[blockIdx.y];
    hi = (int)seg[blockIdx.y + 1];
  } else {
    hi = (int)((counters[C_PAIRS] + kRsPairChunk - 1) / kRsPairChunk);
  }
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + tx;
  const int per = (hi - lo + 31) / 32;
  const int c0 = lo + ty * per, c1 = min(hi, c0 + per);
  uint32_t sum = 0;
  if (col < ncols) {
#pragma unroll 8
    for (int c = c0; c < c1; ++c) sum += tab[(size_t)c * ncols + col];
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
    if (col < ncols) tot[(seg ? (size_t)blockIdx.y * ncols : 0) + col] = run;
  }
  __syncthreads();
  if (col < ncols) {
    uint32_t run = s[ty][tx];
    int c = c0;
    for (; c + 8 <= c1; c += 8) {
      uint32_t v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = tab[(size_t)(c + q) * ncols + col];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        tab[(size_t)(c + q) * ncols + col] = run;
        run += v[q];
      }
    }
    for (; c < c1; ++c) {
      uint32_t* p = tab + (size_t)c * ncols + col;
      const uint32_t v = *p;
      *p = run;
      run += v;
    }
  }
}

// exclusive scan of the per-row entry totals (one CTA): row_start[0..tiles_y]
__global__ void __launch_bounds__(1024) k_rs_rowstart(const uint32_t* __restrict__ rowE, int32_t tiles_y,
                                                      const uint32_t* counters, uint32_t* row_start) {
  __shared__ uint32_t s_w[32];
  if (counters[C_OVERFLOW]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t carry = 0;
  for (int y0 = 0; y0 < tiles_y; y0 += 1024) {
    const int y = y0 + tid;
    const uint32_t v = y < tiles_y ? rowE[y] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t woff = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < warp) woff += s_w[w];
      tot += s_w[w];
    }
    if (y < tiles_y) row_start[y] = carry + woff + incl - v;
    carry += tot;
    __syncthreads();
  }
  if (tid == 0) row_start[tiles_y] = carry;
}

// ---------------------------------------------------------------- emission (A3 and B5)
// One warp emits the items [a, b) of a sequence of sources s = sb, sb + 1, ... (source s
// owns items [off_s, off_s + cnt_s), item j of it falls in bin bin0_s + j), each item to
// position ctr[bin]++ (the warp's counters in shared memory), stably: a 32-item batch is
// ranked by MATCH.ANY on the bin, its lowest lane of each bin reserves the bin's
// positions.  The owner of each item comes from the batch's source heads (one
// OR-reduction).  Sources arrive 32 at a time (a window) through a per-warp ring of
// kRsRing windows in shared memory filled by cp.async (LDGSTS) kRsRing - 1 windows ahead:
// a window of B holds ~3 batches of items, too few to cover a DRAM round trip with one
// window of register prefetch.  The next batch's lookup and peer set are computed while
// the current one commits.
constexpr int kRsRing = 4;

__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_ring() {
  asm volatile("cp.async.wait_group %0;" ::"n"(kRsRing - 1) : "memory");
}

// A: ranks r -> rows (entries); B: entries e -> tile columns (items)
struct RsSrcRanks {
  static constexpr int kWords = 5;
  const uint32_t *pair_off, *rank_h, *rect_words, *sigma;
  int64_t n;
  uint32_t P;
  __device__ __forceinline__ void issue(int64_t r, uint32_t* w) const {  // w[k * 32]: word k
    if (r < n) {
      cp_async4(w, pair_off + r);
      cp_async4(w + 32, rank_h + r);
      cp_async4(w + 64, rect_words + 2 * r);
      cp_async4(w + 96, rect_words + 2 * r + 1);
      cp_async4(w + 128, sigma + r);
    } else {
      w[0] = P;
      w[32] = 0;
    }
  }
  __device__ __forceinline__ void decode(const uint32_t* w, uint32_t& off, uint32_t& cnt, uint32_t& bin0,
                                         uint32_t& p0, uint32_t& p1) const {
    off = w[0];
    cnt = w[32];
    const uint32_t x = w[64], y = w[96];
    bin0 = x >> 16;                      // y0
    p0 = (x & 0xffffu) | (y << 16);      // x0 | w << 16
    p1 = w[128];
  }
};
struct RsSrcEntries {
  static constexpr int kWords = 3;
  const uint32_t *eoff, *ent_xw, *ent_g;
  int64_t e_hi;
  __device__ __forceinline__ void issue(int64_t e, uint32_t* w) const {
    if (e < e_hi) {
      cp_async4(w, eoff + e);
      cp_async4(w + 32, ent_xw + e);
      cp_async4(w + 64, ent_g + e);
    } else {
      w[0] = 0xffffffffu;
      w[32] = 0;
    }
  }
  __device__ __forceinline__ void decode(const uint32_t* w, uint32_t& off, uint32_t& cnt, uint32_t& bin0,
                                         uint32_t& p0, uint32_t& p1) const {
    off = w[0];
    const uint32_t xw = w[32];
    cnt = xw >> 16;
    bin0 = xw & 0xffffu;
    p0 = w[64];
    p1 = 0;
  }
};

// ctr_at / ring_at: word offsets of the warp's counters and source ring in s_rs_dyn
template <class Src, class Emit>
__device__ __forceinline__ void rs_emit_range(const Src& src, int64_t sb, uint32_t a, uint32_t b, int ctr_at,
                                              int ring_at, int lane, Emit emit) {
  const uint32_t lt = lanemask_lt(), le = lt | (1u << lane);
  uint32_t* ring = s_rs_dyn + ring_at + lane;
  constexpr int kSlot = Src::kWords * 32;
#pragma unroll
  for (int q = 0; q < kRsRing - 1; ++q) {
    src.issue(sb + 32 * q + lane, ring + q * kSlot);
    cp_async_commit();
  }
  uint32_t pos = a;
  for (int win = 0; pos < b; ++win) {
    src.issue(sb + 32 * (kRsRing - 1) + lane, ring + ((win + kRsRing - 1) % kRsRing) * kSlot);
    cp_async_commit();
    cp_async_wait_ring();  // this window's copies (this lane's own) have landed
    uint32_t off, cnt, bin0, p0, p1;
    src.decode(ring + (win % kRsRing) * kSlot, off, cnt, bin0, p0, p1);
    const uint32_t end = min(b, __shfl_sync(0xffffffffu, off + cnt, 31));
    int g_prev = __shfl_sync(0xffffffffu, off, 0) == pos ? -1 : 0;  // owner of item pos - 1
    auto locate = [&](uint32_t kb, uint32_t& bin, uint32_t& q0, uint32_t& q1) {
      const uint32_t rel = off - kb;
      const uint32_t heads = __reduce_or_sync(0xffffffffu, (cnt && rel < 32u) ? 1u << rel : 0u);
      const int g = g_prev + __popc(heads & le);
      g_prev += __popc(heads);
      const uint32_t g_off = __shfl_sync(0xffffffffu, off, g);
      bin = __shfl_sync(0xffffffffu, bin0, g) + (kb + lane - g_off);
      q0 = __shfl_sync(0xffffffffu, p0, g);
      q1 = __shfl_sync(0xffffffffu, p1, g);
    };
    uint32_t bin, q0, q1, pm;
    locate(pos, bin, q0, q1);
    pm = __match_any_sync(0xffffffffu, pos + lane < end ? bin : 0x80000000u | (uint32_t)lane);
    for (uint32_t kb = pos; kb < end; kb += 32) {
      const bool valid = kb + lane < end;
      uint32_t bin_n = 0, q0_n = 0, q1_n = 0, pm_n = 0;
      if (kb + 32 < end) {
        locate(kb + 32, bin_n, q0_n, q1_n);
        pm_n = __match_any_sync(0xffffffffu, kb + 32 + lane < end ? bin_n : 0x80000000u | (uint32_t)lane);
      }
      const int leader = valid ? __ffs(pm) - 1 : lane;
      uint32_t got = 0;
      if (valid && leader == lane) {
        got = s_rs_dyn[ctr_at + bin];
        s_rs_dyn[ctr_at + bin] = got + __popc(pm);
      }
      __syncwarp();  // the next batch's leaders read these counters
      const uint32_t base = __shfl_sync(0xffffffffu, got, leader);
      if (valid) emit(base + __popc(pm & lt), q0, q1);
      bin = bin_n;
      q0 = q0_n;
      q1 = q1_n;
      pm = pm_n;
    }
    pos = end;
    sb += 32;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // the ring is reused by the next range
  __syncwarp();
}

// A3: entries, row-major: ent_xw[e] = x0 | w << 16, ent_g[e] = Gaussian
__global__ void __launch_bounds__(kRsThreads) k_rs_pair_emit(int64_t n, const uint32_t* __restrict__ pair_off,
                                                             const uint32_t* __restrict__ rank_h,
                                                             const uint2* __restrict__ rank_rect,
                                                             const uint32_t* __restrict__ sigma, int32_t tiles_y,
                                                             const uint32_t* counters,
                                                             const uint32_t* __restrict__ tabA,
                                                             const uint32_t* __restrict__ chunk_r0,
                                                             const uint32_t* __restrict__ row_start, uint32_t* ent_xw,
                                                             uint32_t* ent_g) {
  if (counters[C_OVERFLOW]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per_warp = kRsRing * RsSrcRanks::kWords * 32 + ((tiles_y + 3) & ~3);
  const int ring_at = warp * per_warp, ctr_at = ring_at + kRsRing * RsSrcRanks::kWords * 32;
  const uint32_t P = counters[C_PAIRS];
  const uint32_t n_chunks = (P + kRsPairChunk - 1) / kRsPairChunk;
  const RsSrcRanks src{pair_off, rank_h, reinterpret_cast<const uint32_t*>(rank_rect), sigma, n, P};
  for (uint32_t c = blockIdx.x * kRsWarps + warp; c < n_chunks; c += gridDim.x * kRsWarps) {
    const uint32_t* row = tabA + (size_t)c * tiles_y;
    for (int y = lane; y < tiles_y; y += 32) s_rs_dyn[ctr_at + y] = row_start[y] + row[y];
    __syncwarp();
    const uint32_t a = c * kRsPairChunk, b = min(P, a + kRsPairChunk);
    rs_emit_range(src, chunk_r0[c], a, b, ctr_at, ring_at, lane, [&](uint32_t e, uint32_t q0, uint32_t q1) {
      ent_xw[e] = q0;
      ent_g[e] = q1;
    });
  }
}

// B0: exclusive scan of the entries' widths (item offset of each entry in the row-major
// item sequence), single pass with decoupled look-back over a persistent grid; the entry
// count P is read on the device.  The total is the key count K.
constexpr int kRsScanThreads = 256, kRsScanItems = 16, kRsScanTile = kRsScanThreads * kRsScanItems;

__global__ void __launch_bounds__(kRsScanThreads) k_rs_width_scan(const uint32_t* __restrict__ ent_xw,
                                                                  uint32_t* __restrict__ eoff,
                                                                  unsigned long long* status, uint32_t* counters) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[kRsScanThreads / 32];
  __shared__ uint32_t s_prefix;
  if (counters[C_OVERFLOW]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t P = counters[C_PAIRS];
  const uint32_t n_tiles = (P + kRsScanTile - 1) / kRsScanTile;
  constexpr unsigned long long kA = 1ull << 62, kP = 2ull << 62, kMask = (1ull << 62) - 1;
  while (true) {
    if (tid == 0) s_tile = atomicAdd(&counters[C_RS_TICKET], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    __syncthreads();
    if (tile >= n_tiles) break;
    const uint32_t base = tile * kRsScanTile + tid * kRsScanItems;
    uint32_t v[kRsScanItems], local = 0;
#pragma unroll
    for (int k = 0; k < kRsScanItems; ++k) {
      v[k] = base + k < P ? ent_xw[base + k] >> 16 : 0u;
      local += v[k];
    }
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t woff = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kRsScanThreads / 32; ++w) {
      if (w < warp) woff += s_warp[w];
      total += s_warp[w];
    }
    if (warp == 0) {
      uint32_t prefix = 0;
      if (tile == 0) {
        if (lane == 0) st_relaxed_u64(&status[0], kP | total);
      } else {
        if (lane == 0) st_relaxed_u64(&status[tile], kA | total);
        int64_t j = (int64_t)tile - 1 - lane;
        while (true) {
          unsigned long long sv = kP;  // virtual inclusive prefix 0 before tile 0
          if (j >= 0) {
            do {
              sv = ld_relaxed_u64(&status[j]);
            } while ((sv >> 62) == 0);
          }
          const uint32_t pmask = __ballot_sync(0xffffffffu, (sv >> 62) == 2);
          const int stop = pmask ? __ffs(pmask) - 1 : 32;
          uint32_t contrib = lane <= stop ? (uint32_t)(sv & kMask) : 0u;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
          prefix += contrib;
          if (pmask) break;
          j -= 32;
        }
        if (lane == 0) st_relaxed_u64(&status[tile], kP | (prefix + total));
      }
      if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    uint32_t run = s_prefix + woff + (incl - local);
#pragma unroll
    for (int k = 0; k < kRsScanItems; ++k) {
      if (base + k < P) eoff[base + k] = run;
      run += v[k];
    }
  }
}

// B1: units = item ranges of <= CB items inside one row (one CTA).  unit_start[y] = first
// unit of row y; units[u] = {row, first item, end item (row-major item sequence)}.
__global__ void __launch_bounds__(1024) k_rs_units(const uint32_t* __restrict__ eoff,
                                                   const uint32_t* __restrict__ row_start, int32_t tiles_y,
                                                   uint32_t* counters, uint32_t* unit_start, uint4* units,
                                                   uint32_t max_units) {
  __shared__ uint32_t s_w[32];
  if (counters[C_OVERFLOW]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t P = counters[C_PAIRS], K = counters[C_K_LO];
  const uint32_t CB = unit_items_of(K);
  auto item_at = [&](uint32_t e) { return e < P ? eoff[e] : K; };
  uint32_t carry = 0;
  for (int y0 = 0; y0 < tiles_y; y0 += 1024) {
    const int y = y0 + tid;
    uint32_t nu = 0, ia = 0, ib = 0;
    if (y < tiles_y) {
      ia = item_at(row_start[y]);
      ib = item_at(row_start[y + 1]);
      nu = (ib - ia + CB - 1) / CB;
    }
    uint32_t incl = nu;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t woff = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < warp) woff += s_w[w];
      tot += s_w[w];
    }
    const uint32_t u0 = carry + woff + incl - nu;
    if (y < tiles_y) {
      unit_start[y] = u0;
      for (uint32_t k = 0; k < nu && u0 + k < max_units; ++k)
        units[u0 + k] = make_uint4((uint32_t)y, ia + k * CB, min(ib, ia + (k + 1) * CB), row_start[y]);
    }
    carry += tot;
    __syncthreads();
  }
  if (tid == 0) {
    unit_start[tiles_y] = carry;
    counters[C_UNITS] = min(carry, max_units);
  }
}

// B2: per-(unit, x) item counts; units[u].w becomes the unit's first entry
__global__ void __launch_bounds__(kRsThreads) k_rs_unit_hist(const uint32_t* __restrict__ eoff,
                                                             const uint32_t* __restrict__ ent_xw,
                                                             const uint32_t* __restrict__ row_start, int32_t tiles_x,
                                                             const uint32_t* counters, uint4* units, uint32_t* tabB) {
  if (counters[C_OVERFLOW]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* D = reinterpret_cast<int32_t*>(s_rs_dyn) + warp * (tiles_x + 1);
  const uint32_t n_units = counters[C_UNITS];
  for (uint32_t u = blockIdx.x * kRsWarps + warp; u < n_units; u += gridDim.x * kRsWarps) {
    for (int k = lane; k <= tiles_x; k += 32) D[k] = 0;
    __syncwarp();
    const uint4 U = units[u];  // {row, a, b, row's first entry}
    const uint32_t y = U.x, a = U.y, b = U.z;
    const int64_t e_hi = row_start[y + 1];
    const int64_t e0 = rs_search(eoff, U.w, e_hi, a, lane);
    if (lane == 0) units[u].w = (uint32_t)e0;
    for (int64_t eb = e0; eb < e_hi; eb += 32) {
      const int64_t e = eb + lane;
      uint32_t off = 0xffffffffu, w = 0, x0 = 0;
      if (e < e_hi) {
        off = eoff[e];
        const uint32_t xw = ent_xw[e];
        w = xw >> 16;
        x0 = xw & 0xffffu;
      }
      const uint32_t s0 = max(a, off), s1 = off == 0xffffffffu ? 0u : min(b, off + w);
      if (w && s0 < s1) {
        atomicAdd(&D[x0 + (s0 - off)], 1);
        atomicAdd(&D[x0 + (s1 - off)], -1);
      }
      const uint32_t last = __shfl_sync(0xffffffffu, e < e_hi ? off + w : 0xffffffffu, 31);
      if (last >= b || eb + 32 >= e_hi) break;
    }
    rs_prefix_out(D, tiles_x, tabB + (size_t)u * tiles_x, lane);
    __syncwarp();
  }
}

// B5: the items, to their tile-major positions: vals[ranges[y tiles_x + x].x + ...] = Gaussian
__global__ void __launch_bounds__(kRsThreads) k_rs_item_emit(const uint32_t* __restrict__ eoff,
                                                             const uint32_t* __restrict__ ent_xw,
                                                             const uint32_t* __restrict__ ent_g, int32_t tiles_x,
                                                             const uint32_t* counters, const uint4* __restrict__ units,
                                                             const uint32_t* __restrict__ tabB,
                                                             const uint32_t* __restrict__ row_start,
                                                             const uint2* __restrict__ ranges, uint32_t* vals) {
  if (counters[C_OVERFLOW]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per_warp = kRsRing * RsSrcEntries::kWords * 32 + ((tiles_x + 3) & ~3);
  const int ring_at = warp * per_warp, ctr_at = ring_at + kRsRing * RsSrcEntries::kWords * 32;
  const uint32_t n_units = counters[C_UNITS];
  for (uint32_t u = blockIdx.x * kRsWarps + warp; u < n_units; u += gridDim.x * kRsWarps) {
    const uint4 U = units[u];
    const uint32_t y = U.x;
    const uint32_t* row = tabB + (size_t)u * tiles_x;
    const uint2* rg = ranges + (size_t)y * tiles_x;
    for (int x = lane; x < tiles_x; x += 32) s_rs_dyn[ctr_at + x] = rg[x].x + row[x];
    __syncwarp();
    const RsSrcEntries src{eoff, ent_xw, ent_g, (int64_t)row_start[y + 1]};
    rs_emit_range(src, U.w, U.y, U.z, ctr_at, ring_at, lane, [&](uint32_t p, uint32_t q0, uint32_t) { vals[p] = q0; });
  }
}

// ---------------------------------------------------------------- launcher
bgs_status launch_rowsplit(Frame* F, cudaStream_t s) {
  bgs_status st;
  const int TX = F->tiles_x, TY = F->tiles_y;
  static int grid = 0;
  if (!grid) {
    grid = num_sms() * kRsCtasPerSm;
    for (auto fn : {(const void*)k_rs_pair_hist, (const void*)k_rs_pair_emit, (const void*)k_rs_unit_hist,
                    (const void*)k_rs_item_emit})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  }
  // (the caller has scanned the ranks' tile counts (K, overflow) and heights (P))
  if (cudaMemsetAsync(F->counters + C_RS_TICKET, 0, 4, s) != cudaSuccess ||
      cudaMemsetAsync(F->rs_status, 0, 8 * (size_t)F->rs_scan_tiles, s) != cudaSuccess)
    return check_launch("rowsplit memset");
  uint32_t* rowE = F->rs_rows;                 // [TY]
  uint32_t* row_start = F->rs_rows + TY;       // [TY + 1]
  uint32_t* unit_start = F->rs_rows + 2 * TY + 1;  // [TY + 1]
  uint32_t* ent_xw = reinterpret_cast<uint32_t*>(F->keys[1]);
  uint32_t* ent_g = ent_xw + F->max_keys;
  uint32_t* eoff = reinterpret_cast<uint32_t*>(F->keys[0]);
  const size_t smY = (size_t)kRsWarps * 4 * (TY + 1), smX = (size_t)kRsWarps * 4 * (TX + 1);
  const size_t smA = (size_t)kRsWarps * 4 * (kRsRing * 5 * 32 + ((TY + 3) & ~3));
  const size_t smB = (size_t)kRsWarps * 4 * (kRsRing * 3 * 32 + ((TX + 3) & ~3));
  k_rs_pair_hist<<<grid, kRsThreads, smY, s>>>(F->n, F->offsets, F->rank_h, F->rank_rect, TY, F->counters,
                                               F->rs_tabA, F->rs_chunk_r0);
  note_launch();
  if ((st = check_launch("k_rs_pair_hist")) != BGS_OK) return st;
  k_rs_colscan<<<dim3((TY + 31) / 32, 1), 1024, 0, s>>>(F->rs_tabA, TY, F->counters, nullptr, rowE);
  note_launch();
  if ((st = check_launch("k_rs_colscan<rows>")) != BGS_OK) return st;
  k_rs_rowstart<<<1, 1024, 0, s>>>(rowE, TY, F->counters, row_start);
  note_launch();
  if ((st = check_launch("k_rs_rowstart")) != BGS_OK) return st;
  k_rs_pair_emit<<<grid, kRsThreads, smA, s>>>(F->n, F->offsets, F->rank_h, F->rank_rect, F->dval[0], TY,
                                               F->counters, F->rs_tabA, F->rs_chunk_r0, row_start, ent_xw, ent_g);
  note_launch();
  if ((st = check_launch("k_rs_pair_emit")) != BGS_OK) return st;
  k_rs_width_scan<<<2 * num_sms(), kRsScanThreads, 0, s>>>(ent_xw, eoff, F->rs_status, F->counters);
  note_launch();
  if ((st = check_launch("k_rs_width_scan")) != BGS_OK) return st;
  k_rs_units<<<1, 1024, 0, s>>>(eoff, row_start, TY, F->counters, unit_start, F->rs_units,
                                (uint32_t)F->rs_max_units);
  note_launch();
  if ((st = check_launch("k_rs_units")) != BGS_OK) return st;
  k_rs_unit_hist<<<grid, kRsThreads, smX, s>>>(eoff, ent_xw, row_start, TX, F->counters, F->rs_units, F->rs_tabB);
  note_launch();
  if ((st = check_launch("k_rs_unit_hist")) != BGS_OK) return st;
  k_rs_colscan<<<dim3((TX + 31) / 32, TY), 1024, 0, s>>>(F->rs_tabB, TX, F->counters, unit_start, F->tile_count);
  note_launch();
  if ((st = check_launch("k_rs_colscan<tiles>")) != BGS_OK) return st;
  if ((st = launch_tile_scan(F, s)) != BGS_OK) return st;
  k_rs_item_emit<<<grid, kRsThreads, smB, s>>>(eoff, ent_xw, ent_g, TX, F->counters, F->rs_units, F->rs_tabB,
                                               row_start, F->ranges, F->vals[0]);
  note_launch();
  return check_launch("k_rs_item_emit");
}

}  // namespace bgs
