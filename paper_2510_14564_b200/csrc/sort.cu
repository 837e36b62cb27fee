// sort.cu -- a4-a6: (tile | depth) key duplication (K9), stable 64-bit LSD radix sort
// (K10, onesweep), tile ranges (K11).
//
// "N denotes the set of Gaussians contributing to the pixel, sorted by depth" (PAPER.md
// l.149, §II-A); per 16x16 tile; ties by Gaussian index.
// Reading R13: key = (ty*tiles_x + tx) << 32 | float_bits(t_z), value = Gaussian index,
// produced in index order with each rect ty-major; a stable ascending sort on bits
// [0, 32 + bit_width(tiles-1)) then yields the lexicographic (tile, depth bits, index).
//
// Onesweep (one kernel per 8-bit digit pass, keys read once and written once per
// pass): a 4096-key tile per CTA iteration, warp-level multi-split ranking with
// __match_any_sync (stable inside a warp's contiguous 512-key slice), warp prefix
// across the CTA, decoupled look-back across tiles for the digit's global offset,
// then a shared-memory reorder so the global writes are digit-contiguous (coalesced).
// A persistent grid takes tiles in ticket order, so a predecessor tile is always
// resident when a successor waits on it.
#include "common.cuh"

namespace bgs {

constexpr int kSortThreads = 256, kSortItems = 16, kSortTile = kSortThreads * kSortItems, kRadix = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr uint32_t kStA = 1u << 30, kStP = 2u << 30, kStMask = (1u << 30) - 1;

__device__ __forceinline__ uint64_t load_k(const uint32_t* counters) {
  return ((uint64_t)counters[C_K_HI] << 32) | counters[C_K_LO];
}

// ---------------------------------------------------------------- K9 duplicate
__global__ void __launch_bounds__(256) k_duplicate(int64_t n, const float4* __restrict__ record,
                                                   const int32_t* __restrict__ radius,
                                                   const float* __restrict__ depth,
                                                   const uint32_t* __restrict__ offsets,
                                                   const uint32_t* __restrict__ tiles_touched, int32_t tiles_x,
                                                   int32_t tiles_y, const uint32_t* counters, uint64_t* keys,
                                                   uint32_t* vals) {
  if (counters[C_OVERFLOW]) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || tiles_touched[i] == 0) return;
  const float4 r0 = record[3 * i];
  const int rad = radius[i];
  // the same canonical rect expression as the preprocess (R11)
  const float tx = (float)tiles_x, ty = (float)tiles_y;
  const int rx0 = (int)fminf(tx, fmaxf(0.0f, floorf((r0.x - (float)rad) * 0.0625f)));
  const int ry0 = (int)fminf(ty, fmaxf(0.0f, floorf((r0.y - (float)rad) * 0.0625f)));
  const int rx1 = (int)fminf(tx, fmaxf(0.0f, floorf((r0.x + (float)(rad + 15)) * 0.0625f)));
  const int ry1 = (int)fminf(ty, fmaxf(0.0f, floorf((r0.y + (float)(rad + 15)) * 0.0625f)));
  const uint64_t lo = (uint64_t)__float_as_uint(depth[i]);
  uint32_t o = offsets[i];
  for (int y = ry0; y < ry1; ++y)
    for (int x = rx0; x < rx1; ++x) {
      keys[o] = ((uint64_t)(uint32_t)(y * tiles_x + x) << 32) | lo;
      vals[o] = (uint32_t)i;
      ++o;
    }
}

// ---------------------------------------------------------------- digit histograms, all passes
__global__ void __launch_bounds__(256) k_sort_hist(const uint64_t* __restrict__ keys, const uint32_t* counters,
                                                   uint32_t* hist, int passes) {
  __shared__ uint32_t sh[8][kRadix];
  for (int k = threadIdx.x; k < 8 * kRadix; k += blockDim.x) (&sh[0][0])[k] = 0;
  __syncthreads();
  if (!counters[C_OVERFLOW]) {
    const int64_t K = (int64_t)load_k(counters);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t key = keys[i];
      for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 0xff], 1u);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < passes * kRadix; k += blockDim.x) {
    const uint32_t v = (&sh[0][0])[k];
    if (v) atomicAdd(&hist[k], v);
  }
}

// ---------------------------------------------------------------- one onesweep pass
struct SortSmem {
  uint64_t keys[kSortTile];
  uint32_t vals[kSortTile];
  uint32_t warp_hist[kSortWarps][kRadix];  // counts, then exclusive prefix over warps
  uint32_t tile_start[kRadix];             // exclusive prefix over digits inside the tile
  uint32_t global_base[kRadix];            // destination of the digit's first key of this tile
  uint32_t hist_excl[kRadix];              // exclusive scan of this pass's global histogram
  uint32_t scan_tmp[kSortWarps];
  uint32_t tile;
};

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(const uint64_t* __restrict__ kin,
                                                            const uint32_t* __restrict__ vin, uint64_t* kout,
                                                            uint32_t* vout, const uint32_t* __restrict__ hist,
                                                            uint32_t* status, uint32_t* ticket,
                                                            const uint32_t* counters, int shift) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& S = *reinterpret_cast<SortSmem*>(smem_raw);
  if (counters[C_OVERFLOW]) return;
  const int64_t K = (int64_t)load_k(counters);
  const int64_t ntiles = (K + kSortTile - 1) / kSortTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // exclusive scan of the pass histogram (thread = digit)
  {
    const uint32_t h = hist[tid];
    uint32_t incl = h;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) S.scan_tmp[warp] = incl;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += S.scan_tmp[w];
    S.hist_excl[tid] = off + incl - h;
    __syncthreads();
  }
  const uint32_t lt = lanemask_lt();
  while (true) {
    if (tid == 0) S.tile = atomicAdd(ticket, 1u);
    for (int k = tid; k < kSortWarps * kRadix; k += kSortThreads) (&S.warp_hist[0][0])[k] = 0;
    __syncthreads();
    const int64_t tile = S.tile;
    if (tile >= ntiles) break;
    const int64_t tbase = tile * kSortTile;
    const int tcount = (int)(K - tbase < kSortTile ? K - tbase : kSortTile);
    // load: warp w owns the contiguous slice [w*512, (w+1)*512) of the tile
    uint64_t key[kSortItems];
    uint32_t val[kSortItems];
    uint16_t rank[kSortItems];
    const int wbase = warp * (kSortItems * 32);
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
      const int idx = wbase + k * 32 + lane;
      if (idx < tcount) {
        key[k] = kin[tbase + idx];
        val[k] = vin[tbase + idx];
      } else {
        key[k] = ~0ull;
        val[k] = 0;
      }
    }
    // warp-level multi-split ranking, in input order (stable)
    uint32_t* wh = S.warp_hist[warp];
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
      const int idx = wbase + k * 32 + lane;
      const bool valid = idx < tcount;
      const uint32_t d = valid ? (uint32_t)((key[k] >> shift) & 0xff) : 0x100u + (uint32_t)lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      uint32_t base = 0;
      if (valid) base = wh[d];
      __syncwarp();
      if (valid) {
        const uint32_t before = __popc(peers & lt);
        if (before == 0) wh[d] = base + __popc(peers);
        rank[k] = (uint16_t)(base + before);
      }
      __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, tile count
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = S.warp_hist[w][tid];
      S.warp_hist[w][tid] = cnt;
      cnt += c;
    }
    // publish the tile aggregate early (decoupled look-back)
    uint32_t* st = status + tile * kRadix;
    if (tile == 0) st_volatile_u32(&st[tid], kStP | cnt);
    else st_volatile_u32(&st[tid], kStA | cnt);
    // exclusive prefix over digits inside the tile
    {
      uint32_t incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
      }
      if (lane == 31) S.scan_tmp[warp] = incl;
      __syncthreads();
      uint32_t off = 0;
      for (int w = 0; w < warp; ++w) off += S.scan_tmp[w];
      S.tile_start[tid] = off + incl - cnt;
    }
    // look-back for digit tid
    uint32_t prefix = 0;
    if (tile > 0) {
      for (int64_t j = tile - 1; j >= 0; --j) {
        uint32_t s;
        do {
          s = ld_volatile_u32(&status[j * kRadix + tid]);
        } while ((s >> 30) == 0);
        prefix += s & kStMask;
        if ((s >> 30) == 2) break;
      }
      st_volatile_u32(&st[tid], kStP | (prefix + cnt));
    }
    S.global_base[tid] = S.hist_excl[tid] + prefix;
    __syncthreads();
    // reorder through shared memory (digit-contiguous)
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
      const int idx = wbase + k * 32 + lane;
      if (idx < tcount) {
        const uint32_t d = (uint32_t)((key[k] >> shift) & 0xff);
        const uint32_t pos = S.tile_start[d] + S.warp_hist[warp][d] + rank[k];
        S.keys[pos] = key[k];
        S.vals[pos] = val[k];
      }
    }
    __syncthreads();
    for (int j = tid; j < tcount; j += kSortThreads) {
      const uint64_t k2 = S.keys[j];
      const uint32_t d = (uint32_t)((k2 >> shift) & 0xff);
      const uint32_t g = S.global_base[d] + (uint32_t)j - S.tile_start[d];
      kout[g] = k2;
      vout[g] = S.vals[j];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K11 ranges
__global__ void __launch_bounds__(256) k_ranges(const uint64_t* __restrict__ keys, const uint32_t* counters,
                                                uint2* ranges) {
  if (counters[C_OVERFLOW]) return;
  const int64_t K = (int64_t)load_k(counters);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(keys[i] >> 32);
    if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[t].x = (uint32_t)i;
    if (i == K - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[t].y = (uint32_t)(i + 1);
  }
}

static int sort_grid() {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sort_pass, kSortThreads, sizeof(SortSmem));
    if (per_sm < 1) per_sm = 1;
    grid = per_sm * num_sms();
  }
  return grid;
}

bgs_status launch_sort(Frame* F, cudaStream_t s) {
  if (cudaMemsetAsync(F->ranges, 0, 8 * (size_t)F->num_tiles, s) != cudaSuccess) return check_launch("ranges memset");
  if (F->n == 0) return BGS_OK;
  const int dup_blocks = (int)((F->n + 255) / 256);
  k_duplicate<<<dup_blocks, 256, 0, s>>>(F->n, F->record, F->radius, F->depth, F->offsets, F->tiles_touched,
                                         F->tiles_x, F->tiles_y, F->counters, F->keys[0], F->vals[0]);
  note_launch();
  bgs_status st = check_launch("k_duplicate");
  if (st != BGS_OK || (F->debug_flags & BGS_DEBUG_SKIP_SORT)) return st;
  const int P = F->sort_passes;
  if (cudaMemsetAsync(F->sort_hist, 0, 4 * 8 * kRadix, s) != cudaSuccess ||
      cudaMemsetAsync(F->counters + C_SORT_TICKET, 0, 4 * 8, s) != cudaSuccess)
    return check_launch("sort memset");
  const int grid = sort_grid();
  k_sort_hist<<<grid, 256, 0, s>>>(F->keys[0], F->counters, F->sort_hist, P);
  note_launch();
  if ((st = check_launch("k_sort_hist")) != BGS_OK) return st;
  for (int p = 0; p < P; ++p) {
    if (cudaMemsetAsync(F->sort_status, 0, 4 * kRadix * (size_t)F->sort_tiles_max, s) != cudaSuccess)
      return check_launch("sort status memset");
    const int a = p & 1, b = (p + 1) & 1;
    k_sort_pass<<<grid, kSortThreads, sizeof(SortSmem), s>>>(F->keys[a], F->vals[a], F->keys[b], F->vals[b],
                                                             F->sort_hist + p * kRadix, F->sort_status,
                                                             F->counters + C_SORT_TICKET + p, F->counters, 8 * p);
    note_launch();
    if ((st = check_launch("k_sort_pass")) != BGS_OK) return st;
  }
  k_ranges<<<4 * num_sms(), 256, 0, s>>>(F->keys[F->final_buf], F->counters, F->ranges);
  note_launch();
  return check_launch("k_ranges");
}

}  // namespace bgs
