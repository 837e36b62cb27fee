// radix.cu -- a5 (K10): one pass of the stable LSD radix sort of (key, value) pairs,
// onesweep style (one kernel per 8-bit digit pass; keys read once and written once).
//
// "N denotes the set of Gaussians contributing to the pixel, sorted by depth" (PAPER.md
// l.149, §II-A); ties by Gaussian index (R13): a stable ascending
// sort of key = tile << 32 | depth bits, fed in index order, yields (tile, depth, index).
//
// A 4096-key tile per CTA iteration: warp-level multi-split ranking with
// ballot-based peer detection (stable inside a warp's contiguous 512-key slice), warp prefix across
// the CTA, decoupled look-back across tiles for the digit's global offset, then a
// shared-memory reorder so the global writes are digit-contiguous (coalesced).  A
// persistent grid takes tiles in ticket order, so a predecessor tile is always resident
// when a successor waits on it.  The pass histograms come from the key duplication
// (depth digits) and the per-tile key counts (tile digits), see sort.cu.
#include "common.cuh"

namespace bgs {

#ifndef BGS_SORT_MINB
#define BGS_SORT_MINB 3
#endif
constexpr int kSortThreads = 256, kSortItems = BGS_SORT_ITEMS, kSortTile = kSortThreads * kSortItems, kRadix = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr uint32_t kStA = 1u << 30, kStP = 2u << 30, kStMask = (1u << 30) - 1;
#ifndef BGS_LOOK_BATCH
#define BGS_LOOK_BATCH 8
#endif
constexpr int kLookBatch = BGS_LOOK_BATCH;

__device__ __forceinline__ uint64_t load_k(const uint32_t* counters) {
  return ((uint64_t)counters[C_K_HI] << 32) | counters[C_K_LO];
}

// ---------------------------------------------------------------- one onesweep pass
template <typename K>
struct SortSmem {
  K keys[kSortTile];
  uint32_t vals[kSortTile];
  uint32_t warp_hist[kSortWarps][kRadix];  // counts, then exclusive prefix over warps
  uint32_t tile_start[kRadix];             // exclusive prefix over digits inside the tile
  uint32_t global_base[kRadix];            // destination of the digit's first key of this tile
  uint32_t hist_excl[kRadix];              // exclusive scan of this pass's global histogram
  uint32_t scan_tmp[kSortWarps];
  uint32_t tile;
  uint32_t tile_valid;
};

// Sorts `count` (key, value) pairs by the digit at `shift`; count = -1 means "read K from
// counters" (the 64-bit tile|depth keys), count = -2 "read the visible count" (the depth
// sort after its first pass), otherwise it is the host-known length.  drop_culled: keys
// ~0 (culled Gaussians) take no slot and are not written (the pass histogram excludes
// them), so the depth sort's first pass compacts the visible Gaussians to [0, V).
// fill_to > 0 (the depth sort's last pass): ranks [V, fill_to) get zero tile counts.
// gen_tt != null (the depth sort's first pass): kin holds the depth bits of every Gaussian,
// the key of Gaussian i is its depth bits if gen_tt[i] (tiles touched) else ~0, its value i.
template <typename KT>
__global__ void __launch_bounds__(kSortThreads, BGS_SORT_MINB) k_sort_pass(const KT* __restrict__ kin,
                                                            const uint32_t* __restrict__ vin, KT* kout,
                                                            uint32_t* vout, const uint32_t* __restrict__ hist,
                                                            uint32_t* status, uint32_t* ticket,
                                                            const uint32_t* counters, int shift, int64_t count,
                                                            const uint2* __restrict__ rect, uint32_t* rank_cnt,
                                                            uint2* rank_rect, uint32_t* rank_h, bool drop_culled,
                                                            int64_t fill_to, const uint32_t* __restrict__ gen_tt) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem<KT>& S = *reinterpret_cast<SortSmem<KT>*>(smem_raw);
  if (counters[C_OVERFLOW]) return;
  const int64_t K = count >= 0 ? count : count == -1 ? (int64_t)load_k(counters) : (int64_t)counters[C_VISIBLE];
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
    const KT culled = (KT)~(KT)0;
    // load: warp w owns the contiguous slice [w*512, (w+1)*512) of the tile
    KT key[kSortItems];
    uint32_t val[kSortItems];
    uint16_t rank[kSortItems];
    const int wbase = warp * (kSortItems * 32);
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
      const int idx = wbase + k * 32 + lane;
      if (idx < tcount) {
        if (gen_tt) {  // the depth sort's first pass: keys from the depths, values = indices
          key[k] = gen_tt[tbase + idx] ? kin[tbase + idx] : culled;
          val[k] = (uint32_t)(tbase + idx);
        } else {
          key[k] = kin[tbase + idx];
          val[k] = vin[tbase + idx];
        }
      } else {
        key[k] = (KT)~(KT)0;
        val[k] = 0;
      }
    }
    // warp-level multi-split ranking, in input order (stable): peers of a digit from 8
    // ballots, the lowest peer reserves the slots with one shared-memory atomic and
    // broadcasts the base by shuffle
    uint32_t* wh = S.warp_hist[warp];
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
      const int idx = wbase + k * 32 + lane;
      const bool valid = idx < tcount && !(drop_culled && key[k] == culled);
      const uint32_t d = (uint32_t)((key[k] >> shift) & 0xff);
      uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
      const int leader = valid ? __ffs(peers) - 1 : lane;
      uint32_t got = 0;
      if (valid && leader == lane) got = atomicAdd(&wh[d], (uint32_t)__popc(peers));
      const uint32_t base = __shfl_sync(0xffffffffu, got, leader);
      rank[k] = (uint16_t)(base + __popc(peers & lt));
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
    if (tile == 0) st_relaxed_u32(&st[tid], kStP | cnt);
    else st_relaxed_u32(&st[tid], kStA | cnt);
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
      if (tid == kRadix - 1) S.tile_valid = off + incl;  // the tile's keys that take a slot
    }
    // look-back for digit tid: the statuses of kLookBatch predecessors are loaded together
    // (independent loads in flight), then consumed in order until an inclusive prefix; an
    // entry not yet published is re-polled alone.  A serial one-at-a-time walk through
    // aggregate-only predecessors cost one L2 round trip per tile in the first wave.
    uint32_t prefix = 0;
    if (tile > 0) {
      int64_t j = tile - 1;
      bool done = false;
      while (!done) {
        uint32_t sv[kLookBatch];
#pragma unroll
        for (int q = 0; q < kLookBatch; ++q)
          sv[q] = (j - q >= 0) ? ld_relaxed_u32(&status[(j - q) * kRadix + tid]) : kStP;
#pragma unroll
        for (int q = 0; q < kLookBatch; ++q) {
          if (done) break;
          uint32_t v = sv[q];
          while ((v >> 30) == 0) v = ld_relaxed_u32(&status[(j - q) * kRadix + tid]);
          prefix += v & kStMask;
          done = (v >> 30) == 2;
        }
        j -= kLookBatch;
      }
      st_relaxed_u32(&st[tid], kStP | (prefix + cnt));
    }
    S.global_base[tid] = S.hist_excl[tid] + prefix;
    __syncthreads();
    // reorder through shared memory (digit-contiguous)
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
      const int idx = wbase + k * 32 + lane;
      if (idx < tcount && !(drop_culled && key[k] == culled)) {
        const uint32_t d = (uint32_t)((key[k] >> shift) & 0xff);
        const uint32_t pos = S.tile_start[d] + S.warp_hist[warp][d] + rank[k];
        S.keys[pos] = key[k];
        S.vals[pos] = val[k];
      }
    }
    __syncthreads();
    const int tvalid = (int)S.tile_valid;
    if (rank_rect) {
      // the depth sort's last pass: per-rank tile count and packed rect, the rect gathers of
      // four keys per thread in flight together
      constexpr int B = 4;
      for (int j0 = tid; j0 < tvalid; j0 += B * kSortThreads) {
        uint32_t gq[B], vq[B];
        uint2 rq[B];
        bool ok[B];
#pragma unroll
        for (int q = 0; q < B; ++q) {
          const int j = j0 + q * kSortThreads;
          ok[q] = j < tvalid;
          const KT k2 = ok[q] ? S.keys[j] : (KT)~(KT)0;
          const uint32_t d = (uint32_t)((k2 >> shift) & 0xff);
          gq[q] = ok[q] ? S.global_base[d] + (uint32_t)j - S.tile_start[d] : 0u;
          vq[q] = ok[q] ? S.vals[j] : 0u;
          rq[q] = make_uint2(0u, 0u);
          if (ok[q]) {
            kout[gq[q]] = k2;
            if ((uint32_t)k2 != 0xffffffffu) rq[q] = __ldg(rect + vq[q]);  // visible: the preprocess's rect
          }
        }
#pragma unroll
        for (int q = 0; q < B; ++q) {
          if (!ok[q]) continue;
          vout[gq[q]] = vq[q];
          const uint32_t w = rq[q].y & 0xffffu, hh = rq[q].y >> 16;
          rank_cnt[gq[q]] = w * hh;
          rank_rect[gq[q]] = make_uint2(rq[q].x, w);
          rank_h[gq[q]] = hh;
        }
      }
    } else
    for (int j = tid; j < tvalid; j += kSortThreads) {
      const KT k2 = S.keys[j];
      const uint32_t d = (uint32_t)((k2 >> shift) & 0xff);
      const uint32_t g = S.global_base[d] + (uint32_t)j - S.tile_start[d];
      const uint32_t v = S.vals[j];
      kout[g] = k2;
      vout[g] = v;
    }
    __syncthreads();
  }
  if (fill_to > K)  // ranks past the visible ones own no tiles
    for (int64_t r = K + (int64_t)blockIdx.x * kSortThreads + tid; r < fill_to; r += (int64_t)gridDim.x * kSortThreads) {
      rank_cnt[r] = 0u;
      rank_rect[r] = make_uint2(0u, 0u);
      rank_h[r] = 0u;
    }
}

template <typename KT>
static int pass_grid() {
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_sort_pass<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem<KT>));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sort_pass<KT>, kSortThreads, sizeof(SortSmem<KT>));
    if (per_sm < 1) per_sm = 1;
    grid = per_sm * num_sms();
  }
  return grid;
}

int sort_pass_grid() { return pass_grid<uint64_t>(); }

bgs_status launch_sort_pass(const uint64_t* kin, const uint32_t* vin, uint64_t* kout, uint32_t* vout,
                            const uint32_t* hist, uint32_t* status, uint32_t* ticket, const uint32_t* counters,
                            int shift, cudaStream_t s) {
  k_sort_pass<uint64_t><<<pass_grid<uint64_t>(), kSortThreads, sizeof(SortSmem<uint64_t>), s>>>(
      kin, vin, kout, vout, hist, status, ticket, counters, shift, -1, nullptr, nullptr, nullptr, nullptr, false, 0,
      nullptr);
  note_launch();
  return check_launch("k_sort_pass<u64>");
}

bgs_status launch_sort_pass32(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                              const uint32_t* hist, uint32_t* status, uint32_t* ticket, const uint32_t* counters,
                              int shift, int64_t count, cudaStream_t s, const uint2* rect, uint32_t* rank_cnt,
                              uint2* rank_rect, uint32_t* rank_h, bool drop_culled, int64_t fill_to,
                              const uint32_t* gen_tt) {
  k_sort_pass<uint32_t><<<pass_grid<uint32_t>(), kSortThreads, sizeof(SortSmem<uint32_t>), s>>>(
      kin, vin, kout, vout, hist, status, ticket, counters, shift, count, rect, rank_cnt, rank_rect, rank_h,
      drop_culled, fill_to, gen_tt);
  note_launch();
  return check_launch("k_sort_pass<u32>");
}

}  // namespace bgs
