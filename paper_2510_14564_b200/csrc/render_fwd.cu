// render_fwd.cu -- a7: front-to-back alpha blend (§II-A l.143-149):
//   C = sum_{i in N} c_i alpha_i prod_{j<i} (1 - alpha_j),  N = the tile's depth-sorted list,
// with readings R14 (skip power > 0; alpha = min(0.99, o G); skip alpha < 1/255),
// R15 (stop before T (1 - alpha) < 1e-4, the crossing Gaussian is not blended),
// R16 (out = C + T_final bg; n_contrib = 1-based position of the last blended entry).
// Decision-bearing arithmetic is the canonical tree of R22 (explicit fmaf, file built
// with --fmad=false); G uses MUFU.EX2 (R23 near-tie rule covers the few-ulp difference).
//
// Workload-balanced mapping (the paper's Challenge-2: with one thread
// per pixel walking in lock-step over a tile, the slowest pixels set the pace):
//  * one CTA per 16x16 tile, heaviest tiles first (k_tile_scan orders tiles by list length);
//  * warp-specialised: a producer warp streams the tile list in 256-entry batches into a
//    4-slot shared-memory ring -- the B200 form of the paper's T3 batch loading of
//    per-Gaussian contiguous RGB into shared memory: 48-byte
//    records {x,y,ex,ey | A,B,C,o | r,g,b,cbits} gathered with 16-byte loads -- and 8
//    consumer warps, one per 8x4 pixel block, each take the batches at their own pace
//    (mbarrier full/empty handshakes), so a warp whose pixels are busy never holds up
//    the others, and the CTA only stops streaming once every warp's pixels are done;
//  * per batch a consumer warp compacts the entries whose conservative alpha >= 1/255
//    box (ex, ey) reaches its block -- the rest would be skipped by all 32 of its pixels --
//    and its pixels walk only those.  List positions are kept, so n_contrib and every
//    decision are those of the plain per-pixel walk.
#include "common.cuh"

namespace bgs {

constexpr int kBatch = 256;
constexpr int kRing = 4;
constexpr int kConsumers = 8;
constexpr int kFwdThreads = (kConsumers + 1) * 32;

struct FwdSmem {
  float4 r0[kRing][kBatch];
  float4 r1[kRing][kBatch];
  float4 r2[kRing][kBatch];
  uint32_t cnt[kRing];
  uint64_t full[kRing];
  uint64_t empty[kRing];
  uint8_t list[kConsumers][kBatch];
  int alive;
  uint32_t cost;
};

__global__ void __launch_bounds__(kFwdThreads) k_render_fwd(const uint2* __restrict__ ranges,
                                                             const uint32_t* __restrict__ values,
                                                             const float4* __restrict__ record,
                                                             const uint32_t* __restrict__ counters, Cam cam,
                                                             const uint32_t* __restrict__ tile_order,
                                                             float* __restrict__ image, float* __restrict__ final_T,
                                                             uint32_t* __restrict__ n_contrib,
                                                             uint32_t* __restrict__ tile_cost) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdSmem& S = *reinterpret_cast<FwdSmem*>(smem_raw);
  const int tile = (int)tile_order[blockIdx.x];
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint2 rg = ranges[tile];
  if (counters[C_OVERFLOW]) rg = make_uint2(0, 0);
  const uint32_t len = rg.y - rg.x;
  const int nb = (int)((len + kBatch - 1) / kBatch);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&S.full[s], 32);         // the producer warp's 32 lanes
      mbar_init(&S.empty[s], kConsumers);  // one arrive per consumer warp
    }
    S.alive = kConsumers;
    S.cost = 0;
  }
  __syncthreads();
  if (warp == kConsumers) {
    // ------------------------------------------------ producer warp
    for (int b = 0; b < nb; ++b) {
      const int slot = b & (kRing - 1);
      if (b >= kRing) mbar_wait(&S.empty[slot], (uint32_t)((b / kRing) - 1) & 1u);
      const int alive = *(volatile int*)&S.alive;
      const int cnt = alive ? (int)min((uint32_t)kBatch, len - (uint32_t)b * kBatch) : 0;
      const uint32_t j0 = rg.x + (uint32_t)b * kBatch;
      for (int e = lane; e < cnt; e += 32) {
        const uint32_t id = __ldg(values + j0 + e);
        S.r0[slot][e] = __ldg(record + 3 * id);
        S.r1[slot][e] = __ldg(record + 3 * id + 1);
        S.r2[slot][e] = __ldg(record + 3 * id + 2);
      }
      if (lane == 0) S.cnt[slot] = (uint32_t)cnt;
      __syncwarp();
      mbar_arrive(&S.full[slot]);
    }
  } else {
    // ------------------------------------------------ consumer warp: one 8x4 pixel block
    const int bx = tx * kTile + (warp & 1) * 8, by = ty * kTile + (warp >> 1) * 4;
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    const float bx0 = (float)bx, by0 = (float)by, bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
    const bool inside = px < cam.W && py < cam.H;
    const float pxf = (float)px, pyf = (float)py;
    const uint32_t lt = lanemask_lt();
    uint8_t* list = S.list[warp];
    bool done = !inside;
    bool reported = false;
    float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
    uint32_t last = 0;
    for (int b = 0; b < nb; ++b) {
      const int slot = b & (kRing - 1);
      mbar_wait(&S.full[slot], (uint32_t)(b / kRing) & 1u);
      const int cnt = (int)S.cnt[slot];
      const bool all_done = __all_sync(0xffffffffu, done);
      if (all_done && !reported) {
        if (lane == 0) atomicSub(&S.alive, 1);
        reported = true;
      }
      if (!all_done && cnt > 0) {
        const float4* r0s = S.r0[slot];
        const float4* r1s = S.r1[slot];
        const float4* r2s = S.r2[slot];
        int m = 0;
        for (int r = 0; r * 32 < cnt; ++r) {
          const int e = r * 32 + lane;
          bool hit = false;
          if (e < cnt) {
            const float4 a = r0s[e];
            hit = a.x + a.z >= bx0 && a.x - a.z <= bx1 && a.y + a.w >= by0 && a.y - a.w <= by1;
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, hit);
          if (hit) list[m + __popc(bal & lt)] = (uint8_t)e;
          m += __popc(bal);
        }
        __syncwarp();
        const uint32_t pos0 = (uint32_t)b * kBatch + 1u;
        for (int k = 0; k < m && !done; ++k) {
          const int e = list[k];
          const float4 r0 = r0s[e];
          const float dx = r0.x - pxf, dy = r0.y - pyf;
          const float4 r1 = r1s[e];
          const float power = fmaf(r1.x, dx * dx, fmaf(r1.z, dy * dy, r1.y * (dx * dy)));
          if (power > 0.0f) continue;
          const float alpha = fminf(0.99f, r1.w * fast_exp(power));
          if (alpha < (1.0f / 255.0f)) continue;
          const float tT = T * (1.0f - alpha);
          if (tT < 1e-4f) {
            done = true;
            break;
          }
          const float w = alpha * T;
          const float4 r2 = r2s[e];
          Cr = fmaf(r2.x, w, Cr);
          Cg = fmaf(r2.y, w, Cg);
          Cb = fmaf(r2.z, w, Cb);
          T = tT;
          last = pos0 + (uint32_t)e;
        }
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(&S.empty[slot]);
    }
    if (inside) {
      const int64_t pix = (int64_t)py * cam.W + px;
      const int64_t plane = (int64_t)cam.W * cam.H;
      image[pix] = fmaf(T, cam.bg[0], Cr);
      image[plane + pix] = fmaf(T, cam.bg[1], Cg);
      image[2 * plane + pix] = fmaf(T, cam.bg[2], Cb);
      final_T[pix] = T;
      n_contrib[pix] = last;
    }
    // the tile's largest n_contrib: the backward's cost estimate for its heavy-first order
    const uint32_t wl = __reduce_max_sync(0xffffffffu, last);
    if (lane == 0 && wl) atomicMax(&S.cost, wl);
  }
  __syncthreads();
  if (threadIdx.x == 0) tile_cost[tile] = S.cost;
}

bgs_status launch_render_fwd(Frame* F, float* image, float* final_T, uint32_t* n_contrib, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_render_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FwdSmem));
    attr = true;
  }
  k_render_fwd<<<F->num_tiles, kFwdThreads, sizeof(FwdSmem), s>>>(F->ranges, F->vals[F->final_buf], F->record,
                                                                   F->counters, F->cam, F->tile_order, image,
                                                                   final_T, n_contrib, F->tile_cost);
  note_launch();
  return check_launch("k_render_fwd");
}

}  // namespace bgs
