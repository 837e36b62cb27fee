// render_fwd.cu -- a7: front-to-back alpha blend (§II-A l.143-149):
//   C = sum_{i in N} c_i alpha_i prod_{j<i} (1 - alpha_j),  N = the tile's depth-sorted list,
// with readings R14 (skip power > 0; alpha = min(0.99, o G); skip alpha < 1/255),
// R15 (stop before T (1 - alpha) < 1e-4, the crossing Gaussian is not blended),
// R16 (out = C + T_final bg; n_contrib = 1-based position of the last blended entry).
// Decision-bearing arithmetic is the canonical tree of R22 (explicit fmaf, file built
// with --fmad=false); G uses MUFU.EX2 (R23 near-tie rule covers the few-ulp difference).
//
// Mapping (B200): one CTA per 16x16 tile, 8 warps, each warp owns an 8x4 pixel block
// (one pixel per lane).  The tile list is streamed in batches of 256 render records
// (48 B: {x,y,ex,ey | A,B,C,o | r,g,b,cbits}) staged into shared memory by the whole CTA
// with 16-byte loads -- the B200 form of the paper's T3 "batch loading into shared
// memory" of per-Gaussian contiguous RGB.  Each warp then
// compacts the batch to the entries whose conservative alpha >= 1/255 bounding box
// (ex, ey from the preprocess) touches its 8x4 block -- every other entry would be
// skipped by all 32 of its pixels anyway -- so a pixel walks only those (about a third
// of the list on the garden workload).  List positions are kept, so n_contrib and every
// decision are those of the plain per-pixel walk.
#include "common.cuh"

namespace bgs {

constexpr int kBatch = kTilePixels;

// pixel of (tile, warp, lane): warp w covers columns (w&1)*8..+7, rows (w>>1)*4..+3
__device__ __forceinline__ void warp_block_pixel(int tx, int ty, int warp, int lane, int& px, int& py) {
  px = tx * kTile + (warp & 1) * 8 + (lane & 7);
  py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
}

__global__ void __launch_bounds__(kTilePixels) k_render_fwd(const uint2* __restrict__ ranges,
                                                            const uint32_t* __restrict__ values,
                                                            const float4* __restrict__ record,
                                                            const uint32_t* __restrict__ counters, Cam cam,
                                                            const uint32_t* __restrict__ tile_order,
                                                            float* __restrict__ image, float* __restrict__ final_T,
                                                            uint32_t* __restrict__ n_contrib,
                                                            uint32_t* __restrict__ tile_cost) {
  __shared__ float4 s_r0[kBatch], s_r1[kBatch], s_r2[kBatch];
  __shared__ uint8_t s_list[kTilePixels / 32][kBatch];
  __shared__ uint32_t s_cost;
  const int tile = (int)tile_order[blockIdx.x];  // heavy tiles first (k_tile_scan)
  if (threadIdx.x == 0) s_cost = 0;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int px, py;
  warp_block_pixel(tx, ty, warp, lane, px, py);
  const bool inside = px < cam.W && py < cam.H;
  const float pxf = (float)px, pyf = (float)py;
  // the warp's pixel block, clipped to the image
  const float bx0 = (float)(tx * kTile + (warp & 1) * 8), by0 = (float)(ty * kTile + (warp >> 1) * 4);
  const float bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
  uint2 rg = ranges[tile];
  if (counters[C_OVERFLOW]) rg = make_uint2(0, 0);
  bool done = !inside;
  float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
  uint32_t last = 0;
  const uint32_t lt = lanemask_lt();
  for (uint32_t start = rg.x; start < rg.y; start += kBatch) {
    if (__syncthreads_count(done) == kTilePixels) break;
    const uint32_t j = start + threadIdx.x;
    if (j < rg.y) {
      const uint32_t id = values[j];
      s_r0[threadIdx.x] = __ldg(record + 3 * id);
      s_r1[threadIdx.x] = __ldg(record + 3 * id + 1);
      s_r2[threadIdx.x] = __ldg(record + 3 * id + 2);
    }
    __syncthreads();
    const int cnt = (int)min(rg.y - start, (uint32_t)kBatch);
    // per-warp compaction of the batch to the entries that can reach this 8x4 block
    int m = 0;
    if (__any_sync(0xffffffffu, !done)) {
#pragma unroll
      for (int r = 0; r < kBatch / 32; ++r) {
        const int e = r * 32 + lane;
        bool hit = false;
        if (e < cnt) {
          const float4 a = s_r0[e];
          hit = a.x + a.z >= bx0 && a.x - a.z <= bx1 && a.y + a.w >= by0 && a.y - a.w <= by1;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, hit);
        if (hit) s_list[warp][m + __popc(bal & lt)] = (uint8_t)e;
        m += __popc(bal);
      }
      __syncwarp();
    }
    for (int k = 0; k < m && !done; ++k) {
      const int e = s_list[warp][k];
      const float4 r0 = s_r0[e];
      const float dx = r0.x - pxf, dy = r0.y - pyf;
      const float4 r1 = s_r1[e];
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
      const float4 r2 = s_r2[e];
      Cr = fmaf(r2.x, w, Cr);
      Cg = fmaf(r2.y, w, Cg);
      Cb = fmaf(r2.z, w, Cb);
      T = tT;
      last = start - rg.x + (uint32_t)e + 1u;
    }
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
  if (lane == 0 && wl) atomicMax(&s_cost, wl);
  __syncthreads();
  if (threadIdx.x == 0) tile_cost[tile] = s_cost;
}

bgs_status launch_render_fwd(Frame* F, float* image, float* final_T, uint32_t* n_contrib, cudaStream_t s) {
  k_render_fwd<<<F->num_tiles, kTilePixels, 0, s>>>(F->ranges, F->vals[F->final_buf], F->record, F->counters, F->cam,
                                                    F->tile_order, image, final_T, n_contrib, F->tile_cost);
  note_launch();
  return check_launch("k_render_fwd");
}

}  // namespace bgs
