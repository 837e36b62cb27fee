// render_fwd.cu -- a7: front-to-back alpha blend (§II-A l.143-149):
//   C = sum_{i in N} c_i alpha_i prod_{j<i} (1 - alpha_j),  N = the tile's depth-sorted list,
// with readings R14 (skip power > 0; alpha = min(0.99, o G); skip alpha < 1/255),
// R15 (stop before T (1 - alpha) < 1e-4, the crossing Gaussian is not blended),
// R16 (out = C + T_final bg; n_contrib = 1-based position of the last blended entry).
// Decision-bearing arithmetic is the canonical tree of R22 (explicit fmaf, file built
// with --fmad=false); G uses MUFU.EX2 (R23 near-tie rule covers the few-ulp difference).
//
// Workload-balanced mapping (the paper's Challenge-2: with one thread
// per pixel walking a tile in lock-step, the slowest pixels and longest tiles set the
// pace): the unit of work is one warp x one 8x4 pixel block of a tile (one pixel per
// lane).  A persistent grid of independent warps pulls these (tile, block) items from a
// global ticket, longest first (by this frame's previous per-block walk lengths when it
// re-renders a view, else by tile list length), so no
// warp waits on another and a warp leaves its tile as soon as its own 32 pixels are done.
// A warp streams its tile's list 32 entries per step: each lane gathers one entry's
// 16-byte cull record {x, y, ex, ey} and tests the conservative alpha >= 1/255 box against
// the block; the hits (about a fifth of the list on the garden workload) are compacted
// with a ballot and their 48-byte records {x,y,ex,ey | A,B,C,o | r,g,b,pthr} staged in the
// warp's slice of shared memory -- the B200 form of the paper's T3 batch loading of
// per-Gaussian contiguous RGB.  The step loop is
// software-pipelined (ids three steps ahead, cull records two, hit records one), so the
// gathers overlap the walk.  List positions are kept, so n_contrib and every decision
// are those of the plain per-pixel walk.
#include "common.cuh"

namespace bgs {

constexpr int kFwdWarps = 4;

__device__ __forceinline__ bool box_hits_f(const float4 a, float bx0, float by0, float bx1, float by1) {
  return a.x + a.z >= bx0 && a.x - a.z <= bx1 && a.y + a.w >= by0 && a.y - a.w <= by1;
}

__global__ void __launch_bounds__(kFwdWarps * 32) k_render_fwd(const uint2* __restrict__ ranges,
                                                                const uint32_t* __restrict__ values,
                                                                const float4* __restrict__ record,
                                                                const uint32_t* __restrict__ counters, Cam cam,
                                                                const uint32_t* __restrict__ item_order,
                                                                uint32_t n_items, uint32_t* ticket,
                                                                float* __restrict__ image, float* __restrict__ final_T,
                                                                uint32_t* __restrict__ n_contrib,
                                                                uint32_t* __restrict__ block_cost) {
  __shared__ float4 s_rec[kFwdWarps][3][32];
  __shared__ uint32_t s_pos[kFwdWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const bool overflow = counters[C_OVERFLOW] != 0;
  float4* sr0 = s_rec[warp][0];
  float4* sr1 = s_rec[warp][1];
  float4* sr2 = s_rec[warp][2];
  uint32_t* spos = s_pos[warp];
  const float4 none = make_float4(-1e30f, -1e30f, -1e30f, -1e30f);
  while (true) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(ticket, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const uint32_t it = item_order[item];
    const int tile = (int)(it >> 3), blk = (int)(it & 7);
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int bx = tx * kTile + (blk & 1) * 8, by = ty * kTile + (blk >> 1) * 4;
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    const float bx0 = (float)bx, by0 = (float)by, bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
    const bool inside = px < cam.W && py < cam.H;
    const float pxf = (float)px, pyf = (float)py;
    uint2 rg = ranges[tile];
    if (overflow) rg = make_uint2(0, 0);
    const int len = (int)(rg.y - rg.x);
    const int nst = (len + 31) / 32;
    bool done = !inside;
    float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
    uint32_t last = 0;
    auto load_id = [&](int s) -> uint32_t {
      const int p = 32 * s + lane;
      return (p < len) ? __ldg(values + rg.x + (uint32_t)p) : 0xffffffffu;
    };
    auto load_cull = [&](uint32_t id) { return id != 0xffffffffu ? __ldg(record + 3 * id) : none; };
    if (nst > 0 && !__all_sync(0xffffffffu, done)) {
      // pipeline prologue: step 0 fully, step 1 cull record, step 2 id
      uint32_t id_c = load_id(0);
      float4 a_c = load_cull(id_c);
      uint32_t id_n = load_id(1);
      float4 a_n = load_cull(id_n);
      uint32_t id_nn = load_id(2);
      bool h_c = box_hits_f(a_c, bx0, by0, bx1, by1);
      float4 r1_c = none, r2_c = none;
      if (h_c) {
        r1_c = __ldg(record + 3 * id_c + 1);
        r2_c = __ldg(record + 3 * id_c + 2);
      }
      for (int s = 0; s < nst; ++s) {
        // (1) commit step s into the warp's shared-memory slice
        const uint32_t bal = __ballot_sync(0xffffffffu, h_c);
        if (h_c) {
          const int q = __popc(bal & lt);
          sr0[q] = a_c;
          sr1[q] = r1_c;
          sr2[q] = r2_c;
          spos[q] = (uint32_t)(32 * s + lane);
        }
        __syncwarp();
        // (2) step s+1 hit test and records; (3) step s+2 cull record, step s+3 id
        const bool h_n = box_hits_f(a_n, bx0, by0, bx1, by1);
        float4 r1_n = none, r2_n = none;
        if (h_n) {
          r1_n = __ldg(record + 3 * id_n + 1);
          r2_n = __ldg(record + 3 * id_n + 2);
        }
        const float4 a_nn = load_cull(id_nn);
        const uint32_t id_nnn = load_id(s + 3);
        // (4) walk step s
        const int m = __popc(bal);
        int lastk = -1;
        for (int k = 0; k < m; ++k) {
          const float4 r0 = sr0[k];
          const float4 r1 = sr1[k];
          const float4 r2 = sr2[k];
          const float dx = r0.x - pxf, dy = r0.y - pyf;
          const float power = fmaf(r1.x, dx * dx, fmaf(r1.z, dy * dy, r1.y * (dx * dy)));
          // one predicate: pixel done, R14's power > 0 guard, or power below the exact
          // alpha < 1/255 bound (pthr, preprocess) -- the last skips the MUFU path
          if (done | (power > 0.0f) | (power < r2.w)) continue;
          const float alpha = fminf(0.99f, r1.w * fast_exp(power));
          if (alpha < (1.0f / 255.0f)) continue;
          const float tT = T * (1.0f - alpha);
          if (tT < 1e-4f) {
            done = true;
            continue;
          }
          const float w = alpha * T;
          Cr = fmaf(r2.x, w, Cr);
          Cg = fmaf(r2.y, w, Cg);
          Cb = fmaf(r2.z, w, Cb);
          T = tT;
          lastk = k;
        }
        if (lastk >= 0) last = spos[lastk] + 1u;
        if (__all_sync(0xffffffffu, done)) break;
        // rotate the pipeline
        id_c = id_n;
        a_c = a_n;
        h_c = h_n;
        r1_c = r1_n;
        r2_c = r2_n;
        id_n = id_nn;
        a_n = a_nn;
        id_nn = id_nnn;
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
    // the block's largest n_contrib: the backward's (and this frame's next forward's) cost
    const uint32_t wl = __reduce_max_sync(0xffffffffu, last);
    if (lane == 0) block_cost[it] = wl;
  }
}

static int fwd_grid() {
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_fwd, kFwdWarps * 32, 0);
    grid = (per_sm < 1 ? 1 : per_sm) * num_sms();
  }
  return grid;
}

bgs_status launch_render_fwd(Frame* F, float* image, float* final_T, uint32_t* n_contrib, cudaStream_t s) {
  if (cudaMemsetAsync(F->counters + C_FWD_TICKET, 0, 4, s) != cudaSuccess)
    return check_launch("render_fwd memset");
  const uint32_t n_items = 8u * (uint32_t)F->num_tiles;
  k_render_fwd<<<fwd_grid(), kFwdWarps * 32, 0, s>>>(F->ranges, F->vals[F->final_buf], F->record, F->counters,
                                                     F->cam, F->order_fwd, n_items, F->counters + C_FWD_TICKET,
                                                     image, final_T, n_contrib, F->block_cost);
  note_launch();
  F->have_cost = 1;
  return check_launch("k_render_fwd");
}

}  // namespace bgs
