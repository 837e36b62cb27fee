// render_bwd.cu -- a9 blend backward (K12).
//
// The paper has no backward; it inherits 3DGS training.  Reading
// R18: the gradient of the forward O1-O14 with every discrete decision frozen (cull,
// rect, power/alpha skips, early stop, the 0.99 alpha clamp -> zero gradient to o and G,
// the SH clamp, the J-clamp branch).
//
// Same workload-balanced mapping as the forward: independent warps of a persistent grid
// pull (tile, 8x4 block) items heaviest first -- by the forward's per-tile largest
// n_contrib -- and each walks its tile list back to front from its own block's largest
// n_contrib, 32 entries at a time, compacted to the entries whose alpha >= 1/255 box
// reaches the block (exact, as in the forward).  Per pixel: T_i = T_{i+1} / (1 - alpha_i),
// the colour behind accumulates S += c alpha T (S starts at T_final bg), and each
// evaluated entry yields 9 partials {dxy(2), dconic(3), dopacity, drgb(3)}, summed across
// the warp with shuffles; lane 0 then issues two 16-byte vector REDs and one scalar RED
// into grad2d[id] -- instead of 3DGS's nine scalar global atomics per evaluated
// (pixel, Gaussian).
//
// K13 (the chain rule to theta) is in preprocess_bwd.cu.
#include "common.cuh"

namespace bgs {

constexpr int kBwdWarpsPerCta = 4;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

__device__ __forceinline__ void red_add_v4(float4* addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(kBwdWarpsPerCta * 32) k_render_bwd(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ values, const float4* __restrict__ record,
    const uint32_t* __restrict__ counters, Cam cam, const uint32_t* __restrict__ tile_order, uint32_t n_items,
    uint32_t* ticket, const float* __restrict__ dl_dimage, const float* __restrict__ final_T,
    const uint32_t* __restrict__ n_contrib, float4* __restrict__ grad2d) {
  __shared__ float4 s_rec[kBwdWarpsPerCta][3][32];
  __shared__ uint32_t s_pos[kBwdWarpsPerCta][32];
  __shared__ uint32_t s_id[kBwdWarpsPerCta][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const bool overflow = counters[C_OVERFLOW] != 0;
  float4* sr0 = s_rec[warp][0];
  float4* sr1 = s_rec[warp][1];
  float4* sr2 = s_rec[warp][2];
  uint32_t* spos = s_pos[warp];
  uint32_t* sid = s_id[warp];
  const int64_t plane = (int64_t)cam.W * cam.H;
  while (true) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(ticket, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const int tile = (int)tile_order[item >> 3], blk = (int)(item & 7);
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int bx = tx * kTile + (blk & 1) * 8, by = ty * kTile + (blk >> 1) * 4;
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    const float bx0 = (float)bx, by0 = (float)by, bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
    const bool inside = px < cam.W && py < cam.H;
    const float pxf = (float)px, pyf = (float)py;
    uint2 rg = ranges[tile];
    if (overflow) rg = make_uint2(0, 0);
    const int64_t pix = (int64_t)py * cam.W + px;
    const uint32_t my_last = inside ? n_contrib[pix] : 0u;
    const uint32_t wmax = min(__reduce_max_sync(0xffffffffu, my_last), rg.y - rg.x);
    if (wmax == 0) continue;
    float T = inside ? final_T[pix] : 1.0f;
    float dLr = 0.f, dLg = 0.f, dLb = 0.f;
    if (inside) {
      dLr = dl_dimage[pix];
      dLg = dl_dimage[plane + pix];
      dLb = dl_dimage[2 * plane + pix];
    }
    float Sr = T * cam.bg[0], Sg = T * cam.bg[1], Sb = T * cam.bg[2];
    for (int end = (int)wmax; end > 0; end -= 32) {
      const int begin = end - 32;  // may be negative: those lanes are idle
      const int posl = begin + lane;
      bool hit = false;
      uint32_t id = 0;
      float4 a;
      if (posl >= 0) {
        id = __ldg(values + rg.x + (uint32_t)posl);
        a = __ldg(record + 3 * id);
        hit = a.x + a.z >= bx0 && a.x - a.z <= bx1 && a.y + a.w >= by0 && a.y - a.w <= by1;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int q = __popc(bal & lt);
        sr0[q] = a;
        sr1[q] = __ldg(record + 3 * id + 1);
        sr2[q] = __ldg(record + 3 * id + 2);
        spos[q] = (uint32_t)posl;
        sid[q] = id;
      }
      __syncwarp();
      const int m = __popc(bal);
      for (int k = m - 1; k >= 0; --k) {
        const uint32_t pos = spos[k];
        bool act = pos < my_last;
        float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f, g5 = 0.f, g6 = 0.f, g7 = 0.f, g8 = 0.f;
        if (act) {
          const float4 r0 = sr0[k];
          const float4 r1 = sr1[k];
          const float dx = r0.x - pxf, dy = r0.y - pyf;
          const float power = fmaf(r1.x, dx * dx, fmaf(r1.z, dy * dy, r1.y * (dx * dy)));
          const float G = fast_exp(power);
          const float og = r1.w * G;
          const float alpha = fminf(0.99f, og);
          if (power > 0.0f || alpha < (1.0f / 255.0f)) {
            act = false;
          } else {
            const float ioma = 1.0f / (1.0f - alpha);
            T = T * ioma;  // transmittance in front of this Gaussian
            const float w = alpha * T;
            const float4 r2 = sr2[k];
            g6 = w * dLr;
            g7 = w * dLg;
            g8 = w * dLb;
            const float dLda =
                dLr * (r2.x * T - Sr * ioma) + dLg * (r2.y * T - Sg * ioma) + dLb * (r2.z * T - Sb * ioma);
            Sr = fmaf(r2.x, w, Sr);
            Sg = fmaf(r2.y, w, Sg);
            Sb = fmaf(r2.z, w, Sb);
            if (og <= 0.99f) {  // unclamped alpha: gradient to opacity and G (R18)
              g5 = dLda * G;
              const float dp = dLda * og;  // dL/dpower
              g0 = dp * (2.0f * r1.x * dx + r1.y * dy);
              g1 = dp * (2.0f * r1.z * dy + r1.y * dx);
              g2 = dp * (-0.5f * dx * dx);
              g3 = dp * (-dx * dy);
              g4 = dp * (-0.5f * dy * dy);
            }
          }
        }
        if (__any_sync(0xffffffffu, act)) {
          g0 = warp_sum(g0); g1 = warp_sum(g1); g2 = warp_sum(g2);
          g3 = warp_sum(g3); g4 = warp_sum(g4); g5 = warp_sum(g5);
          g6 = warp_sum(g6); g7 = warp_sum(g7); g8 = warp_sum(g8);
          if (lane == 0) {
            float4* dst = grad2d + 3 * sid[k];
            red_add_v4(dst, make_float4(g0, g1, g2, g3));
            red_add_v4(dst + 1, make_float4(g4, g5, g6, g7));
            atomicAdd(&dst[2].x, g8);
          }
        }
      }
      __syncwarp();
    }
  }
}

static int bwd_grid() {
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_bwd, kBwdWarpsPerCta * 32, 0);
    grid = (per_sm < 1 ? 1 : per_sm) * num_sms();
  }
  return grid;
}

bgs_status launch_blend_bwd(Frame* F, const float* dL_dimage, const float* final_T, const uint32_t* n_contrib,
                            cudaStream_t s) {
  bgs_status st = launch_tile_order(F->tile_cost, F->num_tiles, F->counters, F->tile_order_bwd, s);
  if (st != BGS_OK) return st;
  if (cudaMemsetAsync(F->counters + C_BWD_TICKET, 0, 4, s) != cudaSuccess) return check_launch("blend_bwd memset");
  k_render_bwd<<<bwd_grid(), kBwdWarpsPerCta * 32, 0, s>>>(
      F->ranges, F->vals[F->final_buf], F->record, F->counters, F->cam, F->tile_order_bwd, 8u * (uint32_t)F->num_tiles,
      F->counters + C_BWD_TICKET, dL_dimage, final_T, n_contrib, F->grad2d);
  note_launch();
  return check_launch("k_render_bwd");
}

bgs_status launch_render_bwd(const bgs_gaussians* g, Frame* F, const float* dL_dimage, const float* final_T,
                             const uint32_t* n_contrib, float* grad, cudaStream_t s) {
  bgs_status st = launch_blend_bwd(F, dL_dimage, final_T, n_contrib, s);
  return st != BGS_OK ? st : launch_preprocess_bwd(g, F, grad, s);
}

}  // namespace bgs
