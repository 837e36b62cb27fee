// render_bwd.cu -- a9 blend backward (K12).
//
// The paper has no backward; it inherits 3DGS training.  Reading
// R18: the gradient of the forward O1-O14 with every discrete decision frozen (cull,
// rect, power/alpha skips, early stop, the 0.99 alpha clamp -> zero gradient to o and G,
// the SH clamp, the J-clamp branch).
//
// One CTA per tile, 8 warps each owning an 8x4 pixel block (as the forward); the tile list
// is walked back to front from the tile's largest n_contrib, in batches of 256 records
// staged in shared memory.  Each warp compacts a batch to the entries that can reach its
// block (the same exact alpha-level-set test as the forward, plus position < the warp's
// largest n_contrib).  Per pixel: T_i = T_{i+1} / (1 - alpha_i), the colour behind
// accumulates S += c alpha T (S starts at T_final bg), and each evaluated entry yields 9
// partials {dxy(2), dconic(3), dopacity, drgb(3)}.  They are summed across the warp with
// shuffles, then across the CTA's 8 warps with shared-memory atomics, and each entry is
// flushed to grad2d[id] once per tile with two 16-byte vector REDs and one scalar RED --
// instead of 3DGS's nine scalar global atomics per evaluated (pixel, Gaussian).
//
// K13 (the chain rule to theta) is in preprocess_bwd.cu.
#include "common.cuh"

namespace bgs {

constexpr int kBatchB = kTilePixels;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

__device__ __forceinline__ void red_add_v4(float4* addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(kTilePixels) k_render_bwd(const uint2* __restrict__ ranges,
                                                            const uint32_t* __restrict__ values,
                                                            const float4* __restrict__ record,
                                                            const uint32_t* __restrict__ counters, Cam cam,
                                                            const uint32_t* __restrict__ tile_order,
                                                            const float* __restrict__ dl_dimage,
                                                            const float* __restrict__ final_T,
                                                            const uint32_t* __restrict__ n_contrib,
                                                            float4* __restrict__ grad2d) {
  __shared__ float4 s_r0[kBatchB], s_r1[kBatchB], s_r2[kBatchB];
  __shared__ uint32_t s_id[kBatchB];
  __shared__ float s_g[9][kBatchB];
  __shared__ uint8_t s_hit[kBatchB];
  __shared__ uint8_t s_list[kTilePixels / 32][kBatchB];
  __shared__ uint32_t s_max;
  const int tile = (int)tile_order[blockIdx.x];  // heavy first, by the forward's tile_cost
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
  const int py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
  const float bx0 = (float)(tx * kTile + (warp & 1) * 8), by0 = (float)(ty * kTile + (warp >> 1) * 4);
  const float bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
  const bool inside = px < cam.W && py < cam.H;
  const float pxf = (float)px, pyf = (float)py;
  uint2 rg = ranges[tile];
  if (counters[C_OVERFLOW]) rg = make_uint2(0, 0);
  const int64_t pix = (int64_t)py * cam.W + px;
  const int64_t plane = (int64_t)cam.W * cam.H;
  const uint32_t my_last = inside ? n_contrib[pix] : 0u;
  float T = inside ? final_T[pix] : 1.0f;
  float dLr = 0.f, dLg = 0.f, dLb = 0.f;
  if (inside) {
    dLr = dl_dimage[pix];
    dLg = dl_dimage[plane + pix];
    dLb = dl_dimage[2 * plane + pix];
  }
  float Sr = T * cam.bg[0], Sg = T * cam.bg[1], Sb = T * cam.bg[2];
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  const uint32_t wmax = __reduce_max_sync(0xffffffffu, my_last);
  if (lane == 0 && wmax) atomicMax(&s_max, wmax);
  __syncthreads();
  const int tile_last = (int)min(s_max, rg.y - rg.x);
  const uint32_t lt = lanemask_lt();
  for (int end = tile_last; end > 0; end -= kBatchB) {
    const int begin = max(0, end - kBatchB);
    const int cnt = end - begin;
    __syncthreads();
    if ((int)threadIdx.x < cnt) {
      const uint32_t id = values[rg.x + begin + threadIdx.x];
      s_id[threadIdx.x] = id;
      s_r0[threadIdx.x] = __ldg(record + 3 * id);
      s_r1[threadIdx.x] = __ldg(record + 3 * id + 1);
      s_r2[threadIdx.x] = __ldg(record + 3 * id + 2);
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) s_g[q][threadIdx.x] = 0.0f;
    s_hit[threadIdx.x] = 0;
    __syncthreads();
    // per-warp compaction: entries that can reach this block, below the warp's largest n_contrib
    int m = 0;
    if (wmax > (uint32_t)begin) {
#pragma unroll
      for (int r = 0; r < kBatchB / 32; ++r) {
        const int e = r * 32 + lane;
        bool hit = false;
        if (e < cnt && (uint32_t)(begin + e) < wmax) {
          const float4 a = s_r0[e];
          const float4 c = s_r2[e];
          hit = a.x + c.z >= bx0 && a.x - c.z <= bx1 && a.y + c.w >= by0 && a.y - c.w <= by1;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, hit);
        if (hit) s_list[warp][m + __popc(bal & lt)] = (uint8_t)e;
        m += __popc(bal);
      }
      __syncwarp();
    }
    for (int k = m - 1; k >= 0; --k) {
      const int e = s_list[warp][k];
      const uint32_t pos = (uint32_t)(begin + e);
      bool act = pos < my_last;
      float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f, g5 = 0.f, g6 = 0.f, g7 = 0.f, g8 = 0.f;
      if (act) {
        const float4 r0 = s_r0[e];
        const float4 r1 = s_r1[e];
        const float dx = r0.x - pxf, dy = r0.y - pyf;
        const float power = fmaf(r0.z, dx * dx, fmaf(r1.x, dy * dy, r0.w * (dx * dy)));
        const float G = fast_exp(power);
        const float og = r1.y * G;
        const float alpha = fminf(0.99f, og);
        if (power > 0.0f || alpha < (1.0f / 255.0f)) {
          act = false;
        } else {
          const float ioma = 1.0f / (1.0f - alpha);
          T = T * ioma;  // transmittance in front of this Gaussian
          const float w = alpha * T;
          const float cr = r1.z, cg = r1.w, cb = s_r2[e].x;
          g6 = w * dLr;
          g7 = w * dLg;
          g8 = w * dLb;
          const float dLda = dLr * (cr * T - Sr * ioma) + dLg * (cg * T - Sg * ioma) + dLb * (cb * T - Sb * ioma);
          Sr = fmaf(cr, w, Sr);
          Sg = fmaf(cg, w, Sg);
          Sb = fmaf(cb, w, Sb);
          if (og <= 0.99f) {  // unclamped alpha: gradient to opacity and G (R18)
            g5 = dLda * G;
            const float dp = dLda * og;  // dL/dpower
            g0 = dp * (2.0f * r0.z * dx + r0.w * dy);
            g1 = dp * (2.0f * r1.x * dy + r0.w * dx);
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
          atomicAdd(&s_g[0][e], g0); atomicAdd(&s_g[1][e], g1); atomicAdd(&s_g[2][e], g2);
          atomicAdd(&s_g[3][e], g3); atomicAdd(&s_g[4][e], g4); atomicAdd(&s_g[5][e], g5);
          atomicAdd(&s_g[6][e], g6); atomicAdd(&s_g[7][e], g7); atomicAdd(&s_g[8][e], g8);
          s_hit[e] = 1;
        }
      }
    }
    __syncthreads();
    // one flush per (tile, entry)
    if ((int)threadIdx.x < cnt && s_hit[threadIdx.x]) {
      const int e = threadIdx.x;
      float4* dst = grad2d + 3 * s_id[e];
      red_add_v4(dst, make_float4(s_g[0][e], s_g[1][e], s_g[2][e], s_g[3][e]));
      red_add_v4(dst + 1, make_float4(s_g[4][e], s_g[5][e], s_g[6][e], s_g[7][e]));
      atomicAdd(&dst[2].x, s_g[8][e]);
    }
  }
}

bgs_status launch_blend_bwd(Frame* F, const float* dL_dimage, const float* final_T, const uint32_t* n_contrib,
                            cudaStream_t s) {
  bgs_status st = launch_tile_order(F->tile_cost, F->num_tiles, F->counters, F->tile_order_bwd, s);
  if (st != BGS_OK) return st;
  k_render_bwd<<<F->num_tiles, kTilePixels, 0, s>>>(F->ranges, F->vals[F->final_buf], F->record, F->counters, F->cam,
                                                    F->tile_order_bwd, dL_dimage, final_T, n_contrib, F->grad2d);
  note_launch();
  return check_launch("k_render_bwd");
}

bgs_status launch_render_bwd(const bgs_gaussians* g, Frame* F, const float* dL_dimage, const float* final_T,
                             const uint32_t* n_contrib, float* grad, cudaStream_t s) {
  bgs_status st = launch_blend_bwd(F, dL_dimage, final_T, n_contrib, s);
  return st != BGS_OK ? st : launch_preprocess_bwd(g, F, grad, s);
}

}  // namespace bgs
