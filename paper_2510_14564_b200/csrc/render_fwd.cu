// render_fwd.cu -- a7: front-to-back alpha blend (§II-A l.143-149):
//   C = sum_{i in N} c_i alpha_i prod_{j<i} (1 - alpha_j),  N = the tile's depth-sorted list,
// with readings R14 (skip power > 0; alpha = min(0.99, o G); skip alpha < 1/255),
// R15 (stop before T (1 - alpha) < 1e-4, the crossing Gaussian is not blended),
// R16 (out = C + T_final bg; n_contrib = 1-based position of the last blended entry).
// Decision-bearing arithmetic is the canonical tree of R22 (explicit fmaf, file built
// with --fmad=false); G uses MUFU.EX2 (R23 near-tie rule covers the few-ulp difference).
//
// Mapping: one CTA per 16x16 tile, one thread per pixel; the tile's list is streamed
// in batches of 256 render records (48 B each, {x,y,A,B | C,o,r,g | b,..}) staged into
// shared memory by the whole CTA with 16-byte loads, then every pixel thread walks the
// batch reading broadcast LDS.128 -- the B200 form of the paper's T3 "batch loading
// into shared memory" of per-Gaussian contiguous RGB.
#include "common.cuh"

namespace bgs {

constexpr int kBatch = kTilePixels;

__global__ void __launch_bounds__(kTilePixels) k_render_fwd(const uint2* __restrict__ ranges,
                                                            const uint32_t* __restrict__ values,
                                                            const float4* __restrict__ record,
                                                            const uint32_t* __restrict__ counters, Cam cam,
                                                            float* __restrict__ image, float* __restrict__ final_T,
                                                            uint32_t* __restrict__ n_contrib) {
  __shared__ float4 s_r0[kBatch], s_r1[kBatch], s_r2[kBatch];
  const int tile = blockIdx.x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
  const bool inside = px < cam.W && py < cam.H;
  const float pxf = (float)px, pyf = (float)py;
  uint2 rg = ranges[tile];
  if (counters[C_OVERFLOW]) rg = make_uint2(0, 0);
  bool done = !inside;
  float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
  uint32_t last = 0;
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
    for (int k = 0; k < cnt && !done; ++k) {
      const float4 r0 = s_r0[k];
      const float dx = r0.x - pxf, dy = r0.y - pyf;
      const float4 r1 = s_r1[k];
      const float power = fmaf(r0.z, dx * dx, fmaf(r1.x, dy * dy, r0.w * (dx * dy)));
      if (power > 0.0f) continue;
      const float alpha = fminf(0.99f, r1.y * fast_exp(power));
      if (alpha < (1.0f / 255.0f)) continue;
      const float tT = T * (1.0f - alpha);
      if (tT < 1e-4f) {
        done = true;
        break;
      }
      const float w = alpha * T;
      Cr = fmaf(r1.z, w, Cr);
      Cg = fmaf(r1.w, w, Cg);
      Cb = fmaf(s_r2[k].x, w, Cb);
      T = tT;
      last = start - rg.x + (uint32_t)k + 1u;
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
}

bgs_status launch_render_fwd(Frame* F, float* image, float* final_T, uint32_t* n_contrib, cudaStream_t s) {
  k_render_fwd<<<F->num_tiles, kTilePixels, 0, s>>>(F->ranges, F->vals[F->final_buf], F->record, F->counters, F->cam,
                                                    image, final_T, n_contrib);
  note_launch();
  return check_launch("k_render_fwd");
}

}  // namespace bgs
