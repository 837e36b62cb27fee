// importance.cu -- NEXT-3: T2's similarity-based sampling (PAPER.md
// §IV-C1, l.253-268) and the importance score "retained for use during rendering"
// (§IV-C3, l.279-284), plus the keep rule NEXT-4's render-only serving applies.
// Readings R37-R40:
//   k_tile_buckets  one CTA per 16x16 tile: each pixel's rendered colour (clamped to
//                   [0, 1]) -> c8 = min(255, floor(256 c)) -> c8 / 16 per channel -> key =
//                   R 256 + G 16 + B; a 4096-slot shared-memory table ("The hash table is
//                   implemented using shared memory", l.265) counts the pixels and sums
//                   their colour and opacity (1 - T_final); occupied buckets are emitted in
//                   ascending key order.
//   k_importance    one warp per (tile, 8x4 block): walks the whole tile list (no early
//                   stop: the score counts every pixel g reaches, occluded or not); per entry
//                   whose alpha >= 1/255 box reaches the block, every pixel with alpha_g >=
//                   1/255 (R14) adds sim(c_g, c_pixel) alpha_g and 1; warp sums go to the
//                   Gaussian's accumulators with one atomic each.
//   keep rule       stable radix sort of (I_g bits, index) ascending (or descending with
//                   `invert`), the first ceil(f n) are kept.
// None of this is on the training hot path (a2-a11); it is an analysis pass per viewpoint.
#include <math.h>

#include "common.cuh"

namespace bgs {

constexpr int kBucketSlots = 4096;

__device__ __forceinline__ uint32_t quant_level(float c) {
  const float u = fminf(fmaxf(c, 0.0f), 1.0f);
  const uint32_t c8 = min(255u, (uint32_t)floorf(u * 256.0f));
  return c8 >> 4;  // floor(c8 / 256 * 16)
}

__global__ void __launch_bounds__(kTilePixels) k_tile_buckets(const float* __restrict__ image,
                                                              const float* __restrict__ final_T, int W, int H,
                                                              int tiles_x, uint32_t* nb, uint16_t* keys,
                                                              uint32_t* counts, float* color_sum,
                                                              float* opacity_sum) {
  extern __shared__ float s_tab[];  // [4096][4] colour sums r, g, b and opacity sum
  __shared__ uint32_t s_cnt[kBucketSlots];
  __shared__ uint32_t s_wsum[kTilePixels / 32];
  const int tile = blockIdx.x, t = threadIdx.x;
  for (int k = t; k < kBucketSlots; k += kTilePixels) {
    s_cnt[k] = 0;
    s_tab[4 * k] = s_tab[4 * k + 1] = s_tab[4 * k + 2] = s_tab[4 * k + 3] = 0.0f;
  }
  __syncthreads();
  const int px = (tile % tiles_x) * kTile + (t & 15), py = (tile / tiles_x) * kTile + (t >> 4);
  if (px < W && py < H) {
    const size_t plane = (size_t)W * H, p = (size_t)py * W + px;
    const float r = fminf(fmaxf(image[p], 0.f), 1.f), g = fminf(fmaxf(image[plane + p], 0.f), 1.f),
                b = fminf(fmaxf(image[2 * plane + p], 0.f), 1.f);
    const uint32_t key = quant_level(r) * 256u + quant_level(g) * 16u + quant_level(b);
    atomicAdd(&s_cnt[key], 1u);
    atomicAdd(&s_tab[4 * key], r);
    atomicAdd(&s_tab[4 * key + 1], g);
    atomicAdd(&s_tab[4 * key + 2], b);
    atomicAdd(&s_tab[4 * key + 3], 1.0f - final_T[p]);
  }
  __syncthreads();
  // compaction in key order: thread t owns slots [16 t, 16 t + 16)
  uint32_t mine = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) mine += s_cnt[16 * t + j] != 0;
  uint32_t inc = mine;
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_wsum[w] = inc;
  __syncthreads();
  uint32_t base = 0;
  for (int k = 0; k < w; ++k) base += s_wsum[k];
  uint32_t at = base + inc - mine;
  const size_t tb = (size_t)tile * kTilePixels;
  for (int j = 0; j < 16; ++j) {
    const int k = 16 * t + j;
    if (!s_cnt[k]) continue;
    keys[tb + at] = (uint16_t)k;
    counts[tb + at] = s_cnt[k];
    color_sum[3 * (tb + at)] = s_tab[4 * k];
    color_sum[3 * (tb + at) + 1] = s_tab[4 * k + 1];
    color_sum[3 * (tb + at) + 2] = s_tab[4 * k + 2];
    opacity_sum[tb + at] = s_tab[4 * k + 3];
    ++at;
  }
  if (t == kTilePixels - 1) nb[tile] = at;
}

__global__ void __launch_bounds__(128) k_importance(const uint2* __restrict__ ranges, const uint32_t* __restrict__ values,
                                                   const float4* __restrict__ record, const uint32_t* counters,
                                                   Cam cam, const float* __restrict__ image, float* sum,
                                                   uint32_t* cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (item >= 8ll * cam.tiles_x * cam.tiles_y || counters[C_OVERFLOW]) return;
  const int tile = (int)(item >> 3), blk = (int)(item & 7);
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int bx = tx * kTile + (blk & 1) * 8, by = ty * kTile + (blk >> 1) * 4;
  const int px = bx + (lane & 7), py = by + (lane >> 3);
  const float bx0 = (float)bx, by0 = (float)by, bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
  const bool inside = px < cam.W && py < cam.H;
  float cr = 0.f, cg = 0.f, cb = 0.f;
  if (inside) {
    const size_t plane = (size_t)cam.W * cam.H, p = (size_t)py * cam.W + px;
    cr = fminf(fmaxf(image[p], 0.f), 1.f);
    cg = fminf(fmaxf(image[plane + p], 0.f), 1.f);
    cb = fminf(fmaxf(image[2 * plane + p], 0.f), 1.f);
  }
  const uint2 rg = ranges[tile];
  const float inv_sqrt3 = 0.57735026918962576f;
  for (uint32_t b = rg.x; b < rg.y; b += 32) {
    const uint32_t e = b + lane;
    uint32_t id = 0xffffffffu;
    bool hit = false;
    if (e < rg.y) {
      id = values[e];
      const float4 a = record[3 * id];
      hit = a.x + a.z >= bx0 && a.x - a.z <= bx1 && a.y + a.w >= by0 && a.y - a.w <= by1;
    }
    uint32_t bal = __ballot_sync(0xffffffffu, hit);
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      const uint32_t g = __shfl_sync(0xffffffffu, id, src);
      const float4 r0 = record[3 * g], r1 = record[3 * g + 1], r2 = record[3 * g + 2];
      float contrib = 0.f, one = 0.f;
      if (inside) {
        const float dx = r0.x - (float)px, dy = r0.y - (float)py;
        const float power = fmaf(r1.x, dx * dx, fmaf(r1.z, dy * dy, r1.y * (dx * dy)));
        const float alpha = fminf(0.99f, r1.w * expf(power));
        if (power <= 0.0f && alpha >= 1.0f / 255.0f) {
          const float er = fminf(r2.x, 1.f) - cr, eg = fminf(r2.y, 1.f) - cg, eb = fminf(r2.z, 1.f) - cb;
          contrib = (1.0f - sqrtf(er * er + eg * eg + eb * eb) * inv_sqrt3) * alpha;
          one = 1.0f;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
        one += __shfl_xor_sync(0xffffffffu, one, o);
      }
      if (lane == 0 && one > 0.f) {
        atomicAdd(&sum[g], contrib);
        atomicAdd(&cnt[g], (uint32_t)one);
      }
    }
  }
}

__global__ void k_importance_finish(int64_t n, const float* sum, const uint32_t* cnt, float* out,
                                    uint32_t* count_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cnt[i];
    out[i] = c ? sum[i] / (float)c : 0.0f;
    if (count_out) count_out[i] = c;
  }
}

// keys for the keep rule: I >= 0, so its float bits sort as unsigned; `invert` flips them
__global__ void __launch_bounds__(256) k_imp_keys(int64_t n, const float* __restrict__ imp, int invert, uint32_t* key,
                                                  uint32_t* val, uint32_t* hist) {
  __shared__ uint32_t s_h[4][256];
  for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) (&s_h[0][0])[k] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = __float_as_uint(fmaxf(imp[i], 0.0f));
    if (invert) k = ~k;
    key[i] = k;
    val[i] = (uint32_t)i;
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&s_h[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x)
    if ((&s_h[0][0])[k]) atomicAdd(&hist[k], (&s_h[0][0])[k]);
}

__global__ void k_keep_mark(int64_t n, int64_t keep_n, const uint32_t* __restrict__ order, uint8_t* keep) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    keep[order[r]] = r < keep_n ? 1 : 0;
}

struct ImpWs {
  float* sum;
  uint32_t *cnt, *key[2], *val[2], *hist, *status, *counters;
  int64_t status_tiles;
};

static size_t imp_align(size_t x) { return (x + 255) & ~(size_t)255; }

static bool imp_layout(int64_t n, char* base, ImpWs* w, size_t* total) {
  if (n < 1 || n >= ((int64_t)1 << 31)) return false;
  const int64_t tiles = (n + 4095) / 4096;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o = imp_align(o + b);
    return at;
  };
  const size_t a_s = take(4 * (size_t)n), a_c = take(4 * (size_t)n), a_k0 = take(4 * (size_t)n),
               a_k1 = take(4 * (size_t)n), a_v0 = take(4 * (size_t)n), a_v1 = take(4 * (size_t)n),
               a_h = take(4 * 4 * 256), a_st = take(4 * 256 * (size_t)tiles), a_co = take(4 * C_NUM);
  if (total) *total = o;
  if (w && base) {
    w->sum = (float*)(base + a_s);
    w->cnt = (uint32_t*)(base + a_c);
    w->key[0] = (uint32_t*)(base + a_k0);
    w->key[1] = (uint32_t*)(base + a_k1);
    w->val[0] = (uint32_t*)(base + a_v0);
    w->val[1] = (uint32_t*)(base + a_v1);
    w->hist = (uint32_t*)(base + a_h);
    w->status = (uint32_t*)(base + a_st);
    w->counters = (uint32_t*)(base + a_co);
    w->status_tiles = tiles;
  }
  return true;
}

}  // namespace bgs

using namespace bgs;

extern "C" {

bgs_status bgs_tile_buckets(const float* image, const float* final_T, int32_t w, int32_t h, uint32_t* nb,
                            uint16_t* keys, uint32_t* counts, float* color_sum, float* opacity_sum, void* stream) {
  if (!image || !final_T || !nb || !keys || !counts || !color_sum || !opacity_sum || w < 1 || h < 1 || w > 16384 ||
      h > 16384)
    return BGS_ERR_INVALID;
  const int tx = (w + kTile - 1) / kTile, ty = (h + kTile - 1) / kTile;
  const size_t smem = (size_t)kBucketSlots * 4 * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tile_buckets, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_tile_buckets<<<tx * ty, kTilePixels, smem, (cudaStream_t)stream>>>(image, final_T, w, h, tx, nb, keys, counts,
                                                                       color_sum, opacity_sum);
  note_launch();
  return check_launch("k_tile_buckets");
}

size_t bgs_importance_workspace_bytes(int64_t n) {
  size_t total = 0;
  return imp_layout(n, nullptr, nullptr, &total) ? total : 0;
}

bgs_status bgs_importance(const bgs_frame* f, const float* image, float* importance, uint32_t* count,
                          void* workspace, size_t bytes, void* stream) {
  ImpWs w;
  size_t total = 0;
  if (!f || !image || !importance || !workspace || ((uintptr_t)workspace & 255u)) return BGS_ERR_INVALID;
  const Frame* F = frame_of(f);
  if (F->magic != kFrameMagic || !F->cam_valid || F->n < 1 || !imp_layout(F->n, (char*)workspace, &w, &total) ||
      bytes < total)
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(w.sum, 0, 4 * (size_t)F->n, s) != cudaSuccess ||
      cudaMemsetAsync(w.cnt, 0, 4 * (size_t)F->n, s) != cudaSuccess)
    return check_launch("importance memset");
  const int64_t warps = 8ll * F->num_tiles;
  k_importance<<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(F->ranges, F->vals[F->final_buf], F->record, F->counters,
                                                          F->cam, image, w.sum, w.cnt);
  note_launch();
  bgs_status st = check_launch("k_importance");
  if (st != BGS_OK) return st;
  k_importance_finish<<<4 * num_sms(), 256, 0, s>>>(F->n, w.sum, w.cnt, importance, count);
  note_launch();
  return check_launch("k_importance_finish");
}

bgs_status bgs_importance_keep(const float* importance, int64_t n, float fraction, int32_t invert, uint8_t* keep,
                               void* workspace, size_t bytes, void* stream) {
  ImpWs w;
  size_t total = 0;
  if (!importance || !keep || !workspace || ((uintptr_t)workspace & 255u) || !(fraction >= 0.0f && fraction <= 1.0f) ||
      !imp_layout(n, (char*)workspace, &w, &total) || bytes < total)
    return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(w.hist, 0, 4 * 4 * 256, s) != cudaSuccess ||
      cudaMemsetAsync(w.counters, 0, 4 * C_NUM, s) != cudaSuccess)
    return check_launch("keep memset");
  const int grid = 4 * num_sms();
  k_imp_keys<<<grid, 256, 0, s>>>(n, importance, invert, w.key[0], w.val[0], w.hist);
  note_launch();
  bgs_status st = check_launch("k_imp_keys");
  if (st != BGS_OK) return st;
  for (int p = 0; p < 4; ++p) {
    if (cudaMemsetAsync(w.status, 0, 4 * 256 * (size_t)w.status_tiles, s) != cudaSuccess)
      return check_launch("keep status memset");
    const int a = p & 1, b = (p + 1) & 1;
    st = launch_sort_pass32(w.key[a], w.val[a], w.key[b], w.val[b], w.hist + 256 * p, w.status, w.counters + 4 + p,
                            w.counters, 8 * p, n, s);
    if (st != BGS_OK) return st;
  }
  const int64_t keep_n = (int64_t)ceil((double)fraction * (double)n);
  k_keep_mark<<<grid, 256, 0, s>>>(n, keep_n, w.val[0], keep);
  note_launch();
  return check_launch("k_keep_mark");
}

bgs_status bgs_frame_set_keep(bgs_frame* f, const uint8_t* keep) {
  if (!f) return BGS_ERR_INVALID;
  Frame* F = frame_of(f);
  if (F->magic != kFrameMagic) return BGS_ERR_INVALID;
  F->keep = keep;
  return BGS_OK;
}

}  // extern "C"
