// adam.cu -- a11 fused Adam (K14), a8 L1 loss gradient (K15), and the workload-count
// kernel behind bgs_frame_stats (not on the timed path).
//
// K14 (R21, PyTorch Adam semantics): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// theta -= (lr / bc1) * m / (sqrt(v) / sqrt(bc2) + eps); g = 0.  One pass over the
// four fp32[59n] buffers with 16-byte vector loads/stores (1888 B per Gaussian, HBM
// bound: SURVEY §8(d)); the learning-rate group of each element follows from its
// offset in theta's segment layout (sh_dc = the first 3 of each Gaussian's 48 SH floats).
#include <algorithm>

#include "common.cuh"

namespace bgs {

struct AdamParams {
  float4* theta;
  float4* grad;
  float4* m;
  float4* v;
  int64_t n, base, total4;  // element i of the pointers is theta element base + i
  float lr[6];
  float b1, b2, eps;
  float step_size[6];  // lr / bc1
  float inv_sqrt_bc2;
  int32_t zero_grad;  // 0: grad is left as it is (the next step's chain rule assigns it)
};

__device__ __forceinline__ int adam_group(int64_t e, int64_t n) {
  if (e < 3 * n) return 0;
  if (e < 6 * n) return 1;
  if (e < 10 * n) return 2;
  if (e < 11 * n) return 3;
  // offset inside the SH segment: in 32 bits while 48n < 2^32 (n < 89.4M; a constant-divisor
  // modulo becomes a multiply-shift instead of a 64-bit division per element), else 64
  const int64_t o = e - 11 * n;
  const uint32_t k = n < (int64_t)(0xffffffffull / 48) ? (uint32_t)o % 48u : (uint32_t)((uint64_t)o % 48u);
  return k < 3u ? 4 : 5;
}

__device__ __forceinline__ void adam_one(float& th, float& g, float& m, float& v, float ss, const AdamParams& p) {
  m = fmaf(p.b1, m, (1.0f - p.b1) * g);
  v = fmaf(p.b2, v, (1.0f - p.b2) * g * g);
  const float denom = sqrtf(v) * p.inv_sqrt_bc2 + p.eps;
  th = th - ss * (m / denom);
  g = 0.0f;
}

__global__ void __launch_bounds__(256) k_adam(AdamParams p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.total4; i += stride) {
    float4 th = p.theta[i], g = p.grad[i], m = p.m[i], v = p.v[i];
    const int64_t e = p.base + 4 * i;
    const int g0 = adam_group(e, p.n), g3 = adam_group(e + 3, p.n);
    if (g0 == g3 && g0 < 4) {
      const float ss = p.step_size[g0];
      adam_one(th.x, g.x, m.x, v.x, ss, p);
      adam_one(th.y, g.y, m.y, v.y, ss, p);
      adam_one(th.z, g.z, m.z, v.z, ss, p);
      adam_one(th.w, g.w, m.w, v.w, ss, p);
    } else {
      adam_one(th.x, g.x, m.x, v.x, p.step_size[adam_group(e, p.n)], p);
      adam_one(th.y, g.y, m.y, v.y, p.step_size[adam_group(e + 1, p.n)], p);
      adam_one(th.z, g.z, m.z, v.z, p.step_size[adam_group(e + 2, p.n)], p);
      adam_one(th.w, g.w, m.w, v.w, p.step_size[adam_group(e + 3, p.n)], p);
    }
    p.theta[i] = th;
    if (p.zero_grad) p.grad[i] = g;
    p.m[i] = m;
    p.v[i] = v;
  }
}

// The scalar tail: local elements [start, end) (the last count mod 4).
__global__ void k_adam_tail(float* theta, float* grad, float* m, float* v, int64_t n, int64_t start, int64_t end,
                            AdamParams p) {
  const int64_t i = start + threadIdx.x;
  if (i >= end) return;
  float g = grad[i];
  adam_one(theta[i], g, m[i], v[i], p.step_size[adam_group(p.base + i, n)], p);
  if (p.zero_grad) grad[i] = g;
}

// Adam over theta elements [begin, begin + count) of the 59n layout; the pointers address
// element `begin` (a shard of a reduce-scattered update, or begin = 0 for all of theta).
// Elements at or past 59n (shard padding) are left untouched.
bgs_status launch_adam(float* theta, float* grad, float* m, float* v, int64_t n, int64_t begin, int64_t count,
                       const bgs_adam_hparams* hp, int64_t step, cudaStream_t s, bool zero_grad) {
  const int64_t total = std::max<int64_t>(0, std::min<int64_t>(count, 59 * n - begin));
  if (total == 0) return BGS_OK;
  AdamParams p;
  p.theta = (float4*)theta;
  p.grad = (float4*)grad;
  p.m = (float4*)m;
  p.v = (float4*)v;
  p.n = n;
  p.base = begin;
  p.total4 = total / 4;  // the tail (total mod 4) is handled below
  const float lr[6] = {hp->lr_means, hp->lr_log_scales, hp->lr_quats, hp->lr_opacity, hp->lr_sh_dc, hp->lr_sh_rest};
  const double bc1 = 1.0 - pow((double)hp->beta1, (double)step);
  const double bc2 = 1.0 - pow((double)hp->beta2, (double)step);
  for (int k = 0; k < 6; ++k) {
    p.lr[k] = lr[k];
    p.step_size[k] = (float)((double)lr[k] / bc1);
  }
  p.b1 = hp->beta1;
  p.b2 = hp->beta2;
  p.eps = hp->eps;
  p.inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
  p.zero_grad = zero_grad ? 1 : 0;
  const int64_t work = p.total4 > 0 ? p.total4 : 1;
  int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)num_sms() * 8);
  k_adam<<<blocks, 256, 0, s>>>(p);
  note_launch();
  bgs_status st = check_launch("k_adam");
  if (st != BGS_OK) return st;
  const int64_t tail = total - 4 * p.total4;
  if (tail > 0) {
    k_adam_tail<<<1, 4, 0, s>>>(theta, grad, m, v, n, 4 * p.total4, total, p);
    note_launch();
    return check_launch("k_adam_tail");
  }
  return BGS_OK;
}

// ---------------------------------------------------------------- fused exchange + Adam (§8(e) 3)
// NVSwitch multicast: grad_mc / theta_mc are multicast addresses of every rank's grad and
// theta (one NVLink-SHARP object each).  Per 4 elements of this rank's shard: the sum of
// all ranks' gradients in one in-switch reduction load (multimem.ld_reduce), the Adam
// update with the shard's moments, the new theta stored to every rank's replica in one
// multicast store (multimem.st), and the shard of every rank's grad zeroed the same way --
// reduce-scatter, Adam and all-gather in a single pass over the shard.
__device__ __forceinline__ float4 mm_ld_reduce_add(const float* mc) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(mc)
               : "memory");
  return r;
}
__device__ __forceinline__ void mm_st(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(256) k_adam_multimem(AdamParams p, float* grad_mc, float* theta_mc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.total4; i += stride) {
    const int64_t e = p.base + 4 * i;
    float4 g = mm_ld_reduce_add(grad_mc + e);
    float4 th = p.theta[i], m = p.m[i], v = p.v[i];
    adam_one(th.x, g.x, m.x, v.x, p.step_size[adam_group(e, p.n)], p);
    adam_one(th.y, g.y, m.y, v.y, p.step_size[adam_group(e + 1, p.n)], p);
    adam_one(th.z, g.z, m.z, v.z, p.step_size[adam_group(e + 2, p.n)], p);
    adam_one(th.w, g.w, m.w, v.w, p.step_size[adam_group(e + 3, p.n)], p);
    mm_st(theta_mc + e, th);
    mm_st(grad_mc + e, z4);
    p.m[i] = m;
    p.v[i] = v;
  }
}

bgs_status launch_adam_multimem(float* theta, float* theta_mc, float* grad_mc, float* m, float* v, int64_t n,
                                int64_t begin, int64_t count, const bgs_adam_hparams* hp, int64_t step,
                                cudaStream_t s) {
  const int64_t total = std::max<int64_t>(0, std::min<int64_t>(count, 59 * n - begin));
  if (total == 0) return BGS_OK;
  AdamParams p;
  p.theta = (float4*)(theta + begin);  // this rank's replica, read; the new values go out by multicast
  p.grad = nullptr;
  p.m = (float4*)m;
  p.v = (float4*)v;
  p.n = n;
  p.base = begin;
  p.total4 = total / 4;
  const float lr[6] = {hp->lr_means, hp->lr_log_scales, hp->lr_quats, hp->lr_opacity, hp->lr_sh_dc, hp->lr_sh_rest};
  const double bc1 = 1.0 - pow((double)hp->beta1, (double)step);
  const double bc2 = 1.0 - pow((double)hp->beta2, (double)step);
  for (int k = 0; k < 6; ++k) {
    p.lr[k] = lr[k];
    p.step_size[k] = (float)((double)lr[k] / bc1);
  }
  p.b1 = hp->beta1;
  p.b2 = hp->beta2;
  p.eps = hp->eps;
  p.inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
  p.zero_grad = 1;  // the multicast form zeroes every rank's shard of grad (multimem.st)
  const int64_t work = p.total4 > 0 ? p.total4 : 1;
  const int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)num_sms() * 8);
  k_adam_multimem<<<blocks, 256, 0, s>>>(p, grad_mc, theta_mc);
  note_launch();
  return check_launch("k_adam_multimem");
}

// ---------------------------------------------------------------- K15 L1 loss gradient
__global__ void __launch_bounds__(256) k_l1(const float* __restrict__ image, const uint8_t* __restrict__ target,
                                            int64_t count, float scale, float* __restrict__ dl, float* loss_sum) {
  float acc = 0.0f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const float d = image[i] - (float)target[i] * (1.0f / 255.0f);
    dl[i] = d > 0.0f ? scale : (d < 0.0f ? -scale : 0.0f);
    acc += fabsf(d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ float s[8];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int w = 0; w < 8; ++w) t += s[w];
    atomicAdd(loss_sum, t);
  }
}

bgs_status launch_l1(const float* image, const uint8_t* target, int32_t w, int32_t h, float scale, float* dl,
                     float* loss_sum, cudaStream_t s) {
  const int64_t count = 3ll * w * h;
  const int blocks = (int)std::min<int64_t>((count + 255) / 256, (int64_t)num_sms() * 4);
  k_l1<<<blocks, 256, 0, s>>>(image, target, count, scale, dl, loss_sum);
  note_launch();
  return check_launch("k_l1");
}

// ---------------------------------------------------------------- workload counters
// E_f per pixel is recomputed by re-walking the list with the forward's decisions; not
// timed (bgs_frame_stats).
__global__ void __launch_bounds__(kTilePixels) k_stats(const uint2* __restrict__ ranges,
                                                       const uint32_t* __restrict__ values,
                                                       const float4* __restrict__ record,
                                                       const uint32_t* __restrict__ counters, Cam cam,
                                                       const uint32_t* __restrict__ n_contrib,
                                                       unsigned long long* out) {
  const int tile = blockIdx.x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the blend kernels' mapping: warp w owns an 8x4 pixel block
  const int px = tx * kTile + (warp & 1) * 8 + (lane & 7), py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
  const float bx0 = (float)(tx * kTile + (warp & 1) * 8), by0 = (float)(ty * kTile + (warp >> 1) * 4);
  const float bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
  const bool inside = px < cam.W && py < cam.H;
  uint2 rg = ranges[tile];
  if (counters[C_OVERFLOW]) rg = make_uint2(0, 0);
  uint32_t walked = 0, nc = 0, blended = 0, walked_c = 0, bwd_c = 0;
  if (inside) {
    nc = n_contrib[(int64_t)py * cam.W + px];
    float T = 1.0f;
    for (uint32_t j = rg.x; j < rg.y; ++j) {
      ++walked;
      const uint32_t id = values[j];
      const float4 r0 = record[3 * id], r1 = record[3 * id + 1], r2 = record[3 * id + 2];
      (void)r2;
      const bool hit = r0.x + r0.z >= bx0 && r0.x - r0.z <= bx1 && r0.y + r0.w >= by0 && r0.y - r0.w <= by1;
      walked_c += hit;
      if (hit && j - rg.x < nc) ++bwd_c;
      const float dx = r0.x - (float)px, dy = r0.y - (float)py;
      const float power = fmaf(r1.x, dx * dx, fmaf(r1.z, dy * dy, r1.y * (dx * dy)));
      if (power > 0.0f) continue;
      const float alpha = fminf(0.99f, r1.w * fast_exp(power));
      if (alpha < (1.0f / 255.0f)) continue;
      const float tT = T * (1.0f - alpha);
      if (tT < 1e-4f) break;
      T = tT;
      ++blended;
    }
  }
  const uint32_t wmax = __reduce_max_sync(0xffffffffu, walked_c);
  unsigned long long f = walked, b = nc, bl = blended, fc = walked_c, bc = bwd_c;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    bl += __shfl_xor_sync(0xffffffffu, bl, o);
    fc += __shfl_xor_sync(0xffffffffu, fc, o);
    bc += __shfl_xor_sync(0xffffffffu, bc, o);
  }
  if (lane == 0) {
    atomicAdd(&out[0], f);
    atomicAdd(&out[1], b);
    atomicAdd(&out[2], 32ull * wmax);
    atomicAdd(&out[5], bl);
    atomicAdd(&out[6], fc);
    atomicAdd(&out[7], bc);
  }
  if (threadIdx.x == 0) atomicMax(&out[3], (unsigned long long)(rg.y - rg.x));
}

__global__ void k_count_visible(const int32_t* radius, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += radius[i] > 0;
  atomicAdd(&out[4], c);
}

bgs_status launch_stats(const Frame* F, const uint32_t* n_contrib, bgs_stats* out, cudaStream_t s) {
  unsigned long long* d = nullptr;
  if (cudaMallocAsync(&d, 8 * 8, s) != cudaSuccess) return check_launch("stats alloc");
  cudaMemsetAsync(d, 0, 64, s);
  k_stats<<<F->num_tiles, kTilePixels, 0, s>>>(F->ranges, F->vals[F->final_buf], F->record, F->counters, F->cam,
                                               n_contrib, d);
  if (F->n > 0) k_count_visible<<<num_sms() * 4, 256, 0, s>>>(F->radius, F->n, d);
  unsigned long long h[8];
  uint32_t c[2];
  cudaMemcpyAsync(h, d, 64, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(c, F->counters, 8, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("stats");
  out->evals_fwd = (int64_t)h[0];
  out->evals_bwd = (int64_t)h[1];
  out->evals_slot = (int64_t)h[2];
  out->max_list = (int64_t)h[3];
  out->visible = (int64_t)h[4];
  out->blended = (int64_t)h[5];
  out->evals_fwd_culled = (int64_t)h[6];
  out->evals_bwd_culled = (int64_t)h[7];
  out->num_keys = (int64_t)(((uint64_t)c[1] << 32) | c[0]);
  return check_launch("k_stats");
}

}  // namespace bgs
