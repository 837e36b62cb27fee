// loss.cu -- NEXT-2: the 3DGS training loss between the blend forward
// (a7) and backward (a9), fused into two tiled kernels:
//   Loss = (1 - lam) mean|x - y| + lam (1 - mean SSIM(x, y)),  lam = 0.2 in 3DGS,
// SSIM per channel with an 11x11 Gaussian window (sigma 1.5, zero padding), C1 = 0.01^2,
// C2 = 0.03^2 (Wang et al. 2004, the quality metric of PAPER.md §VI-A l.394; window per
// SPEC.md l.171; readings R28-R30 in DESIGN.md §3).
//
// The 11-tap passes run two maps at once where they pair ({x, y}, {x^2, y^2}; {dS/dm, dS/dE})
// as paired FP32 (FFMA2): the same rounding per map, half the instructions.
// k_ssim_fwd: per (32x32 tile, channel): x and y = target/255 with a 5-pixel halo staged in
// shared memory, the five window moments {w*x, w*y, w*x^2, w*y^2, w*xy} by a separable
// 11-tap pass (rows, then columns), then per pixel SSIM, |x - y| and the three partials of
// SSIM w.r.t. the raw moments (dS/dm, dS/dE, dS/dP) written to the workspace; each block
// writes its sums of SSIM and |x - y| to its own slot (no same-address atomics).
// k_ssim_bwd: per tile, the three partial maps (halo 5, zero outside the image) correlated
// with the (symmetric) window, and dL/dx = scale ((1 - lam) sign(x - y) - lam (w*dS/dm +
// 2 x w*dS/dE + y w*dS/dP)) / N; block 0 also reduces the per-block sums into the loss.
// HBM traffic per view: image 12 B + target 3 B + 9 partial maps 2 x 36 B + dL 12 B per
// pixel, ~100 B per pixel (0.1 GB at 1237 x 822): a few tens of microseconds.
#include <math.h>

#include "common.cuh"

namespace bgs {

constexpr int kLTx = 32, kLTy = 32, kLR = 5, kLWin = 2 * kLR + 1;
constexpr int kLHx = kLTx + 2 * kLR, kLHy = kLTy + 2 * kLR;  // tile + halo (42 x 42)
constexpr int kLThreads = 256;
constexpr int kLStage = (kLHy * kLHx + kLThreads - 1) / kLThreads;  // staging rounds per thread
// register blocking: the row pass gives each thread 4 consecutive outputs of one halo row
// (14 inputs per map instead of 44), the column pass 4 consecutive outputs of one column
constexpr int kLRun = 4, kLSegs = kLTx / kLRun, kLRowItems = kLHy * kLSegs, kLColRuns = kLTy / kLRun;
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;
static_assert(kLColRuns * kLTx == kLThreads, "one column run per thread");

struct LossWin {
  float w[kLWin];
};

// the 11-tap window over 14 consecutive values -> 4 outputs
__device__ __forceinline__ void win4(const LossWin& win, const float* v, float* o) {
#pragma unroll
  for (int j = 0; j < kLRun; ++j) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < kLWin; ++k) acc = fmaf(win.w[k], v[j + k], acc);
    o[j] = acc;
  }
}

// the same over two maps at once (paired FP32: one FFMA2 per tap, separately rounded halves)
__device__ __forceinline__ void win4x2(const LossWin& win, const float2* v, float2* o) {
#pragma unroll
  for (int j = 0; j < kLRun; ++j) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < kLWin; ++k) acc = __ffma2_rn(make_float2(win.w[k], win.w[k]), v[j + k], acc);
    o[j] = acc;
  }
}

__global__ void __launch_bounds__(kLThreads) k_ssim_fwd(const float* __restrict__ img, const uint8_t* __restrict__ tgt,
                                                        int W, int H, LossWin win, float* __restrict__ part,
                                                        float* __restrict__ acc) {
  // x and y interleaved (the paired window passes load both with one 8-byte access)
  __shared__ float2 s_xy[kLHy][kLHx + 1];
  __shared__ float2 h01[kLHy][kLTx + 1], h23[kLHy][kLTx + 1];  // {w*x, w*y}, {w*x^2, w*y^2} along rows
  __shared__ float h4[kLHy][kLTx + 1];                         // w*xy along rows
  const int ch = blockIdx.z;
  const int x0 = blockIdx.x * kLTx, y0 = blockIdx.y * kLTy;
  const size_t plane = (size_t)W * H;
  const float* xc = img + ch * plane;
  const uint8_t* yc = tgt + ch * plane;
  {
    // the tile + halo in one batch of independent loads per thread (kLStage rounds unrolled:
    // every load in flight before the first store)
    float xv[kLStage], yv[kLStage];
#pragma unroll
    for (int q = 0; q < kLStage; ++q) {
      const int i = threadIdx.x + q * kLThreads;
      const int r = i / kLHx, c = i - r * kLHx;
      const int gx = x0 + c - kLR, gy = y0 + r - kLR;
      xv[q] = 0.f;
      yv[q] = 0.f;
      if (i < kLHy * kLHx && gx >= 0 && gx < W && gy >= 0 && gy < H) {
        xv[q] = __ldg(xc + (size_t)gy * W + gx);
        yv[q] = (float)__ldg(yc + (size_t)gy * W + gx) * (1.0f / 255.0f);
      }
    }
#pragma unroll
    for (int q = 0; q < kLStage; ++q) {
      const int i = threadIdx.x + q * kLThreads;
      if (i < kLHy * kLHx) s_xy[i / kLHx][i % kLHx] = make_float2(xv[q], yv[q]);
    }
  }
  __syncthreads();
  // rows: the 11-tap pass along x of the five moment maps, 4 outputs per thread; (x, y) and
  // (x^2, y^2) as pairs
  for (int it = threadIdx.x; it < kLRowItems; it += kLThreads) {
    const int r = it / kLSegs, c0 = (it - r * kLSegs) * kLRun;
    float2 v[kLRun + kLWin - 1], o[kLRun];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v[k] = s_xy[r][c0 + k];
    win4x2(win, v, o);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) h01[r][c0 + j] = o[j];
    float u[kLRun + kLWin - 1], ou[kLRun];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) u[k] = v[k].x * v[k].y;
    win4(win, u, ou);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) h4[r][c0 + j] = ou[j];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v[k] = __fmul2_rn(v[k], v[k]);
    win4x2(win, v, o);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) h23[r][c0 + j] = o[j];
  }
  __syncthreads();
  // columns (4 consecutive rows of one column per thread), then per pixel SSIM and partials
  const int c = threadIdx.x % kLTx, r0 = (threadIdx.x / kLTx) * kLRun;
  float m[5][kLRun];
  {
    float2 v[kLRun + kLWin - 1], o[kLRun];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v[k] = h01[r0 + k][c];
    win4x2(win, v, o);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) {
      m[0][j] = o[j].x;
      m[1][j] = o[j].y;
    }
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v[k] = h23[r0 + k][c];
    win4x2(win, v, o);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) {
      m[2][j] = o[j].x;
      m[3][j] = o[j].y;
    }
    float u[kLRun + kLWin - 1];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) u[k] = h4[r0 + k][c];
    win4(win, u, m[4]);
  }
  float s_sum = 0.f, l1_sum = 0.f;
  const int gx = x0 + c;
#pragma unroll
  for (int j = 0; j < kLRun; ++j) {
    const int gy = y0 + r0 + j;
    if (gx >= W || gy >= H) continue;
    const float mx = m[0][j], my = m[1][j], exx = m[2][j], eyy = m[3][j], exy = m[4][j];
    const float sxx = exx - mx * mx, syy = eyy - my * my, sxy = exy - mx * my;
    const float a1 = 2.f * mx * my + kC1, a2 = 2.f * sxy + kC2;
    const float b1 = mx * mx + my * my + kC1, b2 = sxx + syy + kC2;
    // b1, b2 >= C1, C2 > 0: MUFU reciprocals (~1 ulp), far inside the loss tolerance
    const float ib1 = __frcp_rn(b1), ib2 = __frcp_rn(b2);
    const float ib = ib1 * ib2;
    const float s = a1 * a2 * ib;
    const float d_e = -s * ib2;
    const float d_p = 2.f * a1 * ib;
    const float d_m = 2.f * my * a2 * ib - 2.f * mx * s * ib1 + 2.f * mx * s * ib2 - 2.f * my * a1 * ib;
    const size_t p = (size_t)gy * W + gx;
    part[(0 * 3 + ch) * plane + p] = d_m;
    part[(1 * 3 + ch) * plane + p] = d_e;
    part[(2 * 3 + ch) * plane + p] = d_p;
    s_sum += s;
    const float2 q = s_xy[r0 + j + kLR][c + kLR];
    l1_sum += fabsf(q.x - q.y);
  }
  // block sums -> this block's slot of the partial-sum array (no same-address atomics)
  __shared__ float s_red[2][kLThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
    l1_sum += __shfl_xor_sync(0xffffffffu, l1_sum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_red[0][threadIdx.x >> 5] = l1_sum;
    s_red[1][threadIdx.x >> 5] = s_sum;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    float t = 0.f;
    for (int k = 0; k < kLThreads / 32; ++k) t += s_red[threadIdx.x][k];
    const int b = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    acc[2 * b + threadIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kLThreads) k_ssim_bwd(const float* __restrict__ img, const uint8_t* __restrict__ tgt,
                                                        int W, int H, LossWin win, const float* __restrict__ part,
                                                        float lam, float scale, float* __restrict__ dl,
                                                        const float* __restrict__ acc, float* loss_sum) {
  // the partial maps dS/dm, dS/dE (paired) and dS/dP
  __shared__ float2 sg01[kLHy][kLHx + 1];
  __shared__ float sg2[kLHy][kLHx + 1];
  __shared__ float2 hg01[kLHy][kLTx + 1];
  __shared__ float hg2[kLHy][kLTx + 1];
  const int ch = blockIdx.z;
  const int x0 = blockIdx.x * kLTx, y0 = blockIdx.y * kLTy;
  const size_t plane = (size_t)W * H;
  const double n = 3.0 * (double)plane;
  if (blockIdx.x == 0 && blockIdx.y == 0 && ch == 0) {
    // the loss from k_ssim_fwd's per-block partial sums (in double, fixed order per lane)
    __shared__ double s_acc[2][kLThreads / 32];
    const int nb = gridDim.x * gridDim.y * gridDim.z;
    double l1 = 0.0, ss = 0.0;
    for (int b = threadIdx.x; b < nb; b += kLThreads) {
      l1 += (double)acc[2 * b];
      ss += (double)acc[2 * b + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if ((threadIdx.x & 31) == 0) {
      s_acc[0][threadIdx.x >> 5] = l1;
      s_acc[1][threadIdx.x >> 5] = ss;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      l1 = ss = 0.0;
      for (int k = 0; k < kLThreads / 32; ++k) {
        l1 += s_acc[0][k];
        ss += s_acc[1][k];
      }
      atomicAdd(loss_sum, (float)(scale * ((1.0 - lam) * l1 / n + lam * (1.0 - ss / n))));
    }
  }
  // this thread's output pixels' image and target values, loaded now (used after the passes)
  const int oc = threadIdx.x % kLTx, or0 = (threadIdx.x / kLTx) * kLRun;
  float pxv[kLRun], pyv[kLRun];
#pragma unroll
  for (int j = 0; j < kLRun; ++j) {
    const int gx = x0 + oc, gy = y0 + or0 + j;
    const bool in = gx < W && gy < H;
    const size_t p = (size_t)gy * W + gx;
    pxv[j] = in ? __ldg(img + ch * plane + p) : 0.f;
    pyv[j] = in ? (float)__ldg(tgt + ch * plane + p) * (1.0f / 255.0f) : 0.f;
  }
  {
    float a0[kLStage], a1[kLStage], a2[kLStage];  // all loads in flight before the stores
#pragma unroll
    for (int q = 0; q < kLStage; ++q) {
      const int i = threadIdx.x + q * kLThreads;
      const int r = i / kLHx, c = i - r * kLHx;
      const int gx = x0 + c - kLR, gy = y0 + r - kLR;
      const bool in = i < kLHy * kLHx && gx >= 0 && gx < W && gy >= 0 && gy < H;
      const size_t p = (size_t)gy * W + gx;
      a0[q] = in ? __ldg(part + (0 * 3 + ch) * plane + p) : 0.f;
      a1[q] = in ? __ldg(part + (1 * 3 + ch) * plane + p) : 0.f;
      a2[q] = in ? __ldg(part + (2 * 3 + ch) * plane + p) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kLStage; ++q) {
      const int i = threadIdx.x + q * kLThreads;
      if (i < kLHy * kLHx) {
        sg01[i / kLHx][i % kLHx] = make_float2(a0[q], a1[q]);
        sg2[i / kLHx][i % kLHx] = a2[q];
      }
    }
  }
  __syncthreads();
  for (int it = threadIdx.x; it < kLRowItems; it += kLThreads) {
    const int r = it / kLSegs, c0 = (it - r * kLSegs) * kLRun;
    float2 v2[kLRun + kLWin - 1], o2[kLRun];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v2[k] = sg01[r][c0 + k];
    win4x2(win, v2, o2);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) hg01[r][c0 + j] = o2[j];
    float v[kLRun + kLWin - 1], o[kLRun];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v[k] = sg2[r][c0 + k];
    win4(win, v, o);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) hg2[r][c0 + j] = o[j];
  }
  __syncthreads();
  const int c = threadIdx.x % kLTx, r0 = (threadIdx.x / kLTx) * kLRun;
  float m[3][kLRun];
  {
    float2 v2[kLRun + kLWin - 1], o2[kLRun];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v2[k] = hg01[r0 + k][c];
    win4x2(win, v2, o2);
#pragma unroll
    for (int j = 0; j < kLRun; ++j) {
      m[0][j] = o2[j].x;
      m[1][j] = o2[j].y;
    }
    float v[kLRun + kLWin - 1];
#pragma unroll
    for (int k = 0; k < kLRun + kLWin - 1; ++k) v[k] = hg2[r0 + k][c];
    win4(win, v, m[2]);
  }
  const float inv_n = (float)(1.0 / n);
  const int gx = x0 + c;
#pragma unroll
  for (int j = 0; j < kLRun; ++j) {
    const int gy = y0 + r0 + j;
    if (gx >= W || gy >= H) continue;
    const size_t p = (size_t)gy * W + gx;
    const float xv = pxv[j], yv = pyv[j];
    const float d = xv - yv;
    const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    const float dssim = m[0][j] + 2.f * xv * m[1][j] + yv * m[2][j];
    dl[ch * plane + p] = scale * inv_n * ((1.0f - lam) * sgn - lam * dssim);
  }
}

static LossWin make_window() {
  // R29: g_k ~ exp(-(k - 5)^2 / (2 * 1.5^2)), normalised, in double, rounded once
  LossWin lw;
  double g[kLWin], sum = 0.0;
  for (int k = 0; k < kLWin; ++k) {
    const double d = (double)(k - kLR);
    g[k] = exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += g[k];
  }
  for (int k = 0; k < kLWin; ++k) lw.w[k] = (float)(g[k] / sum);
  return lw;
}

static size_t loss_blocks(int32_t w, int32_t h) {
  return (size_t)((w + kLTx - 1) / kLTx) * (size_t)((h + kLTy - 1) / kLTy) * 3;
}

// [per-block partial sums: 2 floats per k_ssim_fwd block, 256-B padded][9 partial maps]
static size_t loss_acc_bytes(int32_t w, int32_t h) { return (2 * sizeof(float) * loss_blocks(w, h) + 255) & ~(size_t)255; }

size_t loss_workspace_bytes(int32_t w, int32_t h) {
  return loss_acc_bytes(w, h) + (size_t)9 * (size_t)w * (size_t)h * sizeof(float);
}

bgs_status launch_l1_dssim(const float* image, const uint8_t* target, int32_t w, int32_t h, float lam, float scale,
                           float* dl, float* loss_sum, void* workspace, cudaStream_t s) {
  static const LossWin win = make_window();
  float* acc = reinterpret_cast<float*>(workspace);
  float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) + loss_acc_bytes(w, h));
  const dim3 grid((w + kLTx - 1) / kLTx, (h + kLTy - 1) / kLTy, 3);
  k_ssim_fwd<<<grid, kLThreads, 0, s>>>(image, target, w, h, win, part, acc);
  note_launch();
  bgs_status st = check_launch("k_ssim_fwd");
  if (st != BGS_OK) return st;
  k_ssim_bwd<<<grid, kLThreads, 0, s>>>(image, target, w, h, win, part, lam, scale, dl, acc, loss_sum);
  note_launch();
  return check_launch("k_ssim_bwd");
}

}  // namespace bgs
