// render_bwd.cu -- a9 blend backward (K12) and a10 preprocess backward (K13).
//
// The paper has no backward; it inherits 3DGS training.  Reading
// R18: the gradient of the forward O1-O14 with every discrete decision frozen (cull,
// rect, power/alpha skips, early stop, the 0.99 alpha clamp -> zero gradient to o and G,
// the SH clamp, the J-clamp branch).
//
// K12: one CTA per tile, one thread per pixel, walking the tile list back to front
// from the tile's largest n_contrib; T is recovered as T_i = T_{i+1} / (1 - alpha_i)
// and the colour "behind" accumulates S += c alpha T (S starts at T_final bg).  Per
// list entry each pixel produces 9 partials {dxy(2), dconic(3), dopacity, drgb(3)};
// they are summed across the warp with shuffles (skipped when no lane contributes)
// and lane 0 issues three 16-byte vector REDs into grad2d[id] -- instead of 3DGS's nine
// scalar atomics per pixel.
//
// K13: one thread per visible Gaussian: conic -> (a, b, c) of Sigma' -> Sigma and T = J W
// -> (s, q) and t -> mu; xy -> mu through the projection; rgb -> SH coefficients and the
// view direction -> mu; opacity -> logit.  grad[59n] += (views are summed, R20).
// grad2d was zeroed for the visible Gaussians by this view's preprocess.
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
                                                            const float* __restrict__ dl_dimage,
                                                            const float* __restrict__ final_T,
                                                            const uint32_t* __restrict__ n_contrib,
                                                            float4* __restrict__ grad2d) {
  __shared__ float4 s_r0[kBatchB], s_r1[kBatchB];
  __shared__ float s_b[kBatchB];
  __shared__ uint32_t s_id[kBatchB];
  __shared__ uint32_t s_max;
  const int tile = blockIdx.x;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
  const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
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
  if ((threadIdx.x & 31) == 0 && wmax) atomicMax(&s_max, wmax);
  __syncthreads();
  const int tile_last = (int)min(s_max, rg.y - rg.x);
  const int lane = threadIdx.x & 31;
  for (int end = tile_last; end > 0; end -= kBatchB) {
    const int begin = max(0, end - kBatchB);
    const int cnt = end - begin;
    __syncthreads();
    if ((int)threadIdx.x < cnt) {
      const uint32_t id = values[rg.x + begin + threadIdx.x];
      s_id[threadIdx.x] = id;
      s_r0[threadIdx.x] = __ldg(record + 3 * id);
      s_r1[threadIdx.x] = __ldg(record + 3 * id + 1);
      s_b[threadIdx.x] = __ldg(record + 3 * id + 2).x;
    }
    __syncthreads();
    for (int k = cnt - 1; k >= 0; --k) {
      const uint32_t pos = (uint32_t)(begin + k);
      bool act = pos < my_last;
      float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f, g5 = 0.f, g6 = 0.f, g7 = 0.f, g8 = 0.f;
      if (act) {
        const float4 r0 = s_r0[k];
        const float4 r1 = s_r1[k];
        const float dx = r0.x - pxf, dy = r0.y - pyf;
        const float power = fmaf(r0.z, dx * dx, fmaf(r1.x, dy * dy, r0.w * (dx * dy)));
        const float G = fast_exp(power);
        const float og = r1.y * G;
        const float alpha = fminf(0.99f, og);
        if (power > 0.0f || alpha < (1.0f / 255.0f)) {
          act = false;
        } else {
          const float oma = 1.0f - alpha;
          const float ioma = 1.0f / oma;
          T = T * ioma;  // transmittance in front of this Gaussian
          const float w = alpha * T;
          const float cr = r1.z, cg = r1.w, cb = s_b[k];
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
          float4* dst = grad2d + 3 * s_id[k];
          red_add_v4(dst, make_float4(g0, g1, g2, g3));
          red_add_v4(dst + 1, make_float4(g4, g5, g6, g7));
          atomicAdd(&dst[2].x, g8);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K13
__constant__ float bC0 = 0.28209479177387814f;
__constant__ float bC1 = 0.4886025119029199f;
__constant__ float bC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                             -1.0925484305920792f, 0.5462742152960396f};
__constant__ float bC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                             0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                             -0.5900435899266435f};

struct PreBwdParams {
  Cam cam;
  const float* means;
  const float* log_scales;
  const float4* quats;
  const float* ologits;
  const float* sh;
  int64_t n;
  int32_t deg;
  const int32_t* radius;
  const float4* record;
  const float4* grad2d;
  float* grad;  // theta layout
};

__global__ void __launch_bounds__(128) k_preprocess_bwd(PreBwdParams p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n || p.radius[i] <= 0) return;
  const int64_t n = p.n;
  const Cam& c = p.cam;
  const float4* g2 = p.grad2d + 3 * i;
  const float4 ga4 = g2[0], gb4 = g2[1], gc4 = g2[2];
  const float gx = ga4.x, gy = ga4.y, gcx = ga4.z, gcy = ga4.w, gcz = gb4.x, gop = gb4.y;
  const uint32_t cb = __float_as_uint(p.record[3 * i + 2].y);
  const float grc[3] = {(cb & CB_R) ? 0.f : gb4.z, (cb & CB_G) ? 0.f : gb4.w, (cb & CB_B) ? 0.f : gc4.x};
  const float mx = p.means[3 * i], my = p.means[3 * i + 1], mz = p.means[3 * i + 2];
  const float* V = c.V;
  const float* P = c.P;
  const float t0 = V[0] * mx + V[4] * my + V[8] * mz + V[12];
  const float t1 = V[1] * mx + V[5] * my + V[9] * mz + V[13];
  const float t2 = V[2] * mx + V[6] * my + V[10] * mz + V[14];
  float dmx = 0.f, dmy = 0.f, dmz = 0.f;
  // ---- colour: SH coefficients and view direction
  {
    const float dxw = mx - c.campos[0], dyw = my - c.campos[1], dzw = mz - c.campos[2];
    const float il = rsqrtf(dxw * dxw + dyw * dyw + dzw * dzw);
    const float x = dxw * il, y = dyw * il, z = dzw * il;
    const float* sh = p.sh + 48 * i;
    float* gsh = p.grad + 11 * n + 48 * i;
    float Y[16], dY[16][3];
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[0] = bC0;
    dY[0][0] = dY[0][1] = dY[0][2] = 0.f;
    int nc = 1;
    if (p.deg > 0) {
      nc = 4;
      Y[1] = -bC1 * y; dY[1][0] = 0.f; dY[1][1] = -bC1; dY[1][2] = 0.f;
      Y[2] = bC1 * z;  dY[2][0] = 0.f; dY[2][1] = 0.f;  dY[2][2] = bC1;
      Y[3] = -bC1 * x; dY[3][0] = -bC1; dY[3][1] = 0.f; dY[3][2] = 0.f;
      if (p.deg > 1) {
        nc = 9;
        Y[4] = bC2[0] * x * y; dY[4][0] = bC2[0] * y; dY[4][1] = bC2[0] * x; dY[4][2] = 0.f;
        Y[5] = bC2[1] * y * z; dY[5][0] = 0.f; dY[5][1] = bC2[1] * z; dY[5][2] = bC2[1] * y;
        Y[6] = bC2[2] * (2.f * zz - xx - yy);
        dY[6][0] = -2.f * bC2[2] * x; dY[6][1] = -2.f * bC2[2] * y; dY[6][2] = 4.f * bC2[2] * z;
        Y[7] = bC2[3] * x * z; dY[7][0] = bC2[3] * z; dY[7][1] = 0.f; dY[7][2] = bC2[3] * x;
        Y[8] = bC2[4] * (xx - yy); dY[8][0] = 2.f * bC2[4] * x; dY[8][1] = -2.f * bC2[4] * y; dY[8][2] = 0.f;
        if (p.deg > 2) {
          nc = 16;
          Y[9] = bC3[0] * y * (3.f * xx - yy);
          dY[9][0] = 6.f * bC3[0] * x * y; dY[9][1] = bC3[0] * 3.f * (xx - yy); dY[9][2] = 0.f;
          Y[10] = bC3[1] * x * y * z;
          dY[10][0] = bC3[1] * y * z; dY[10][1] = bC3[1] * x * z; dY[10][2] = bC3[1] * x * y;
          Y[11] = bC3[2] * y * (4.f * zz - xx - yy);
          dY[11][0] = -2.f * bC3[2] * x * y; dY[11][1] = bC3[2] * (4.f * zz - xx - 3.f * yy);
          dY[11][2] = 8.f * bC3[2] * y * z;
          Y[12] = bC3[3] * z * (2.f * zz - 3.f * xx - 3.f * yy);
          dY[12][0] = -6.f * bC3[3] * x * z; dY[12][1] = -6.f * bC3[3] * y * z;
          dY[12][2] = bC3[3] * (6.f * zz - 3.f * xx - 3.f * yy);
          Y[13] = bC3[4] * x * (4.f * zz - xx - yy);
          dY[13][0] = bC3[4] * (4.f * zz - 3.f * xx - yy); dY[13][1] = -2.f * bC3[4] * x * y;
          dY[13][2] = 8.f * bC3[4] * x * z;
          Y[14] = bC3[5] * z * (xx - yy);
          dY[14][0] = 2.f * bC3[5] * x * z; dY[14][1] = -2.f * bC3[5] * y * z; dY[14][2] = bC3[5] * (xx - yy);
          Y[15] = bC3[6] * x * (xx - 3.f * yy);
          dY[15][0] = bC3[6] * 3.f * (xx - yy); dY[15][1] = -6.f * bC3[6] * x * y; dY[15][2] = 0.f;
        }
      }
    }
    float ddx = 0.f, ddy = 0.f, ddz = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < nc) {
        const float s0 = sh[3 * k], s1 = sh[3 * k + 1], s2 = sh[3 * k + 2];
        gsh[3 * k] += Y[k] * grc[0];
        gsh[3 * k + 1] += Y[k] * grc[1];
        gsh[3 * k + 2] += Y[k] * grc[2];
        const float shg = s0 * grc[0] + s1 * grc[1] + s2 * grc[2];
        ddx += dY[k][0] * shg;
        ddy += dY[k][1] * shg;
        ddz += dY[k][2] * shg;
      }
    }
    const float dot = ddx * x + ddy * y + ddz * z;
    dmx += (ddx - x * dot) * il;
    dmy += (ddy - y * dot) * il;
    dmz += (ddz - z * dot) * il;
  }
  // ---- opacity
  {
    const float o = 1.0f / (1.0f + expf(-p.ologits[i]));
    p.grad[10 * n + i] += gop * o * (1.0f - o);
  }
  // ---- covariance chain
  const float s[3] = {expf(p.log_scales[3 * i]), expf(p.log_scales[3 * i + 1]), expf(p.log_scales[3 * i + 2])};
  const float4 qh = p.quats[i];
  const float qn = sqrtf(qh.x * qh.x + qh.y * qh.y + qh.z * qh.z + qh.w * qh.w);
  const float iq = 1.0f / qn;
  const float w = qh.x * iq, x = qh.y * iq, y = qh.z * iq, z = qh.w * iq;
  float R[3][3];
  R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
  R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
  R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
  float M[3][3], Sg[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) M[a][k] = R[a][k] * s[k];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) {
      Sg[a][b] = M[a][0] * M[b][0] + M[a][1] * M[b][1] + M[a][2] * M[b][2];
      Sg[b][a] = Sg[a][b];
    }
  float u = t0 / t2, v = t1 / t2;
  if (cb & CB_JX) u = (cb & CB_JX_NEG) ? -c.limx : c.limx;
  if (cb & CB_JY) v = (cb & CB_JY_NEG) ? -c.limy : c.limy;
  const float itz = 1.0f / t2, itz2 = itz * itz;
  const float j00 = c.fx * itz, j02 = -c.fx * u * itz, j11 = c.fy * itz, j12 = -c.fy * v * itz;
  float Tm[2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    Tm[0][k] = j00 * V[0 + 4 * k] + j02 * V[2 + 4 * k];
    Tm[1][k] = j11 * V[1 + 4 * k] + j12 * V[2 + 4 * k];
  }
  float TS[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) TS[a][k] = Tm[a][0] * Sg[0][k] + Tm[a][1] * Sg[1][k] + Tm[a][2] * Sg[2][k];
  const float A = TS[0][0] * Tm[0][0] + TS[0][1] * Tm[0][1] + TS[0][2] * Tm[0][2] + 0.3f;
  const float B = TS[0][0] * Tm[1][0] + TS[0][1] * Tm[1][1] + TS[0][2] * Tm[1][2];
  const float Cc = TS[1][0] * Tm[1][0] + TS[1][1] * Tm[1][1] + TS[1][2] * Tm[1][2] + 0.3f;
  const float det = A * Cc - B * B;
  const float id2 = 1.0f / (det * det);
  const float gA = (-Cc * Cc * gcx + B * Cc * gcy - B * B * gcz) * id2;
  const float gB = (2.f * B * Cc * gcx - (A * Cc + B * B) * gcy + 2.f * A * B * gcz) * id2;
  const float gC = (-B * B * gcx + A * B * gcy - A * A * gcz) * id2;
  const float Gp[2][2] = {{gA, 0.5f * gB}, {0.5f * gB, gC}};
  // dL/dSigma = T^T G' T ; dL/dT = 2 G' (T Sigma)
  float GS[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q)
      GS[r][q] = Tm[0][r] * (Gp[0][0] * Tm[0][q] + Gp[0][1] * Tm[1][q]) +
                 Tm[1][r] * (Gp[1][0] * Tm[0][q] + Gp[1][1] * Tm[1][q]);
  float gT[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) gT[a][k] = 2.f * (Gp[a][0] * TS[0][k] + Gp[a][1] * TS[1][k]);
  float gj00 = 0.f, gj02 = 0.f, gj11 = 0.f, gj12 = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gj00 += gT[0][k] * V[0 + 4 * k];
    gj02 += gT[0][k] * V[2 + 4 * k];
    gj11 += gT[1][k] * V[1 + 4 * k];
    gj12 += gT[1][k] * V[2 + 4 * k];
  }
  float gt0 = 0.f, gt1 = 0.f, gt2 = -(gj00 * c.fx + gj11 * c.fy) * itz2;
  if (cb & CB_JX) {
    gt2 += gj02 * c.fx * u * itz2;
  } else {
    gt0 += -gj02 * c.fx * itz2;
    gt2 += gj02 * 2.f * c.fx * t0 * itz2 * itz;
  }
  if (cb & CB_JY) {
    gt2 += gj12 * c.fy * v * itz2;
  } else {
    gt1 += -gj12 * c.fy * itz2;
    gt2 += gj12 * 2.f * c.fy * t1 * itz2 * itz;
  }
  dmx += V[0] * gt0 + V[1] * gt1 + V[2] * gt2;
  dmy += V[4] * gt0 + V[5] * gt1 + V[6] * gt2;
  dmz += V[8] * gt0 + V[9] * gt1 + V[10] * gt2;
  // ---- projected mean (O3)
  {
    const float c0 = P[0] * mx + P[4] * my + P[8] * mz + P[12];
    const float c1 = P[1] * mx + P[5] * my + P[9] * mz + P[13];
    const float c3 = P[3] * mx + P[7] * my + P[11] * mz + P[15];
    const float ic3 = 1.0f / c3, ic32 = ic3 * ic3;
    const float hx = 0.5f * (float)c.W * gx * ic32, hy = 0.5f * (float)c.H * gy * ic32;
    dmx += hx * (P[0] * c3 - P[3] * c0) + hy * (P[1] * c3 - P[3] * c1);
    dmy += hx * (P[4] * c3 - P[7] * c0) + hy * (P[5] * c3 - P[7] * c1);
    dmz += hx * (P[8] * c3 - P[11] * c0) + hy * (P[9] * c3 - P[11] * c1);
  }
  float* gm = p.grad + 3 * i;
  gm[0] += dmx;
  gm[1] += dmy;
  gm[2] += dmz;
  // ---- Sigma = M M^T, M = R diag(s)
  float gR[3][3];
  float* gls = p.grad + 3 * n + 3 * i;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float gsk = 0.f;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const float gM = 2.f * (GS[r][0] * M[0][k] + GS[r][1] * M[1][k] + GS[r][2] * M[2][k]);
      gsk += gM * R[r][k];
      gR[r][k] = gM * s[k];
    }
    gls[k] += gsk * s[k];
  }
  float gw = 2.f * (-z * gR[0][1] + y * gR[0][2] + z * gR[1][0] - x * gR[1][2] - y * gR[2][0] + x * gR[2][1]);
  float gx_ = 2.f * (y * gR[0][1] + z * gR[0][2] + y * gR[1][0] - 2.f * x * gR[1][1] - w * gR[1][2] +
                     z * gR[2][0] + w * gR[2][1] - 2.f * x * gR[2][2]);
  float gy_ = 2.f * (-2.f * y * gR[0][0] + x * gR[0][1] + w * gR[0][2] + x * gR[1][0] + z * gR[1][2] -
                     w * gR[2][0] + z * gR[2][1] - 2.f * y * gR[2][2]);
  float gz_ = 2.f * (-2.f * z * gR[0][0] - w * gR[0][1] + x * gR[0][2] + w * gR[1][0] - 2.f * z * gR[1][1] +
                     y * gR[1][2] + x * gR[2][0] + y * gR[2][1]);
  const float qd = gw * w + gx_ * x + gy_ * y + gz_ * z;
  float* gq = p.grad + 6 * n + 4 * i;
  gq[0] += (gw - w * qd) * iq;
  gq[1] += (gx_ - x * qd) * iq;
  gq[2] += (gy_ - y * qd) * iq;
  gq[3] += (gz_ - z * qd) * iq;
}

bgs_status launch_blend_bwd(Frame* F, const float* dL_dimage, const float* final_T, const uint32_t* n_contrib,
                            cudaStream_t s) {
  k_render_bwd<<<F->num_tiles, kTilePixels, 0, s>>>(F->ranges, F->vals[F->final_buf], F->record, F->counters, F->cam,
                                                    dL_dimage, final_T, n_contrib, F->grad2d);
  note_launch();
  return check_launch("k_render_bwd");
}

bgs_status launch_preprocess_bwd(const bgs_gaussians* g, Frame* F, float* grad, cudaStream_t s) {
  if (F->n == 0) return BGS_OK;
  PreBwdParams p;
  p.cam = F->cam;
  p.means = g->means;
  p.log_scales = g->log_scales;
  p.quats = (const float4*)g->quats;
  p.ologits = g->opacity_logits;
  p.sh = g->sh;
  p.n = F->n;
  p.deg = g->sh_degree;
  p.radius = F->radius;
  p.record = F->record;
  p.grad2d = F->grad2d;
  p.grad = grad;
  k_preprocess_bwd<<<(unsigned)((F->n + 127) / 128), 128, 0, s>>>(p);
  note_launch();
  return check_launch("k_preprocess_bwd");
}

bgs_status launch_render_bwd(const bgs_gaussians* g, Frame* F, const float* dL_dimage, const float* final_T,
                             const uint32_t* n_contrib, float* grad, cudaStream_t s) {
  bgs_status st = launch_blend_bwd(F, dL_dimage, final_T, n_contrib, s);
  return st != BGS_OK ? st : launch_preprocess_bwd(g, F, grad, s);
}

}  // namespace bgs
