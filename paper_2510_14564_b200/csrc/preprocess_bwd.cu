// preprocess_bwd.cu -- a10 (K13): the chain rule from the per-view blend gradients to theta.
//
// The paper has no backward (it inherits 3DGS training); reading R18: the
// derivative of O1-O9 with the forward's decisions frozen (J-clamp branch and rgb clamp,
// both taken from the cbits the preprocess stored in the render record).  Per visible
// Gaussian: conic -> (a, b, c) of Sigma' -> Sigma and T = J W -> (s, q) and t -> mu;
// xy -> mu through the projection; rgb -> SH coefficients and the view direction -> mu;
// opacity -> logit.  grad[59n] += (views are summed, R20).
//
// Numerics: Sigma, Sigma' = T Sigma T^T, det = ac - b^2 and dL/d(a,b,c) are evaluated in
// FP64 -- det cancels badly for edge-on footprints (ac ~ b^2), and in FP32 that cost
// ~1e-3 relative on the log_scales gradient; everything downstream of dL/dSigma' and the
// SH part are FP32 (B200 runs FP64 at half the FP32 rate; this kernel is HBM-bound).
//
// Batching (bgs_preprocess_bwd_batch): the theta-side work and the grad read-modify-write
// are per Gaussian, the camera-side work per (Gaussian, view); one launch serves up to 16
// views, so theta and grad cross HBM once per batch instead of once per view.
//
// Memory: one thread per Gaussian, 2 warps per CTA.  The 192-byte SH block and the
// 192-byte SH-gradient block of a warp's 32 Gaussians are contiguous (6 KB each), so the
// warp reads the SH coefficients and read-modify-writes the SH gradients as coalesced
// float4 passes staged through shared memory (two padded 49-float rows per Gaussian: the
// coefficients, and dL/dsh summed over the views); the per-thread parts (means, scales,
// quats, opacity) are naturally coalesced.
#include "common.cuh"

namespace bgs {

struct PreBwdView {
  Cam cam;
  const int32_t* radius;
  const uint8_t* cbits;
  const float4* grad2d;
  float4* grad2d_zero;  // non-null: zero each slot after reading it (the frame's grad2d is then clean)
};

struct PreBwdParams {
  const float* means;
  const float* log_scales;
  const float* quats;
  const float* ologits;
  const float* sh;  // [n][16][3]
  int64_t n;
  int64_t i0, i1;  // the Gaussians [i0, i1) this launch processes
  int32_t deg, nviews;
  bool quat_vec4, sh_vec4, gq_vec4, gsh_vec4;  // 16-byte aligned -> vector paths
  float* grad;  // theta layout (fused Adam: the partial sums of earlier launches, or null)
  // fused Adam (R21; bgs_preprocess_bwd_batch_adam): theta += Adam(sum of the gradient)
  bool adam;
  bool assign;  // grad = (not +=) this launch's sum; unseen Gaussians get 0
  float* theta;  // writable theta (the buffer the pointers above view)
  float* m;
  float* v;
  float step_size[6], b1, b2, eps, inv_sqrt_bc2;
  PreBwdView view[kPreBwdMaxViews];
};

// One gradient element e of theta's layout: grad[e] += g, or (fused) the Adam update of
// theta[e] with g plus the partial sum of earlier launches (R21, adam.cu's arithmetic).
__device__ __forceinline__ void put_grad(const PreBwdParams& p, int64_t e, float g, int grp) {
  if (!p.adam) {
    if (p.assign) p.grad[e] = g;
    else p.grad[e] += g;
    return;
  }
  if (p.grad) {
    g += p.grad[e];
    p.grad[e] = 0.0f;
  }
  // explicit roundings (this file is built with FMA contraction; adam.cu is not): the fused
  // update stays bit-identical to bgs_adam_step's
  float m = p.m[e], v = p.v[e];
  m = fmaf(p.b1, m, __fmul_rn(1.0f - p.b1, g));
  v = fmaf(p.b2, v, __fmul_rn(__fmul_rn(1.0f - p.b2, g), g));
  const float denom = __fadd_rn(__fmul_rn(sqrtf(v), p.inv_sqrt_bc2), p.eps);
  p.theta[e] = __fsub_rn(p.theta[e], __fmul_rn(p.step_size[grp], m / denom));
  p.m[e] = m;
  p.v[e] = v;
}

constexpr int kBwdThreads = 64;
constexpr int kRow = 52;  // padded row stride (floats) of the staged SH block: 16-byte rows,
                          // conflict-free for 16-byte accesses (8 lanes of a phase: 20 l mod 32)

// Real SH constants (R12).
constexpr float kC0 = 0.28209479177387814f, kC1 = 0.4886025119029199f;
constexpr float kC20 = 1.0925484305920792f, kC21 = -1.0925484305920792f, kC22 = 0.31539156525252005f,
                kC23 = -1.0925484305920792f, kC24 = 0.5462742152960396f;
constexpr float kC30 = -0.5900435899266435f, kC31 = 2.890611442640554f, kC32 = -0.4570457994644658f,
                kC33 = 0.3731763325901154f, kC34 = -0.4570457994644658f, kC35 = 1.445305721320277f,
                kC36 = -0.5900435899266435f;

// One thread per Gaussian, looping over the batch's views (one launch per <= 16 views).
// The view-independent parts -- Sigma = M M^T (FP64), the quaternion/scale chain, the
// sigmoid, the theta loads and the grad read-modify-write -- are done once per Gaussian;
// per view only the camera-dependent terms are evaluated, and dL/dSigma, dL/dmu,
// dL/dopacity and dL/dsh are summed in registers / shared memory across the views.
__global__ void __launch_bounds__(kBwdThreads, 8) k_preprocess_bwd(const __grid_constant__ PreBwdParams p) {
  __shared__ __align__(16) float s_sh[kBwdThreads / 32][32 * kRow];   // SH coefficients (read-only)
  __shared__ __align__(16) float s_dsh[kBwdThreads / 32][32 * kRow];  // dL/dsh, summed over the views
  __shared__ int s_vis[kBwdThreads / 32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = p.n;
  const int64_t wbase = p.i0 + ((int64_t)blockIdx.x * kBwdThreads) + warp * 32;
  const int64_t i = wbase + lane;
  uint32_t vmask = 0;  // views in which Gaussian i is visible
  if (i < p.i1)
    for (int v = 0; v < p.nviews; ++v) vmask |= (p.view[v].radius[i] > 0 ? 1u : 0u) << v;
  const bool valid = vmask != 0;
  s_vis[warp][lane] = valid;
  float* row = &s_sh[warp][lane * kRow];
  float* drow = &s_dsh[warp][lane * kRow];
  const int ncoef = (p.deg + 1) * (p.deg + 1);
  const int64_t nvalid = p.i1 - wbase < 32 ? p.i1 - wbase : 32;
  for (int k = 0; k < 12; ++k) reinterpret_cast<float4*>(drow)[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
  // ---- coalesced load of the warp's SH block into shared memory
  if (p.sh_vec4) {
    const float4* src = reinterpret_cast<const float4*>(p.sh) + 12 * wbase;
    for (int c = lane; c < 12 * nvalid; c += 32) {
      const int g = c / 12, e = 4 * (c % 12);
      if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
      const float4 v = __ldg(src + c);
      *reinterpret_cast<float4*>(&s_sh[warp][g * kRow + e]) = v;
    }
  } else {
    const float* src = p.sh + 48 * wbase;
    for (int c = lane; c < 48 * nvalid; c += 32) {
      const int g = c / 48, e = c % 48;
      if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
      s_sh[warp][g * kRow + e] = __ldg(src + c);
    }
  }
  __syncwarp();
  if (valid) {
    const float mx = p.means[3 * i], my = p.means[3 * i + 1], mz = p.means[3 * i + 2];
    const float s[3] = {expf(p.log_scales[3 * i]), expf(p.log_scales[3 * i + 1]), expf(p.log_scales[3 * i + 2])};
    const float4 qh = p.quat_vec4 ? __ldg(reinterpret_cast<const float4*>(p.quats) + i)
                                  : make_float4(p.quats[4 * i], p.quats[4 * i + 1], p.quats[4 * i + 2],
                                                p.quats[4 * i + 3]);
    const float qn = sqrtf(qh.x * qh.x + qh.y * qh.y + qh.z * qh.z + qh.w * qh.w);
    const float iq = 1.0f / qn;
    const float w = qh.x * iq, x = qh.y * iq, y = qh.z * iq, z = qh.w * iq;
    float R[3][3];
    R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
    R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
    R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
    float M[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k) M[a][k] = R[a][k] * s[k];
    // Sigma (FP64; symmetric, 6 entries)
    double S00, S01, S02, S11, S12, S22;
    {
      auto sg = [&](int a, int b) {
        return (double)M[a][0] * M[b][0] + (double)M[a][1] * M[b][1] + (double)M[a][2] * M[b][2];
      };
      S00 = sg(0, 0); S01 = sg(0, 1); S02 = sg(0, 2); S11 = sg(1, 1); S12 = sg(1, 2); S22 = sg(2, 2);
    }
    float dmx = 0.f, dmy = 0.f, dmz = 0.f, gop = 0.f;
    float GS00 = 0.f, GS01 = 0.f, GS02 = 0.f, GS11 = 0.f, GS12 = 0.f, GS22 = 0.f;  // dL/dSigma (sym.)
    // the next view's blend gradients and clamp bits are loaded one view ahead (in flight
    // during this view's arithmetic)
    float4 na = make_float4(0.f, 0.f, 0.f, 0.f), nb = na, nc = na;
    uint32_t ncb = 0;
    auto fetch = [&](int v) {
      if (v < p.nviews && ((vmask >> v) & 1u)) {
        const PreBwdView& q = p.view[v];
        na = q.grad2d[3 * i];
        nb = q.grad2d[3 * i + 1];
        nc = q.grad2d[3 * i + 2];
        ncb = q.cbits[i];
      }
    };
    fetch(0);
    for (int vi = 0; vi < p.nviews; ++vi) {
      const float4 ga4 = na, gb4 = nb, gc4 = nc;
      const uint32_t cb = ncb;
      fetch(vi + 1);
      if (!((vmask >> vi) & 1u)) continue;
      const PreBwdView& pv = p.view[vi];
      const Cam& c = pv.cam;
      const float* V = c.V;
      const float* P = c.P;
      const float gx = ga4.x, gy = ga4.y;
      gop += gb4.y;
      const float g_r = (cb & CB_R) ? 0.f : gb4.z, g_g = (cb & CB_G) ? 0.f : gb4.w, g_b = (cb & CB_B) ? 0.f : gc4.x;
      // ---- colour: per SH term, dL/dd from the coefficients, dL/dsh_k += Y_k dL/drgb
      //      (masked by the frozen clamp, R12)
      {
        const float dxw = mx - c.campos[0], dyw = my - c.campos[1], dzw = mz - c.campos[2];
        const float il = rsqrtf(dxw * dxw + dyw * dyw + dzw * dzw);
        const float x = dxw * il, y = dyw * il, z = dzw * il;
        const float xx = x * x, yy = y * y, zz = z * z;
        float ddx = 0.f, ddy = 0.f, ddz = 0.f;
        // the coefficients in groups of four (12 floats = 3 16-byte chunks of the staged row
        // and of the gradient row): 36 shared-memory accesses per view instead of 144
        float rv[12], dv[12];
        auto load_group = [&](int j) {
          const float4* r4 = reinterpret_cast<const float4*>(row) + 3 * j;
          const float4* d4 = reinterpret_cast<const float4*>(drow) + 3 * j;
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 a = r4[q], b = d4[q];
            rv[4 * q] = a.x; rv[4 * q + 1] = a.y; rv[4 * q + 2] = a.z; rv[4 * q + 3] = a.w;
            dv[4 * q] = b.x; dv[4 * q + 1] = b.y; dv[4 * q + 2] = b.z; dv[4 * q + 3] = b.w;
          }
        };
        auto store_group = [&](int j) {
          float4* d4 = reinterpret_cast<float4*>(drow) + 3 * j;
#pragma unroll
          for (int q = 0; q < 3; ++q) d4[q] = make_float4(dv[4 * q], dv[4 * q + 1], dv[4 * q + 2], dv[4 * q + 3]);
        };
        auto term = [&](int k, float Y, float dYx, float dYy, float dYz) {
          const int e = 3 * (k & 3);
          const float shg = rv[e] * g_r + rv[e + 1] * g_g + rv[e + 2] * g_b;
          ddx = fmaf(dYx, shg, ddx);
          ddy = fmaf(dYy, shg, ddy);
          ddz = fmaf(dYz, shg, ddz);
          dv[e] = fmaf(Y, g_r, dv[e]);
          dv[e + 1] = fmaf(Y, g_g, dv[e + 1]);
          dv[e + 2] = fmaf(Y, g_b, dv[e + 2]);
        };
        load_group(0);
        term(0, kC0, 0.f, 0.f, 0.f);
        if (p.deg > 0) {
          term(1, -kC1 * y, 0.f, -kC1, 0.f);
          term(2, kC1 * z, 0.f, 0.f, kC1);
          term(3, -kC1 * x, -kC1, 0.f, 0.f);
        }
        store_group(0);
        if (p.deg > 1) {
          load_group(1);
          term(4, kC20 * x * y, kC20 * y, kC20 * x, 0.f);
          term(5, kC21 * y * z, 0.f, kC21 * z, kC21 * y);
          term(6, kC22 * (2.f * zz - xx - yy), -2.f * kC22 * x, -2.f * kC22 * y, 4.f * kC22 * z);
          term(7, kC23 * x * z, kC23 * z, 0.f, kC23 * x);
          store_group(1);
          load_group(2);
          term(8, kC24 * (xx - yy), 2.f * kC24 * x, -2.f * kC24 * y, 0.f);
          if (p.deg > 2) {
            term(9, kC30 * y * (3.f * xx - yy), 6.f * kC30 * x * y, 3.f * kC30 * (xx - yy), 0.f);
            term(10, kC31 * x * y * z, kC31 * y * z, kC31 * x * z, kC31 * x * y);
            term(11, kC32 * y * (4.f * zz - xx - yy), -2.f * kC32 * x * y, kC32 * (4.f * zz - xx - 3.f * yy),
                 8.f * kC32 * y * z);
          }
          store_group(2);
          if (p.deg > 2) {
            load_group(3);
            term(12, kC33 * z * (2.f * zz - 3.f * xx - 3.f * yy), -6.f * kC33 * x * z, -6.f * kC33 * y * z,
                 kC33 * (6.f * zz - 3.f * xx - 3.f * yy));
            term(13, kC34 * x * (4.f * zz - xx - yy), kC34 * (4.f * zz - 3.f * xx - yy), -2.f * kC34 * x * y,
                 8.f * kC34 * x * z);
            term(14, kC35 * z * (xx - yy), 2.f * kC35 * x * z, -2.f * kC35 * y * z, kC35 * (xx - yy));
            term(15, kC36 * x * (xx - 3.f * yy), 3.f * kC36 * (xx - yy), -6.f * kC36 * x * y, 0.f);
            store_group(3);
          }
        }
        const float dot = ddx * x + ddy * y + ddz * z;
        dmx += (ddx - x * dot) * il;
        dmy += (ddy - y * dot) * il;
        dmz += (ddz - z * dot) * il;
      }
      // ---- covariance chain: FP64 through Sigma', det and dL/d(a, b, c)
      const float t0 = V[0] * mx + V[4] * my + V[8] * mz + V[12];
      const float t1 = V[1] * mx + V[5] * my + V[9] * mz + V[13];
      const float t2 = V[2] * mx + V[6] * my + V[10] * mz + V[14];
      const float fx = c.fx, fy = c.fy;
      // MUFU reciprocals (~1 ulp): the decisions are the forward's (frozen), and the gradient
      // tolerance (1e-3 relative) is far above the rounding of an IEEE division
      const float itz = fast_rcp(t2), itz2 = itz * itz;
      float u = t0 * itz, v = t1 * itz;
      if (cb & CB_JX) u = (cb & CB_JX_NEG) ? -c.limx : c.limx;
      if (cb & CB_JY) v = (cb & CB_JY_NEG) ? -c.limy : c.limy;
      const float j00 = fx * itz, j02 = -fx * u * itz, j11 = fy * itz, j12 = -fy * v * itz;
      float Tm[2][3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        Tm[0][k] = j00 * V[0 + 4 * k] + j02 * V[2 + 4 * k];
        Tm[1][k] = j11 * V[1 + 4 * k] + j12 * V[2 + 4 * k];
      }
      float TS[2][3];
      double Gp00, Gp01, Gp11;
      {
        const double Sg[3][3] = {{S00, S01, S02}, {S01, S11, S12}, {S02, S12, S22}};
        double TSd[2][3];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            TSd[a][k] = (double)Tm[a][0] * Sg[0][k] + (double)Tm[a][1] * Sg[1][k] + (double)Tm[a][2] * Sg[2][k];
            TS[a][k] = (float)TSd[a][k];
          }
        const double A = TSd[0][0] * Tm[0][0] + TSd[0][1] * Tm[0][1] + TSd[0][2] * Tm[0][2] + 0.3;
        const double B = TSd[0][0] * Tm[1][0] + TSd[0][1] * Tm[1][1] + TSd[0][2] * Tm[1][2];
        const double Cc = TSd[1][0] * Tm[1][0] + TSd[1][1] * Tm[1][1] + TSd[1][2] * Tm[1][2] + 0.3;
        const double det = A * Cc - B * B;
        const float idet = fast_rcp((float)det);  // det itself stays FP64 (it cancels)
        const double id2 = (double)idet * (double)idet;
        const double gcx = ga4.z, gcy = ga4.w, gcz = gb4.x;
        Gp00 = (-Cc * Cc * gcx + B * Cc * gcy - B * B * gcz) * id2;
        Gp01 = 0.5 * (2.0 * B * Cc * gcx - (A * Cc + B * B) * gcy + 2.0 * A * B * gcz) * id2;
        Gp11 = (-B * B * gcx + A * B * gcy - A * A * gcz) * id2;
      }
      const float G00 = (float)Gp00, G01 = (float)Gp01, G11 = (float)Gp11;
      // dL/dSigma += T^T G' T ; dL/dT = 2 G' (T Sigma)
      auto gs = [&](int r, int q) {
        return Tm[0][r] * (G00 * Tm[0][q] + G01 * Tm[1][q]) + Tm[1][r] * (G01 * Tm[0][q] + G11 * Tm[1][q]);
      };
      GS00 += gs(0, 0); GS01 += gs(0, 1); GS02 += gs(0, 2); GS11 += gs(1, 1); GS12 += gs(1, 2); GS22 += gs(2, 2);
      float gj00 = 0.f, gj02 = 0.f, gj11 = 0.f, gj12 = 0.f;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float gT0 = 2.f * (G00 * TS[0][k] + G01 * TS[1][k]);
        const float gT1 = 2.f * (G01 * TS[0][k] + G11 * TS[1][k]);
        gj00 += gT0 * V[0 + 4 * k];
        gj02 += gT0 * V[2 + 4 * k];
        gj11 += gT1 * V[1 + 4 * k];
        gj12 += gT1 * V[2 + 4 * k];
      }
      float gt0 = 0.f, gt1 = 0.f, gt2 = -(gj00 * fx + gj11 * fy) * itz2;
      if (cb & CB_JX) {
        gt2 += gj02 * fx * u * itz2;
      } else {
        gt0 += -gj02 * fx * itz2;
        gt2 += gj02 * 2.f * fx * t0 * itz2 * itz;
      }
      if (cb & CB_JY) {
        gt2 += gj12 * fy * v * itz2;
      } else {
        gt1 += -gj12 * fy * itz2;
        gt2 += gj12 * 2.f * fy * t1 * itz2 * itz;
      }
      dmx += V[0] * gt0 + V[1] * gt1 + V[2] * gt2;
      dmy += V[4] * gt0 + V[5] * gt1 + V[6] * gt2;
      dmz += V[8] * gt0 + V[9] * gt1 + V[10] * gt2;
      // ---- projected mean (O3)
      {
        const float c0 = P[0] * mx + P[4] * my + P[8] * mz + P[12];
        const float c1 = P[1] * mx + P[5] * my + P[9] * mz + P[13];
        const float c3 = P[3] * mx + P[7] * my + P[11] * mz + P[15];
        const float ic3 = fast_rcp(c3), ic32 = ic3 * ic3;
        const float hx = 0.5f * (float)c.W * gx * ic32, hy = 0.5f * (float)c.H * gy * ic32;
        dmx += hx * (P[0] * c3 - P[3] * c0) + hy * (P[1] * c3 - P[3] * c1);
        dmy += hx * (P[4] * c3 - P[7] * c0) + hy * (P[5] * c3 - P[7] * c1);
        dmz += hx * (P[8] * c3 - P[11] * c0) + hy * (P[9] * c3 - P[11] * c1);
      }
    }
    // ---- opacity
    {
      const float o = 1.0f / (1.0f + expf(-p.ologits[i]));
      put_grad(p, 10 * n + i, gop * o * (1.0f - o), 3);
    }
    put_grad(p, 3 * i, dmx, 0);
    put_grad(p, 3 * i + 1, dmy, 0);
    put_grad(p, 3 * i + 2, dmz, 0);
    // ---- Sigma = M M^T, M = R diag(s): the summed dL/dSigma to (s, q) once
    const float GS[3][3] = {{GS00, GS01, GS02}, {GS01, GS11, GS12}, {GS02, GS12, GS22}};
    float gR[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      float gsk = 0.f;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float gM = 2.f * (GS[r][0] * M[0][k] + GS[r][1] * M[1][k] + GS[r][2] * M[2][k]);
        gsk += gM * R[r][k];
        gR[r][k] = gM * s[k];
      }
      put_grad(p, 3 * n + 3 * i + k, gsk * s[k], 1);
    }
    const float gw = 2.f * (-z * gR[0][1] + y * gR[0][2] + z * gR[1][0] - x * gR[1][2] - y * gR[2][0] + x * gR[2][1]);
    const float gx_ = 2.f * (y * gR[0][1] + z * gR[0][2] + y * gR[1][0] - 2.f * x * gR[1][1] - w * gR[1][2] +
                             z * gR[2][0] + w * gR[2][1] - 2.f * x * gR[2][2]);
    const float gy_ = 2.f * (-2.f * y * gR[0][0] + x * gR[0][1] + w * gR[0][2] + x * gR[1][0] + z * gR[1][2] -
                             w * gR[2][0] + z * gR[2][1] - 2.f * y * gR[2][2]);
    const float gz_ = 2.f * (-2.f * z * gR[0][0] - w * gR[0][1] + x * gR[0][2] + w * gR[1][0] - 2.f * z * gR[1][1] +
                             y * gR[1][2] + x * gR[2][0] + y * gR[2][1]);
    const float qd = gw * w + gx_ * x + gy_ * y + gz_ * z;
    const float d0 = (gw - w * qd) * iq, d1 = (gx_ - x * qd) * iq, d2 = (gy_ - y * qd) * iq, d3 = (gz_ - z * qd) * iq;
    if (p.adam) {
      put_grad(p, 6 * n + 4 * i, d0, 2);
      put_grad(p, 6 * n + 4 * i + 1, d1, 2);
      put_grad(p, 6 * n + 4 * i + 2, d2, 2);
      put_grad(p, 6 * n + 4 * i + 3, d3, 2);
    } else if (p.gq_vec4 && p.assign) {
      reinterpret_cast<float4*>(p.grad + 6 * n)[i] = make_float4(d0, d1, d2, d3);
    } else if (p.gq_vec4) {
      float4* gq = reinterpret_cast<float4*>(p.grad + 6 * n) + i;
      float4 q4 = *gq;
      q4.x += d0;
      q4.y += d1;
      q4.z += d2;
      q4.w += d3;
      *gq = q4;
    } else {
      float* gq = p.grad + 6 * n + 4 * i;
      gq[0] += d0;
      gq[1] += d1;
      gq[2] += d2;
      gq[3] += d3;
    }
  }
  else if ((p.adam || p.assign) && i < p.i1) {
    // fused Adam is dense (R26): a Gaussian no view sees still takes g = 0 (and an assigning
    // launch writes its zero gradient)
    for (int e = 0; e < 3; ++e) put_grad(p, 3 * i + e, 0.0f, 0);
    for (int e = 0; e < 3; ++e) put_grad(p, 3 * n + 3 * i + e, 0.0f, 1);
    for (int e = 0; e < 4; ++e) put_grad(p, 6 * n + 4 * i + e, 0.0f, 2);
    put_grad(p, 10 * n + i, 0.0f, 3);
  }
  __syncwarp();
  // ---- coalesced read-modify-write of the warp's contiguous SH-gradient block
  //      (coefficients above the active degree stay zero in the row: no gradient, R12)
  if (p.adam) {  // every coefficient of every Gaussian (dense Adam); group sh_dc = first 3
    for (int c = lane; c < 48 * nvalid; c += 32) {
      const int g = c / 48, e = c % 48;
      put_grad(p, 11 * n + 48 * wbase + c, s_dsh[warp][g * kRow + e], e < 3 ? 4 : 5);
    }
  } else if (p.assign) {  // every coefficient of every Gaussian (the row is zero where unseen)
    if (p.gsh_vec4) {
      float4* dst = reinterpret_cast<float4*>(p.grad + 11 * n) + 12 * wbase;
      for (int c = lane; c < 12 * nvalid; c += 32) {
        const int g = c / 12, e = 4 * (c % 12);
        dst[c] = *reinterpret_cast<const float4*>(&s_dsh[warp][g * kRow + e]);
      }
    } else {
      float* dst = p.grad + 11 * n + 48 * wbase;
      for (int c = lane; c < 48 * nvalid; c += 32) dst[c] = s_dsh[warp][(c / 48) * kRow + c % 48];
    }
  } else if (p.gsh_vec4) {
    float4* dst = reinterpret_cast<float4*>(p.grad + 11 * n) + 12 * wbase;
    for (int c = lane; c < 12 * nvalid; c += 32) {
      const int g = c / 12, e = 4 * (c % 12);
      if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
      const float4 r = *reinterpret_cast<const float4*>(&s_dsh[warp][g * kRow + e]);
      float4 v = dst[c];
      v.x += r.x;
      v.y += r.y;
      v.z += r.z;
      v.w += r.w;
      dst[c] = v;
    }
  } else {
    float* dst = p.grad + 11 * n + 48 * wbase;
    for (int c = lane; c < 48 * nvalid; c += 32) {
      const int g = c / 48, e = c % 48;
      if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
      dst[c] += s_dsh[warp][g * kRow + e];
    }
  }
  // a consuming frame: the blend-gradient slots read above are left zero for its next
  // backward (after all the arithmetic: the stores stay off the loads' pipeline; a warp's
  // slots of one view are 1.5 KB contiguous)
  for (int v = 0; v < p.nviews; ++v) {
    float4* z = p.view[v].grad2d_zero;
    if (z && ((vmask >> v) & 1u)) {
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      z[3 * i] = z4;
      z[3 * i + 1] = z4;
      z[3 * i + 2] = z4;
    }
  }
}

// a10 over a batch of views: grad += sum over the frames of each view's chain rule; with
// `adam` (hp != null) the last launch applies Adam instead of writing grad (grad may then be
// null when one launch covers all views).
bgs_status launch_preprocess_bwd_batch_impl(const bgs_gaussians* g, Frame* const* frames, int nviews, float* grad,
                                            float* theta, float* m, float* v, const bgs_adam_hparams* hp,
                                            int64_t step, cudaStream_t s, int64_t i0, int64_t i1, bool assign) {
  const int64_t n = frames[0]->n;
  if (i1 < 0) i1 = n;
  if (n == 0 || i1 <= i0) return BGS_OK;
  PreBwdParams p;
  p.adam = false;
  p.assign = false;
  p.theta = theta;
  p.m = m;
  p.v = v;
  if (hp) {
    const float lr[6] = {hp->lr_means, hp->lr_log_scales, hp->lr_quats, hp->lr_opacity, hp->lr_sh_dc,
                         hp->lr_sh_rest};
    const double bc1 = 1.0 - pow((double)hp->beta1, (double)step);
    const double bc2 = 1.0 - pow((double)hp->beta2, (double)step);
    for (int k = 0; k < 6; ++k) p.step_size[k] = (float)((double)lr[k] / bc1);
    p.b1 = hp->beta1;
    p.b2 = hp->beta2;
    p.eps = hp->eps;
    p.inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
  }
  p.means = g->means;
  p.log_scales = g->log_scales;
  p.quats = g->quats;
  p.ologits = g->opacity_logits;
  p.sh = g->sh;
  p.n = n;
  p.i0 = i0;
  p.i1 = i1;
  p.deg = g->sh_degree;
  auto al16 = [](const void* q) { return ((uintptr_t)q & 15u) == 0; };
  p.quat_vec4 = al16(g->quats);
  p.sh_vec4 = al16(g->sh);
  p.gq_vec4 = grad && al16(grad + 6 * n);
  p.gsh_vec4 = grad && al16(grad + 11 * n);
  p.grad = grad;
  for (int v0 = 0; v0 < nviews; v0 += kPreBwdMaxViews) {
    p.nviews = nviews - v0 < kPreBwdMaxViews ? nviews - v0 : kPreBwdMaxViews;
    p.adam = hp != nullptr && v0 + p.nviews >= nviews;  // the last launch applies Adam
    p.assign = assign && v0 == 0;                        // the first launch assigns grad
    for (int v = 0; v < p.nviews; ++v) {
      const Frame* F = frames[v0 + v];
      p.view[v].cam = F->cam;
      p.view[v].radius = F->radius;
      p.view[v].cbits = F->cbits;
      p.view[v].grad2d = F->grad2d;
      // a consuming frame (bgs_frame_set_consume): a launch over every Gaussian zeroes what it
      // reads, so the next preprocess of the frame need not (a partial range leaves the frame
      // to the preprocess's zeroing)
      p.view[v].grad2d_zero = (F->consume_g2 && i0 == 0 && i1 == n) ? F->grad2d : nullptr;
    }
    k_preprocess_bwd<<<(unsigned)((i1 - i0 + kBwdThreads - 1) / kBwdThreads), kBwdThreads, 0, s>>>(p);
    note_launch();
    bgs_status st = check_launch("k_preprocess_bwd");
    if (st != BGS_OK) return st;
    for (int v = 0; v < p.nviews; ++v)  // one backward's slots zeroed: all zero again
      if (p.view[v].grad2d_zero) frames[v0 + v]->grad2d_clean = frames[v0 + v]->grad2d_clean == 2 ? 1 : 0;
  }
  return BGS_OK;
}

bgs_status launch_preprocess_bwd_batch(const bgs_gaussians* g, Frame* const* frames, int nviews, float* grad,
                                       cudaStream_t s) {
  return launch_preprocess_bwd_batch_impl(g, frames, nviews, grad, nullptr, nullptr, nullptr, nullptr, 0, s);
}

bgs_status launch_preprocess_bwd(const bgs_gaussians* g, Frame* F, float* grad, cudaStream_t s) {
  Frame* const frames[1] = {F};
  return launch_preprocess_bwd_batch(g, frames, 1, grad, s);
}

}  // namespace bgs
