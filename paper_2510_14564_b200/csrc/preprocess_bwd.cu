// preprocess_bwd.cu -- a10 (K13): the chain rule from the per-view blend gradients to theta.
//
// The paper has no backward (it inherits 3DGS training); reading R18: the
// derivative of O1-O9 with the forward's decisions frozen (J-clamp branch and rgb clamp,
// both taken from the cbits the preprocess stored in the render record).  Per visible
// Gaussian: conic -> (a, b, c) of Sigma' -> Sigma and T = J W -> (s, q) and t -> mu;
// xy -> mu through the projection; rgb -> SH coefficients and the view direction -> mu;
// opacity -> logit.  grad[59n] += (views are summed, R20).
//
// Numerics: evaluated in FP64 (B200 runs FP64 at half the FP32 rate and this kernel is
// HBM-bound, ~744 B per visible Gaussian); the float version lost ~1e-3 relative on
// log_scales through cancellation in dL/dSigma' -> dL/dSigma for ill-conditioned footprints.
//
// Memory: one thread per Gaussian, 4 warps per CTA.  The 192-byte SH block and the
// 192-byte SH-gradient block of the warp's 32 Gaussians are contiguous (6 KB each), so the
// warp reads the SH coefficients and read-modify-writes the SH gradients as coalesced
// float4 passes staged through shared memory; the per-thread parts (means, scales,
// quats, opacity) are naturally coalesced.
#include "common.cuh"

namespace bgs {

__constant__ double dC0 = 0.28209479177387814;
__constant__ double dC1 = 0.4886025119029199;
__constant__ double dC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                              0.5462742152960396};
__constant__ double dC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                              -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

struct PreBwdParams {
  Cam cam;
  const float* means;
  const float* log_scales;
  const float* quats;
  const float* ologits;
  const float* sh;  // [n][16][3]
  int64_t n;
  int32_t deg;
  bool quat_vec4, sh_vec4, gq_vec4, gsh_vec4;  // 16-byte aligned -> vector paths
  const int32_t* radius;
  const float4* record;
  const float4* grad2d;
  float* grad;  // theta layout
};

constexpr int kBwdThreads = 128;
constexpr int kRow = 49;  // padded row stride (floats) of the staged SH block: conflict-free

__global__ void __launch_bounds__(kBwdThreads) k_preprocess_bwd(PreBwdParams p) {
  __shared__ float s_sh[kBwdThreads / 32][32 * kRow];
  __shared__ int s_vis[kBwdThreads / 32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = p.n;
  const int64_t wbase = ((int64_t)blockIdx.x * kBwdThreads) + warp * 32;
  const int64_t i = wbase + lane;
  const bool valid = i < n && p.radius[i] > 0;
  s_vis[warp][lane] = valid;
  float* row = &s_sh[warp][lane * kRow];
  const int ncoef = (p.deg + 1) * (p.deg + 1);
  // ---- coalesced load of the warp's SH block into shared memory
  {
    const int64_t nvalid = n - wbase < 32 ? n - wbase : 32;
    if (p.sh_vec4) {
      const float4* src = reinterpret_cast<const float4*>(p.sh) + 12 * wbase;
      for (int c = lane; c < 12 * nvalid; c += 32) {
        const int g = c / 12, e = 4 * (c % 12);
        if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
        const float4 v = __ldg(src + c);
        float* r = &s_sh[warp][g * kRow + e];
        r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
      }
    } else {
      const float* src = p.sh + 48 * wbase;
      for (int c = lane; c < 48 * nvalid; c += 32) {
        const int g = c / 48, e = c % 48;
        if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
        s_sh[warp][g * kRow + e] = __ldg(src + c);
      }
    }
  }
  __syncwarp();
  double dsh_scale[3] = {0.0, 0.0, 0.0};
  double Y[16];
  if (valid) {
    const Cam& c = p.cam;
    const float4 ga4 = p.grad2d[3 * i], gb4 = p.grad2d[3 * i + 1], gc4 = p.grad2d[3 * i + 2];
    const double gx = ga4.x, gy = ga4.y, gcx = ga4.z, gcy = ga4.w, gcz = gb4.x, gop = gb4.y;
    const uint32_t cb = __float_as_uint(p.record[3 * i + 2].y);
    const double grc[3] = {(cb & CB_R) ? 0.0 : (double)gb4.z, (cb & CB_G) ? 0.0 : (double)gb4.w,
                           (cb & CB_B) ? 0.0 : (double)gc4.x};
    const double mx = p.means[3 * i], my = p.means[3 * i + 1], mz = p.means[3 * i + 2];
    double V[16], P[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      V[k] = c.V[k];
      P[k] = c.P[k];
    }
    const double t0 = V[0] * mx + V[4] * my + V[8] * mz + V[12];
    const double t1 = V[1] * mx + V[5] * my + V[9] * mz + V[13];
    const double t2 = V[2] * mx + V[6] * my + V[10] * mz + V[14];
    double dmx = 0.0, dmy = 0.0, dmz = 0.0;
    // ---- colour: SH basis at the view direction; dL/dsh = Y grc (written below), dL/dd
    {
      const double dxw = mx - c.campos[0], dyw = my - c.campos[1], dzw = mz - c.campos[2];
      const double il = 1.0 / sqrt(dxw * dxw + dyw * dyw + dzw * dzw);
      const double x = dxw * il, y = dyw * il, z = dzw * il;
      const double xx = x * x, yy = y * y, zz = z * z;
      double dY[16][3];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        Y[k] = 0.0;
        dY[k][0] = dY[k][1] = dY[k][2] = 0.0;
      }
      Y[0] = dC0;
      if (p.deg > 0) {
        Y[1] = -dC1 * y; dY[1][1] = -dC1;
        Y[2] = dC1 * z;  dY[2][2] = dC1;
        Y[3] = -dC1 * x; dY[3][0] = -dC1;
        if (p.deg > 1) {
          Y[4] = dC2[0] * x * y; dY[4][0] = dC2[0] * y; dY[4][1] = dC2[0] * x;
          Y[5] = dC2[1] * y * z; dY[5][1] = dC2[1] * z; dY[5][2] = dC2[1] * y;
          Y[6] = dC2[2] * (2.0 * zz - xx - yy);
          dY[6][0] = -2.0 * dC2[2] * x; dY[6][1] = -2.0 * dC2[2] * y; dY[6][2] = 4.0 * dC2[2] * z;
          Y[7] = dC2[3] * x * z; dY[7][0] = dC2[3] * z; dY[7][2] = dC2[3] * x;
          Y[8] = dC2[4] * (xx - yy); dY[8][0] = 2.0 * dC2[4] * x; dY[8][1] = -2.0 * dC2[4] * y;
          if (p.deg > 2) {
            Y[9] = dC3[0] * y * (3.0 * xx - yy);
            dY[9][0] = 6.0 * dC3[0] * x * y; dY[9][1] = 3.0 * dC3[0] * (xx - yy);
            Y[10] = dC3[1] * x * y * z;
            dY[10][0] = dC3[1] * y * z; dY[10][1] = dC3[1] * x * z; dY[10][2] = dC3[1] * x * y;
            Y[11] = dC3[2] * y * (4.0 * zz - xx - yy);
            dY[11][0] = -2.0 * dC3[2] * x * y; dY[11][1] = dC3[2] * (4.0 * zz - xx - 3.0 * yy);
            dY[11][2] = 8.0 * dC3[2] * y * z;
            Y[12] = dC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            dY[12][0] = -6.0 * dC3[3] * x * z; dY[12][1] = -6.0 * dC3[3] * y * z;
            dY[12][2] = dC3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
            Y[13] = dC3[4] * x * (4.0 * zz - xx - yy);
            dY[13][0] = dC3[4] * (4.0 * zz - 3.0 * xx - yy); dY[13][1] = -2.0 * dC3[4] * x * y;
            dY[13][2] = 8.0 * dC3[4] * x * z;
            Y[14] = dC3[5] * z * (xx - yy);
            dY[14][0] = 2.0 * dC3[5] * x * z; dY[14][1] = -2.0 * dC3[5] * y * z; dY[14][2] = dC3[5] * (xx - yy);
            Y[15] = dC3[6] * x * (xx - 3.0 * yy);
            dY[15][0] = 3.0 * dC3[6] * (xx - yy); dY[15][1] = -6.0 * dC3[6] * x * y;
          }
        }
      }
      double ddx = 0.0, ddy = 0.0, ddz = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k < ncoef) {
          const double shg = (double)row[3 * k] * grc[0] + (double)row[3 * k + 1] * grc[1] +
                             (double)row[3 * k + 2] * grc[2];
          ddx += dY[k][0] * shg;
          ddy += dY[k][1] * shg;
          ddz += dY[k][2] * shg;
        }
      }
      const double dot = ddx * x + ddy * y + ddz * z;
      dmx += (ddx - x * dot) * il;
      dmy += (ddy - y * dot) * il;
      dmz += (ddz - z * dot) * il;
      dsh_scale[0] = grc[0];
      dsh_scale[1] = grc[1];
      dsh_scale[2] = grc[2];
    }
    // ---- opacity
    {
      const double o = 1.0 / (1.0 + exp(-(double)p.ologits[i]));
      p.grad[10 * n + i] += (float)(gop * o * (1.0 - o));
    }
    // ---- covariance chain
    const double s[3] = {exp((double)p.log_scales[3 * i]), exp((double)p.log_scales[3 * i + 1]),
                         exp((double)p.log_scales[3 * i + 2])};
    const float4 qh = p.quat_vec4 ? __ldg(reinterpret_cast<const float4*>(p.quats) + i)
                                  : make_float4(p.quats[4 * i], p.quats[4 * i + 1], p.quats[4 * i + 2],
                                                p.quats[4 * i + 3]);
    const double qn = sqrt((double)qh.x * qh.x + (double)qh.y * qh.y + (double)qh.z * qh.z + (double)qh.w * qh.w);
    const double iq = 1.0 / qn;
    const double w = qh.x * iq, x = qh.y * iq, y = qh.z * iq, z = qh.w * iq;
    double R[3][3];
    R[0][0] = 1.0 - 2.0 * (y * y + z * z); R[0][1] = 2.0 * (x * y - w * z); R[0][2] = 2.0 * (x * z + w * y);
    R[1][0] = 2.0 * (x * y + w * z); R[1][1] = 1.0 - 2.0 * (x * x + z * z); R[1][2] = 2.0 * (y * z - w * x);
    R[2][0] = 2.0 * (x * z - w * y); R[2][1] = 2.0 * (y * z + w * x); R[2][2] = 1.0 - 2.0 * (x * x + y * y);
    double M[3][3], Sg[3][3];
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
    const double fx = c.fx, fy = c.fy;
    double u = t0 / t2, v = t1 / t2;
    if (cb & CB_JX) u = (cb & CB_JX_NEG) ? -(double)c.limx : (double)c.limx;
    if (cb & CB_JY) v = (cb & CB_JY_NEG) ? -(double)c.limy : (double)c.limy;
    const double itz = 1.0 / t2, itz2 = itz * itz;
    const double j00 = fx * itz, j02 = -fx * u * itz, j11 = fy * itz, j12 = -fy * v * itz;
    double Tm[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      Tm[0][k] = j00 * V[0 + 4 * k] + j02 * V[2 + 4 * k];
      Tm[1][k] = j11 * V[1 + 4 * k] + j12 * V[2 + 4 * k];
    }
    double TS[2][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k) TS[a][k] = Tm[a][0] * Sg[0][k] + Tm[a][1] * Sg[1][k] + Tm[a][2] * Sg[2][k];
    const double A = TS[0][0] * Tm[0][0] + TS[0][1] * Tm[0][1] + TS[0][2] * Tm[0][2] + 0.3;
    const double B = TS[0][0] * Tm[1][0] + TS[0][1] * Tm[1][1] + TS[0][2] * Tm[1][2];
    const double Cc = TS[1][0] * Tm[1][0] + TS[1][1] * Tm[1][1] + TS[1][2] * Tm[1][2] + 0.3;
    const double det = A * Cc - B * B;
    const double id2 = 1.0 / (det * det);
    const double gA = (-Cc * Cc * gcx + B * Cc * gcy - B * B * gcz) * id2;
    const double gB = (2.0 * B * Cc * gcx - (A * Cc + B * B) * gcy + 2.0 * A * B * gcz) * id2;
    const double gC = (-B * B * gcx + A * B * gcy - A * A * gcz) * id2;
    const double Gp[2][2] = {{gA, 0.5 * gB}, {0.5 * gB, gC}};
    // dL/dSigma = T^T G' T ; dL/dT = 2 G' (T Sigma)
    double GS[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        GS[r][q] = Tm[0][r] * (Gp[0][0] * Tm[0][q] + Gp[0][1] * Tm[1][q]) +
                   Tm[1][r] * (Gp[1][0] * Tm[0][q] + Gp[1][1] * Tm[1][q]);
    double gT[2][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k) gT[a][k] = 2.0 * (Gp[a][0] * TS[0][k] + Gp[a][1] * TS[1][k]);
    double gj00 = 0.0, gj02 = 0.0, gj11 = 0.0, gj12 = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      gj00 += gT[0][k] * V[0 + 4 * k];
      gj02 += gT[0][k] * V[2 + 4 * k];
      gj11 += gT[1][k] * V[1 + 4 * k];
      gj12 += gT[1][k] * V[2 + 4 * k];
    }
    double gt0 = 0.0, gt1 = 0.0, gt2 = -(gj00 * fx + gj11 * fy) * itz2;
    if (cb & CB_JX) {
      gt2 += gj02 * fx * u * itz2;
    } else {
      gt0 += -gj02 * fx * itz2;
      gt2 += gj02 * 2.0 * fx * t0 * itz2 * itz;
    }
    if (cb & CB_JY) {
      gt2 += gj12 * fy * v * itz2;
    } else {
      gt1 += -gj12 * fy * itz2;
      gt2 += gj12 * 2.0 * fy * t1 * itz2 * itz;
    }
    dmx += V[0] * gt0 + V[1] * gt1 + V[2] * gt2;
    dmy += V[4] * gt0 + V[5] * gt1 + V[6] * gt2;
    dmz += V[8] * gt0 + V[9] * gt1 + V[10] * gt2;
    // ---- projected mean (O3)
    {
      const double c0 = P[0] * mx + P[4] * my + P[8] * mz + P[12];
      const double c1 = P[1] * mx + P[5] * my + P[9] * mz + P[13];
      const double c3 = P[3] * mx + P[7] * my + P[11] * mz + P[15];
      const double ic3 = 1.0 / c3, ic32 = ic3 * ic3;
      const double hx = 0.5 * (double)c.W * gx * ic32, hy = 0.5 * (double)c.H * gy * ic32;
      dmx += hx * (P[0] * c3 - P[3] * c0) + hy * (P[1] * c3 - P[3] * c1);
      dmy += hx * (P[4] * c3 - P[7] * c0) + hy * (P[5] * c3 - P[7] * c1);
      dmz += hx * (P[8] * c3 - P[11] * c0) + hy * (P[9] * c3 - P[11] * c1);
    }
    float* gm = p.grad + 3 * i;
    gm[0] += (float)dmx;
    gm[1] += (float)dmy;
    gm[2] += (float)dmz;
    // ---- Sigma = M M^T, M = R diag(s)
    double gR[3][3];
    float* gls = p.grad + 3 * n + 3 * i;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double gsk = 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const double gM = 2.0 * (GS[r][0] * M[0][k] + GS[r][1] * M[1][k] + GS[r][2] * M[2][k]);
        gsk += gM * R[r][k];
        gR[r][k] = gM * s[k];
      }
      gls[k] += (float)(gsk * s[k]);
    }
    const double gw = 2.0 * (-z * gR[0][1] + y * gR[0][2] + z * gR[1][0] - x * gR[1][2] - y * gR[2][0] + x * gR[2][1]);
    const double gx_ = 2.0 * (y * gR[0][1] + z * gR[0][2] + y * gR[1][0] - 2.0 * x * gR[1][1] - w * gR[1][2] +
                              z * gR[2][0] + w * gR[2][1] - 2.0 * x * gR[2][2]);
    const double gy_ = 2.0 * (-2.0 * y * gR[0][0] + x * gR[0][1] + w * gR[0][2] + x * gR[1][0] + z * gR[1][2] -
                              w * gR[2][0] + z * gR[2][1] - 2.0 * y * gR[2][2]);
    const double gz_ = 2.0 * (-2.0 * z * gR[0][0] - w * gR[0][1] + x * gR[0][2] + w * gR[1][0] -
                              2.0 * z * gR[1][1] + y * gR[1][2] + x * gR[2][0] + y * gR[2][1]);
    const double qd = gw * w + gx_ * x + gy_ * y + gz_ * z;
    const float d0 = (float)((gw - w * qd) * iq), d1 = (float)((gx_ - x * qd) * iq);
    const float d2 = (float)((gy_ - y * qd) * iq), d3 = (float)((gz_ - z * qd) * iq);
    if (p.gq_vec4) {
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
  __syncwarp();
  // ---- stage this thread's dL/dsh row (Y_k * grc_ch) in shared memory, then a coalesced
  //      float4 read-modify-write of the warp's contiguous SH-gradient block
  if (valid) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      row[3 * k] = (float)(Y[k] * dsh_scale[0]);
      row[3 * k + 1] = (float)(Y[k] * dsh_scale[1]);
      row[3 * k + 2] = (float)(Y[k] * dsh_scale[2]);
    }
  }
  __syncwarp();
  const int64_t nvalid = n - wbase < 32 ? n - wbase : 32;
  if (p.gsh_vec4) {
    float4* dst = reinterpret_cast<float4*>(p.grad + 11 * n) + 12 * wbase;
    for (int c = lane; c < 12 * nvalid; c += 32) {
      const int g = c / 12, e = 4 * (c % 12);
      if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
      const float* r = &s_sh[warp][g * kRow + e];
      float4 v = dst[c];
      v.x += r[0];
      v.y += r[1];
      v.z += r[2];
      v.w += r[3];
      dst[c] = v;
    }
  } else {
    float* dst = p.grad + 11 * n + 48 * wbase;
    for (int c = lane; c < 48 * nvalid; c += 32) {
      const int g = c / 48, e = c % 48;
      if (!s_vis[warp][g] || e >= 3 * ncoef) continue;
      dst[c] += s_sh[warp][g * kRow + e];
    }
  }
}

bgs_status launch_preprocess_bwd(const bgs_gaussians* g, Frame* F, float* grad, cudaStream_t s) {
  if (F->n == 0) return BGS_OK;
  PreBwdParams p;
  p.cam = F->cam;
  p.means = g->means;
  p.log_scales = g->log_scales;
  p.quats = g->quats;
  p.ologits = g->opacity_logits;
  p.sh = g->sh;
  auto al16 = [](const void* q) { return ((uintptr_t)q & 15u) == 0; };
  p.quat_vec4 = al16(g->quats);
  p.sh_vec4 = al16(g->sh);
  p.gq_vec4 = al16(grad + 6 * F->n);
  p.gsh_vec4 = al16(grad + 11 * F->n);
  p.n = F->n;
  p.deg = g->sh_degree;
  p.radius = F->radius;
  p.record = F->record;
  p.grad2d = F->grad2d;
  p.grad = grad;
  k_preprocess_bwd<<<(unsigned)((F->n + kBwdThreads - 1) / kBwdThreads), kBwdThreads, 0, s>>>(p);
  note_launch();
  return check_launch("k_preprocess_bwd");
}

}  // namespace bgs
