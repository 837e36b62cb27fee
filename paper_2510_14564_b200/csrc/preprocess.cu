// preprocess.cu -- a1-a3: per-Gaussian projection (K7) + exclusive scan of tiles_touched (K8).
//
// PAPER.md §II-A l.128-142: G(x) = exp(-1/2 (x-mu)^T Sigma^-1 (x-mu)), Sigma' = J W Sigma W^T J^T;
// l.59: colour from SH coefficients.  Readings R1-R13 and the canonical expression tree
// R22: every decision-bearing value (depth, xy, Sigma', conic, radius,
// rect) is computed with explicit fmaf() and IEEE div/sqrt, and this file is compiled
// with --fmad=false so nvcc contracts nothing else.  rgb/SH is free-order.
//
// Layout: theta segments are read as coalesced vectors (quats float4,
// SH 12 x float4 per Gaussian, only for Gaussians that survive the culls); outputs are
// the 48-byte render record {x, y, ex, ey | A, B, C, o | r, g, b, pthr} that the blend
// kernels stage through shared memory (the B200 form of the paper's T3 RGB
// reordering), plus radius, depth and tiles_touched.
#include "common.cuh"

namespace bgs {

// Real SH constants (R12).
__constant__ float kC0 = 0.28209479177387814f;
__constant__ float kC1 = 0.4886025119029199f;
__constant__ float kC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                             -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                             0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                             -0.5900435899266435f};

// One view's camera and output buffers.
struct PreView {
  Cam cam;
  int32_t* radius;
  float* depth;
  float4* record;
  uint32_t* tiles_touched;
  uint2* rect;              // {x0 | y0 << 16, w | h << 16} of visible Gaussians (depth-first sort)
  float4* grad2d;
  uint8_t* cbits;
  const uint8_t* keep;      // NEXT-4 keep mask or null
  int32_t square;           // R10 / R11's square rect instead of R11' (BGS_DEBUG_SQUARE_RECT)
  int32_t zero_g2;          // zero the visible Gaussians' blend-gradient slots (not already zero)
};

// Up to kPreMaxViews views per launch: theta is read once per Gaussian for all of them
// (the views of a training batch share theta, R20), so HBM traffic per view is the
// outputs plus 1/nviews of theta instead of all of theta.
struct PreParams {
  const float* means;
  const float* log_scales;
  const float* quats;
  const float* ologits;
  const float* sh;  // [n][16][3]
  int64_t n;
  int32_t deg, nviews;
  bool quat_vec4, sh_vec4;  // 16-byte aligned segments -> vector loads
  PreView view[kPreMaxViews];
};

// Sigma = (R diag s)(R diag s)^T (R5, R6) and the opacity, from theta: view independent.
struct Sigma3 {
  float S00, S01, S02, S11, S12, S22, o;
};

__device__ __forceinline__ Sigma3 sigma3(const PreParams& p, int64_t i) {
  // activations (R5): double transcendental, rounded once
  const float s0 = (float)exp((double)p.log_scales[3 * i]);
  const float s1 = (float)exp((double)p.log_scales[3 * i + 1]);
  const float s2 = (float)exp((double)p.log_scales[3 * i + 2]);
  Sigma3 r;
  r.o = (float)(1.0 / (1.0 + exp(-(double)p.ologits[i])));
  float4 q;
  if (p.quat_vec4) {
    q = __ldg(reinterpret_cast<const float4*>(p.quats) + i);
  } else {
    q = make_float4(p.quats[4 * i], p.quats[4 * i + 1], p.quats[4 * i + 2], p.quats[4 * i + 3]);
  }
  const float n2 = fmaf(q.x, q.x, fmaf(q.y, q.y, fmaf(q.z, q.z, q.w * q.w)));
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(n2));
  const float qw = q.x * inv, qx = q.y * inv, qy = q.z * inv, qz = q.w * inv;
  const float xx = qx * qx, yy = qy * qy, zz = qz * qz, xy = qx * qy, xz = qx * qz, yz = qy * qz;
  const float wx = qw * qx, wy = qw * qy, wz = qw * qz;
  const float M00 = (1.0f - 2.0f * (yy + zz)) * s0, M01 = (2.0f * (xy - wz)) * s1, M02 = (2.0f * (xz + wy)) * s2;
  const float M10 = (2.0f * (xy + wz)) * s0, M11 = (1.0f - 2.0f * (xx + zz)) * s1, M12 = (2.0f * (yz - wx)) * s2;
  const float M20 = (2.0f * (xz - wy)) * s0, M21 = (2.0f * (yz + wx)) * s1, M22 = (1.0f - 2.0f * (xx + yy)) * s2;
  r.S00 = fmaf(M02, M02, fmaf(M01, M01, M00 * M00));
  r.S01 = fmaf(M02, M12, fmaf(M01, M11, M00 * M10));
  r.S02 = fmaf(M02, M22, fmaf(M01, M21, M00 * M20));
  r.S11 = fmaf(M12, M12, fmaf(M11, M11, M10 * M10));
  r.S12 = fmaf(M12, M22, fmaf(M11, M21, M10 * M20));
  r.S22 = fmaf(M22, M22, fmaf(M21, M21, M20 * M20));
  return r;
}

// One view's geometry of a Gaussian in front of the near plane: pixel position, Sigma',
// conic, radius, tile rect.  Writes every output but the colour (rec[2]) and the clamp
// bits; returns the J clamp bits (CB_J*), or 0xffffffff when the Gaussian is culled.
__device__ __forceinline__ uint32_t project_view(const PreView& pv, int64_t i, float mx, float my, float mz,
                                                 float t0, float t1, float t2, const Sigma3& g, float tau) {
  const Cam& c = pv.cam;
  // clip, perspective divide (R4), pixel coordinates (R1)
  const float c0 = fmaf(c.P[8], mz, fmaf(c.P[4], my, fmaf(c.P[0], mx, c.P[12])));
  const float c1 = fmaf(c.P[9], mz, fmaf(c.P[5], my, fmaf(c.P[1], mx, c.P[13])));
  const float c3 = fmaf(c.P[11], mz, fmaf(c.P[7], my, fmaf(c.P[3], mx, c.P[15])));
  const float ndx = __fdiv_rn(c0, c3), ndy = __fdiv_rn(c1, c3);
  const float px = 0.5f * fmaf(ndx + 1.0f, (float)c.W, -1.0f);
  const float py = 0.5f * fmaf(ndy + 1.0f, (float)c.H, -1.0f);
  // EWA: T = J W3 (R7 clamp), Sigma' = T Sigma T^T + 0.3 I (R8)
  uint32_t cb = 0;
  float u = __fdiv_rn(t0, t2), v = __fdiv_rn(t1, t2);
  if (u > c.limx) cb |= CB_JX;
  if (u < -c.limx) cb |= CB_JX | CB_JX_NEG;
  if (v > c.limy) cb |= CB_JY;
  if (v < -c.limy) cb |= CB_JY | CB_JY_NEG;
  u = fminf(c.limx, fmaxf(-c.limx, u));
  v = fminf(c.limy, fmaxf(-c.limy, v));
  const float tpx = u * t2, tpy = v * t2;
  const float tz2 = t2 * t2;
  const float j00 = __fdiv_rn(c.fx, t2), j02 = -__fdiv_rn(c.fx * tpx, tz2);
  const float j11 = __fdiv_rn(c.fy, t2), j12 = -__fdiv_rn(c.fy * tpy, tz2);
  // W_ik = V[i + 4k]
  const float T00 = fmaf(j02, c.V[2], j00 * c.V[0]);
  const float T01 = fmaf(j02, c.V[6], j00 * c.V[4]);
  const float T02 = fmaf(j02, c.V[10], j00 * c.V[8]);
  const float T10 = fmaf(j12, c.V[2], j11 * c.V[1]);
  const float T11 = fmaf(j12, c.V[6], j11 * c.V[5]);
  const float T12 = fmaf(j12, c.V[10], j11 * c.V[9]);
  // L = T Sigma (row i, column k): L_ik = fma(T_i2, S_2k, fma(T_i1, S_1k, T_i0 S_0k))
  const float L00 = fmaf(T02, g.S02, fmaf(T01, g.S01, T00 * g.S00));
  const float L01 = fmaf(T02, g.S12, fmaf(T01, g.S11, T00 * g.S01));
  const float L02 = fmaf(T02, g.S22, fmaf(T01, g.S12, T00 * g.S02));
  const float L10 = fmaf(T12, g.S02, fmaf(T11, g.S01, T10 * g.S00));
  const float L11 = fmaf(T12, g.S12, fmaf(T11, g.S11, T10 * g.S01));
  const float L12 = fmaf(T12, g.S22, fmaf(T11, g.S12, T10 * g.S02));
  const float a = fmaf(L02, T02, fmaf(L01, T01, L00 * T00)) + 0.3f;
  const float b = fmaf(L02, T12, fmaf(L01, T11, L00 * T10));
  const float cc = fmaf(L12, T12, fmaf(L11, T11, L10 * T10)) + 0.3f;
  // det, conic (R9), radius (R10)
  const float det = fmaf(a, cc, -(b * b));
  if (det <= 0.0f) return 0xffffffffu;
  const float idet = __fdiv_rn(1.0f, det);
  const float conx = cc * idet, cony = -(b * idet), conz = a * idet;
  const float mid = 0.5f * (a + cc);
  const float lam = mid + __fsqrt_rn(fmaxf(0.1f, mid * mid - det));
  const int rad = (int)ceilf(3.0f * __fsqrt_rn(lam));
  // Conservative half-extents of the alpha >= 1/255 level set, d^T conic d <= 2 ln(255 o)
  // (R14): AABB half-widths sqrt(2 tau a), sqrt(2 tau c) with tau = ln(255 o) raised by 1e-3
  // (the threshold lowered by e^-1e-3) and a 1e-3 relative + 1e-3 px margin, so every pixel
  // outside it gets alpha < 1/255 in the blend's own float arithmetic (its G error is ~2^-20
  // relative).  The tile rect (R11') and the blend kernels' per-block skips use it; it never
  // changes a blend decision.
  float ex = -1e30f, ey = -1e30f;
  if (tau > 0.0f) {
    ex = __fsqrt_rn(2.0f * tau * a) * 1.001f + 1e-3f;
    ey = __fsqrt_rn(2.0f * tau * cc) * 1.001f + 1e-3f;
  }
  // rect, floor then clamp; culled if empty.  R11' (default): the tiles the alpha box
  // reaches -- every tile with a pixel that can blend the Gaussian, no other (a Gaussian with
  // o < 1/255 blends nowhere).  R10 / R11 (BGS_DEBUG_SQUARE_RECT): 3DGS's square of half-width
  // radius, which also holds tiles no pixel of which blends it and cuts the alpha set of an
  // opaque Gaussian (sqrt(2 ln 255) = 3.33 sigma > 3 sigma).
  const float tx = (float)c.tiles_x, ty = (float)c.tiles_y;
  int rx0, ry0, rx1, ry1;
  if (pv.square) {
    rx0 = (int)fminf(tx, fmaxf(0.0f, floorf((px - (float)rad) * 0.0625f)));
    ry0 = (int)fminf(ty, fmaxf(0.0f, floorf((py - (float)rad) * 0.0625f)));
    rx1 = (int)fminf(tx, fmaxf(0.0f, floorf((px + (float)(rad + 15)) * 0.0625f)));
    ry1 = (int)fminf(ty, fmaxf(0.0f, floorf((py + (float)(rad + 15)) * 0.0625f)));
  } else {
    if (!(tau > 0.0f)) return 0xffffffffu;
    rx0 = (int)fminf(tx, fmaxf(0.0f, floorf((px - ex) * 0.0625f)));
    ry0 = (int)fminf(ty, fmaxf(0.0f, floorf((py - ey) * 0.0625f)));
    rx1 = (int)fminf(tx, fmaxf(0.0f, floorf((px + ex) * 0.0625f) + 1.0f));
    ry1 = (int)fminf(ty, fmaxf(0.0f, floorf((py + ey) * 0.0625f) + 1.0f));
  }
  const uint32_t area = (uint32_t)(rx1 - rx0) * (uint32_t)(ry1 - ry0);
  if (area == 0) return 0xffffffffu;
  pv.radius[i] = rad;
  pv.depth[i] = t2;
  pv.tiles_touched[i] = area;
  pv.rect[i] = make_uint2((uint32_t)rx0 | ((uint32_t)ry0 << 16), (uint32_t)(rx1 - rx0) | ((uint32_t)(ry1 - ry0) << 16));
  float4* rec = pv.record + 3 * i;
  rec[1] = make_float4(-0.5f * conx, -cony, -0.5f * conz, g.o);
  rec[0] = make_float4(px, py, ex, ey);  // everything the per-warp cull test reads
  // this view's blend-gradient accumulator (render_bwd REDs into it), unless the frame's
  // grad2d is known to be all zero (a consuming frame)
  if (pv.zero_g2) {
    float4* g2 = pv.grad2d + 3 * i;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    g2[0] = z4;
    g2[1] = z4;
    g2[2] = z4;
  }
  return cb;
}

__device__ __forceinline__ void load_sh(const PreParams& p, int64_t i, float* sh) {
  if (p.sh_vec4) {
    const float4* shp = reinterpret_cast<const float4*>(p.sh) + 12 * i;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      const float4 f4 = __ldg(shp + k);
      sh[4 * k] = f4.x; sh[4 * k + 1] = f4.y; sh[4 * k + 2] = f4.z; sh[4 * k + 3] = f4.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 48; ++k) sh[k] = __ldg(p.sh + 48 * i + k);
  }
}

// SH colour (R12), free order, + 0.5, clamped below; writes rec[2] = {rgb, pthr} and the
// clamp bits (cb = the view's J bits).
__device__ __forceinline__ void colour_view(const PreView& pv, const PreParams& p, int64_t i, float mx, float my,
                                            float mz, const float* sh, float tau, uint32_t cb) {
  const Cam& c = pv.cam;
  const float dxw = mx - c.campos[0], dyw = my - c.campos[1], dzw = mz - c.campos[2];
  const float il = rsqrtf(dxw * dxw + dyw * dyw + dzw * dzw);
  const float x = dxw * il, y = dyw * il, z = dzw * il;
  float rgb[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) rgb[ch] = kC0 * sh[ch];
  if (p.deg > 0) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      rgb[ch] += -kC1 * y * sh[3 + ch] + kC1 * z * sh[6 + ch] - kC1 * x * sh[9 + ch];
    if (p.deg > 1) {
      const float xx_ = x * x, yy_ = y * y, zz_ = z * z;
      const float b4 = kC2[0] * x * y, b5 = kC2[1] * y * z, b6 = kC2[2] * (2.0f * zz_ - xx_ - yy_);
      const float b7 = kC2[3] * x * z, b8 = kC2[4] * (xx_ - yy_);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch)
        rgb[ch] += b4 * sh[12 + ch] + b5 * sh[15 + ch] + b6 * sh[18 + ch] + b7 * sh[21 + ch] + b8 * sh[24 + ch];
      if (p.deg > 2) {
        const float b9 = kC3[0] * y * (3.0f * xx_ - yy_), b10 = kC3[1] * x * y * z;
        const float b11 = kC3[2] * y * (4.0f * zz_ - xx_ - yy_);
        const float b12 = kC3[3] * z * (2.0f * zz_ - 3.0f * xx_ - 3.0f * yy_);
        const float b13 = kC3[4] * x * (4.0f * zz_ - xx_ - yy_), b14 = kC3[5] * z * (xx_ - yy_);
        const float b15 = kC3[6] * x * (xx_ - 3.0f * yy_);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
          rgb[ch] += b9 * sh[27 + ch] + b10 * sh[30 + ch] + b11 * sh[33 + ch] + b12 * sh[36 + ch] +
                     b13 * sh[39 + ch] + b14 * sh[42 + ch] + b15 * sh[45 + ch];
      }
    }
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    rgb[ch] += 0.5f;
    if (rgb[ch] < 0.0f) {
      cb |= (1u << ch);
      rgb[ch] = 0.0f;
    }
  }
  // the same bound as ex/ey per pixel: power < -tau  =>  o exp(power) < e^-1e-3 / 255, so
  // the blend's alpha (G within 2^-20 relative) is < 1/255 -- skipped without evaluating G
  const float pthr = tau > 0.0f ? -tau : 3.0e38f;
  pv.record[3 * i + 2] = make_float4(rgb[0], rgb[1], rgb[2], pthr);
  pv.cbits[i] = (uint8_t)cb;
}

// camera-space position (O2)
__device__ __forceinline__ void to_camera(const Cam& c, float mx, float my, float mz, float& t0, float& t1,
                                          float& t2) {
  t0 = fmaf(c.V[8], mz, fmaf(c.V[4], my, fmaf(c.V[0], mx, c.V[12])));
  t1 = fmaf(c.V[9], mz, fmaf(c.V[5], my, fmaf(c.V[1], mx, c.V[13])));
  t2 = fmaf(c.V[10], mz, fmaf(c.V[6], my, fmaf(c.V[2], mx, c.V[14])));
}

// One view (view[0]).
__global__ void __launch_bounds__(256, 4) k_preprocess(const __grid_constant__ PreParams p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const PreView& pv = p.view[0];
  const float mx = p.means[3 * i], my = p.means[3 * i + 1], mz = p.means[3 * i + 2];
  float t0, t1, t2;
  to_camera(pv.cam, mx, my, mz, t0, t1, t2);
  pv.radius[i] = 0;
  pv.tiles_touched[i] = 0;
  if (t2 <= pv.cam.near_plane) return;  // near cull (R3)
  if (pv.keep && !pv.keep[i]) return;   // NEXT-4: dropped by the importance keep rule (R40)
  const Sigma3 g = sigma3(p, i);
  const float tau = (float)log((double)(255.0f * g.o)) + 1e-3f;  // double, rounded once (R5)
  const uint32_t cb = project_view(pv, i, mx, my, mz, t0, t1, t2, g, tau);
  if (cb == 0xffffffffu) return;
  float sh[48];
  load_sh(p, i, sh);
  colour_view(pv, p, i, mx, my, mz, sh, tau, cb);
}

// Up to kPreMaxViews views per thread: Sigma and the opacity once, the SH coefficients
// loaded once and held in registers across the view loop; each view's record is written
// whole (its sectors complete in L2).  Measured alternatives: loading theta
// lazily at the first view that needs it (three dependent DRAM round trips: 3.17 vs 2.96 ms
// per 16 views), all geometry first and the colours after (records written in two halves
// far apart: partial sectors leave L2), re-reading the SH per view from L1/L2 and 3 CTAs
// per SM (spills) were slower.  Bit-identical to k_preprocess per view.
__global__ void __launch_bounds__(256, 2) k_preprocess_views(const __grid_constant__ PreParams p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const float mx = p.means[3 * i], my = p.means[3 * i + 1], mz = p.means[3 * i + 2];
  // every theta load is issued up front (one DRAM round trip instead of three dependent
  // ones): across a batch of views almost every Gaussian is visible in some view
  const Sigma3 g = sigma3(p, i);
  const float tau = (float)log((double)(255.0f * g.o)) + 1e-3f;  // double, rounded once (R5)
  float sh[48];
  load_sh(p, i, sh);
#pragma unroll 1
  for (int v = 0; v < p.nviews; ++v) {
    const PreView& pv = p.view[v];
    float t0, t1, t2;
    to_camera(pv.cam, mx, my, mz, t0, t1, t2);
    pv.radius[i] = 0;
    pv.tiles_touched[i] = 0;
    if (t2 <= pv.cam.near_plane) continue;
    if (pv.keep && !pv.keep[i]) continue;
    const uint32_t cb = project_view(pv, i, mx, my, mz, t0, t1, t2, g, tau);
    if (cb == 0xffffffffu) continue;
    colour_view(pv, p, i, mx, my, mz, sh, tau, cb);
  }
}

// ---------------------------------------------------------------------------
// K8: single-pass exclusive scan with decoupled look-back (dynamic tile ids).
// status word: bits 62-63 = flag (1 aggregate, 2 inclusive prefix), bits 0-61 = value.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kScanThreads) k_scan(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                      int64_t n, unsigned long long* status, uint32_t* counters,
                                                      uint32_t* ticket, int64_t max_keys, int32_t num_tiles,
                                                      bool publish_k) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  __shared__ unsigned long long s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kScanTile + (int64_t)tid * kScanItems;
  uint32_t v[kScanItems];
  unsigned long long local = 0;
  const bool full = base + kScanItems <= n;  // 16-byte vector loads (in is 256-byte aligned)
  if (full) {
#pragma unroll
    for (int k = 0; k < kScanItems / 4; ++k) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + base) + k);
      v[4 * k] = q.x;
      v[4 * k + 1] = q.y;
      v[4 * k + 2] = q.z;
      v[4 * k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = (base + k < n) ? in[base + k] : 0u;
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) local += v[k];
  // block exclusive scan of per-thread totals
  unsigned long long incl = local;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  unsigned long long warp_off = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    if (w < warp) warp_off += s_warp[w];
    total += s_warp[w];
  }
  // look-back by warp 0
  if (warp == 0) {
    unsigned long long prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed_u64(&status[0], kFlagP | total);
    } else {
      if (lane == 0) st_relaxed_u64(&status[tile], kFlagA | total);
      int64_t j = tile - 1 - lane;  // window of 32 predecessors
      while (true) {
        unsigned long long s = 0;
        if (j >= 0) {
          do {
            s = ld_relaxed_u64(&status[j]);
          } while ((s >> 62) == 0);
        } else {
          s = kFlagP;  // virtual inclusive prefix 0 before tile 0
        }
        const uint32_t pmask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        const int stop = pmask ? __ffs(pmask) - 1 : 32;
        unsigned long long contrib = (lane <= stop) ? (s & kValMask) : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, d);
        prefix += contrib;
        if (pmask) break;
        j -= 32;
      }
      if (lane == 0) st_relaxed_u64(&status[tile], kFlagP | (prefix + total));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  unsigned long long run = s_prefix + warp_off + (incl - local);
  uint32_t o[kScanItems];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    o[k] = (uint32_t)(run > 0xffffffffull ? 0xffffffffull : run);
    run += v[k];
  }
  if (full) {
#pragma unroll
    for (int k = 0; k < kScanItems / 4; ++k)
      reinterpret_cast<uint4*>(out + base)[k] = make_uint4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (base + k < n) out[base + k] = o[k];
  }
  if (tile == num_tiles - 1 && tid == 0) {
    const unsigned long long K = s_prefix + total;
    if (publish_k) {
      counters[C_K_LO] = (uint32_t)K;
      counters[C_K_HI] = (uint32_t)(K >> 32);
      counters[C_OVERFLOW] = K > (unsigned long long)max_keys ? 1u : 0u;
      if (K > (unsigned long long)max_keys) counters[C_OVF_STICKY] = 1u;
    }
    counters[C_SCAN_TOTAL] = (uint32_t)K;
  }
}

bgs_status launch_scan(const uint32_t* in, uint32_t* out, int64_t n, Frame* F, bool publish_k, cudaStream_t s) {
  const int tiles = (int)((n + kScanTile - 1) / kScanTile);
  if (tiles == 0) return BGS_OK;
  if (cudaMemsetAsync(F->scan_status, 0, 8 * (size_t)tiles, s) != cudaSuccess ||
      cudaMemsetAsync(F->counters + C_SCAN_TICKET, 0, 4, s) != cudaSuccess)
    return check_launch("scan memset");
  k_scan<<<tiles, kScanThreads, 0, s>>>(in, out, n, F->scan_status, F->counters, F->counters + C_SCAN_TICKET,
                                        F->max_keys, tiles, publish_k);
  note_launch();
  return check_launch("k_scan");
}

bgs_status launch_preprocess_batch(const bgs_gaussians* g, Frame* const* F, int nviews, cudaStream_t s) {
  for (int v = 0; v < nviews; ++v) {  // every word but the sticky overflow flag (zeroed once)
    if (cudaMemsetAsync(F[v]->counters, 0, 4 * (F[v]->counters_init ? C_OVF_STICKY : C_NUM), s) != cudaSuccess)
      return check_launch("preprocess memset");
    F[v]->counters_init = 1;
  }
  if (F[0]->n == 0) return BGS_OK;
  PreParams p;
  p.means = g->means;
  p.log_scales = g->log_scales;
  p.quats = g->quats;
  p.ologits = g->opacity_logits;
  p.sh = g->sh;
  p.quat_vec4 = ((uintptr_t)g->quats & 15u) == 0;
  p.sh_vec4 = ((uintptr_t)g->sh & 15u) == 0;
  p.n = F[0]->n;
  p.deg = g->sh_degree;
  const int64_t blocks = (p.n + 255) / 256;
  for (int v = 0; v < nviews; ++v) {
    // a consuming frame (bgs_frame_set_consume) keeps grad2d all zero between backwards: once
    // it is in an unknown state, one memset restores that; a non-consuming frame has the
    // kernel zero its visible Gaussians' slots every time
    Frame* f = F[v];
    if (f->consume_g2 && f->grad2d_clean != 1) {
      if (cudaMemsetAsync(f->grad2d, 0, 48 * (size_t)f->n, s) != cudaSuccess) return check_launch("grad2d memset");
      f->grad2d_clean = 1;
    } else if (!f->consume_g2) {
      f->grad2d_clean = 0;
    }
  }
  for (int v0 = 0; v0 < nviews; v0 += kPreMaxViews) {
    p.nviews = nviews - v0 < kPreMaxViews ? nviews - v0 : kPreMaxViews;
    for (int k = 0; k < p.nviews; ++k) {
      const Frame* f = F[v0 + k];
      PreView& pv = p.view[k];
      pv.cam = f->cam;
      pv.radius = f->radius;
      pv.depth = f->depth;
      pv.record = f->record;
      pv.tiles_touched = f->tiles_touched;
      pv.rect = f->rect;
      pv.grad2d = f->grad2d;
      pv.cbits = f->cbits;
      pv.keep = f->keep;
      pv.square = (f->debug_flags & BGS_DEBUG_SQUARE_RECT) ? 1 : 0;
      pv.zero_g2 = f->grad2d_clean == 1 ? 0 : 1;
    }
    if (p.nviews == 1)
      k_preprocess<<<(unsigned)blocks, 256, 0, s>>>(p);
    else
      k_preprocess_views<<<(unsigned)blocks, 256, 0, s>>>(p);
    note_launch();
    bgs_status st = check_launch("k_preprocess");
    if (st != BGS_OK) return st;
  }
  // the key count K (and the capacity check) comes from the sort's scan: of tiles_touched
  // in index order (64-bit reference path), or of the tile counts in depth order
  return BGS_OK;
}

bgs_status launch_preprocess(const bgs_gaussians* g, Frame* F, cudaStream_t s) {
  return launch_preprocess_batch(g, &F, 1, s);
}

}  // namespace bgs
