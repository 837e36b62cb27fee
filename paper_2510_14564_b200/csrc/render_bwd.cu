// render_bwd.cu -- a9 blend backward (K12).
//
// The paper has no backward; it inherits 3DGS training.  Reading
// R18: the gradient of the forward O1-O14 with every discrete decision frozen (cull,
// rect, power/alpha skips, early stop, the 0.99 alpha clamp -> zero gradient to o and G,
// the SH clamp, the J-clamp branch).
//
// Workload-balanced mapping: independent warps of a persistent grid pull (tile, 8x4 block)
// items heaviest first -- by the forward's per-tile largest n_contrib -- so no warp waits
// on another.  A warp walks its tile list back to front from its own block's largest
// n_contrib, 32 entries per step, compacted to the entries whose alpha >= 1/255 box
// reaches the block (exact, as in the forward).  The step loop is software-pipelined:
// list ids are fetched three steps ahead, the 16-byte cull records {x,y,ex,ey} two steps
// ahead, and the full records of the hits one step ahead, so the gathers overlap the
// walk.  Per pixel: T_i = T_{i+1} / (1 - alpha_i), and the colour behind, S += c alpha T
// (S starts at T_final bg), is carried only as the scalar DS = dL/dC . S it contributes.
// Each evaluated entry yields 9 partials: dL/dxy (2), dp {dx^2, dx dy, dy^2} (dp =
// dL/dpower), the opacity part and w dL/dC.  A reduce-scatter butterfly (12 shuffles) leaves
// the 9 warp totals on 9 lanes, which scale the conic ones and add all 9 into grad2d[id]
// with one 9-lane RED instruction -- instead of 3DGS's nine scalar global
// atomics per evaluated pair.
//
// K13 (the chain rule to theta) is in preprocess_bwd.cu.
#include "common.cuh"

namespace bgs {

constexpr int kBwdWarpsPerCta = 4;
// entries taken by at most this many lanes are added by per-lane REDs instead of the warp
// reduce-scatter
#ifndef BGS_BWD_RED_LANES
#define BGS_BWD_RED_LANES 6
#endif

// Reduce-scatter of 9 per-lane values over the warp: each butterfly step halves the set of
// values a lane carries (5 -> 3 -> 2 -> 1 -> 1 shuffles: 12 instead of 9 x 5 = 45).  On
// return lane l holds the warp total of value `idx`, or idx = -1 (padding / duplicate).
__device__ __forceinline__ float warp_reduce_scatter9(const float v[9], int lane, int& idx) {
  const bool a = lane & 16, b = lane & 8, c = lane & 4, d = lane & 2;
  // each step: the lane keeps one half of its values and sends the other to its partner;
  // the sums of a step go pairwise through FADD2
  float k5[5], r5[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const float lo = v[j], hi = j < 4 ? v[5 + j] : 0.0f;
    k5[j] = a ? hi : lo;
    r5[j] = __shfl_xor_sync(0xffffffffu, a ? lo : hi, 16);
  }
  const float2 s01 = __fadd2_rn(make_float2(k5[0], k5[1]), make_float2(r5[0], r5[1]));
  const float2 s23 = __fadd2_rn(make_float2(k5[2], k5[3]), make_float2(r5[2], r5[3]));
  const float s[5] = {s01.x, s01.y, s23.x, s23.y, k5[4] + r5[4]};
  float k3[3], r3[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float lo = s[j], hi = j < 2 ? s[3 + j] : 0.0f;
    k3[j] = b ? hi : lo;
    r3[j] = __shfl_xor_sync(0xffffffffu, b ? lo : hi, 8);
  }
  const float2 t01 = __fadd2_rn(make_float2(k3[0], k3[1]), make_float2(r3[0], r3[1]));
  const float t[3] = {t01.x, t01.y, k3[2] + r3[2]};
  float k2[2], r2[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const float lo = t[j], hi = j < 1 ? t[2] : 0.0f;
    k2[j] = c ? hi : lo;
    r2[j] = __shfl_xor_sync(0xffffffffu, c ? lo : hi, 4);
  }
  const float2 u = __fadd2_rn(make_float2(k2[0], k2[1]), make_float2(r2[0], r2[1]));
  float w = (d ? u.y : u.x) + __shfl_xor_sync(0xffffffffu, d ? u.x : u.y, 2);
  w += __shfl_xor_sync(0xffffffffu, w, 1);
  const int slot = (b ? 3 : 0) + (c ? 2 : 0) + (d ? 1 : 0);
  const bool valid = (b ? !c : !(c && d)) && !(a && slot == 4) && !(lane & 1);
  idx = valid ? (a ? 5 : 0) + slot : -1;
  return w;
}

__device__ __forceinline__ uint64_t f2_to_u64(float2 a) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a.x), "f"(a.y));
  return d;
}
__device__ __forceinline__ float2 f2_from_u64(uint64_t a) {
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(a));
  return d;
}
__device__ __forceinline__ void f2_mul_inplace(uint64_t& a, uint64_t b) {
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(b));
}

__device__ __forceinline__ bool box_hits(const float4 a, float bx0, float by0, float bx1, float by1) {
  return a.x + a.z >= bx0 && a.x - a.z <= bx1 && a.y + a.w >= by0 && a.y - a.w <= by1;
}

// PPL = pixels per lane: 1 -> the unit is an 8x4 block (one forward item), 2 -> an 8x8
// block (two vertically adjacent forward items, lane l on pixels (x, y) and (x, y + 4)):
// each entry's staging, shared-memory record reads and 9-value warp reduction then serve
// 64 pixels instead of 32.
template <int PPL, bool CANON>
__global__ void __launch_bounds__(kBwdWarpsPerCta * 32) k_render_bwd(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ values, const float4* __restrict__ record,
    const uint32_t* __restrict__ counters, Cam cam, const uint32_t* __restrict__ units, uint32_t* ticket,
    const float* __restrict__ dl_dimage, const float* __restrict__ final_T, const uint32_t* __restrict__ n_contrib,
    float4* __restrict__ grad2d, int32_t seg_len, const uint32_t* __restrict__ ck_table,
    const float4* __restrict__ ck_pool) {
  __shared__ float4 s_rec[kBwdWarpsPerCta][32 * 3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const bool overflow = counters[C_OVERFLOW] != 0;
  float4* srec = s_rec[warp];
  const int64_t plane = (int64_t)cam.W * cam.H;
  const float4 none = make_float4(-1e30f, -1e30f, -1e30f, -1e30f);
  const uint32_t n_units = counters[C_BWD_UNITS];
  // the factor this lane's reduced value takes (warp_reduce_scatter9's idx depends on the
  // lane only): the conic partials dp {dx^2, dx dy, dy^2} -> dL/dconic = (-1/2, -1, -1/2) x
  float red_mul = 1.0f;
  {
    int idx;
    const float zero[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    (void)warp_reduce_scatter9(zero, lane, idx);
    red_mul = idx == 3 ? -1.0f : (idx == 2 || idx == 4) ? -0.5f : 1.0f;
  }
  while (true) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(ticket, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_units) break;
    // unit = (tile << log2(8 / PPL) | block) | segment k << 25 | last segment << 31
    const uint32_t code = units[item];
    const uint32_t it = code & ((1u << 25) - 1u);
    const int seg = (int)((code >> 25) & 63u);
    const bool last_seg = (code >> 31) != 0;
    const int per_tile = 8 / PPL;
    const int tile = (int)(it / per_tile), blk = (int)(it % per_tile);
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int bx = tx * kTile + (blk & 1) * 8, by = ty * kTile + (blk >> 1) * 4 * PPL;
    const int px = bx + (lane & 7);
    const float bx0 = (float)bx, by0 = (float)by, bx1 = bx0 + 7.0f, by1 = by0 + (float)(4 * PPL - 1);
    const float pxf = (float)px;
    uint2 rg = ranges[tile];
    if (overflow) rg = make_uint2(0, 0);
    // per pixel h of the lane: forward item (8x4 block) fit[h], pixel (px, py[h])
    bool inside[PPL];
    int64_t pix[PPL];
    uint32_t my_last[PPL], fit[PPL];
    float pyf[PPL];
    uint32_t lmax = 0;
#pragma unroll
    for (int h = 0; h < PPL; ++h) {
      const int py = by + 4 * h + (lane >> 3);
      fit[h] = PPL == 1 ? it : (uint32_t)tile * 8u + (uint32_t)((blk & 1) + 4 * (blk >> 1) + 2 * h);
      inside[h] = px < cam.W && py < cam.H;
      pix[h] = (int64_t)py * cam.W + px;
      pyf[h] = (float)py;
      my_last[h] = inside[h] ? n_contrib[pix[h]] : 0u;
      lmax = max(lmax, my_last[h]);
    }
    const int wmax = (int)min(__reduce_max_sync(0xffffffffu, lmax), rg.y - rg.x);
    // this unit walks list positions [lo, top): segment seg of the block's walk
    const int lo = seg * seg_len;
    const int top = last_seg ? wmax : min(wmax, lo + seg_len);
    if (top <= lo) continue;
    float T[PPL], dLr[PPL], dLg[PPL], dLb[PPL], DS[PPL];
#pragma unroll
    for (int h = 0; h < PPL; ++h) {
      T[h] = inside[h] ? final_T[pix[h]] : 1.0f;
      dLr[h] = dLg[h] = dLb[h] = 0.f;
      if (inside[h]) {
        dLr[h] = dl_dimage[pix[h]];
        dLg[h] = dl_dimage[plane + pix[h]];
        dLb[h] = dl_dimage[2 * plane + pix[h]];
      }
      // the colour behind the current entry enters the gradient only as DS = dL/dC . S
      DS[h] = T[h] * (dLr[h] * cam.bg[0] + dLg[h] * cam.bg[1] + dLb[h] * cam.bg[2]);
      if (!last_seg && (int)my_last[h] > top) {
        // the pixel's walk continues past this segment: start from the forward's checkpoint
        // {T, colour behind} at boundary seg + 1 of its own forward item
        const float4 c = ck_pool[(size_t)ck_table[(size_t)fit[h] * kCkMax + seg] * 32 + lane];
        T[h] = c.x;
        DS[h] = dLr[h] * c.y + dLg[h] * c.z + dLb[h] * c.w;
      }
    }
    // PPL == 2: the two pixels' state as pairs for the FP32x2 instructions (FFMA2 / FMUL2 /
    // FADD2 of sm_100: one instruction, two separately rounded results)
    // (T2 is carried as one 64-bit register pair: as a float2 the allocator split it over two
    // unrelated registers and copied it into a pair around every entry)
    uint64_t T2u = f2_to_u64(make_float2(T[0], T[PPL - 1]));
    float2 DS2 = make_float2(DS[0], DS[PPL - 1]);
    const float2 dLr2 = make_float2(dLr[0], dLr[PPL - 1]), dLg2 = make_float2(dLg[0], dLg[PPL - 1]),
                 dLb2 = make_float2(dLb[0], dLb[PPL - 1]), npy2 = make_float2(-pyf[0], -pyf[PPL - 1]);
    const int nst = (top - lo + 31) / 32;
    // lane's list position in step s (back to front; below lo = no entry)
    auto pos_of = [&](int s) { return top - 32 * (s + 1) + lane; };
    auto load_id = [&](int s) -> uint32_t {
      const int p = pos_of(s);
      return (s < nst && p >= lo) ? __ldg(values + rg.x + (uint32_t)p) : 0xffffffffu;
    };
    auto load_cull = [&](uint32_t id) { return id != 0xffffffffu ? __ldg(record + 3 * id) : none; };
    // pipeline prologue: step 0 fully, step 1 cull record, step 2 id
    uint32_t id_c = load_id(0);
    float4 a_c = load_cull(id_c);
    uint32_t id_n = load_id(1);
    float4 a_n = load_cull(id_n);
    uint32_t id_nn = load_id(2);
    bool h_c = box_hits(a_c, bx0, by0, bx1, by1);
    float4 r1_c, r2_c;  // loaded (and read) only for a hit
    if (h_c) {
      r1_c = __ldg(record + 3 * id_c + 1);
      r2_c = __ldg(record + 3 * id_c + 2);
    }
    for (int s = 0; s < nst; ++s) {
      // (1) commit step s into the warp's shared-memory slice
      // exact ellipse-vs-block cull of the box hits (their full records are loaded)
      if (h_c) h_c = ellipse_hits_block(a_c.x, a_c.y, r1_c.x, r1_c.y, r1_c.z, r2_c.w, bx0, by0, bx1, by1);
      const uint32_t bal = __ballot_sync(0xffffffffu, h_c);
      if (h_c) {
        const int q = __popc(bal & lt);
        srec[3 * q] = make_float4(a_c.x, a_c.y, __uint_as_float((uint32_t)pos_of(s)), __uint_as_float(id_c));
        srec[3 * q + 1] = r1_c;
        srec[3 * q + 2] = r2_c;
      }
      __syncwarp();
      // (2) step s+1: hit test and its full records; (3) step s+2 cull record, s+3 id
      const bool h_n = box_hits(a_n, bx0, by0, bx1, by1);
      float4 r1_n, r2_n;
      if (h_n) {
        r1_n = __ldg(record + 3 * id_n + 1);
        r2_n = __ldg(record + 3 * id_n + 2);
      }
      const float4 a_nn = load_cull(id_nn);
      const uint32_t id_nnn = load_id(s + 3);
      // (4) walk step s, back to front.  Per entry and pixel the partials are
      //   dL/dxy = dp (2A dx + B dy, 2C dy + B dx), dp {dx^2, dx dy, dy^2}, dL/do-part, w dL/dC
      // (dp = dL/dpower), summed over the lane's pixels; the conic's factors (-1/2, -1, -1/2)
      // are applied to the warp totals
      const int m = __popc(bal);
      for (int k = m - 1; k >= 0; --k) {
        // entry k of the step: {x, y, list position, id}, {A, B, C, o}, {r, g, b, pthr}
        const float4 r0 = srec[3 * k];
        const float4 r1 = srec[3 * k + 1];
        const float4 r2 = srec[3 * k + 2];
        const uint32_t pos = __float_as_uint(r0.z);
        bool any_act = false;
        float g0, g1, g2, g3, g4, g5, g6, g7, g8;
        if constexpr (PPL == 2) {
          // both pixels of the lane at once, without per-pixel branches: a pixel that does not
          // take the entry gets alpha = 0 (1 / (1 - 0) = 1 exactly, weight 0), so its T, DS and
          // partials are unchanged; an entry no pixel of the warp takes is skipped uniformly
          const float dx = r0.x - pxf;
          const float dxx = dx * dx;
          const float2 dx2 = make_float2(dx, dx);
          const float2 dy2 = __fadd2_rn(make_float2(r0.y, r0.y), npy2);
          const float2 dyy2 = __fmul2_rn(dy2, dy2), dxy2 = __fmul2_rn(dx2, dy2);
          const float2 pw = __ffma2_rn(make_float2(r1.x, r1.x), make_float2(dxx, dxx),
                                       __ffma2_rn(make_float2(r1.z, r1.z), dyy2,
                                                  __fmul2_rn(make_float2(r1.y, r1.y), dxy2)));
          // the pixel's walk reaches the entry, and the power is neither below the exact
          // alpha < 1/255 bound (pthr) nor above R14's power > 0 guard
          const bool c0 = (pos < my_last[0]) & !(pw.x > 0.0f) & !(pw.x < r2.w);
          const bool c1 = (pos < my_last[1]) & !(pw.y > 0.0f) & !(pw.y < r2.w);
          if (!__any_sync(0xffffffffu, c0 | c1)) continue;
          // min(power, 0): G <= 1 is finite for the pixels that skip the entry too, so their
          // zeroed dL/dalpha zeroes every partial (power <= 0 wherever the entry is taken)
          const float G0 = CANON ? canon_exp(fminf(pw.x, 0.0f)) : fast_exp(fminf(pw.x, 0.0f));
          const float G1 = CANON ? canon_exp(fminf(pw.y, 0.0f)) : fast_exp(fminf(pw.y, 0.0f));
          const float2 og2 = __fmul2_rn(make_float2(r1.w, r1.w), make_float2(G0, G1));
          const float al0 = fminf(0.99f, og2.x), al1 = fminf(0.99f, og2.y);
          const bool t0 = c0 & (al0 >= (1.0f / 255.0f)), t1 = c1 & (al1 >= (1.0f / 255.0f));
          any_act = t0 | t1;
          const float2 al2 = make_float2(t0 ? al0 : 0.0f, t1 ? al1 : 0.0f);
          const float2 om2 = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-al2.x, -al2.y));
          // MUFU reciprocal (1 - alpha >= 0.01): ~2^-22 relative per step, far inside the
          // 1e-3 gradient tolerance, instead of the multi-instruction IEEE division
          const float2 io2 = make_float2(fast_rcp(om2.x), fast_rcp(om2.y));
          f2_mul_inplace(T2u, f2_to_u64(io2));  // transmittance in front of this Gaussian
          const float2 T2 = f2_from_u64(T2u);
          const float2 w2 = __fmul2_rn(al2, T2);
          const float2 p6 = __fmul2_rn(w2, dLr2), p7 = __fmul2_rn(w2, dLg2), p8 = __fmul2_rn(w2, dLb2);
          // dL/dalpha = T (dL . c) - DS / (1 - alpha); DS += (dL . c) w
          const float2 dLc2 = __ffma2_rn(dLb2, make_float2(r2.z, r2.z),
                                         __ffma2_rn(dLg2, make_float2(r2.y, r2.y),
                                                    __fmul2_rn(dLr2, make_float2(r2.x, r2.x))));
          const float2 dsi = __fmul2_rn(DS2, io2);
          const float2 dLda2 = __ffma2_rn(T2, dLc2, make_float2(-dsi.x, -dsi.y));
          DS2 = __ffma2_rn(dLc2, w2, DS2);
          // unclamped alpha: gradient to opacity and G (R18)
          const bool u0 = t0 & (og2.x <= 0.99f), u1 = t1 & (og2.y <= 0.99f);
          const float2 dl2 = make_float2(u0 ? dLda2.x : 0.0f, u1 ? dLda2.y : 0.0f);
          const float2 p5 = __fmul2_rn(dl2, make_float2(G0, G1));
          const float2 dp2 = __fmul2_rn(dl2, og2);  // dL/dpower
          const float2 e0 = __ffma2_rn(make_float2(2.0f * r1.x, 2.0f * r1.x), dx2,
                                       __fmul2_rn(make_float2(r1.y, r1.y), dy2));
          const float2 e1 = __ffma2_rn(make_float2(2.0f * r1.z, 2.0f * r1.z), dy2,
                                       __fmul2_rn(make_float2(r1.y, r1.y), dx2));
          const float2 p0 = __fmul2_rn(dp2, e0), p1 = __fmul2_rn(dp2, e1);
          const float2 p2 = __fmul2_rn(dp2, make_float2(dxx, dxx)), p3 = __fmul2_rn(dp2, dxy2),
                       p4 = __fmul2_rn(dp2, dyy2);
          g0 = p0.x + p0.y;
          g1 = p1.x + p1.y;
          g2 = p2.x + p2.y;
          g3 = p3.x + p3.y;
          g4 = p4.x + p4.y;
          g5 = p5.x + p5.y;
          g6 = p6.x + p6.y;
          g7 = p7.x + p7.y;
          g8 = p8.x + p8.y;
        } else {
          g0 = g1 = g2 = g3 = g4 = g5 = g6 = g7 = g8 = 0.0f;
          if (pos < my_last[0]) {
            const float dx = r0.x - pxf;
            const float dxx = dx * dx;
            const float dy = r0.y - pyf[0];
            const float dyy = dy * dy, dxy = dx * dy;
            const float power = fmaf(r1.x, dxx, fmaf(r1.z, dyy, r1.y * dxy));
            // power below the exact alpha < 1/255 bound (pthr): skipped without the MUFU path
            if (!(power > 0.0f || power < r2.w)) {
              const float G = CANON ? canon_exp(power) : fast_exp(power);
              const float og = r1.w * G;
              const float alpha = fminf(0.99f, og);
              if (alpha >= (1.0f / 255.0f)) {
                any_act = true;
                const float ioma = __fdividef(1.0f, 1.0f - alpha);
                T[0] = T[0] * ioma;  // transmittance in front of this Gaussian
                const float w = alpha * T[0];
                g6 = w * dLr[0];
                g7 = w * dLg[0];
                g8 = w * dLb[0];
                // dL/dalpha = sum_c dL_c (c_c T - S_c / (1 - alpha)) = T (dL . c) - DS / (1 - alpha)
                const float dLc = fmaf(dLb[0], r2.z, fmaf(dLg[0], r2.y, dLr[0] * r2.x));
                const float dLda = fmaf(T[0], dLc, -(DS[0] * ioma));
                DS[0] = fmaf(dLc, w, DS[0]);  // S += c w
                if (og <= 0.99f) {  // unclamped alpha: gradient to opacity and G (R18)
                  g5 = dLda * G;
                  const float dp = dLda * og;  // dL/dpower
                  g0 = dp * fmaf(2.0f * r1.x, dx, r1.y * dy);
                  g1 = dp * fmaf(2.0f * r1.z, dy, r1.y * dx);
                  g2 = dp * dxx;
                  g3 = dp * dxy;
                  g4 = dp * dyy;
                }
              }
            }
          }
        }
        const uint32_t actm = __ballot_sync(0xffffffffu, any_act);
        const uint32_t id = __float_as_uint(r0.w);
        if (__popc(actm) > BGS_BWD_RED_LANES) {
          const float gv[9] = {g0, g1, g2, g3, g4, g5, g6, g7, g8};
          int idx;
          const float tot = warp_reduce_scatter9(gv, lane, idx);
          // 9 lanes, 9 consecutive floats of grad2d[id]: one RED instruction (the conic
          // partials take their constant factor here, once per entry)
          if (idx >= 0) atomicAdd(reinterpret_cast<float*>(grad2d + 3 * id) + idx, tot * red_mul);
        } else if (any_act) {
          // at most 8 active lanes (an entry at the edge of its footprint): 9 REDs from each
          // instead of the 12-shuffle reduce-scatter.  Garden: blend bwd 20.65 -> 20.4 ms per
          // step at <= 8; <= 16 lanes is slower (22.6 ms: same-address L2 atomics)
          float* dst = reinterpret_cast<float*>(grad2d + 3 * id);
          atomicAdd(dst + 0, g0);
          atomicAdd(dst + 1, g1);
          atomicAdd(dst + 2, -0.5f * g2);
          atomicAdd(dst + 3, -g3);
          atomicAdd(dst + 4, -0.5f * g4);
          atomicAdd(dst + 5, g5);
          atomicAdd(dst + 6, g6);
          atomicAdd(dst + 7, g7);
          atomicAdd(dst + 8, g8);
        }
      }
      __syncwarp();
      // rotate the pipeline
      id_c = id_n;
      a_c = a_n;
      h_c = h_n;
      r1_c = r1_n;
      r2_c = r2_n;
      id_n = id_nn;
      a_n = a_nn;
      id_nn = id_nnn;
    }
  }
}

template <int PPL, bool CANON>
static int bwd_grid() {
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_bwd<PPL, CANON>, kBwdWarpsPerCta * 32, 0);
    grid = (per_sm < 1 ? 1 : per_sm) * num_sms();
  }
  return grid;
}

// Backward work units, longest first: every (tile, 8x4 block) item with a non-empty walk
// (block_cost = its largest n_contrib, from the forward) contributes one unit per segment:
// segments [k seg_len, (k + 1) seg_len) for each consecutive recorded boundary, and a last
// segment up to the walk's end.  Bucketed by length (4 buckets per octave) in three grid
// steps like the forward's plan (k_plan_scan is in render_fwd.cu).
__global__ void __launch_bounds__(kPlanBuckets) k_plan_scan(uint32_t* plan, uint32_t* counters, int units_slot,
                                                           int reset0, int reset1);

// segments of unit t (its PPL forward items fit = first + 2 h): boundaries b = 1.. with
// b seg_len < the unit's walk, where every item whose own walk crosses b has a checkpoint
__device__ __forceinline__ void bwd_unit(int t, int ppl, const uint32_t* block_cost, bool overflow, uint32_t& wl,
                                         uint32_t* fit) {
  wl = 0;
  const int per_tile = 8 / ppl, tile = t / per_tile, blk = t % per_tile;
  for (int h = 0; h < ppl; ++h) {
    fit[h] = ppl == 1 ? (uint32_t)t : (uint32_t)tile * 8u + (uint32_t)((blk & 1) + 4 * (blk >> 1) + 2 * h);
    wl = max(wl, overflow ? 0u : block_cost[fit[h]]);
  }
}

__device__ __forceinline__ int bwd_nseg(const uint32_t* fit, int ppl, uint32_t wl, const uint32_t* block_cost,
                                        const uint32_t* ck_table, uint32_t ck_cap, int seg_len) {
  int nb = 0;
  while (nb < kCkMax && (uint32_t)(nb + 1) * (uint32_t)seg_len < wl) {
    bool ok = true;
    for (int h = 0; h < ppl; ++h)
      if (block_cost[fit[h]] > (uint32_t)(nb + 1) * (uint32_t)seg_len)
        ok &= ck_table[(size_t)fit[h] * kCkMax + nb] < ck_cap;
    if (!ok) break;
    ++nb;
  }
  return nb + 1;
}

__global__ void __launch_bounds__(256) k_bwd_plan_count(const uint32_t* __restrict__ block_cost, int32_t n_units,
                                                       int32_t ppl, const uint32_t* __restrict__ ck_table,
                                                       uint32_t ck_cap, int32_t seg_len, const uint32_t* counters,
                                                       uint32_t* plan) {
  __shared__ uint32_t s_b[kPlanBuckets];
  for (int k = threadIdx.x; k < kPlanBuckets; k += blockDim.x) s_b[k] = 0;
  __syncthreads();
  const bool overflow = counters[C_OVERFLOW] != 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_units; t += gridDim.x * blockDim.x) {
    uint32_t wl, fit[2];
    bwd_unit(t, ppl, block_cost, overflow, wl, fit);
    if (!wl) continue;
    const int ns = bwd_nseg(fit, ppl, wl, block_cost, ck_table, ck_cap, seg_len);
    if (ns > 1) atomicAdd(&s_b[cost_bucket((uint32_t)seg_len)], (uint32_t)(ns - 1));
    atomicAdd(&s_b[cost_bucket(wl - (uint32_t)(ns - 1) * (uint32_t)seg_len)], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kPlanBuckets; k += blockDim.x)
    if (s_b[k]) atomicAdd(&plan[k], s_b[k]);
}

__global__ void __launch_bounds__(256) k_bwd_plan_place(const uint32_t* __restrict__ block_cost, int32_t n_units,
                                                       int32_t ppl, const uint32_t* __restrict__ ck_table,
                                                       uint32_t ck_cap, int32_t seg_len, const uint32_t* counters,
                                                       uint32_t* plan, uint32_t* units) {
  const bool overflow = counters[C_OVERFLOW] != 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_units; t += gridDim.x * blockDim.x) {
    uint32_t wl, fit[2];
    bwd_unit(t, ppl, block_cost, overflow, wl, fit);
    if (!wl) continue;
    const int ns = bwd_nseg(fit, ppl, wl, block_cost, ck_table, ck_cap, seg_len);
    if (ns > 1) {
      const uint32_t base = atomicAdd(&plan[kPlanBuckets + cost_bucket((uint32_t)seg_len)], (uint32_t)(ns - 1));
      for (int k = 0; k < ns - 1; ++k) units[base + k] = (uint32_t)t | ((uint32_t)k << 25);
    }
    const uint32_t pos =
        atomicAdd(&plan[kPlanBuckets + cost_bucket(wl - (uint32_t)(ns - 1) * (uint32_t)seg_len)], 1u);
    units[pos] = (uint32_t)t | ((uint32_t)(ns - 1) << 25) | (1u << 31);
  }
}

bgs_status launch_bwd_plan(Frame* F, cudaStream_t s) {
  const uint32_t cap = (uint32_t)(F->ck_cap < 0xffffffffll ? F->ck_cap : 0xffffffffll);
  const int ppl = (F->debug_flags & BGS_DEBUG_BWD_8X4) ? 1 : 2;
  const int n_units = 8 / ppl * F->num_tiles;
  const int pgrid = (n_units + 255) / 256 < 2 * num_sms() ? (n_units + 255) / 256 : 2 * num_sms();
  if (cudaMemsetAsync(F->plan, 0, 4 * kPlanWords, s) != cudaSuccess) return check_launch("bwd plan memset");
  k_bwd_plan_count<<<pgrid, 256, 0, s>>>(F->block_cost, n_units, ppl, F->ck_table, cap, F->seg_len, F->counters,
                                         F->plan);
  k_plan_scan<<<1, kPlanBuckets, 0, s>>>(F->plan, F->counters, C_BWD_UNITS, C_BWD_TICKET, -1);
  k_bwd_plan_place<<<pgrid, 256, 0, s>>>(F->block_cost, n_units, ppl, F->ck_table, cap, F->seg_len, F->counters,
                                         F->plan, F->order_bwd);
  note_launch(3);
  const bgs_status st = check_launch("k_bwd_plan");
  F->bwd_planned = st == BGS_OK;
  return st;
}

bgs_status launch_blend_bwd(Frame* F, const float* dL_dimage, const float* final_T, const uint32_t* n_contrib,
                            cudaStream_t s) {
  // 8x8 units (two pixels per lane) unless BGS_DEBUG_BWD_8X4 asks for the 8x4 ones; the work
  // units built ahead by bgs_blend_bwd_plan, else now
  const int ppl = (F->debug_flags & BGS_DEBUG_BWD_8X4) ? 1 : 2;
  if (!F->bwd_planned) {
    const bgs_status st = launch_bwd_plan(F, s);
    if (st != BGS_OK) return st;
  }
  F->bwd_planned = 0;
  // the REDs below accumulate into the slots of this view's visible Gaussians
  F->grad2d_clean = F->grad2d_clean == 1 ? 2 : 0;
  const bool canon = (F->debug_flags & BGS_DEBUG_PARITY_EXP) != 0;
#define BGS_BWD_LAUNCH(P, C)                                                                                    \
  k_render_bwd<P, C><<<bwd_grid<P, C>(), kBwdWarpsPerCta * 32, 0, s>>>(                                         \
      F->ranges, F->vals[F->final_buf], F->record, F->counters, F->cam, F->order_bwd, F->counters + C_BWD_TICKET, \
      dL_dimage, final_T, n_contrib, F->grad2d, F->seg_len, F->ck_table, F->ck_pool)
  if (ppl == 2) {
    if (canon) BGS_BWD_LAUNCH(2, true);
    else BGS_BWD_LAUNCH(2, false);
  } else {
    if (canon) BGS_BWD_LAUNCH(1, true);
    else BGS_BWD_LAUNCH(1, false);
  }
#undef BGS_BWD_LAUNCH
  note_launch();
  return check_launch("k_render_bwd");
}

bgs_status launch_render_bwd(const bgs_gaussians* g, Frame* F, const float* dL_dimage, const float* final_T,
                             const uint32_t* n_contrib, float* grad, cudaStream_t s) {
  bgs_status st = launch_blend_bwd(F, dL_dimage, final_T, n_contrib, s);
  return st != BGS_OK ? st : launch_preprocess_bwd(g, F, grad, s);
}

}  // namespace bgs
