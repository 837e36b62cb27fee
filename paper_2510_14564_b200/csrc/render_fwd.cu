// render_fwd.cu -- a7: front-to-back alpha blend (§II-A l.143-149):
//   C = sum_{i in N} c_i alpha_i prod_{j<i} (1 - alpha_j),  N = the tile's depth-sorted list,
// with readings R14 (skip power > 0; alpha = min(0.99, o G); skip alpha < 1/255),
// R15 (stop before T (1 - alpha) < 1e-4, the crossing Gaussian is not blended),
// R16 (out = C + T_final bg; n_contrib = 1-based position of the last blended entry).
// Decision-bearing arithmetic is the canonical tree of R22 (explicit fmaf, file built
// with --fmad=false); G uses MUFU.EX2 (R23 near-tie rule covers the few-ulp difference).
//
// Workload-balanced mapping (the paper's Challenge-2: with one thread
// per pixel walking a tile in lock-step, the slowest pixels and longest tiles set the
// pace): the unit of work is one warp x one 8x4 pixel block of a tile (one pixel per
// lane).  A persistent grid of independent warps pulls these (tile, block) items from a
// global ticket, longest first (by this frame's previous per-block walk lengths when it
// re-renders a view, else by tile list length), so no
// warp waits on another and a warp leaves its tile as soon as its own 32 pixels are done.
// A warp streams its tile's list 32 entries per step: each lane gathers one entry's
// 16-byte cull record {x, y, ex, ey} and tests the conservative alpha >= 1/255 box against
// the block; the hits (about a fifth of the list on the garden workload) are compacted
// with a ballot and their 48-byte records {x,y,ex,ey | A,B,C,o | r,g,b,pthr} staged in the
// warp's slice of shared memory -- the B200 form of the paper's T3 batch loading of
// per-Gaussian contiguous RGB.  The step loop is
// software-pipelined (ids three steps ahead, cull records two, hit records one), so the
// gathers overlap the walk.  List positions are kept, so n_contrib and every decision
// are those of the plain per-pixel walk.
//
// Long walks are split (the tail of the longest items otherwise sets the kernel's length):
// when the frame re-renders its view, k_fwd_plan splits every item whose previous walk
// exceeded 2 seg_len into list segments [k seg_len, (k + 1) seg_len).  Segment 0 walks
// exactly; segments k >= 1 walk speculatively from T = 1 (the blend is a product, so each
// yields {prod (1 - alpha), sum c alpha T_local, last}, and a local stop T_local (1 - alpha)
// < 1e-4 implies the global one).  The last warp to finish an item merges the segments in
// order -- C += T C_k, T *= P_k -- and re-walks exactly the segment in which a pixel stops
// (T P_k < 1e-4 or a local stop), then continues exactly past the last segment.  Decisions
// equal the plain walk's except where T's rounding order moves a T (1 - alpha) = 1e-4
// comparison, i.e. inside the R23 near-tie margin.  Every exact walk records each pixel's
// {T, C} at the segment boundaries for the backward (k_render_bwd's segment split).
#include "common.cuh"

namespace bgs {

#ifndef BGS_FWD_CULL
#define BGS_FWD_CULL 0
#endif
constexpr int kFwdWarps = 4;
// a hinted forward splits a walk into speculative segments when its hinted length exceeds
// this many segment lengths
#ifndef BGS_FWD_SPLIT_MUL
#define BGS_FWD_SPLIT_MUL 4
#endif
// The forward keeps a one-CTA planner: it places a tile's eight blocks next to each other
// inside their cost bucket, and the tile list they share stays hot in L2 (a grid-wide
// planner with atomics per bucket scattered them: forward 13.6 -> 14.0 ms per step).
constexpr int kFwdPlanThreads = 1024, kFwdPlanBuckets = 128;

__device__ __forceinline__ bool box_hits_f(const float4 a, float bx0, float by0, float bx1, float by1) {
  return a.x + a.z >= bx0 && a.x - a.z <= bx1 && a.y + a.w >= by0 && a.y - a.w <= by1;
}

struct FwdArgs {
  const uint2* ranges;
  const uint32_t* values;
  const float4* record;
  const uint32_t* counters;
  const uint32_t* units;     // (tile << 3 | block) | segment << 25 | split << 31
  uint32_t* ticket;
  float* image;
  float* final_T;
  uint32_t* n_contrib;
  uint32_t* block_cost;
  int32_t seg_len;
  uint32_t ck_cap;
  uint32_t* ck_bump;
  uint32_t* ck_table;
  float4* ck_pool;
  const uint32_t* spec_base;  // first state slot of a split item (segment k -> slot base + k)
  const uint32_t* spec_n;     // segments of a split item
  uint32_t* arrive;           // segments of a split item finished so far
  float4* spec_state;         // [slot][32] {T or prod(1 - alpha), C rgb}
  uint32_t* spec_last;        // [slot][32] last | stopped << 31
};

template <bool CANON>
__global__ void __launch_bounds__(kFwdWarps * 32) k_render_fwd(const FwdArgs a, const Cam cam) {
  __shared__ float4 s_rec[kFwdWarps][3][32];
  __shared__ uint32_t s_pos[kFwdWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const bool overflow = a.counters[C_OVERFLOW] != 0;
  const uint32_t n_units = a.counters[C_FWD_UNITS];
  const int seg_steps = a.seg_len / 32;
  float4* sr0 = s_rec[warp][0];
  float4* sr1 = s_rec[warp][1];
  float4* sr2 = s_rec[warp][2];
  uint32_t* spos = s_pos[warp];
  const float4 none = make_float4(-1e30f, -1e30f, -1e30f, -1e30f);
  while (true) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(a.ticket, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= n_units) break;
    const uint32_t code = a.units[u];
    const uint32_t it = code & ((1u << 25) - 1u);
    const int seg = (int)((code >> 25) & 63u);
    const bool split = (code >> 31) != 0;
    const int nseg = split ? (int)a.spec_n[it] : 1;
    const uint32_t sbase = split ? a.spec_base[it] : 0u;
    const int tile = (int)(it >> 3), blk = (int)(it & 7);
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int bx = tx * kTile + (blk & 1) * 8, by = ty * kTile + (blk >> 1) * 4;
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    const float bx0 = (float)bx, by0 = (float)by, bx1 = bx0 + 7.0f, by1 = by0 + 3.0f;
    const bool inside = px < cam.W && py < cam.H;
    const float pxf = (float)px, pyf = (float)py;
    uint2 rg = a.ranges[tile];
    if (overflow) rg = make_uint2(0, 0);
    const int len = (int)(rg.y - rg.x);
    const int nst_all = (len + 31) / 32;
    bool done = !inside;
    float T = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f;
    uint32_t last = 0;
    int nck = 0;  // segment boundaries recorded for this item
    // record every lane's {T, C} at boundary nck + 1 (state before list position (nck + 1) seg_len)
    auto record_ck = [&]() {
      uint32_t slot = 0;
      if (lane == 0) slot = atomicAdd(a.ck_bump, 1u);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (slot < a.ck_cap) a.ck_pool[(size_t)slot * 32 + lane] = make_float4(T, Cr, Cg, Cb);
      if (lane == 0) a.ck_table[(size_t)it * kCkMax + nck] = slot < a.ck_cap ? slot : 0xffffffffu;
      ++nck;
    };
    // the phase to walk: steps [s_lo, s_hi); `exact` walks record boundaries
    int s_lo = split ? seg * seg_steps : 0;
    int s_hi = split ? min(nst_all, (seg + 1) * seg_steps) : nst_all;
    bool exact = !split || seg == 0;
    bool combining = false, rewalking = false, emit = true, rw = false;
    int mk = 1;
    float sT = 0.f, sR = 0.f, sG = 0.f, sB = 0.f;
    uint32_t sLast = 0;
    bool sDone = false;
    while (true) {
      if (s_lo < s_hi && !__all_sync(0xffffffffu, done)) {
        auto load_id = [&](int s) -> uint32_t {
          const int p = 32 * s + lane;
          return (s < s_hi && p < len) ? __ldg(a.values + rg.x + (uint32_t)p) : 0xffffffffu;
        };
        auto load_cull = [&](uint32_t id) { return id != 0xffffffffu ? __ldg(a.record + 3 * id) : none; };
        // pipeline prologue: step s_lo fully, s_lo + 1 cull record, s_lo + 2 id
        uint32_t id_c = load_id(s_lo);
        float4 a_c = load_cull(id_c);
        uint32_t id_n = load_id(s_lo + 1);
        float4 a_n = load_cull(id_n);
        uint32_t id_nn = load_id(s_lo + 2);
        bool h_c = box_hits_f(a_c, bx0, by0, bx1, by1);
        float4 r1_c, r2_c;  // loaded (and read) only for a hit
        if (h_c) {
          r1_c = __ldg(a.record + 3 * id_c + 1);
          r2_c = __ldg(a.record + 3 * id_c + 2);
        }
        // the next segment boundary this (exact) walk records, or -1
        int ck_step = (exact && nck < kCkMax) ? (nck + 1) * seg_steps : -1;
        for (int s = s_lo; s < s_hi; ++s) {
          // (0) segment boundary: record {T, C} before it
          if (s == ck_step) {
            record_ck();
            ck_step = nck < kCkMax ? (nck + 1) * seg_steps : -1;
          }
          // (1) commit step s into the warp's shared-memory slice
#if BGS_FWD_CULL == 1
          if (h_c) h_c = ellipse_hits_block(a_c.x, a_c.y, r1_c.x, r1_c.y, r1_c.z, r2_c.w, bx0, by0, bx1, by1);
#elif BGS_FWD_CULL == 2
          if (h_c) h_c = bound_hits_block(a_c.x, a_c.y, r1_c.x, r1_c.y, r1_c.z, r2_c.w, bx0 + 3.5f, by0 + 1.5f, 3.5f, 1.5f);
#endif
          const uint32_t bal = __ballot_sync(0xffffffffu, h_c);
          if (h_c) {
            const int q = __popc(bal & lt);
            sr0[q] = a_c;
            sr1[q] = r1_c;
            sr2[q] = r2_c;
            spos[q] = (uint32_t)(32 * s + lane);
          }
          __syncwarp();
          // (2) step s+1 hit test and records; (3) step s+2 cull record, step s+3 id
          const bool h_n = box_hits_f(a_n, bx0, by0, bx1, by1);
          float4 r1_n, r2_n;
          if (h_n) {
            r1_n = __ldg(a.record + 3 * id_n + 1);
            r2_n = __ldg(a.record + 3 * id_n + 2);
          }
          const float4 a_nn = load_cull(id_nn);
          const uint32_t id_nnn = load_id(s + 3);
          // (4) walk step s.  A finished pixel skips every entry through doff = -inf (power +
          // doff < pthr), so one compare pair carries "done", R14's power > 0 guard and the
          // exact alpha < 1/255 bound (pthr, preprocess; it skips the MUFU path)
          const int m = __popc(bal);
          int lastk = -1;
          float doff = done ? -INFINITY : 0.0f;
          for (int k = 0; k < m; ++k) {
            const float4 r0 = sr0[k];
            const float4 r1 = sr1[k];
            const float4 r2 = sr2[k];
            const float dx = r0.x - pxf, dy = r0.y - pyf;
            const float power = fmaf(r1.x, dx * dx, fmaf(r1.z, dy * dy, r1.y * (dx * dy)));
            if ((power > 0.0f) | (power + doff < r2.w)) continue;
            const float alpha = fminf(0.99f, r1.w * (CANON ? canon_exp(power) : fast_exp(power)));
            if (alpha < (1.0f / 255.0f)) continue;
            const float tT = T * (1.0f - alpha);
            if (tT < 1e-4f) {
              doff = -INFINITY;
              continue;
            }
            const float w = alpha * T;
            Cr = fmaf(r2.x, w, Cr);
            Cg = fmaf(r2.y, w, Cg);
            Cb = fmaf(r2.z, w, Cb);
            T = tT;
            lastk = k;
          }
          done = doff < 0.0f;
          if (lastk >= 0) last = spos[lastk] + 1u;
          __syncwarp();
          if (__all_sync(0xffffffffu, done)) break;
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
      if (rewalking) {  // lanes that sat the re-walk out get their state back
        if (!rw) {
          T = sT;
          Cr = sR;
          Cg = sG;
          Cb = sB;
          last = sLast;
          done = sDone;
        }
        rewalking = false;
      }
      if (!split) break;
      if (!combining) {
        // publish this segment's result; the last of the item's segments merges them
        const size_t slot = (size_t)(sbase + seg) * 32 + lane;
        a.spec_state[slot] = make_float4(T, Cr, Cg, Cb);
        a.spec_last[slot] = last | (done ? 0x80000000u : 0u);
        __threadfence();
        __syncwarp();
        uint32_t old = 0;
        if (lane == 0) old = atomicAdd(a.arrive + it, 1u);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old != (uint32_t)nseg - 1u) {
          emit = false;
          break;
        }
        __threadfence();
        combining = true;
        const float4 h = __ldcg(a.spec_state + (size_t)sbase * 32 + lane);
        const uint32_t hl = __ldcg(a.spec_last + (size_t)sbase * 32 + lane);
        T = h.x;
        Cr = h.y;
        Cg = h.z;
        Cb = h.w;
        last = hl & 0x7fffffffu;
        done = (hl >> 31) != 0;
        nck = 0;
        mk = 1;
      } else if (mk > nseg) {
        break;  // the exact continuation past the last segment is done
      }
      // merge the speculative segments mk, mk + 1, ... in list order
      bool need = false;
      while (mk < nseg) {
        if (__all_sync(0xffffffffu, done)) {
          mk = nseg;
          break;
        }
        if (nck == mk - 1 && nck < kCkMax) record_ck();  // exact state at boundary mk
        const size_t slot = (size_t)(sbase + mk) * 32 + lane;
        const float4 p = __ldcg(a.spec_state + slot);
        const uint32_t pl = __ldcg(a.spec_last + slot);
        rw = !done && ((pl >> 31) != 0 || T * p.x < 1e-4f);
        if (!done && !rw) {
          Cr = fmaf(T, p.y, Cr);
          Cg = fmaf(T, p.z, Cg);
          Cb = fmaf(T, p.w, Cb);
          T = T * p.x;
          if (pl & 0x7fffffffu) last = pl & 0x7fffffffu;
        }
        ++mk;
        if (__any_sync(0xffffffffu, rw)) {
          need = true;
          break;
        }
      }
      if (need) {
        // the pixels that stop inside segment mk - 1 re-walk it exactly
        sT = T;
        sR = Cr;
        sG = Cg;
        sB = Cb;
        sLast = last;
        sDone = done;
        if (!rw) done = true;
        rewalking = true;
        s_lo = (mk - 1) * seg_steps;
        s_hi = min(nst_all, mk * seg_steps);
        exact = false;
        continue;
      }
      // all segments merged: continue exactly past the last one (records boundary nseg on
      // its first step)
      s_lo = nseg * seg_steps;
      s_hi = nst_all;
      exact = true;
      mk = nseg + 1;
    }
    if (!emit) continue;
    const float outr = fmaf(T, cam.bg[0], Cr), outg = fmaf(T, cam.bg[1], Cg), outb = fmaf(T, cam.bg[2], Cb);
    if (inside) {
      const int64_t pix = (int64_t)py * cam.W + px;
      const int64_t plane = (int64_t)cam.W * cam.H;
      a.image[pix] = outr;
      a.image[plane + pix] = outg;
      a.image[2 * plane + pix] = outb;
      a.final_T[pix] = T;
      a.n_contrib[pix] = last;
    }
    // the block's largest n_contrib: the backward's (and this frame's next forward's) cost
    const uint32_t wl = __reduce_max_sync(0xffffffffu, last);
    if (lane == 0) a.block_cost[it] = wl;
    // checkpoints hold {T, colour behind the boundary} = {T_b, out - C_b} for the backward
    for (int b = 0; b < nck; ++b) {
      const uint32_t slot = a.ck_table[(size_t)it * kCkMax + b];
      if (slot < a.ck_cap) {
        float4* c = a.ck_pool + (size_t)slot * 32 + lane;
        const float4 v = *c;
        *c = make_float4(v.x, outr - v.y, outg - v.z, outb - v.w);
      }
    }
  }
}

// Forward work units, longest first.  With this frame's previous per-block walk lengths
// (the same view re-rendered), an item that walked more than 2 seg_len entries becomes
// ceil(walk / seg_len) segment units (at most kCkMax + 1, as the state pool allows);
// without them, items are ordered by their tile's list length.  One CTA; it also resets
// the forward's counters.
__global__ void __launch_bounds__(kFwdPlanThreads) k_fwd_plan(const uint32_t* __restrict__ cost, int32_t shift,
                                                             int32_t hinted, int32_t n_items, int32_t seg_len,
                                                             uint32_t cap, uint32_t* counters, uint32_t* units,
                                                             uint32_t* spec_base, uint32_t* spec_n,
                                                             uint32_t* arrive) {
  __shared__ uint32_t s_b[kFwdPlanBuckets];
  __shared__ uint32_t s_bump;
  for (int k = threadIdx.x; k < kFwdPlanBuckets; k += blockDim.x) s_b[k] = 0;
  if (threadIdx.x == 0) {
    s_bump = 0;
    counters[C_FWD_TICKET] = 0;
    counters[C_CK_BUMP] = 0;
  }
  __syncthreads();
  const bool overflow = counters[C_OVERFLOW] != 0;
  const int seg_b = cost_bucket((uint32_t)seg_len);
  // kPlanPF items per thread per round, their loads issued together: one global round trip
  // per round instead of one per item (a lone CTA is latency-bound)
  constexpr int kPlanPF = 8;
  const int stride = kPlanPF * blockDim.x;
  for (int t0 = 0; t0 < n_items; t0 += stride) {
    uint32_t hq[kPlanPF];
#pragma unroll
    for (int q = 0; q < kPlanPF; ++q) {
      const int t = t0 + q * blockDim.x + threadIdx.x;
      hq[q] = (t < n_items && !overflow) ? cost[t >> shift] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kPlanPF; ++q) {
      const int t = t0 + q * blockDim.x + threadIdx.x;
      if (t >= n_items) continue;
      const uint32_t h = hq[q];
      uint32_t ns = 1, base = 0;
      if (hinted && h > (uint32_t)BGS_FWD_SPLIT_MUL * (uint32_t)seg_len) {
        ns = min((h + (uint32_t)seg_len - 1u) / (uint32_t)seg_len, (uint32_t)kCkMax + 1u);
        base = atomicAdd(&s_bump, ns);
        if (base + ns > cap) ns = 1;
      }
      spec_base[t] = base;
      spec_n[t] = ns;
      arrive[t] = 0;
      atomicAdd(&s_b[ns > 1 ? seg_b : cost_bucket(h)], ns);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int b = 0; b < kFwdPlanBuckets; ++b) {
      const uint32_t c = s_b[b];
      s_b[b] = run;
      run += c;
    }
    counters[C_FWD_UNITS] = run;
  }
  __syncthreads();
  for (int t0 = 0; t0 < n_items; t0 += stride) {
    uint32_t nq[kPlanPF], hq[kPlanPF];
#pragma unroll
    for (int q = 0; q < kPlanPF; ++q) {
      const int t = t0 + q * blockDim.x + threadIdx.x;
      nq[q] = t < n_items ? spec_n[t] : 0u;
      hq[q] = (t < n_items && !overflow) ? cost[t >> shift] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kPlanPF; ++q) {
      const int t = t0 + q * blockDim.x + threadIdx.x;
      if (t >= n_items) continue;
      const uint32_t ns = nq[q];
      const uint32_t pos = atomicAdd(&s_b[ns > 1 ? seg_b : cost_bucket(hq[q])], ns);
      if (ns > 1)
        for (uint32_t k = 0; k < ns; ++k) units[pos + k] = (uint32_t)t | (k << 25) | (1u << 31);
      else
        units[pos] = (uint32_t)t;
    }
  }
}

// (the backward's planner, render_bwd.cu, uses this scan of its bucket counts)
// exclusive scan of the bucket counts into plan[128..]; the unit count and the tickets
__global__ void __launch_bounds__(kPlanBuckets) k_plan_scan(uint32_t* plan, uint32_t* counters, int units_slot,
                                                           int reset0, int reset1) {
  __shared__ uint32_t s_w[kPlanBuckets / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t x = plan[t];
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  uint32_t base = 0;
  for (int k = 0; k < w; ++k) base += s_w[k];
  plan[kPlanBuckets + t] = base + inc - x;
  if (t == kPlanBuckets - 1) {
    counters[units_slot] = base + inc;
    counters[reset0] = 0;
    if (reset1 >= 0) counters[reset1] = 0;
  }
}

static int fwd_grid() {
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_fwd<false>, kFwdWarps * 32, 0);
    grid = (per_sm < 1 ? 1 : per_sm) * num_sms();
  }
  return grid;
}

bgs_status launch_fwd_plan(Frame* F, cudaStream_t s) {
  const int n_items = 8 * F->num_tiles;
  const uint32_t cap = (uint32_t)(F->ck_cap < 0xffffffffll ? F->ck_cap : 0xffffffffll);
  // parity mode: no speculative segments (their merges re-associate T, R23)
  const bool parity = (F->debug_flags & BGS_DEBUG_PARITY_EXP) != 0;
  const bool hinted = F->have_cost != 0 && !parity;
  k_fwd_plan<<<1, kFwdPlanThreads, 0, s>>>(hinted ? F->block_cost : F->tile_count, hinted ? 0 : 3, hinted ? 1 : 0,
                                           n_items, F->seg_len, cap, F->counters, F->order_fwd, F->spec_base,
                                           F->spec_n, F->arrive);
  note_launch();
  bgs_status st = check_launch("k_fwd_plan");
  F->fwd_planned = st == BGS_OK;
  return st;
}

bgs_status launch_render_fwd(Frame* F, float* image, float* final_T, uint32_t* n_contrib, cudaStream_t s) {
  // the work units: built ahead by bgs_render_fwd_plan, else now
  if (!F->fwd_planned) {
    const bgs_status st = launch_fwd_plan(F, s);
    if (st != BGS_OK) return st;
  }
  F->fwd_planned = 0;
  F->bwd_planned = 0;  // a new forward: the backward's plan follows it
  const uint32_t cap = (uint32_t)(F->ck_cap < 0xffffffffll ? F->ck_cap : 0xffffffffll);
  const bool parity = (F->debug_flags & BGS_DEBUG_PARITY_EXP) != 0;
  FwdArgs a;
  a.ranges = F->ranges;
  a.values = F->vals[F->final_buf];
  a.record = F->record;
  a.counters = F->counters;
  a.units = F->order_fwd;
  a.ticket = F->counters + C_FWD_TICKET;
  a.image = image;
  a.final_T = final_T;
  a.n_contrib = n_contrib;
  a.block_cost = F->block_cost;
  a.seg_len = F->seg_len;
  a.ck_cap = cap;
  a.ck_bump = F->counters + C_CK_BUMP;
  a.ck_table = F->ck_table;
  a.ck_pool = F->ck_pool;
  a.spec_base = F->spec_base;
  a.spec_n = F->spec_n;
  a.arrive = F->arrive;
  a.spec_state = F->spec_state;
  a.spec_last = F->spec_last;
  if (parity) k_render_fwd<true><<<fwd_grid(), kFwdWarps * 32, 0, s>>>(a, F->cam);
  else k_render_fwd<false><<<fwd_grid(), kFwdWarps * 32, 0, s>>>(a, F->cam);
  note_launch();
  F->have_cost = 1;
  return check_launch("k_render_fwd");
}

}  // namespace bgs
