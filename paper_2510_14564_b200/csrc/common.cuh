// common.cuh -- internal declarations shared by libbgs's kernels (NOT shared with oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bgs.h"

namespace bgs {

constexpr int kTile = BGS_TILE;       // 16 x 16 pixel tiles
constexpr int kTilePixels = kTile * kTile;
// Long (tile, 8x4 block) walks are split into list segments of seg_len entries: the forward
// records each block's per-pixel state at every segment boundary b * seg_len (b = 1..kCkMax)
// it crosses, and the backward processes the segments as independent work units.
constexpr int kCkMax = 63;
// default segment length by frame size: a frame with fewer tiles has fewer (tile, block)
// units to spread over the ~3000 resident warps, so its long walks are cut finer (measured,
// bench views/s: T&T-train 980x545, 2170 tiles: 2048 -> 1336, 4096 -> 1317; garden
// 1237x822, 4056 tiles: 2048 -> 384, 4096 -> 391; DB-playroom 4108 tiles: equal)
constexpr int kSegLenSmallFrame = 2048, kSegLenLargeFrame = 4096, kSegLenTilesLarge = 3000;
constexpr int kCkPoolSeg = 2048;
// direct tile split (sort.cu): chunks of 2048..16384 items (a power of two chosen on the
// device from K so that there are >= kChunkTarget chunks: one warp each); per-warp
// shared-memory tile counters
// keys per CTA tile of the onesweep pass (radix.cu): 256 threads x BGS_SORT_ITEMS; the
// look-back status buffers (frame.cu) are sized by it
#ifndef BGS_SORT_ITEMS
#define BGS_SORT_ITEMS 16
#endif
constexpr int kSortTileKeys = 256 * BGS_SORT_ITEMS;
constexpr int kChunkItemsMin = 2048, kChunkItemsMax = 16384, kChunkTarget = 2048;
__host__ __device__ __forceinline__ uint32_t chunk_items_of(uint32_t K) {
  uint32_t c = kChunkItemsMax;
  while (c > (uint32_t)kChunkItemsMin && K / c < (uint32_t)kChunkTarget) c >>= 1;
  return c;
}
// row split (rowsplit.cu): entry chunks of kRsPairChunk (row, rank) pairs; item units of
// unit_items_of(K) items inside one tile row (a power of two in [1024, 8192], >= 2048 units
// when K allows)
constexpr int kRsPairChunk = 4096;
constexpr uint32_t kRsUnitMin = 1024, kRsUnitMax = 8192, kRsUnitTarget = 2048;
__host__ __device__ __forceinline__ uint32_t unit_items_of(uint32_t K) {
  uint32_t c = kRsUnitMax;
  while (c > kRsUnitMin && K / c < kRsUnitTarget) c >>= 1;
  return c;
}
constexpr int kRsMaxTiles = 4096;  // tiles_x, tiles_y bound of the row split (else the radix split)
constexpr int kDirectMaxCells = 12800;  // (tiles_x + 1)(tiles_y + 1) bound  // the checkpoint / state pools are sized for seg_len >= this

// blend work-unit planning (k_*_plan_*): 128 cost buckets (4 per octave, costliest first),
// plan[0..127] counts, plan[128..255] offsets, plan[256] the split-state bump
constexpr int kPlanBuckets = 128, kPlanWords = 2 * kPlanBuckets + 32;

// counters[] slots (u32 words in the workspace)
enum : int {
  C_K_LO = 0, C_K_HI = 1,     // K as u64
  C_OVERFLOW = 2,             // K > max_keys
  C_SCAN_TICKET = 3,          // dynamic tile ids for the decoupled-lookback scan
  C_SORT_TICKET = 4,          // 8 slots: one per radix pass
  C_VISIBLE = 12,
  C_FWD_TICKET = 13,          // work-item tickets of the warp-persistent blend kernels
  C_CK_BUMP = 14,             // checkpoint slots taken by the forward (reset with C_FWD_TICKET)
  C_BWD_TICKET = 15,
  C_SCAN_TOTAL = 16,          // total of a scan that does not define K (depth-first sort)
  C_SORT32_TICKET = 17,       // 8 slots: the depth-first path's 32-bit passes
  C_BWD_UNITS = 25,           // number of backward work units (k_bwd_plan)
  C_FWD_UNITS = 26,           // number of forward work units (k_fwd_plan)
  C_PAIRS = C_SCAN_TOTAL,     // row split: number of (row, rank) entries (the height scan's total)
  C_UNITS = 27,               // row split: number of item units
  C_RS_TICKET = 28,           // row split: tile ticket of the width scan
  C_OVF_STICKY = 31,          // set by any overflow since the last bgs_frame_status (not reset by preprocess)
  C_NUM = 32
};

// clamp bits stored in record word 9 (decisions frozen for the backward, R18)
enum : uint32_t {
  CB_R = 1u, CB_G = 2u, CB_B = 4u, CB_JX = 8u, CB_JX_NEG = 16u, CB_JY = 32u, CB_JY_NEG = 64u
};

// Camera as the kernels see it (derived constants computed once on the host with the
// canonical float expressions of R22: fx = (float)W / (2 tan_fovx), lim = 1.3 tan_fov).
struct Cam {
  float V[16], P[16];
  float campos[3];
  float fx, fy, limx, limy, near_plane;
  float bg[3];
  int32_t W, H, tiles_x, tiles_y;
};

// Library-private frame layout, stored in bgs_frame::opaque.
struct Frame {
  uint64_t magic;
  int64_t n, max_keys;
  int32_t W, H, tiles_x, tiles_y, num_tiles, sort_bits, sort_passes, scan_tiles;
  int64_t sort_tiles_max;
  int32_t cam_valid, final_buf, debug_flags, sort_mode;  // sort_mode: 0 depth-first, 1 onesweep64
  Cam cam;
  int32_t* radius;
  float* depth;
  float4* record;          // [n][3]
  uint32_t* tiles_touched;
  uint2* rect;             // [n] packed tile rect of visible Gaussians
  uint32_t* offsets;
  uint64_t* keys[2];
  uint32_t* vals[2];
  uint2* ranges;
  unsigned long long* scan_status;  // [scan_tiles]
  uint32_t* sort_hist;     // [8][256]
  uint32_t* sort_status;   // [sort_tiles_max][256]
  uint32_t* counters;      // [C_NUM]
  uint32_t* plan;          // [kPlanWords] work-unit planning: bucket counts, offsets, bump
  float4* grad2d;          // [n][3]
  uint32_t* tile_count;    // [num_tiles] keys per tile (from the duplication)
  uint32_t* order_fwd;     // [8 tiles] forward work items (tile << 3 | 8x4 block), longest first
  uint32_t* order_bwd;     // [8 tiles] backward work items, longest first
  uint32_t* block_cost;    // [8 tiles] each block's largest n_contrib in the last forward
  int32_t have_cost, seg_len;  // block_cost holds this frame's previous forward; list segment length
  int32_t fwd_planned, bwd_planned;  // the next fwd's / bwd's work units are already built (plan-ahead)
  // grad2d state of a consuming frame: 0 unknown (some slots may be non-zero), 1 all zero,
  // 2 non-zero only in the slots of the last preprocess's visible Gaussians (one backward)
  int32_t grad2d_clean;
  int32_t consume_g2;    // bgs_frame_set_consume: the chain rule zeroes the blend gradients it reads
  int32_t counters_init;   // the sticky overflow word has been zeroed (first preprocess)
  uint32_t* ck_table;      // [8 tiles][kCkMax] pool slot of boundary b = 1..kCkMax of each block's walk
  float4* ck_pool;         // [ck_cap][32 lanes] {T, colour behind r, g, b} at a boundary
  int64_t ck_cap;          // slots of ck_pool, and of spec_state / spec_last
  uint32_t* spec_base;     // [8 tiles] forward split: first state slot of the item's segments
  uint32_t* spec_n;        // [8 tiles] forward split: number of segments (1 = not split)
  uint32_t* arrive;        // [8 tiles] forward split: segments finished
  float4* spec_state;      // [ck_cap][32] per-segment {T or prod(1 - alpha), C rgb}
  uint32_t* spec_last;     // [ck_cap][32] per-segment last | stopped << 31
  uint32_t* chunk_cnt;     // [max_keys / 16384][tiles] direct tile split (null when the grid is too large)
  // depth-first sort path (sort.cu): Gaussians stable-sorted by depth bits, then the
  // rank-ordered tile items stable-split by tile -- the same order as the 64-bit sort
  uint32_t* dkey[2];       // [n] depth bits (0xffffffff for culled)
  uint32_t* dval[2];       // [n] Gaussian index; dval[0] = depth order after 4 passes
  uint32_t* rank_cnt;      // [n] tiles_touched in depth order
  uint32_t* item_off;      // [n] exclusive scan of rank_cnt
  uint2* rank_rect;        // [n] packed tile rect per depth rank
  uint8_t* cbits;          // [n] frozen clamp decisions (rgb / J) for the backward (R18)
  const uint8_t* keep;     // [n] NEXT-4 keep mask (device, caller-owned) or null: keep[i] == 0 culls i
  // row split (rowsplit.cu)
  uint32_t* rank_h;        // [n] tile rows of each depth rank's rect
  uint32_t* rs_tabA;       // [rs_max_chunks][tiles_y] entry counts, then offsets, per (pair chunk, row)
  uint32_t* rs_chunk_r0;   // [rs_max_chunks] first rank of each pair chunk
  uint32_t* rs_rows;       // [3 tiles_y + 2] row entry totals, row entry starts, row unit starts
  uint4* rs_units;         // [rs_max_units] {row, first item, end item, first entry}
  uint32_t* rs_tabB;       // [rs_max_units][tiles_x] item counts, then offsets, per (unit, x)
  unsigned long long* rs_status;  // [rs_scan_tiles] look-back words of the width scan
  int64_t rs_max_units, rs_scan_tiles;
};
static_assert(sizeof(Frame) <= sizeof(bgs_frame), "Frame must fit in bgs_frame::opaque");
constexpr uint64_t kFrameMagic = 0xB6500F7A3E5ull;

inline Frame* frame_of(bgs_frame* f) { return reinterpret_cast<Frame*>(f->opaque); }
inline const Frame* frame_of(const bgs_frame* f) { return reinterpret_cast<const Frame*>(f->opaque); }

// launch bookkeeping (frame.cu)
void note_launch(int k = 1);
bgs_status check_launch(const char* what);
void set_error(const char* msg);

// stage launchers (one .cu each)
bgs_status launch_preprocess(const bgs_gaussians* g, Frame* F, cudaStream_t s);
bgs_status launch_preprocess_batch(const bgs_gaussians* g, Frame* const* F, int nviews, cudaStream_t s);
bgs_status launch_sort(Frame* F, cudaStream_t s);
bgs_status launch_render_fwd(Frame* F, float* image, float* final_T, uint32_t* n_contrib, cudaStream_t s);
bgs_status launch_blend_bwd(Frame* F, const float* dL_dimage, const float* final_T, const uint32_t* n_contrib,
                            cudaStream_t s);
bgs_status launch_preprocess_bwd(const bgs_gaussians* g, Frame* F, float* grad, cudaStream_t s);
constexpr int kPreMaxViews = 16;     // views per k_preprocess launch (kernel-parameter cameras)
constexpr int kPreBwdMaxViews = 16;  // views per k_preprocess_bwd launch (kernel-parameter cameras)
bgs_status launch_preprocess_bwd_batch(const bgs_gaussians* g, Frame* const* frames, int nviews, float* grad,
                                       cudaStream_t s);
bgs_status launch_preprocess_bwd_batch_impl(const bgs_gaussians* g, Frame* const* frames, int nviews, float* grad,
                                            float* theta, float* m, float* v, const bgs_adam_hparams* hp,
                                            int64_t step, cudaStream_t s, int64_t i0 = 0, int64_t i1 = -1,
                                            bool assign = false);
bgs_status launch_render_bwd(const bgs_gaussians* g, Frame* F, const float* dL_dimage, const float* final_T,
                             const uint32_t* n_contrib, float* grad, cudaStream_t s);
bgs_status launch_adam(float* theta, float* grad, float* m, float* v, int64_t n, int64_t begin, int64_t count,
                       const bgs_adam_hparams* hp, int64_t step, cudaStream_t s, bool zero_grad = true);
bgs_status launch_l1(const float* image, const uint8_t* target, int32_t w, int32_t h, float scale, float* dl,
                     float* loss_sum, cudaStream_t s);
size_t loss_workspace_bytes(int32_t w, int32_t h);
bgs_status launch_l1_dssim(const float* image, const uint8_t* target, int32_t w, int32_t h, float lam, float scale,
                           float* dl, float* loss_sum, void* workspace, cudaStream_t s);
bgs_status launch_fwd_plan(Frame* F, cudaStream_t s);
bgs_status launch_bwd_plan(Frame* F, cudaStream_t s);
bgs_status launch_validate(const Frame* F, unsigned long long* out, cudaStream_t s);
bgs_status launch_stats(const Frame* F, const uint32_t* n_contrib, bgs_stats* out, cudaStream_t s);

int num_sms();
int sort_pass_grid();
bgs_status launch_sort_pass(const uint64_t* kin, const uint32_t* vin, uint64_t* kout, uint32_t* vout,
                            const uint32_t* hist, uint32_t* status, uint32_t* ticket, const uint32_t* counters,
                            int shift, cudaStream_t s);
bgs_status launch_sort_pass32(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                              const uint32_t* hist, uint32_t* status, uint32_t* ticket, const uint32_t* counters,
                              int shift, int64_t count, cudaStream_t s, const uint2* rect = nullptr,
                              uint32_t* rank_cnt = nullptr, uint2* rank_rect = nullptr,
                              uint32_t* rank_h = nullptr, bool drop_culled = false, int64_t fill_to = 0,
                              const uint32_t* gen_tt = nullptr);
bgs_status launch_scan(const uint32_t* in, uint32_t* out, int64_t n, Frame* F, bool publish_k, cudaStream_t s);
bgs_status launch_rowsplit(Frame* F, cudaStream_t s);
bgs_status launch_adam_multimem(float* theta, float* theta_mc, float* grad_mc, float* m, float* v, int64_t n,
                                int64_t begin, int64_t count, const bgs_adam_hparams* hp, int64_t step,
                                cudaStream_t s);
bgs_status launch_tile_scan(Frame* F, cudaStream_t s);

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ float fast_exp(float x) {
  // ex2.approx of x*log2(e): MUFU.EX2; differs from a correctly rounded exp by a few
  // ulp, which only moves decisions inside the R23 near-tie margins.
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
  return y;
}

// MUFU.RCP alone (rcp.approx: ~1 ulp; __fdividef(1, x) adds a multiply by the numerator)
__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The parity mode's exponential (BGS_DEBUG_PARITY_EXP; R23): a fixed expression tree that
// the oracle evaluates identically (oracle/bgs_oracle.cpp, canon_exp), so alpha -- and every
// blend decision -- is bit-identical on both sides: 2^x with x = power * log2(e) (one float
// multiply), x = n + f (n = floor x, f exact), 2^f by the degree-8 Taylor polynomial of
// e^(f ln 2) in Horner form with fmaf, scaled by 2^n exactly (ldexpf).  Relative error vs
// exp <= 1.5e-6 (mostly the rounding of x), inside the pre-skip and culling margins.
__device__ __forceinline__ float canon_exp(float power) {
  const float x = power * 1.4426950408889634f;
  const float n = floorf(x);
  const float f = x - n;
  float p = 1.3215487e-6f;
  p = fmaf(p, f, 1.5252734e-5f);
  p = fmaf(p, f, 1.5403530e-4f);
  p = fmaf(p, f, 1.3333558e-3f);
  p = fmaf(p, f, 9.6181291e-3f);
  p = fmaf(p, f, 5.5504109e-2f);
  p = fmaf(p, f, 2.4022651e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.0f);
  return ldexpf(p, (int)n);
}

// look-back status words: relaxed, GPU-scope (L2-coherent; no .sys-scope round trip).  A
// status word carries its own flag bits, so no ordering with other data is needed.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async (LDGSTS): global -> shared copies that bypass the registers; completion per
// thread by commit groups
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Exact-up-to-margin cull of one list entry against an 8x4 pixel block: can any pixel
// centre p of [bx0, bx1] x [by0, by1] reach power(p - mu) = A dx^2 + B dx dy + C dy^2 >= thr
// (the alpha >= 1/255 level set, thr = pthr)?  The power is concave, so its maximum over
// the rectangle is at mu when mu is inside, else on the edge(s) facing mu, where it is a
// clamped 1-D vertex.  The margin covers the float error of both this bound and the
// blend's own per-pixel power (each <= 2^-22 of the terms' magnitude), so no entry the
// blend would evaluate as power >= thr is ever dropped.
__device__ __forceinline__ bool ellipse_hits_block(float mx, float my, float A, float B, float C, float thr,
                                                   float bx0, float by0, float bx1, float by1) {
  const float lx = bx0 - mx, hx = bx1 - mx, ly = by0 - my, hy = by1 - my;
  const bool in_x = lx <= 0.0f && hx >= 0.0f, in_y = ly <= 0.0f && hy >= 0.0f;
  if (in_x && in_y) return true;
  float best = -3.0e38f;
  if (!in_x) {
    const float dx = lx > 0.0f ? lx : hx;
    const float dy = fminf(fmaxf(__fdividef(-B * dx, 2.0f * C), ly), hy);
    best = fmaxf(best, A * dx * dx + B * dx * dy + C * dy * dy);
  }
  if (!in_y) {
    const float dy = ly > 0.0f ? ly : hy;
    const float dx = fminf(fmaxf(__fdividef(-B * dy, 2.0f * A), lx), hx);
    best = fmaxf(best, A * dx * dx + B * dx * dy + C * dy * dy);
  }
  const float ex = fmaxf(-lx, hx), ey = fmaxf(-ly, hy);
  const float margin = 1e-3f + 1e-5f * (fabsf(A) * ex * ex + fabsf(C) * ey * ey);
  return best >= thr - margin;
}

// Cheaper conservative form of the same test: the power is a negative-definite quadratic
// q, so over the block (centre c, half-extents hx, hy) q(mu - p) = q(d_c) - grad q(d_c) . e
// + q(e) <= q(d_c) + hx |dq/dx| + hy |dq/dy| (q(e) <= 0).  When even that bound is below
// thr (with the same rounding margin), no pixel of the block reaches the level set.
__device__ __forceinline__ bool bound_hits_block(float mx, float my, float A, float B, float C, float thr,
                                                 float cx, float cy, float hx, float hy) {
  const float dx = mx - cx, dy = my - cy;
  const float gx = fmaf(2.0f * A, dx, B * dy), gy = fmaf(2.0f * C, dy, B * dx);
  const float q = fmaf(A, dx * dx, fmaf(C, dy * dy, B * (dx * dy)));
  const float bound = fmaf(hx, fabsf(gx), fmaf(hy, fabsf(gy), q));
  const float ex = fabsf(dx) + hx, ey = fabsf(dy) + hy;
  const float margin = 1e-3f + 2e-5f * (fabsf(A) * ex * ex + fabsf(C) * ey * ey);
  return bound >= thr - margin;
}

// work-unit ordering: bucket of a cost, 4 buckets per octave, costliest first (0..127)
__device__ __forceinline__ int cost_bucket(uint32_t cost) {
  const int b = (int)(__float_as_uint((float)cost + 1.0f) >> 21) - (127 << 2);  // 4 log2(cost + 1)
  return 127 - (b < 127 ? b : 127);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace bgs
