/* bgs.h -- C ABI of libbgs: the BalanceGS (arXiv 2510.14564) hot path on B200.
 *
 * The path is the 3DGS differentiable tile rasterizer that the paper's system
 * and mapping techniques accelerate ("Gaussian projection ...
 * color splatting", §II-A l.128-149), one training iteration per view:
 *
 *   theta[59n] + camera -> bgs_preprocess -> bgs_sort -> bgs_render_fwd
 *        -> (dL/dimage from the caller, e.g. bgs_l1_loss_grad)
 *        -> bgs_render_bwd (grad += ) -> [caller: NCCL all-reduce] -> bgs_adam_step
 *
 * Conventions (DESIGN.md §3 lists every reading R1-R27 cited below):
 *  - Every pointer is a DEVICE pointer unless marked (host).  Every call that
 *    takes a stream is asynchronous on it; no call allocates, frees or
 *    synchronises, except bgs_frame_status / bgs_frame_stats, which read a few
 *    device words back and must be called after the caller synchronised.
 *  - Ownership: the caller owns theta, grad, exp_avg, exp_avg_sq, images and
 *    the workspace; the library keeps no global device state.  A bgs_frame is a
 *    caller-allocated HOST struct describing one view's workspace.
 *  - Errors: host-side validation happens before any launch; an invalid call
 *    returns BGS_ERR_INVALID and launches nothing.  A CUDA launch error returns
 *    BGS_ERR_CUDA (text via bgs_status_string / bgs_last_error).  Key overflow
 *    (K > max_keys) is detected on the device: later stages of that frame become
 *    no-ops and bgs_frame_status reports BGS_ERR_CAPACITY with the required K.
 *  - Concurrency: frames on different streams may share theta read-only; calls
 *    that accumulate into the same grad must be stream-ordered.  preprocess,
 *    sort and render_fwd are deterministic (bit-reproducible); render_bwd is not
 *    (float atomics; BASELINE.json north_star).
 */
#ifndef BGS_H
#define BGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BGS_OK = 0,
  BGS_ERR_INVALID = -1,
  BGS_ERR_CAPACITY = -2,
  BGS_ERR_CUDA = -3,
  BGS_ERR_UNSUPPORTED = -4
} bgs_status;

#define BGS_TILE 16            /* "16 x 16 pixel blocks" (§IV-C1) */
#define BGS_FLOATS_PER_GAUSSIAN 59
#define BGS_MAX_KEYS_LIMIT ((int64_t)1 << 30)

/* Views into theta[59n] (caller-owned; segments 4-byte aligned, 16-byte aligned ones take
 * the vector load paths -- one contiguous buffer with n % 4 == 0 is fully aligned):
 *   [means 3n | log_scales 3n | quats 4n (w,x,y,z) | opacity_logits n | sh 48n ([n][16][3], k = 0 is DC)]
 * Raw optimiser parameters; exp / normalise / sigmoid are fused (R5).  The
 * primitive is G(x) = exp(-1/2 (x-mu)^T Sigma^-1 (x-mu)) with Sigma = R S S^T R^T
 * (§II-A).  sh_degree = active SH degree 0..3 (R12). */
typedef struct {
  int64_t n;
  int32_t sh_degree;
  int32_t _pad;
  const float *means, *log_scales, *quats, *opacity_logits, *sh;
} bgs_gaussians;

/* Camera (host struct, copied into kernel parameters).  `view` is W of
 * Sigma' = J W Sigma W^T J^T, world -> camera, column-major
 * (t_r = sum_k view[r+4k] mu_k + view[12+r]); `proj` = P . view world -> clip,
 * column-major (R2).  Pixel (x, y) is sampled at integer coordinates (R1). */
typedef struct {
  float view[16];
  float proj[16];
  float campos[3];
  float tan_fovx, tan_fovy;
  int32_t width, height;  /* 1..16384 each; edge tiles may be partial (R1) */
  float bg[3];            /* background colour: out = C + T_final * bg (R16) */
  float near_plane;       /* cull iff t_z <= near_plane; 0.2 by default (R3) */
} bgs_camera;

/* Adam hyper-parameters (R21, PyTorch semantics). lr per group. */
typedef struct {
  float lr_means, lr_log_scales, lr_quats, lr_opacity, lr_sh_dc, lr_sh_rest;
  float beta1, beta2, eps;
} bgs_adam_hparams;

/* One view's workspace (host struct; fields are library-private).  Sized by
 * bgs_workspace_bytes, carved by bgs_frame_init out of ONE caller allocation
 * (>= 256-byte aligned). */
typedef struct {
  uint64_t opaque[128];
} bgs_frame;

/* Device pointers into a frame's workspace, for the parity tests (host struct). */
typedef struct {
  int32_t* radius;          /* [n]  0 = culled ("absent")                       */
  float* depth;             /* [n]  camera-space t_z; its bits are the key low word  */
  float* record;            /* [n][12] {x, y, ex, ey | A, B, C, opacity | r, g, b, pthr}
                               with (A, B, C) = (-conic.x/2, -conic.y, -conic.z/2);
                               (ex, ey) conservative half-extents of the alpha >= 1/255
                               level set and pthr = -(ln(255 o) + 1e-3): the blend kernels'
                               exact per-block and per-pixel skip tests                 */
  uint32_t* tiles_touched;  /* [n]                                                   */
  uint32_t* offsets;        /* [n]  exclusive scan of tiles_touched (R13)            */
  uint64_t* keys_unsorted;  /* [max_keys] (tile << 32 | depth bits), index order     */
  uint32_t* values_unsorted;/* [max_keys] Gaussian index                             */
  uint64_t* keys_sorted;    /* [max_keys] stable ascending                           */
  uint32_t* values_sorted;  /* [max_keys]                                            */
  uint32_t* ranges;         /* [tiles][2] [start, end) per tile, (0,0) if empty      */
  float* grad2d;            /* [n][12] per-view blend grads {dx, dy, dconic x,y,z, do,
                               dr, dg, db, 0, 0, 0}; zeroed by the preprocess (or, on a
                               consuming frame, by the chain rule that reads it) */
  int64_t n, max_keys;
  int32_t tiles_x, tiles_y, sort_bits, sort_passes;
  int32_t sort_mode;        /* 0 depth-first (keys_* hold 32-bit tile ids), 1 onesweep64 */
  int32_t _pad;
  uint8_t* cbits;           /* [n] frozen clamp decisions: rgb clamped (bits 0-2), J clamp
                               x (bit 3, side bit 4), y (bit 5, side bit 6) (R7, R12, R18) */
} bgs_frame_views;

/* Per-frame workload counters (bgs_frame_stats; not on the hot path). */
typedef struct {
  int64_t visible;      /* V: Gaussians with radius > 0                       */
  int64_t num_keys;     /* K                                                  */
  int64_t evals_fwd;    /* E_f: (pixel, list entry) pairs the forward visits  */
  int64_t evals_bwd;    /* E_b: sum over pixels of n_contrib                  */
  int64_t evals_slot;   /* E_slot: sum over 8x4-pixel warps of 32 * max_lane(culled visits) */
  int64_t max_list;     /* longest tile list                                  */
  int64_t blended;      /* (pixel, Gaussian) pairs blended in the forward      */
  int64_t evals_fwd_culled; /* E_f restricted to entries whose alpha level-set box
                               reaches the pixel's 8x4 warp block (what the fwd evaluates) */
  int64_t evals_bwd_culled; /* the same for the backward (positions < n_contrib) */
} bgs_stats;

/* ---------------------------------------------------------------- sizing */
/* Workspace bytes for n Gaussians, a w x h view and a key capacity max_keys
 * (1 <= max_keys < BGS_MAX_KEYS_LIMIT = 2^30: the sort's look-back words hold 30-bit
 * counts; R25).  n < 2^31, 1 <= w, h <= 16384.  Returns 0 on invalid sizes. */
size_t bgs_workspace_bytes(int64_t n, int32_t w, int32_t h, int64_t max_keys);

/* Carve `workspace` (device, `bytes` >= bgs_workspace_bytes) into frame `f`.
 * Does not touch device memory.  BGS_ERR_INVALID on bad sizes or alignment. */
bgs_status bgs_frame_init(bgs_frame* f /*host*/, void* workspace, size_t bytes, int64_t n, int32_t w, int32_t h,
                          int64_t max_keys);

/* ---------------------------------------------------------------- the hot path */
/* a1-a3: activations, view transform, near cull, projection, Sigma' = J W Sigma W^T J^T
 * + 0.3 I, conic, radius, tile rect, SH -> rgb, tiles_touched, and the exclusive scan
 * into offsets / K (§II-A; P:59 SH colour; readings R1-R13, R22).
 * Requires g->n == the frame's n and cam->width/height == the frame's w/h.  n = 0 is
 * valid.  The camera is remembered in the frame for the later calls. */
bgs_status bgs_preprocess(const bgs_gaussians* g /*host*/, const bgs_camera* cam /*host*/, bgs_frame* f /*host*/,
                          void* stream);

/* a1-a3 over a batch of views: cams[nframes] (host array) and frames[nframes] (host array
 * of distinct host frame pointers, 1 <= nframes <= 4096, all of the same n, each
 * cams[v] matching frames[v]'s w/h).  Bit-identical to calling bgs_preprocess(g, &cams[v],
 * frames[v]) for each v, but theta is read once per 16 views instead of once per view
 * (the views of a training batch share theta, R20).  Any invalid camera or frame ->
 * BGS_ERR_INVALID before anything launches. */
bgs_status bgs_preprocess_batch(const bgs_gaussians* g /*host*/, const bgs_camera* cams /*host*/,
                                bgs_frame* const* frames /*host*/, int32_t nframes, void* stream);

/* a4-a6: duplicate (tile | depth) keys (values = Gaussian index), stable 64-bit LSD
 * radix sort on bits [0, 32 + bit_width(tiles - 1)), tile ranges.  Result order =
 * (tile, depth bits, index): "N ... sorted by depth", ties by index
 * (R13). */
bgs_status bgs_sort(bgs_frame* f /*host*/, void* stream);

/* a7: per pixel, front-to-back over its tile's list: alpha = min(0.99, o G), skip
 * alpha < 1/255, stop before T (1 - alpha) < 1e-4, C += c alpha T (PAPER.md l.143-149,
 * §II-A; R14-R16).  Outputs planar image[3][h][w], final_T[h][w] and n_contrib[h][w] =
 * 1-based list position of the last blended Gaussian (0 if none). */
bgs_status bgs_render_fwd(bgs_frame* f /*host*/, float* image, float* final_T, uint32_t* n_contrib, void* stream);
/* Optional plan-ahead of the blend kernels' schedules (a launch-order aid; results are
 * unchanged).  bgs_render_fwd_plan builds the work units of the frame's NEXT bgs_render_fwd
 * (heaviest first and split by its scheduling hint, else ordered by tile list length): call
 * it after bgs_sort and bgs_frame_load_hint, e.g. on another stream while other views blend.
 * bgs_blend_bwd_plan builds the NEXT bgs_blend_bwd's units from the frame's last forward:
 * call it after bgs_render_fwd, e.g. on another stream while the loss runs.  A plan is
 * discarded by bgs_preprocess(_batch), bgs_sort, bgs_frame_load_hint, bgs_frame_set_debug,
 * bgs_frame_set_seg_len (and a forward plan by the forward that uses it, a backward plan by
 * the next bgs_render_fwd); without one, bgs_render_fwd / bgs_blend_bwd plan for themselves.
 * The caller orders the plan before its kernel across streams (events).  Asynchronous. */
bgs_status bgs_render_fwd_plan(bgs_frame* f /*host*/, void* stream);
bgs_status bgs_blend_bwd_plan(bgs_frame* f /*host*/, void* stream);

/* a9-a10: blend backward (back to front, decisions of the forward frozen, R18) and
 * the chain rule conic -> Sigma' -> Sigma/(s, q) and J -> t -> mu, xy -> mu,
 * rgb -> SH / view direction -> mu, opacity -> logit.  grad[59n] += dL/dtheta in
 * theta's layout (the sum over views, R20).  dL_dimage is planar [3][h][w]. */
bgs_status bgs_render_bwd(const bgs_gaussians* g /*host*/, bgs_frame* f /*host*/, const float* dL_dimage,
                          const float* final_T, const uint32_t* n_contrib, float* grad, void* stream);
/* The two halves of bgs_render_bwd, for per-stage timing: a9 accumulates the per-view
 * blend gradients {dxy, dconic, dopacity, drgb} into the frame's grad2d; a10 applies the
 * chain rule to theta's layout (grad +=).  bgs_render_bwd == blend_bwd then preprocess_bwd. */
bgs_status bgs_blend_bwd(bgs_frame* f /*host*/, const float* dL_dimage, const float* final_T,
                         const uint32_t* n_contrib, void* stream);
bgs_status bgs_preprocess_bwd(const bgs_gaussians* g /*host*/, bgs_frame* f /*host*/, float* grad, void* stream);
/* a10 over a batch of views (R20: grad += the sum over views): frames[nframes] (host array
 * of host frame pointers, 1 <= nframes <= 4096, all of the same n, each after its own
 * bgs_preprocess + bgs_blend_bwd for this theta) -> grad[59n] +=.  Equal to calling
 * bgs_preprocess_bwd on each frame up to float summation order, but theta is read and grad
 * read-modified-written once per 16 views instead of once per view. */
bgs_status bgs_preprocess_bwd_batch(const bgs_gaussians* g /*host*/, bgs_frame* const* frames /*host*/,
                                    int32_t nframes, float* grad, void* stream);

/* bgs_preprocess_bwd_batch with grad ASSIGNED, not accumulated: grad[59n] = the sum over the
 * frames of each view's chain rule, every element written (0 for a Gaussian no frame sees,
 * and for SH coefficients above the degree).  With nframes > 16 the first launch assigns
 * and the later ones accumulate.  grad's previous contents are never read, so a caller whose
 * step has one chain-rule pass per rank needs no zeroing between steps (pair it with
 * bgs_adam_step_keep_grad): theta and grad cross HBM once less.  Value-equal to
 * bgs_preprocess_bwd_batch into a zero grad (tests/test_gpu_parity.py).  Errors as
 * bgs_preprocess_bwd_batch. */
bgs_status bgs_preprocess_bwd_batch_assign(const bgs_gaussians* g /*host*/, bgs_frame* const* frames /*host*/,
                                           int32_t nframes, float* grad, void* stream);

/* bgs_preprocess_bwd_batch restricted to the Gaussians [begin, begin + count): grad +=
 * their 59 elements (in each theta segment the sub-range of those Gaussians) and nothing
 * else.  Consecutive ranges covering [0, n) sum to bgs_preprocess_bwd_batch's gradient
 * (bit-identical: each element is written by one Gaussian's thread).  A multi-GPU caller
 * processes the Gaussians in chunks and starts each chunk's gradient exchange (an
 * all-reduce of its five segment sub-ranges) while the next chunk
 * computes.  BGS_ERR_INVALID if the range is not inside [0, n). */
bgs_status bgs_preprocess_bwd_batch_range(const bgs_gaussians* g /*host*/, bgs_frame* const* frames /*host*/,
                                          int32_t nframes, float* grad, int64_t begin, int64_t count,
                                          void* stream);

/* a10 + a11 fused for one GPU (no collective between them): the batched chain rule of
 * bgs_preprocess_bwd_batch, then -- in the same kernel, per Gaussian -- the Adam update of
 * bgs_adam_step with the batch's gradient, which is never written to memory (dense: a
 * Gaussian no view sees takes g = 0, R26).  theta (device) must be the buffer g views
 * (g->means == theta); exp_avg / exp_avg_sq [59n] (device).  With nframes > 16 the earlier
 * launches accumulate into grad [59n] (device, zero on entry, zeroed on exit), else grad may
 * be NULL.  Bit-identical to bgs_preprocess_bwd_batch into a zero grad + bgs_adam_step. */
bgs_status bgs_preprocess_bwd_batch_adam(const bgs_gaussians* g /*host*/, bgs_frame* const* frames /*host*/,
                                         int32_t nframes, float* theta, float* grad, float* exp_avg,
                                         float* exp_avg_sq, const bgs_adam_hparams* hp /*host*/, int64_t step,
                                         void* stream);

/* a11: fused Adam over theta[59n] (R21, PyTorch semantics: bias-corrected, eps after
 * sqrt), per-group learning rate, grad zeroed on exit.  step is 1-based. */
bgs_status bgs_adam_step(float* theta, float* grad, float* exp_avg, float* exp_avg_sq, int64_t n,
                         const bgs_adam_hparams* hp /*host*/, int64_t step, void* stream);

/* bgs_adam_step leaving grad as it is (read only): the same theta / exp_avg / exp_avg_sq
 * update, bit for bit, for a caller whose next chain rule assigns grad
 * (bgs_preprocess_bwd_batch_assign).  Errors as bgs_adam_step. */
bgs_status bgs_adam_step_keep_grad(float* theta, const float* grad, float* exp_avg, float* exp_avg_sq, int64_t n,
                                   const bgs_adam_hparams* hp /*host*/, int64_t step, void* stream);

/* a11 on a shard (reduce-scatter -> Adam on 1/G of theta -> all-gather):
 * the same update as bgs_adam_step restricted to theta elements [begin, begin + count) of the
 * 59n layout.  The four device pointers address element `begin` (shard buffers, or offsets
 * into the full buffers); the learning-rate group of element i is that of begin + i.
 * Elements at or past 59n (the caller's shard padding) are not touched.  begin must be a
 * multiple of 4 and the pointers 16-byte aligned, else BGS_ERR_INVALID (nothing launched). */
bgs_status bgs_adam_step_range(float* theta, float* grad, float* exp_avg, float* exp_avg_sq, int64_t n,
                               int64_t begin, int64_t count, const bgs_adam_hparams* hp /*host*/, int64_t step,
                               void* stream);

/* SURVEY.md §8(e) 3, the exchange fused with Adam over NVSwitch multicast (NVLink SHARP):
 * theta_mc / grad_mc are multicast addresses (CUDA driver cuMulticastCreate / BindMem /
 * MemMap; the caller owns the objects) of every rank's theta[59n] and grad[59n]; theta is
 * this rank's replica.  For the theta elements [begin, begin + count) of this rank's shard:
 * g = the sum of all ranks' grad (one multimem.ld_reduce per 4 elements, reduced in the
 * switch), Adam with the shard's exp_avg / exp_avg_sq [count] (as bgs_adam_step_range), the
 * new theta stored to every rank's replica (multimem.st) and every rank's grad over the
 * shard zeroed (multimem.st) -- reduce-scatter + Adam + all-gather in one pass.  The caller
 * orders it between device-wide barriers across the ranks (every grad complete before,
 * every store visible after).  begin and count multiples of 4 (elements past 59n are not
 * touched), pointers 16-byte aligned, else BGS_ERR_INVALID.  One rank's call updates only
 * its shard; all ranks' calls together update every replica. */
bgs_status bgs_adam_step_multimem(float* theta, float* theta_mc, float* grad_mc, float* exp_avg, float* exp_avg_sq,
                                  int64_t n, int64_t begin, int64_t count, const bgs_adam_hparams* hp /*host*/,
                                  int64_t step, void* stream);

/* Zero `count` floats at device pointer p (cudaMemsetAsync on `stream`): resets a gradient
 * buffer whose shard bgs_adam_step_range consumed after a reduce-scatter (the rest of the
 * buffer still holds this rank's partial sums).  BGS_ERR_INVALID on p = NULL with count > 0. */
bgs_status bgs_zero(float* p, int64_t count, void* stream);

/* a8 (caller-side helper): L1 loss gradient against an 8-bit target [3][h][w]
 * (R19): dL_dimage = scale * sign(image - target/255); loss_sum += sum |image - target/255|
 * (loss_sum: one device float, accumulated).  scale = 1/(3 h w B) for a batch mean (R20). */
bgs_status bgs_l1_loss_grad(const float* image, const uint8_t* target, int32_t w, int32_t h, float scale,
                            float* dL_dimage, float* loss_sum, void* stream);

/* ---------------------------------------------------------------- NEXT-2: the 3DGS training loss */
/* Workspace bytes for bgs_l1_dssim_loss_grad at w x h (0 on invalid sizes). */
size_t bgs_loss_workspace_bytes(int32_t w, int32_t h);

/* The 3DGS training loss and its gradient between a7 and a9:
 *   Loss = (1 - lambda) mean|x - y| + lambda (1 - mean SSIM(x, y)),  lambda = 0.2 in 3DGS,
 * x = image [3][h][w] (device), y = target [3][h][w] (device, 8-bit, read as t/255), means
 * over the 3 h w values; SSIM per channel with an 11x11 Gaussian window (sigma 1.5, zero
 * padding), C1 = 0.01^2, C2 = 0.03^2 (Wang et al. 2004; the paper's quality metric, PAPER.md
 * §VI-A l.394; window per SPEC.md l.171; readings R28-R30).  Outputs: dL_dimage (device,
 * [3][h][w], overwritten) = scale * dLoss/dx, and loss_sum (one device float) += scale *
 * Loss (scale = 1/B gives the batch mean, R20).  workspace: device, 256-byte aligned, >=
 * bgs_loss_workspace_bytes(w, h); no state is kept in it between calls.  BGS_ERR_INVALID on
 * null pointers, bad sizes, lambda outside [0, 1] or a short/unaligned workspace. */
bgs_status bgs_l1_dssim_loss_grad(const float* image, const uint8_t* target, int32_t w, int32_t h, float lambda,
                                  float scale, float* dL_dimage, float* loss_sum, void* workspace, size_t bytes,
                                  void* stream);

/* ---------------------------------------------------------------- NEXT-1: T1 density statistics */
/* Workspace bytes for bgs_local_density over n points (0 on invalid n: 1 <= n < 2^30). */
size_t bgs_density_workspace_bytes(int64_t n);

/* The paper's statistical density thresholding (§III-C1 l.181-186): for every
 * point p of means[n][3] (device, e.g. theta's means segment), counts[n] (device, out) =
 * rho(p) = number of other points q with |q - p| <= r, exact (squared distance evaluated
 * ((dx*dx + dy*dy) + dz*dz) in float against r*r; hashed uniform grid);
 * stats[4] (device doubles, out) = {mu_rho, sigma_rho (population), rho_low = mu - alpha
 * sigma, rho_high = mu + beta sigma}.  workspace: device, >= bgs_density_workspace_bytes(n)
 * bytes, 256-byte aligned.  BGS_ERR_INVALID on bad arguments (nothing launched). */
bgs_status bgs_local_density(const float* means, int64_t n, float r, float alpha, float beta, uint32_t* counts,
                             double* stats, void* workspace, size_t bytes, void* stream);

/* ---------------------------------------------------------------- NEXT-1: the density-control step */
/* PAPER.md §III-C2-C4 (l.188-228): merge dense pairs, densify sparse points, every few
 * thousand iterations (l.228).  Readings R31-R36. */
typedef struct {
  float r;            /* local-density radius (world units, > 0) */
  float alpha, beta;  /* rho_low / rho_high factors */
  float gamma;        /* d_merge = mu_d + gamma sigma_d */
  float alpha_sigma;  /* densification spread sigma_p = alpha_sigma d_bar_p (> 1) */
  float delta;        /* jitter half-width */
  int32_t k;          /* neighbours for d_bar_p and mu_d / sigma_d (1..16; 8) */
  int32_t max_new;    /* children per sparse point cap per round (0..64; 4) */
} bgs_density_params;

typedef struct {      /* filled on the device by bgs_density_plan */
  int64_t n_in, n_out, n_pairs, n_children;
  double mu_rho, sigma_rho, rho_low, rho_high, mu_d, sigma_d, d_merge;
  int64_t n_sparse;   /* points with rho < rho_low (rho_low > 0): the densification parents */
} bgs_density_report;

/* Workspace bytes for the density step over n Gaussians (0 on invalid n: 1 <= n < 2^30). */
size_t bgs_density_step_workspace_bytes(int64_t n);
/* Plan (asynchronous): on theta[59n] (device; the means segment is read): rho and the k
 * nearest neighbours per point (exact; rings of grid cells), the statistics and d_merge
 * (R31-R32; neighbour distances truncated at 3 r), mutual-nearest dense pairs within d_merge (R33), the children of sparse points
 * (R35), the output offsets and n_out -- all kept in the workspace (device, 256-byte
 * aligned, >= bgs_density_step_workspace_bytes(n)). */
bgs_status bgs_density_plan(const float* theta, int64_t n, const bgs_density_params* p /*host*/, void* workspace,
                            size_t bytes, void* stream);
/* After the caller synchronised the plan's stream: the report (host out; n_out and
 * n_children size the apply call's buffers) and the number of points with fewer than k
 * neighbours within 3 r (their missing distances count as 3 r, R32). */
bgs_status bgs_density_result(const void* workspace, int64_t n, bgs_density_report* out /*host*/,
                              uint32_t* short_knn /*host, may be NULL*/);
/* Apply (asynchronous): theta_out / exp_avg_out / exp_avg_sq_out [59 n_out] (device) =
 * survivors in index order (a merged pair's result at its lower index, R34), then the
 * children in (parent, j) order (R35); Adam moments kept for unmerged survivors, zero for
 * merged Gaussians and children (R36).  normals / uniforms: device [n_children][3] N(0,1)
 * and U(-1,1) variates (the method's random draws, supplied by the caller). */
bgs_status bgs_density_apply(const float* theta, const float* exp_avg, const float* exp_avg_sq, int64_t n,
                             const void* workspace, const bgs_density_params* p /*host*/, const float* normals,
                             const float* uniforms, int64_t n_children, float* theta_out, float* exp_avg_out,
                             float* exp_avg_sq_out, int64_t n_out, void* stream);
/* Further densification rounds (R35'; §III-C2 l.206 "This process is repeated
 * iteratively until the desired density is achieved"; SPEC.md l.247 max_rounds).
 * bgs_density_parents (asynchronous, after bgs_density_plan): the report's n_sparse sparse
 * points as parents[n_sparse] (device u32, out) = their indices in bgs_density_apply's
 * output (index order; sparse points are never merged) and sigma[n_sparse] (device double,
 * out) = alpha_sigma d_bar_p (R35).  A round on the current scene of n_t points: the
 * caller counts rho of every point (bgs_local_density on its means, radius p->r), then
 * bgs_density_round_plan: parent p below rho_low spawns min(max_new, ceil(rho_low - rho_p))
 * children (exclusive offsets in the round workspace, device, >=
 * bgs_density_round_workspace_bytes(n_parents) bytes, 256-byte aligned);
 * bgs_density_round_result (after the caller synchronised): the round's child count (0: the
 * desired density is reached, stop); bgs_density_round_apply: the n_t points (moments kept)
 * then the children in (parent, j) order, child at p + sigma_p z + delta u (z, u: device
 * [n_children][3] N(0,1) / U(-1,1) variates), attributes copied from the parent, zero
 * moments; outputs [59 (n_t + n_children)]. */
bgs_status bgs_density_parents(const void* workspace, int64_t n, const bgs_density_params* p /*host*/,
                               uint32_t* parents, double* sigma, void* stream);
size_t bgs_density_round_workspace_bytes(int64_t n_parents);
bgs_status bgs_density_round_plan(const uint32_t* rho, int64_t n_t, const uint32_t* parents, int64_t n_parents,
                                  double rho_low, int32_t max_new, void* workspace, size_t bytes, void* stream);
bgs_status bgs_density_round_result(const void* workspace, int64_t n_parents, int64_t* n_children /*host*/);
bgs_status bgs_density_round_apply(const float* theta, const float* exp_avg, const float* exp_avg_sq, int64_t n_t,
                                   const uint32_t* parents, const double* sigma, int64_t n_parents,
                                   const void* workspace, float delta, const float* normals, const float* uniforms,
                                   int64_t n_children, float* theta_out, float* exp_avg_out, float* exp_avg_sq_out,
                                   void* stream);

/* ---------------------------------------------------------------- NEXT-3 / NEXT-4: T2 sampling */
/* PAPER.md §IV-C1 (l.253-268): per 16x16 tile, each pixel's rendered colour (clamped to
 * [0,1]) quantised to 16 levels per channel (c8 = min(255, floor(256 c)), level = c8 / 16),
 * key = R 256 + G 16 + B, aggregated in a 4096-slot shared-memory table (R37-R38).  Outputs
 * (device): nb[tiles] = occupied buckets; for bucket j < nb[t] of tile t, at [t * 256 + j]
 * in ascending key order: keys (u16), counts (pixels), color_sum[3], opacity_sum
 * (sum of 1 - final_T).  image [3][h][w], final_T [h][w] (device). */
bgs_status bgs_tile_buckets(const float* image, const float* final_T, int32_t w, int32_t h, uint32_t* nb,
                            uint16_t* keys, uint32_t* counts, float* color_sum, float* opacity_sum, void* stream);
/* Workspace bytes for bgs_importance / bgs_importance_keep over n Gaussians (0 if n < 1). */
size_t bgs_importance_workspace_bytes(int64_t n);
/* PAPER.md §IV-C3 (l.279-284): I_g = (1/N_g) sum_i sim(c_g, c_i) alpha_g(i) over the pixels
 * of g's tiles where alpha_g(i) >= 1/255, sim = 1 - |c_g - c_i| / sqrt(3) (R39), for the
 * frame's last bgs_sort and the image it rendered (device [3][h][w]).  importance[n] and
 * count[n] (N_g; may be NULL) out (device).  Not on the training hot path. */
bgs_status bgs_importance(const bgs_frame* f /*host*/, const float* image, float* importance, uint32_t* count,
                          void* workspace, size_t bytes, void* stream);
/* R40: keep[i] = 1 for the first ceil(fraction n) Gaussians by ascending
 * importance (descending if invert), ties by index; 0 for the rest (device u8 [n] out). */
bgs_status bgs_importance_keep(const float* importance, int64_t n, float fraction, int32_t invert, uint8_t* keep,
                               void* workspace, size_t bytes, void* stream);
/* NEXT-4 render-only serving: later bgs_preprocess calls on this frame cull every Gaussian
 * with keep[i] == 0 ("the precomputed importance information is retained for use during
 * rendering", l.284).  keep: device u8 [n], caller-owned, or NULL to render all. */
bgs_status bgs_frame_set_keep(bgs_frame* f /*host*/, const uint8_t* keep);

/* ---------------------------------------------------------------- status / debug */
/* After the caller synchronised the frame's stream: K of the last preprocess (host out)
 * and BGS_OK, or BGS_ERR_CAPACITY when K > max_keys in ANY preprocess of this frame since
 * the previous bgs_frame_status call (a sticky device flag, cleared by this call: a
 * training loop can check once per many steps without losing an overflowed view, whose
 * image is background and gradient zero); re-run with a larger workspace. */
bgs_status bgs_frame_status(const bgs_frame* f /*host*/, int64_t* num_keys /*host*/);
/* Per-camera scheduling hint: the per-(tile, 8x4 block) walk costs of the frame's last
 * forward, which order (heaviest first) and split the next forward's work items.  A
 * trainer rendering many cameras through a few frames saves a camera's hint after its
 * forward and loads it before that camera's next render (src NULL: no hint, work ordered
 * by list length).  Results are identical with any hint; only the schedule changes.
 * dst / src: device, bgs_frame_hint_bytes(f) bytes, caller-owned; asynchronous. */
size_t bgs_frame_hint_bytes(const bgs_frame* f /*host*/);
bgs_status bgs_frame_save_hint(const bgs_frame* f /*host*/, void* dst, void* stream);
bgs_status bgs_frame_load_hint(bgs_frame* f /*host*/, const void* src, void* stream);
bgs_status bgs_frame_debug(const bgs_frame* f /*host*/, bgs_frame_views* out /*host*/);
/* Failure detection, not on the hot path.  Structural check of the frame's
 * last bgs_sort (a4-a6, §II-A, SPEC.md l.123 / R13): out (device,
 * caller-owned, 8-byte aligned u64[5]) receives {range errors (a range outside [0, K),
 * a non-empty tile not starting where the previous one ended, the last not ending at K,
 * an empty tile not (0, 0)), membership errors (an entry that is not a visible Gaussian
 * whose tile rect covers the tile), order errors (adjacent entries not strictly increasing
 * in (depth bits, index)), count error (1 if sum tiles_touched != K), sum tiles_touched}.
 * The first four all zero prove every tile list is exactly its Gaussians in order.
 * Asynchronous on `stream`; BGS_ERR_INVALID on a bad frame or pointer. */
bgs_status bgs_frame_validate(const bgs_frame* f /*host*/, uint64_t* out, void* stream);
/* Non-finite check (e.g. of a gradient before Adam): out (device, caller-owned, 8-byte
 * aligned u64[2]) receives {number of NaN / Inf entries of x[0, count), smallest such
 * index or UINT64_MAX}.  x: device, 16-byte aligned.  Asynchronous on `stream`. */
bgs_status bgs_nonfinite(const float* x, int64_t count, uint64_t* out, void* stream);
/* Workload counters of the last fwd (runs a counting kernel and synchronises). */
bgs_status bgs_frame_stats(const bgs_frame* f /*host*/, const uint32_t* n_contrib, bgs_stats* out /*host*/,
                           void* stream);

/* Test-only knob: flags & BGS_DEBUG_SKIP_SORT makes bgs_sort stop after the key
 * duplication (a4), so the unsorted keys/values stay readable via bgs_frame_debug. */
#define BGS_DEBUG_SKIP_SORT 1
/* Selects the reference sort path: materialised 64-bit (tile | depth) keys and the
 * onesweep LSD sort over all 32 + bit_width(tiles - 1) bits (keys_sorted is then valid).
 * The default depth-first path produces bit-identical values and ranges. */
#define BGS_DEBUG_SORT_ONESWEEP64 2
/* Depth-first path with the radix tile split (two 8-bit onesweep passes over the K items)
 * instead of the direct chunked split; same values and ranges. */
#define BGS_DEBUG_SORT_RADIX_SPLIT 4
/* Kept selectable: the blend backward on 8x4-pixel units (one pixel per lane) instead of
 * the default 8x8 units (two pixels per lane). */
#define BGS_DEBUG_BWD_8X4 8
/* Depth-first path with the row split (rowsplit.cu: the (row, Gaussian) entries stably
 * split by tile row, then each row's items by tile column, one warp per chunk with a
 * position counter per row / column in shared memory) instead of the default one-pass
 * direct tile split (a position counter per tile of the image per warp); same values and
 * ranges; measured slower. */
#define BGS_DEBUG_SORT_ROWSPLIT 16
/* Parity mode (R23): the blend kernels evaluate exp with the canonical expression tree the
 * oracle also uses (instead of MUFU.EX2) and the forward does not split walks, so every
 * blend decision, n_contrib and the image are bit-identical to the oracle's. */
#define BGS_DEBUG_PARITY_EXP 64
/* R10 / R11: 3DGS's square tile rect of half-width radius = ceil(3 sqrt(lambda_1)) instead of
 * the default R11' rect (the tiles the alpha >= 1/255 box reaches): the 3DGS key
 * set, longer lists, and images that cut opaque Gaussians at 3 sigma. */
#define BGS_DEBUG_SQUARE_RECT 128
bgs_status bgs_frame_set_debug(bgs_frame* f /*host*/, int32_t flags);

/* Scheduling parameter of the blend kernels (default 4096 for frames of >= 3000 tiles, 2048
 * below: fewer units to balance, finer cuts): a (tile, 8x4 pixel block) work
 * item whose back-to-front walk is longer than seg_len list entries is split, in the
 * backward, into segments of seg_len entries processed independently, each starting from
 * the per-pixel {T, colour behind} the forward recorded at the segment boundary (up to 63
 * boundaries per item, as many as the frame's checkpoint pool holds; the rest of a walk
 * stays in its last segment).  Results agree with the unsplit walk to float rounding.
 * seg_len: multiple of 32 in [32, 65536].  BGS_ERR_INVALID otherwise. */
/* Consuming frame (on != 0): every chain rule over all Gaussians (bgs_preprocess_bwd,
 * _batch, _batch_adam, bgs_render_bwd) zeroes the frame's per-view blend gradients as it reads
 * them, and the next bgs_preprocess of the frame then skips zeroing them (48 B per visible
 * Gaussian of HBM writes).  A second chain rule over the same backward then sees zeros:
 * leave it off (the default) to run several chain rules from one bgs_blend_bwd. */
bgs_status bgs_frame_set_consume(bgs_frame* f /*host*/, int32_t on);
bgs_status bgs_frame_set_seg_len(bgs_frame* f /*host*/, int32_t seg_len);

const char* bgs_status_string(bgs_status s);
const char* bgs_last_error(void);
/* Number of kernels this library launched since load (host counter; bench evidence). */
uint64_t bgs_launch_count(void);
int32_t bgs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BGS_H */
