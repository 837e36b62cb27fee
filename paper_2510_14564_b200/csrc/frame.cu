// frame.cu -- libbgs C ABI: workspace sizing, frame carving, validation, status, debug.
// The entry points are declared (with their paper citations) in include/bgs.h.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "common.cuh"

namespace bgs {

static std::atomic<uint64_t> g_launches{0};
static thread_local char g_err[512] = "";

void note_launch(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }
void set_error(const char* msg) { snprintf(g_err, sizeof(g_err), "%s", msg); }

bgs_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return BGS_ERR_CUDA;
  }
  return BGS_OK;
}

int num_sms() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  });
  return sms;
}

static inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t radius, depth, record, tiles_touched, rect, offsets, keys0, keys1, vals0, vals1, ranges, scan_status, sort_hist,
      sort_status, counters, plan, grad2d, tile_count, order_fwd, order_bwd, block_cost, ck_table, ck_pool, spec_base, spec_n,
      arrive, spec_state, spec_last, chunk_cnt, dkey0, dkey1,
      dval0, dval1, rank_cnt, item_off, rank_rect, cbits, rank_h, rs_tabA, rs_chunk_r0, rs_rows, rs_units, rs_tabB,
      rs_status, total;
  int64_t rs_max_chunks, rs_max_units, rs_scan_tiles;
  int64_t ck_cap;
  int32_t tiles_x, tiles_y, num_tiles, sort_bits, sort_passes, scan_tiles;
  int64_t sort_tiles_max;
  bool direct;
};

constexpr int kScanTile = 4096;  // = kScanThreads * kScanItems of k_scan (preprocess.cu)
constexpr int kSortTile = kSortTileKeys;

static bool make_layout(int64_t n, int32_t w, int32_t h, int64_t max_keys, Layout& L) {
  if (n < 0 || n > ((int64_t)1 << 31) - 1 || w < 1 || h < 1 || w > 16384 || h > 16384 || max_keys < 1 ||
      max_keys >= BGS_MAX_KEYS_LIMIT)
    return false;
  L.tiles_x = (w + kTile - 1) / kTile;
  L.tiles_y = (h + kTile - 1) / kTile;
  L.num_tiles = L.tiles_x * L.tiles_y;
  int b = 0;
  while (((int64_t)1 << b) < (int64_t)L.num_tiles) ++b;  // bit_width(num_tiles - 1)
  L.sort_bits = 32 + b;
  L.sort_passes = (L.sort_bits + 7) / 8;
  L.scan_tiles = (int32_t)((n + kScanTile - 1) / kScanTile);
  if (L.scan_tiles < 1) L.scan_tiles = 1;
  // look-back status words: enough for the K-key passes and the N-key depth passes
  L.sort_tiles_max = ((max_keys > n ? max_keys : n) + kSortTile - 1) / kSortTile;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + (bytes ? bytes : 1));
    return at;
  };
  const size_t N = (size_t)n, K = (size_t)max_keys;
  L.radius = take(4 * N);
  L.depth = take(4 * N);
  L.record = take(48 * N);
  L.tiles_touched = take(4 * N);
  L.rect = take(8 * N);
  L.offsets = take(4 * N);
  L.keys0 = take(8 * K);
  L.keys1 = take(8 * K);
  L.vals0 = take(4 * K);
  L.vals1 = take(4 * K);
  L.ranges = take(8 * (size_t)L.num_tiles);
  L.scan_status = take(8 * (size_t)L.scan_tiles);
  L.sort_hist = take(4 * 8 * 256);
  L.sort_status = take(4 * 256 * (size_t)L.sort_tiles_max);
  L.counters = take(4 * C_NUM);
  L.plan = take(4 * kPlanWords);
  L.grad2d = take(48 * N);
  const size_t NT = (size_t)L.num_tiles;
  L.tile_count = take(4 * NT);
  // checkpoint pool: walks total at most 8 K entries (8 blocks per tile list), so the
  // segment length kCkPoolSeg needs at most 8 K / kCkPoolSeg boundary slots (+ slack)
  L.ck_cap = 2 * 8 * (int64_t)NT + 8 * ((max_keys > n ? max_keys : n) / kCkPoolSeg) + 64;
  L.order_fwd = take(4 * (8 * NT + (size_t)L.ck_cap));  // forward units: items + segments
  L.order_bwd = take(4 * (8 * NT + (size_t)L.ck_cap));  // backward units: items + boundaries
  L.block_cost = take(4 * 8 * NT);
  L.ck_table = take(4 * 8 * NT * kCkMax);
  L.ck_pool = take(512 * (size_t)L.ck_cap);
  L.spec_base = take(4 * 8 * NT);
  L.spec_n = take(4 * 8 * NT);
  L.arrive = take(4 * 8 * NT);
  L.spec_state = take(512 * (size_t)L.ck_cap);
  L.spec_last = take(128 * (size_t)L.ck_cap);
  L.direct = (int64_t)(L.tiles_x + 1) * (L.tiles_y + 1) <= kDirectMaxCells;
  L.chunk_cnt = L.direct ? take(4 * NT * (size_t)((max_keys + kChunkItemsMin - 1) / kChunkItemsMin)) : 0;
  L.dkey0 = take(4 * N);
  L.dkey1 = take(4 * N);
  L.dval0 = take(4 * N);
  L.dval1 = take(4 * N);
  L.rank_cnt = take(4 * N);
  L.item_off = take(4 * N);
  L.rank_rect = take(8 * N);
  L.cbits = take(N);
  L.rank_h = take(4 * N);
  L.rs_max_chunks = (max_keys + kRsPairChunk - 1) / kRsPairChunk + 1;
  L.rs_max_units = max_keys / kRsUnitMin + L.tiles_y + 1;
  L.rs_scan_tiles = (max_keys + 4095) / 4096 + 1;
  L.rs_tabA = take(4 * (size_t)L.rs_max_chunks * L.tiles_y);
  L.rs_chunk_r0 = take(4 * (size_t)L.rs_max_chunks);
  L.rs_rows = take(4 * (3 * (size_t)L.tiles_y + 2));
  L.rs_units = take(16 * (size_t)L.rs_max_units);
  L.rs_tabB = take(4 * (size_t)L.rs_max_units * L.tiles_x);
  L.rs_status = take(8 * (size_t)L.rs_scan_tiles);
  L.total = o;
  return true;
}

static Cam make_cam(const bgs_camera& c, int32_t tiles_x, int32_t tiles_y) {
  Cam k;
  memcpy(k.V, c.view, sizeof(k.V));
  memcpy(k.P, c.proj, sizeof(k.P));
  memcpy(k.campos, c.campos, sizeof(k.campos));
  // canonical float expressions (R22): separately rounded binary32 ops
  volatile float two_tx = 2.0f * c.tan_fovx, two_ty = 2.0f * c.tan_fovy;
  k.fx = (float)c.width / two_tx;
  k.fy = (float)c.height / two_ty;
  k.limx = 1.3f * c.tan_fovx;
  k.limy = 1.3f * c.tan_fovy;
  k.near_plane = c.near_plane;
  memcpy(k.bg, c.bg, sizeof(k.bg));
  k.W = c.width;
  k.H = c.height;
  k.tiles_x = tiles_x;
  k.tiles_y = tiles_y;
  return k;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static bgs_status validate_camera(const bgs_camera* cam, const Frame* F) {
  if (!cam) return BGS_ERR_INVALID;
  if (cam->width != F->W || cam->height != F->H) return BGS_ERR_INVALID;
  if (!(cam->tan_fovx > 0.0f) || !(cam->tan_fovy > 0.0f) || !(cam->near_plane >= 0.0f)) return BGS_ERR_INVALID;
  // view 3x3 must be orthonormal, tolerance 1e-5
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double d = 0;
      for (int k = 0; k < 3; ++k) d += (double)cam->view[a + 4 * k] * (double)cam->view[b + 4 * k];
      if (fabs(d - (a == b ? 1.0 : 0.0)) > 1e-5) return BGS_ERR_INVALID;
    }
  for (int k = 0; k < 16; ++k)
    if (!isfinite(cam->view[k]) || !isfinite(cam->proj[k])) return BGS_ERR_INVALID;
  return BGS_OK;
}

static bgs_status validate_gaussians(const bgs_gaussians* g, const Frame* F) {
  if (!g || g->n != F->n || g->sh_degree < 0 || g->sh_degree > 3) return BGS_ERR_INVALID;
  if (g->n > 0) {
    if (!g->means || !g->log_scales || !g->quats || !g->opacity_logits || !g->sh) return BGS_ERR_INVALID;
    // 4-byte alignment suffices; kernels take their 16-byte vector paths when the
    // segment pointers allow it (any n with one contiguous theta buffer works)
    auto a4 = [](const void* q) { return ((uintptr_t)q & 3u) == 0; };
    if (!a4(g->quats) || !a4(g->sh) || !a4(g->means) || !a4(g->log_scales) || !a4(g->opacity_logits))
      return BGS_ERR_INVALID;
  }
  return BGS_OK;
}

static bool frame_ok(const bgs_frame* f) { return f && frame_of(f)->magic == kFrameMagic; }

}  // namespace bgs

using namespace bgs;

extern "C" {

int32_t bgs_version(void) { return 1; }
uint64_t bgs_launch_count(void) { return g_launches.load(); }
const char* bgs_last_error(void) { return g_err; }

const char* bgs_status_string(bgs_status s) {
  switch (s) {
    case BGS_OK: return "ok";
    case BGS_ERR_INVALID: return "invalid argument";
    case BGS_ERR_CAPACITY: return "key capacity exceeded (K > max_keys)";
    case BGS_ERR_CUDA: return g_err[0] ? g_err : "CUDA error";
    case BGS_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

size_t bgs_workspace_bytes(int64_t n, int32_t w, int32_t h, int64_t max_keys) {
  Layout L;
  return make_layout(n, w, h, max_keys, L) ? L.total : 0;
}

bgs_status bgs_frame_init(bgs_frame* f, void* workspace, size_t bytes, int64_t n, int32_t w, int32_t h,
                          int64_t max_keys) {
  Layout L;
  if (!f || !workspace || ((uintptr_t)workspace & 255u) || !make_layout(n, w, h, max_keys, L) || bytes < L.total)
    return BGS_ERR_INVALID;
  memset(f, 0, sizeof(*f));
  Frame* F = frame_of(f);
  char* base = (char*)workspace;
  F->magic = kFrameMagic;
  F->n = n;
  F->max_keys = max_keys;
  F->W = w;
  F->H = h;
  F->tiles_x = L.tiles_x;
  F->tiles_y = L.tiles_y;
  F->num_tiles = L.num_tiles;
  F->sort_bits = L.sort_bits;
  F->sort_passes = L.sort_passes;
  F->scan_tiles = L.scan_tiles;
  F->sort_tiles_max = L.sort_tiles_max;
  F->radius = (int32_t*)(base + L.radius);
  F->depth = (float*)(base + L.depth);
  F->record = (float4*)(base + L.record);
  F->tiles_touched = (uint32_t*)(base + L.tiles_touched);
  F->rect = (uint2*)(base + L.rect);
  F->offsets = (uint32_t*)(base + L.offsets);
  F->keys[0] = (uint64_t*)(base + L.keys0);
  F->keys[1] = (uint64_t*)(base + L.keys1);
  F->vals[0] = (uint32_t*)(base + L.vals0);
  F->vals[1] = (uint32_t*)(base + L.vals1);
  F->ranges = (uint2*)(base + L.ranges);
  F->scan_status = (unsigned long long*)(base + L.scan_status);
  F->sort_hist = (uint32_t*)(base + L.sort_hist);
  F->sort_status = (uint32_t*)(base + L.sort_status);
  F->counters = (uint32_t*)(base + L.counters);
  F->plan = (uint32_t*)(base + L.plan);
  F->grad2d = (float4*)(base + L.grad2d);
  F->tile_count = (uint32_t*)(base + L.tile_count);
  F->order_fwd = (uint32_t*)(base + L.order_fwd);
  F->order_bwd = (uint32_t*)(base + L.order_bwd);
  F->block_cost = (uint32_t*)(base + L.block_cost);
  F->have_cost = 0;
  F->fwd_planned = F->bwd_planned = 0;
  F->grad2d_clean = 0;
  F->consume_g2 = 0;
  F->seg_len = L.num_tiles >= kSegLenTilesLarge ? kSegLenLargeFrame : kSegLenSmallFrame;
  F->ck_table = (uint32_t*)(base + L.ck_table);
  F->ck_pool = (float4*)(base + L.ck_pool);
  F->ck_cap = L.ck_cap;
  F->spec_base = (uint32_t*)(base + L.spec_base);
  F->spec_n = (uint32_t*)(base + L.spec_n);
  F->arrive = (uint32_t*)(base + L.arrive);
  F->spec_state = (float4*)(base + L.spec_state);
  F->spec_last = (uint32_t*)(base + L.spec_last);
  F->chunk_cnt = L.direct ? (uint32_t*)(base + L.chunk_cnt) : nullptr;
  F->dkey[0] = (uint32_t*)(base + L.dkey0);
  F->dkey[1] = (uint32_t*)(base + L.dkey1);
  F->dval[0] = (uint32_t*)(base + L.dval0);
  F->dval[1] = (uint32_t*)(base + L.dval1);
  F->rank_cnt = (uint32_t*)(base + L.rank_cnt);
  F->item_off = (uint32_t*)(base + L.item_off);
  F->rank_rect = (uint2*)(base + L.rank_rect);
  F->cbits = (uint8_t*)(base + L.cbits);
  F->rank_h = (uint32_t*)(base + L.rank_h);
  F->rs_tabA = (uint32_t*)(base + L.rs_tabA);
  F->rs_chunk_r0 = (uint32_t*)(base + L.rs_chunk_r0);
  F->rs_rows = (uint32_t*)(base + L.rs_rows);
  F->rs_units = (uint4*)(base + L.rs_units);
  F->rs_tabB = (uint32_t*)(base + L.rs_tabB);
  F->rs_status = (unsigned long long*)(base + L.rs_status);
  F->rs_max_units = L.rs_max_units;
  F->rs_scan_tiles = L.rs_scan_tiles;
  F->final_buf = L.sort_passes & 1;  // pass p reads buf p&1, writes buf (p+1)&1
  return BGS_OK;
}

bgs_status bgs_preprocess(const bgs_gaussians* g, const bgs_camera* cam, bgs_frame* f, void* stream) {
  if (!frame_ok(f)) return BGS_ERR_INVALID;
  Frame* F = frame_of(f);
  bgs_status st = validate_gaussians(g, F);
  if (st != BGS_OK) return st;
  if ((st = validate_camera(cam, F)) != BGS_OK) return st;
  F->cam = make_cam(*cam, F->tiles_x, F->tiles_y);
  F->cam_valid = 1;
  F->fwd_planned = F->bwd_planned = 0;
  return launch_preprocess(g, F, (cudaStream_t)stream);
}

bgs_status bgs_preprocess_batch(const bgs_gaussians* g, const bgs_camera* cams, bgs_frame* const* frames,
                                int32_t nframes, void* stream) {
  if (!cams || !frames || nframes < 1 || nframes > 4096) return BGS_ERR_INVALID;
  static thread_local Frame* F[4096];
  for (int v = 0; v < nframes; ++v) {
    if (!frame_ok(frames[v])) return BGS_ERR_INVALID;
    F[v] = frame_of(frames[v]);
    if (F[v]->n != F[0]->n) return BGS_ERR_INVALID;
    for (int u = 0; u < v; ++u)
      if (F[u] == F[v]) return BGS_ERR_INVALID;  // one frame twice would race on its outputs
  }
  bgs_status st = validate_gaussians(g, F[0]);
  if (st != BGS_OK) return st;
  for (int v = 0; v < nframes; ++v)
    if ((st = validate_camera(&cams[v], F[v])) != BGS_OK) return st;
  for (int v = 0; v < nframes; ++v) {
    F[v]->cam = make_cam(cams[v], F[v]->tiles_x, F[v]->tiles_y);
    F[v]->cam_valid = 1;
    F[v]->fwd_planned = F[v]->bwd_planned = 0;
  }
  return launch_preprocess_batch(g, F, nframes, (cudaStream_t)stream);
}

bgs_status bgs_sort(bgs_frame* f, void* stream) {
  if (!frame_ok(f) || !frame_of(f)->cam_valid) return BGS_ERR_INVALID;
  frame_of(f)->fwd_planned = frame_of(f)->bwd_planned = 0;
  return launch_sort(frame_of(f), (cudaStream_t)stream);
}

bgs_status bgs_render_fwd_plan(bgs_frame* f, void* stream) {
  if (!frame_ok(f) || !frame_of(f)->cam_valid) return BGS_ERR_INVALID;
  return launch_fwd_plan(frame_of(f), (cudaStream_t)stream);
}

bgs_status bgs_blend_bwd_plan(bgs_frame* f, void* stream) {
  if (!frame_ok(f) || !frame_of(f)->cam_valid) return BGS_ERR_INVALID;
  return launch_bwd_plan(frame_of(f), (cudaStream_t)stream);
}

bgs_status bgs_render_fwd(bgs_frame* f, float* image, float* final_T, uint32_t* n_contrib, void* stream) {
  if (!frame_ok(f) || !frame_of(f)->cam_valid || !image || !final_T || !n_contrib) return BGS_ERR_INVALID;
  return launch_render_fwd(frame_of(f), image, final_T, n_contrib, (cudaStream_t)stream);
}

bgs_status bgs_render_bwd(const bgs_gaussians* g, bgs_frame* f, const float* dL_dimage, const float* final_T,
                          const uint32_t* n_contrib, float* grad, void* stream) {
  if (!frame_ok(f) || !frame_of(f)->cam_valid || !dL_dimage || !final_T || !n_contrib) return BGS_ERR_INVALID;
  Frame* F = frame_of(f);
  bgs_status st = validate_gaussians(g, F);
  if (st != BGS_OK) return st;
  if (F->n > 0 && (!grad || ((uintptr_t)grad & 3u))) return BGS_ERR_INVALID;
  return launch_render_bwd(g, F, dL_dimage, final_T, n_contrib, grad, (cudaStream_t)stream);
}

bgs_status bgs_blend_bwd(bgs_frame* f, const float* dL_dimage, const float* final_T, const uint32_t* n_contrib,
                         void* stream) {
  if (!frame_ok(f) || !frame_of(f)->cam_valid || !dL_dimage || !final_T || !n_contrib) return BGS_ERR_INVALID;
  return launch_blend_bwd(frame_of(f), dL_dimage, final_T, n_contrib, (cudaStream_t)stream);
}

bgs_status bgs_preprocess_bwd(const bgs_gaussians* g, bgs_frame* f, float* grad, void* stream) {
  if (!frame_ok(f) || !frame_of(f)->cam_valid) return BGS_ERR_INVALID;
  Frame* F = frame_of(f);
  bgs_status st = validate_gaussians(g, F);
  if (st != BGS_OK) return st;
  if (F->n > 0 && (!grad || ((uintptr_t)grad & 3u))) return BGS_ERR_INVALID;
  return launch_preprocess_bwd(g, F, grad, (cudaStream_t)stream);
}

bgs_status bgs_preprocess_bwd_batch(const bgs_gaussians* g, bgs_frame* const* frames, int32_t nframes, float* grad,
                                    void* stream) {
  if (!frames || nframes < 1 || nframes > 4096) return BGS_ERR_INVALID;
  static thread_local Frame* F[4096];
  for (int v = 0; v < nframes; ++v) {
    if (!frame_ok(frames[v]) || !frame_of(frames[v])->cam_valid) return BGS_ERR_INVALID;
    F[v] = frame_of(frames[v]);
    if (F[v]->n != F[0]->n) return BGS_ERR_INVALID;
  }
  bgs_status st = validate_gaussians(g, F[0]);
  if (st != BGS_OK) return st;
  if (F[0]->n > 0 && (!grad || ((uintptr_t)grad & 3u))) return BGS_ERR_INVALID;
  return launch_preprocess_bwd_batch(g, F, nframes, grad, (cudaStream_t)stream);
}

bgs_status bgs_preprocess_bwd_batch_assign(const bgs_gaussians* g, bgs_frame* const* frames, int32_t nframes,
                                           float* grad, void* stream) {
  if (!frames || nframes < 1 || nframes > 4096) return BGS_ERR_INVALID;
  static thread_local Frame* F[4096];
  for (int v = 0; v < nframes; ++v) {
    if (!frame_ok(frames[v]) || !frame_of(frames[v])->cam_valid) return BGS_ERR_INVALID;
    F[v] = frame_of(frames[v]);
    if (F[v]->n != F[0]->n) return BGS_ERR_INVALID;
  }
  bgs_status st = validate_gaussians(g, F[0]);
  if (st != BGS_OK) return st;
  if (F[0]->n > 0 && (!grad || ((uintptr_t)grad & 3u))) return BGS_ERR_INVALID;
  return launch_preprocess_bwd_batch_impl(g, F, nframes, grad, nullptr, nullptr, nullptr, nullptr, 0,
                                          (cudaStream_t)stream, 0, -1, true);
}

bgs_status bgs_preprocess_bwd_batch_range(const bgs_gaussians* g, bgs_frame* const* frames, int32_t nframes,
                                          float* grad, int64_t begin, int64_t count, void* stream) {
  if (!frames || nframes < 1 || nframes > 4096 || begin < 0 || count < 0) return BGS_ERR_INVALID;
  static thread_local Frame* F[4096];
  for (int v = 0; v < nframes; ++v) {
    if (!frame_ok(frames[v]) || !frame_of(frames[v])->cam_valid) return BGS_ERR_INVALID;
    F[v] = frame_of(frames[v]);
    if (F[v]->n != F[0]->n) return BGS_ERR_INVALID;
  }
  if (begin + count > F[0]->n) return BGS_ERR_INVALID;
  bgs_status st = validate_gaussians(g, F[0]);
  if (st != BGS_OK) return st;
  if (count > 0 && (!grad || ((uintptr_t)grad & 3u))) return BGS_ERR_INVALID;
  return launch_preprocess_bwd_batch_impl(g, F, nframes, grad, nullptr, nullptr, nullptr, nullptr, 0,
                                          (cudaStream_t)stream, begin, begin + count);
}

bgs_status bgs_preprocess_bwd_batch_adam(const bgs_gaussians* g, bgs_frame* const* frames, int32_t nframes,
                                         float* theta, float* grad, float* exp_avg, float* exp_avg_sq,
                                         const bgs_adam_hparams* hp, int64_t step, void* stream) {
  if (!frames || nframes < 1 || nframes > 4096 || !hp || step < 1) return BGS_ERR_INVALID;
  static thread_local Frame* F[4096];
  for (int v = 0; v < nframes; ++v) {
    if (!frame_ok(frames[v]) || !frame_of(frames[v])->cam_valid) return BGS_ERR_INVALID;
    F[v] = frame_of(frames[v]);
    if (F[v]->n != F[0]->n) return BGS_ERR_INVALID;
  }
  bgs_status st = validate_gaussians(g, F[0]);
  if (st != BGS_OK) return st;
  const int64_t n = F[0]->n;
  if (n == 0) return BGS_OK;
  if (!theta || !exp_avg || !exp_avg_sq || (const float*)g->means != theta) return BGS_ERR_INVALID;
  if (nframes > kPreBwdMaxViews && (!grad || ((uintptr_t)grad & 3u))) return BGS_ERR_INVALID;
  if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f && hp->beta2 >= 0.0f && hp->beta2 < 1.0f && hp->eps >= 0.0f))
    return BGS_ERR_INVALID;
  return launch_preprocess_bwd_batch_impl(g, F, nframes, nframes > kPreBwdMaxViews ? grad : nullptr, theta,
                                          exp_avg, exp_avg_sq, hp, step, (cudaStream_t)stream);
}

bgs_status bgs_adam_step(float* theta, float* grad, float* exp_avg, float* exp_avg_sq, int64_t n,
                         const bgs_adam_hparams* hp, int64_t step, void* stream) {
  if (n < 0 || !hp || step < 1) return BGS_ERR_INVALID;
  if (n == 0) return BGS_OK;
  if (!theta || !grad || !exp_avg || !exp_avg_sq) return BGS_ERR_INVALID;
  if (!aligned16(theta) || !aligned16(grad) || !aligned16(exp_avg) || !aligned16(exp_avg_sq)) return BGS_ERR_INVALID;
  if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f && hp->beta2 >= 0.0f && hp->beta2 < 1.0f && hp->eps >= 0.0f))
    return BGS_ERR_INVALID;
  return launch_adam(theta, grad, exp_avg, exp_avg_sq, n, 0, 59 * n, hp, step, (cudaStream_t)stream);
}

bgs_status bgs_adam_step_keep_grad(float* theta, const float* grad, float* exp_avg, float* exp_avg_sq, int64_t n,
                                   const bgs_adam_hparams* hp, int64_t step, void* stream) {
  if (n < 0 || !hp || step < 1) return BGS_ERR_INVALID;
  if (n == 0) return BGS_OK;
  if (!theta || !grad || !exp_avg || !exp_avg_sq) return BGS_ERR_INVALID;
  if (!aligned16(theta) || !aligned16(grad) || !aligned16(exp_avg) || !aligned16(exp_avg_sq)) return BGS_ERR_INVALID;
  if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f && hp->beta2 >= 0.0f && hp->beta2 < 1.0f && hp->eps >= 0.0f))
    return BGS_ERR_INVALID;
  return launch_adam(theta, const_cast<float*>(grad), exp_avg, exp_avg_sq, n, 0, 59 * n, hp, step,
                     (cudaStream_t)stream, false);
}

bgs_status bgs_adam_step_range(float* theta, float* grad, float* exp_avg, float* exp_avg_sq, int64_t n,
                               int64_t begin, int64_t count, const bgs_adam_hparams* hp, int64_t step,
                               void* stream) {
  if (n < 0 || begin < 0 || count < 0 || (begin & 3) || !hp || step < 1) return BGS_ERR_INVALID;
  if (n == 0 || count == 0 || begin >= 59 * n) return BGS_OK;
  if (!theta || !grad || !exp_avg || !exp_avg_sq) return BGS_ERR_INVALID;
  if (!aligned16(theta) || !aligned16(grad) || !aligned16(exp_avg) || !aligned16(exp_avg_sq)) return BGS_ERR_INVALID;
  if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f && hp->beta2 >= 0.0f && hp->beta2 < 1.0f && hp->eps >= 0.0f))
    return BGS_ERR_INVALID;
  return launch_adam(theta, grad, exp_avg, exp_avg_sq, n, begin, count, hp, step, (cudaStream_t)stream);
}

bgs_status bgs_adam_step_multimem(float* theta, float* theta_mc, float* grad_mc, float* exp_avg, float* exp_avg_sq,
                                  int64_t n, int64_t begin, int64_t count, const bgs_adam_hparams* hp,
                                  int64_t step, void* stream) {
  if (n < 0 || begin < 0 || count < 0 || (begin & 3) || (count & 3) || !hp || step < 1) return BGS_ERR_INVALID;
  if (n == 0 || count == 0 || begin >= 59 * n) return BGS_OK;
  if (!theta || !theta_mc || !grad_mc || !exp_avg || !exp_avg_sq) return BGS_ERR_INVALID;
  if (!aligned16(theta) || !aligned16(theta_mc) || !aligned16(grad_mc) || !aligned16(exp_avg) ||
      !aligned16(exp_avg_sq) || ((59 * n - begin) < count && ((59 * n - begin) & 3)))
    return BGS_ERR_INVALID;
  if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f && hp->beta2 >= 0.0f && hp->beta2 < 1.0f && hp->eps >= 0.0f))
    return BGS_ERR_INVALID;
  return launch_adam_multimem(theta, theta_mc, grad_mc, exp_avg, exp_avg_sq, n, begin, count, hp, step,
                              (cudaStream_t)stream);
}

bgs_status bgs_zero(float* p, int64_t count, void* stream) {
  if (count < 0 || (count > 0 && !p)) return BGS_ERR_INVALID;
  if (count == 0) return BGS_OK;
  if (cudaMemsetAsync(p, 0, (size_t)count * sizeof(float), (cudaStream_t)stream) != cudaSuccess)
    return check_launch("bgs_zero");
  return BGS_OK;
}

bgs_status bgs_l1_loss_grad(const float* image, const uint8_t* target, int32_t w, int32_t h, float scale,
                            float* dL_dimage, float* loss_sum, void* stream) {
  if (!image || !target || !dL_dimage || !loss_sum || w < 1 || h < 1 || w > 16384 || h > 16384)
    return BGS_ERR_INVALID;
  return launch_l1(image, target, w, h, scale, dL_dimage, loss_sum, (cudaStream_t)stream);
}

size_t bgs_loss_workspace_bytes(int32_t w, int32_t h) {
  if (w < 1 || h < 1 || w > 16384 || h > 16384) return 0;
  return loss_workspace_bytes(w, h);
}

bgs_status bgs_l1_dssim_loss_grad(const float* image, const uint8_t* target, int32_t w, int32_t h, float lambda,
                                  float scale, float* dL_dimage, float* loss_sum, void* workspace, size_t bytes,
                                  void* stream) {
  if (!image || !target || !dL_dimage || !loss_sum || !workspace || w < 1 || h < 1 || w > 16384 || h > 16384)
    return BGS_ERR_INVALID;
  if (((uintptr_t)workspace & 255u) || bytes < loss_workspace_bytes(w, h)) return BGS_ERR_INVALID;
  if (!(lambda >= 0.0f && lambda <= 1.0f)) return BGS_ERR_INVALID;
  return launch_l1_dssim(image, target, w, h, lambda, scale, dL_dimage, loss_sum, workspace, (cudaStream_t)stream);
}

bgs_status bgs_frame_status(const bgs_frame* f, int64_t* num_keys) {
  if (!frame_ok(f) || !num_keys) return BGS_ERR_INVALID;
  const Frame* F = frame_of(f);
  uint32_t c[C_NUM];
  if (cudaMemcpy(c, F->counters, sizeof(c), cudaMemcpyDeviceToHost) != cudaSuccess)
    return check_launch("bgs_frame_status");
  *num_keys = (int64_t)(((uint64_t)c[C_K_HI] << 32) | c[C_K_LO]);
  const bool sticky = F->counters_init && c[C_OVF_STICKY];
  if (sticky && cudaMemset(F->counters + C_OVF_STICKY, 0, 4) != cudaSuccess) return check_launch("bgs_frame_status");
  return (c[C_OVERFLOW] || sticky) ? BGS_ERR_CAPACITY : BGS_OK;
}

size_t bgs_frame_hint_bytes(const bgs_frame* f) {
  return frame_ok(f) ? 4 * 8 * (size_t)frame_of(f)->num_tiles : 0;
}

bgs_status bgs_frame_save_hint(const bgs_frame* f, void* dst, void* stream) {
  if (!frame_ok(f) || !dst) return BGS_ERR_INVALID;
  const Frame* F = frame_of(f);
  if (cudaMemcpyAsync(dst, F->block_cost, bgs_frame_hint_bytes(f), cudaMemcpyDeviceToDevice,
                      (cudaStream_t)stream) != cudaSuccess)
    return check_launch("bgs_frame_save_hint");
  return BGS_OK;
}

bgs_status bgs_frame_load_hint(bgs_frame* f, const void* src, void* stream) {
  if (!frame_ok(f)) return BGS_ERR_INVALID;
  Frame* F = frame_of(f);
  F->fwd_planned = 0;
  if (!src) {
    F->have_cost = 0;
    return BGS_OK;
  }
  if (cudaMemcpyAsync(F->block_cost, src, bgs_frame_hint_bytes(f), cudaMemcpyDeviceToDevice,
                      (cudaStream_t)stream) != cudaSuccess)
    return check_launch("bgs_frame_load_hint");
  F->have_cost = 1;
  return BGS_OK;
}

bgs_status bgs_frame_debug(const bgs_frame* f, bgs_frame_views* out) {
  if (!frame_ok(f) || !out) return BGS_ERR_INVALID;
  const Frame* F = frame_of(f);
  out->radius = F->radius;
  out->depth = F->depth;
  out->record = (float*)F->record;
  out->tiles_touched = F->tiles_touched;
  out->offsets = F->offsets;
  out->keys_unsorted = F->keys[0];
  out->values_unsorted = F->vals[0];
  out->keys_sorted = F->keys[F->final_buf];
  out->values_sorted = F->vals[F->final_buf];
  out->ranges = (uint32_t*)F->ranges;
  out->grad2d = (float*)F->grad2d;
  out->n = F->n;
  out->max_keys = F->max_keys;
  out->tiles_x = F->tiles_x;
  out->tiles_y = F->tiles_y;
  out->sort_bits = F->sort_bits;
  out->sort_passes = F->sort_passes;
  out->sort_mode = F->sort_mode;
  out->cbits = F->cbits;
  return BGS_OK;
}

bgs_status bgs_frame_set_debug(bgs_frame* f, int32_t flags) {
  if (!frame_ok(f)) return BGS_ERR_INVALID;
  frame_of(f)->debug_flags = flags;
  frame_of(f)->fwd_planned = frame_of(f)->bwd_planned = 0;
  return BGS_OK;
}

bgs_status bgs_frame_set_consume(bgs_frame* f, int32_t on) {
  if (!frame_ok(f)) return BGS_ERR_INVALID;
  frame_of(f)->consume_g2 = on ? 1 : 0;
  frame_of(f)->grad2d_clean = 0;  // unknown until the next preprocess zeroes it
  return BGS_OK;
}

bgs_status bgs_frame_set_seg_len(bgs_frame* f, int32_t seg_len) {
  if (!frame_ok(f) || seg_len < 32 || seg_len > 65536 || (seg_len & 31)) return BGS_ERR_INVALID;
  frame_of(f)->seg_len = seg_len;
  frame_of(f)->fwd_planned = frame_of(f)->bwd_planned = 0;
  return BGS_OK;
}

bgs_status bgs_frame_validate(const bgs_frame* f, uint64_t* out, void* stream) {
  if (!frame_ok(f) || !out || (reinterpret_cast<uintptr_t>(out) & 7u)) return BGS_ERR_INVALID;
  return launch_validate(frame_of(f), reinterpret_cast<unsigned long long*>(out), (cudaStream_t)stream);
}

bgs_status bgs_frame_stats(const bgs_frame* f, const uint32_t* n_contrib, bgs_stats* out, void* stream) {
  if (!frame_ok(f) || !n_contrib || !out) return BGS_ERR_INVALID;
  return launch_stats(frame_of(f), n_contrib, out, (cudaStream_t)stream);
}

}  // extern "C"
