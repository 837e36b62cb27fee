// check.cu -- failure detection: a structural check of a frame's sorted tile
// lists and a non-finite count for gradients.  Neither is on the hot path; both are
// device-side, asynchronous, and report counts into a caller-owned device buffer.
//
// The list check restates what a4-a6 must produce (§II-A: "N denotes the
// set of Gaussians contributing to the pixel, sorted by depth"; per 16x16 tile; ties
// by index, R13): every tile's list holds exactly the visible Gaussians whose
// tile rect covers the tile, in strictly increasing (depth bits, index) order, and the
// ranges cut [0, K) into consecutive per-tile runs in tile order.  Distinct members (strict
// order) of each tile's true set whose counts sum to K = sum of tiles_touched are each tile's
// whole set, so the four counts below being zero proves the lists.
#include "common.cuh"

namespace bgs {

constexpr int kValThreads = 256;

__device__ __forceinline__ uint64_t load_k64(const uint32_t* counters) {
  return ((uint64_t)counters[C_K_HI] << 32) | counters[C_K_LO];
}

// one CTA per tile: membership and order of the tile's list
__global__ void __launch_bounds__(kValThreads) k_validate_lists(const uint2* __restrict__ ranges,
                                                                const uint32_t* __restrict__ vals,
                                                                const int32_t* __restrict__ radius,
                                                                const float* __restrict__ depth,
                                                                const uint2* __restrict__ rect, int64_t n,
                                                                int32_t tiles_x, const uint32_t* counters,
                                                                unsigned long long* out) {
  const int t = blockIdx.x;
  const uint64_t K = load_k64(counters);
  const uint2 rg = ranges[t];
  const uint32_t tx = (uint32_t)(t % tiles_x), ty = (uint32_t)(t / tiles_x);
  if (rg.x > rg.y || rg.y > K) return;  // a range outside [0, K): counted by k_validate_ranges
  unsigned long long member = 0, order = 0;
  for (uint32_t p = rg.x + threadIdx.x; p < rg.y; p += kValThreads) {
    const uint32_t id = vals[p];
    bool ok = (int64_t)id < n && radius[id] > 0;
    if (ok) {
      const uint2 q = rect[id];  // {x0 | y0 << 16, w | h << 16}
      const uint32_t x0 = q.x & 0xffffu, y0 = q.x >> 16, w = q.y & 0xffffu, h = q.y >> 16;
      ok = tx >= x0 && tx < x0 + w && ty >= y0 && ty < y0 + h;
    }
    member += !ok;
    if (p + 1 < rg.y && ok) {
      const uint32_t id2 = vals[p + 1];
      if ((int64_t)id2 < n) {
        const uint32_t d1 = __float_as_uint(depth[id]), d2 = __float_as_uint(depth[id2]);
        order += !(d1 < d2 || (d1 == d2 && id < id2));
      }
    }
  }
  if (member) atomicAdd(&out[1], member);
  if (order) atomicAdd(&out[2], order);
}

// one CTA: the ranges are consecutive in tile order and cover [0, K); K = sum tiles_touched
__global__ void __launch_bounds__(1024) k_validate_ranges(const uint2* __restrict__ ranges, int32_t nt,
                                                          const uint32_t* counters, unsigned long long* out) {
  __shared__ uint32_t s_first[1024], s_last[1024];
  __shared__ unsigned long long s_bad;
  const uint64_t K = load_k64(counters);
  const int per = (nt + 1023) / 1024;
  const int t0 = threadIdx.x * per, t1 = min(nt, t0 + per);
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  uint32_t first = 0xffffffffu, last = 0xffffffffu;  // first start / last end of the chunk's non-empty tiles
  unsigned long long bad = 0;
  for (int t = t0; t < t1; ++t) {
    const uint2 rg = ranges[t];
    if (rg.x > rg.y || rg.y > K) {
      ++bad;
      continue;
    }
    if (rg.x == rg.y) {
      bad += rg.x != 0;  // empty tiles hold (0, 0)
      continue;
    }
    if (first == 0xffffffffu) first = rg.x;
    else bad += rg.x != last;
    last = rg.y;
  }
  s_first[threadIdx.x] = first;
  s_last[threadIdx.x] = last;
  if (bad) atomicAdd(&s_bad, bad);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t end = 0;  // where the next non-empty tile must start
    unsigned long long b = s_bad;
    for (int c = 0; c < 1024; ++c) {
      if (s_first[c] == 0xffffffffu) continue;
      b += s_first[c] != end;
      end = s_last[c];
    }
    b += (uint64_t)end != K;
    out[0] = b;
  }
}

// sum of tiles_touched (R11': the keys the preprocess asked for) against K
__global__ void k_validate_count(const uint32_t* __restrict__ tiles_touched, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += tiles_touched[i];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&out[4], c);
}

__global__ void k_validate_finish(const uint32_t* counters, unsigned long long* out) {
  out[3] = out[4] != load_k64(counters) ? 1ull : 0ull;
}

bgs_status launch_validate(const Frame* F, unsigned long long* out, cudaStream_t s) {
  if (cudaMemsetAsync(out, 0, 5 * sizeof(unsigned long long), s) != cudaSuccess) return check_launch("validate memset");
  k_validate_ranges<<<1, 1024, 0, s>>>(F->ranges, F->num_tiles, F->counters, out);
  k_validate_lists<<<F->num_tiles, kValThreads, 0, s>>>(F->ranges, F->vals[F->final_buf], F->radius, F->depth,
                                                        F->rect, F->n, F->tiles_x, F->counters, out);
  if (F->n > 0) k_validate_count<<<num_sms() * 4, 256, 0, s>>>(F->tiles_touched, F->n, out);
  k_validate_finish<<<1, 1, 0, s>>>(F->counters, out);
  note_launch(F->n > 0 ? 4 : 3);
  return check_launch("k_validate");
}

// ---------------------------------------------------------------- non-finite values
__global__ void k_nonfinite(const float* __restrict__ x, int64_t count, unsigned long long* out) {
  unsigned long long c = 0, first = ~0ull;
  const int64_t n4 = count / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = x4[i];
    const bool b0 = !isfinite(v.x), b1 = !isfinite(v.y), b2 = !isfinite(v.z), b3 = !isfinite(v.w);
    c += (unsigned)b0 + b1 + b2 + b3;
    if (b0 | b1 | b2 | b3) {
      const unsigned long long f = 4 * (unsigned long long)i + (b0 ? 0 : b1 ? 1 : b2 ? 2 : 3);
      first = f < first ? f : first;
    }
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) {
      ++c;
      first = (unsigned long long)i < first ? (unsigned long long)i : first;
    }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, d);
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, first, d);
    first = o < first ? o : first;
  }
  if ((threadIdx.x & 31) == 0 && c) {
    atomicAdd(&out[0], c);
    atomicMin(&out[1], first);
  }
}

}  // namespace bgs

extern "C" {

bgs_status bgs_nonfinite(const float* x, int64_t count, uint64_t* out64, void* stream) {
  using namespace bgs;
  unsigned long long* out = reinterpret_cast<unsigned long long*>(out64);
  if (count < 0 || !out || (count > 0 && !x) || (reinterpret_cast<uintptr_t>(x) & 15u)) return BGS_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(out, 0, 8, s) != cudaSuccess || cudaMemsetAsync(out + 1, 0xff, 8, s) != cudaSuccess)
    return check_launch("nonfinite init");
  if (count == 0) return BGS_OK;
  k_nonfinite<<<num_sms() * 8, 256, 0, s>>>(x, count, out);
  note_launch();
  return check_launch("k_nonfinite");
}

}  // extern "C"
