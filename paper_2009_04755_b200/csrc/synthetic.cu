// SyntheticApp compare (bit-exact restatement of apps.py:201-208) and the
// deterministic PRNU-like pattern generator used for synthetic workloads.
#include <math.h>

#include <algorithm>

#include "internal.h"

namespace rk {

// splitmix64 rounds of rng.mix64 (/root/reference/pkg/src/allpairs/rng.py:15-25).
__host__ __device__ __forceinline__ uint64_t mix_round(uint64_t x, uint64_t v) {
  x = x + v + 0x9E3779B97F4A7C15ull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
__host__ __device__ __forceinline__ uint64_t mix64_4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t x = 0x9E3779B97F4A7C15ull;
  x = mix_round(x, a);
  x = mix_round(x, b);
  x = mix_round(x, c);
  return mix_round(x, d);
}

namespace {

// value = mix64(seed, 0xC0403A3E, i, j) / 2^64 ; Python converts the int to the
// nearest double (ties to even) before the exact power-of-two division.
__global__ void synth_compare_kernel(PairBatch b, uint64_t seed, double* __restrict__ out, uint8_t* __restrict__ flags,
                                     double threshold, const LedgerRef ledger) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= b.npairs) return;
  const uint64_t h = mix64_4(seed, 0xC0403A3Eull, (uint64_t)(int64_t)b.key_i[p], (uint64_t)(int64_t)b.key_j[p]);
  const double v = __ull2double_rn(h) * 0x1p-64;
  out[b.pid[p]] = v;
  ledger_mark(ledger, b.pid[p]);
  if (flags) flags[b.pid[p]] = isnan(threshold) ? 0 : (uint8_t)(1 | (v >= threshold ? 2 : 0));
}

// Dense-range variant used by tiles: every pair (i, j) with r0 <= i < r1, c0 <= j < c1, i < j.
__global__ void synth_tile_kernel(int64_t n, int32_t r0, int32_t r1, int32_t c0, int32_t c1, uint64_t seed,
                                  double* __restrict__ out, uint8_t* __restrict__ flags, double threshold,
                                  const LedgerRef ledger) {
  const int64_t w = c1 - c0;
  const int64_t total = (int64_t)(r1 - r0) * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = r0 + t / w, j = c0 + t % w;
    if (i >= j) continue;
    const uint64_t h = mix64_4(seed, 0xC0403A3Eull, (uint64_t)i, (uint64_t)j);
    const double v = __ull2double_rn(h) * 0x1p-64;
    const int64_t pid = pair_id(n, i, j);
    out[pid] = v;
    ledger_mark(ledger, pid);
    if (flags) flags[pid] = isnan(threshold) ? 0 : (uint8_t)(1 | (v >= threshold ? 2 : 0));
  }
}

__device__ __forceinline__ float normal_from_hash(uint64_t h) {
  // two 24-bit uniforms in (0,1), Box-Muller (cos branch)
  const float u1 = ((float)(h >> 40) + 0.5f) * 0x1p-24f;
  const float u2 = ((float)((h >> 16) & 0xFFFFFFull) + 0.5f) * 0x1p-24f;
  return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

constexpr float kPrnuGain = 0.2f;  // PRNU amplitude relative to unit-variance noise

// One CTA row (blockIdx.y) per item: the key / camera are per-thread constants
// (no 64-bit division per element); four consecutive pixels per thread, one
// float4 store.  The values are those of the scalar definition bit for bit.
__global__ void __launch_bounds__(256) synth_prnu_kernel(int64_t hw, int32_t first_key, int32_t cameras,
                                                         uint64_t seed, float* __restrict__ out) {
  const int64_t key = first_key + (int64_t)blockIdx.y;
  const uint64_t cam = (uint64_t)(key % cameras);
  float* o = out + (int64_t)blockIdx.y * hw;
  for (int64_t p4 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; p4 < hw;
       p4 += (int64_t)gridDim.x * blockDim.x * 4) {
    float r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t pix = (uint64_t)(p4 + q);
      const float k = normal_from_hash(mix64_4(seed, 0x50524E55ull, cam, pix));
      const float e = normal_from_hash(mix64_4(seed, 0x4E4F4953ull, (uint64_t)key, pix));
      r[q] = fmaf(kPrnuGain, k, e);
    }
    if (p4 + 3 < hw) {
      *reinterpret_cast<float4*>(o + p4) = make_float4(r[0], r[1], r[2], r[3]);
    } else {
      for (int q = 0; q < 4 && p4 + q < hw; ++q) o[p4 + q] = r[q];
    }
  }
}

}  // namespace

rk_status synth_compare(rk_app* app, const PairBatch& b, double* d_out, uint8_t* d_flags, cudaStream_t s) {
  synth_compare_kernel<<<(b.npairs + 63) / 64, 64, 0, s>>>(b, app->p.seed, d_out, d_flags, threshold_or_nan(app), app->ledger);
  app->launches += 1;
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

rk_status synth_tile(rk_app* app, int32_t r0, int32_t r1, int32_t c0, int32_t c1, double* d_out, uint8_t* d_flags,
                     cudaStream_t s) {
  const int64_t total = (int64_t)(r1 - r0) * (c1 - c0);
  if (total <= 0) return RK_OK;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  synth_tile_kernel<<<blocks, 256, 0, s>>>(app->p.n, r0, r1, c0, c1, app->p.seed, d_out, d_flags,
                                           threshold_or_nan(app), app->ledger);
  app->launches += 1;
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

rk_status synth_prnu(int32_t h, int32_t w, int32_t first_key, int32_t n_items, int32_t cameras, uint64_t seed,
                     float* d_out, cudaStream_t s) {
  const int64_t hw = (int64_t)h * w;
  if (n_items <= 0 || hw <= 0) return RK_OK;
  if (((uintptr_t)d_out & 15) != 0 || hw % 4 != 0)
    return set_error(RK_ERR_VALUE, "synthetic patterns: 16-byte aligned output and h*w % 4 == 0 required");
  int bx = (int)std::min<int64_t>((hw / 4 + 255) / 256, std::max<int64_t>(1, 148 * 8 / std::max(1, n_items)));
  bx = std::max(bx, 1);
  for (int32_t i0 = 0; i0 < n_items; i0 += 65535) {
    const int32_t m = std::min(65535, n_items - i0);
    synth_prnu_kernel<<<dim3(bx, m), 256, 0, s>>>(hw, first_key + i0, cameras, seed, d_out + (int64_t)i0 * hw);
  }
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

}  // namespace rk
