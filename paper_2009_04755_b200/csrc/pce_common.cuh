// Device helpers shared by the PCE compare kernels (pce.cu: 256^2 / 1024^2,
// pce2k.cu: 2048^2).  See pce.cu for the definitions of the score.
#pragma once

#include <math.h>
#include <stdint.h>

#include "fft.cuh"

namespace rk {
namespace pcek {

constexpr int kWin = 11;                // PCE exclusion neighbourhood side
constexpr int kHalfWin = kWin / 2;
constexpr int kMeanParts = 64;          // CTAs per item in the mean reduction

// Refilling a staging buffer that other threads have just READ with generic
// loads: the barrier before the refill orders the loads' issue, not their
// completion, so the TMA (async proxy) write can overtake a load still in flight
// (measured: without a fence 2-3 of 2,556 PCE values per 256^2 job differed from
// run to run, up to 5e-4 relative; tools/pce_determinism.py).  The issuing thread
// therefore fences generic -> async proxy on shared memory before every refill
// (1, default: fence.proxy.async.shared::cta; 2: the full fence.proxy.async;
// 0: none -- racy, kept only for the A/B record in DESIGN.md).
#ifndef PCE_REFILL_FENCE
#define PCE_REFILL_FENCE 1
#endif
__device__ __forceinline__ void refill_fence() {
  if (PCE_REFILL_FENCE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (PCE_REFILL_FENCE == 2) fence_proxy_async();
}

// Row-phase unpack and energy sums on packed pairs (with RK_F32X2).
#ifndef PCE_X2_ROWS
#define PCE_X2_ROWS 1
#endif

__device__ __forceinline__ bool better(float v, int idx, float bv, int bidx) {
  return v > bv || (v == bv && idx < bidx);
}

// ---------------------------------------------------------------------------
// T (the column pass output) layout per pair: blocks of 8 rows; block rb holds
// all N/2 columns x 8 rows, the 8 rows of one column in 64 contiguous bytes
// whose four 16-byte row-pair chunks are XOR-swizzled by ((column >> 1) & 3), so
// eight consecutive columns of one row pair hit eight distinct bank groups.  A
// column FFT stores four 64-B segments per warp instruction; an 8-row block is
// one contiguous bulk copy (TMA) feeding four warps, one row pair each.
template <int N>
__device__ __forceinline__ size_t t_index8(int r, int c) {
  const int rb = r >> 3, rr = r & 7;
  const int pos = (((rr >> 1) ^ ((c >> 1) & 3)) << 1) | (rr & 1);
  return ((size_t)rb * (N / 2) + c) * 8 + pos;
}

// Z[k] = A[k] + i*B[k] for row pair rp (rows 2rp, 2rp+1) of a staged 8-row block
// ([c][8] with the chunk swizzle), Hermitian-extended; column 0 packs DC + i*Nyquist.
template <int R>
__device__ __forceinline__ void block8_rows_z(float2 (&v)[R], const float2* blk, int rp, int lane) {
  constexpr int N = R * R;
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    const int k = lane + R * n2;
    int kk = (n2 < R / 2) ? k : N - k;
    if (kk >= N / 2) kk = 0;   // lane 0 at k = N/2: the Nyquist value lives in column 0
    const float4 q = *reinterpret_cast<const float4*>(blk + kk * 8 + 2 * (rp ^ ((kk >> 1) & 3)));
    float2 a = make_float2(q.x, q.y), c = make_float2(q.z, q.w);
    if (n2 >= R / 2) {
      a.y = -a.y;
      c.y = -c.y;
    }
    if (kk == 0) {
      a = make_float2(n2 == 0 ? q.x : q.y, 0.f);
      c = make_float2(n2 == 0 ? q.z : q.w, 0.f);
    }
#if PCE_X2_ROWS
    v[n2] = c_add(a, make_float2(-c.y, c.x));   // a + i*c
#else
    v[n2] = make_float2(a.x - c.y, a.y + c.x);
#endif
  }
}

// ---------------------------------------------------------------------------
// Round barrier of the persistent compare grids.  Round k of a launch is pairs
// [k*G, (k+1)*G) (one per CTA); with `rounds` set, a CTA starts its round-k pair
// only when all G CTAs have finished round k-1, so the in-flight pairs (which the
// engine's leaf order draws from a few items) read the same spectrum columns at
// the same time and share them through L2 instead of drifting apart.  It is a
// timing barrier only: a CTA stops waiting after kRoundSpin cycles, so partial
// residency (another kernel holding SMs) can slow it but never deadlock it.
#ifndef PCE_ROUND_SPIN
#define PCE_ROUND_SPIN 200000
#endif
constexpr long long kRoundSpin = PCE_ROUND_SPIN;
// Round-barrier slack, % of the grid (measured: 10 at 1024^2 +0.6 %;
// at 2048^2 any slack loses L2 reuse: 0).
#ifndef PCE_ROUND_SLACK_PCT
#define PCE_ROUND_SLACK_PCT 10
#endif
#ifndef PCE2K_ROUND_SLACK_PCT
#define PCE2K_ROUND_SLACK_PCT 0
#endif
__device__ __forceinline__ void round_wait(const unsigned* rounds, int pi, int G, int tid, int slack_pct) {
  if (rounds == nullptr || pi < G) return;
  if (tid == 0) {
    // arrivals of rounds 0 .. k-1, less a slack of slack_pct % of the grid (a CTA
    // may start round k while the last few CTAs finish round k-1)
    const unsigned slack = (unsigned)(G * slack_pct / 100);
    const unsigned target = (unsigned)(pi / G) * (unsigned)G - slack;
    const long long t0 = clock64();
    while (ld_acquire(rounds) < target && clock64() - t0 < kRoundSpin) __nanosleep(64);
  }
  __syncthreads();
}
__device__ __forceinline__ void round_arrive(unsigned* rounds, int tid) {
  if (rounds != nullptr && tid == 0) red_release_add(rounds, 1u);
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

struct ArgMax {
  float v;
  int idx;
};

__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, a.v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, a.idx, o);
    if (better(ov, oi, a.v, a.idx)) {
      a.v = ov;
      a.idx = oi;
    }
  }
  return a;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Running (max, first index, sum of squares) over one row pair of C.
template <int R>
__device__ __forceinline__ void argmax_update(const float2 (&v)[R], int ra, int lane, float& m, int& idx, float& ss) {
  constexpr int N = R * R;
  float lm = -INFINITY;
#if RK_F32X2 && PCE_X2_ROWS
  float2 s2 = make_float2(0.f, 0.f);   // even / odd row sums, one FFMA2 per element
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) {
    s2 = __ffma2_rn(v[k2], v[k2], s2);
    lm = fmaxf(lm, fmaxf(v[k2].x, v[k2].y));
  }
  ss += s2.x + s2.y;
#else
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) {
    ss = fmaf(v[k2].x, v[k2].x, ss);
    ss = fmaf(v[k2].y, v[k2].y, ss);
    lm = fmaxf(lm, fmaxf(v[k2].x, v[k2].y));
  }
#endif
  if (lm >= m) {
    int li = 0x7fffffff;
#pragma unroll
    for (int k2 = R - 1; k2 >= 0; --k2)
      if (v[k2].x == lm) li = ra * N + lane + R * k2;
    if (li == 0x7fffffff) {
#pragma unroll
      for (int k2 = R - 1; k2 >= 0; --k2)
        if (v[k2].y == lm) li = (ra + 1) * N + lane + R * k2;
    }
    if (lm > m || li < idx) {
      m = lm;
      idx = li;
    }
  }
}

}  // namespace pcek
}  // namespace rk
