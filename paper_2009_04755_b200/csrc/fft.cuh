// Warp-resident complex FFT building blocks for sm_100a.
//
// An N-point transform with N = R*R is computed by a "group" of R lanes
// (R = 32: one warp; R = 16: half a warp) as a four-step FFT:
//   lane n1 holds x[n1 + R*n2] for n2 = 0..R-1 in registers,
//   (1) R-point DFT over n2 in registers (fully unrolled radix-2, constant twiddles),
//   (2) twiddle by W_N^(n1*k1) from a [k1][n1] table (bank-conflict free),
//   (3) transpose through a padded (R+1)-stride shared buffer,
//   (4) R-point DFT over n1 in registers.
// On exit lane k1 holds X[k1 + R*k2] in v[k2] -- the same distribution as the
// input, so callers load/store with lane-contiguous (coalesced) addresses.
//
// The transforms are unnormalised. Forward uses W = exp(-2*pi*i/N), inverse
// exp(+2*pi*i/N), matching numpy.fft (minus numpy's 1/N on the inverse).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rk {

__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 c_mulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 c_conj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 c_scale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

// (cos, sin)(2*pi*m/32) for m in [0, 16); m is a compile-time constant after unrolling.
__device__ __forceinline__ float2 unit32(int m) {
  switch (m) {
    case 1: return make_float2(9.807852804e-01f, 1.950903220e-01f);
    case 2: return make_float2(9.238795325e-01f, 3.826834324e-01f);
    case 3: return make_float2(8.314696123e-01f, 5.555702330e-01f);
    case 4: return make_float2(7.071067812e-01f, 7.071067812e-01f);
    case 5: return make_float2(5.555702330e-01f, 8.314696123e-01f);
    case 6: return make_float2(3.826834324e-01f, 9.238795325e-01f);
    case 7: return make_float2(1.950903220e-01f, 9.807852804e-01f);
    case 9: return make_float2(-1.950903220e-01f, 9.807852804e-01f);
    case 10: return make_float2(-3.826834324e-01f, 9.238795325e-01f);
    case 11: return make_float2(-5.555702330e-01f, 8.314696123e-01f);
    case 12: return make_float2(-7.071067812e-01f, 7.071067812e-01f);
    case 13: return make_float2(-8.314696123e-01f, 5.555702330e-01f);
    case 14: return make_float2(-9.238795325e-01f, 3.826834324e-01f);
    case 15: return make_float2(-9.807852804e-01f, 1.950903220e-01f);
    default: return make_float2(1.0f, 0.0f);
  }
}

// d * W_32^m with W = exp(-+2*pi*i/32); trivial angles are special-cased so the
// unrolled butterflies carry no multiplications by 0 or 1.
template <bool INV>
__device__ __forceinline__ float2 tw32_mul(float2 d, int m) {
  constexpr float kH = 7.071067812e-01f;
  if (m == 0) return d;
  if (m == 8) return INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
  if (m == 4) return INV ? make_float2(kH * (d.x - d.y), kH * (d.x + d.y))
                         : make_float2(kH * (d.x + d.y), kH * (d.y - d.x));
  if (m == 12) return INV ? make_float2(-kH * (d.x + d.y), kH * (d.x - d.y))
                          : make_float2(kH * (d.y - d.x), -kH * (d.x + d.y));
  float2 w = unit32(m);
  if (!INV) w.y = -w.y;
  return c_mul(d, w);
}

__host__ __device__ constexpr int bitrev_const(int i, int logn) {
  int r = 0;
  for (int b = 0; b < logn; ++b) r |= ((i >> b) & 1) << (logn - 1 - b);
  return r;
}

template <int N>
struct Log2 {
  static constexpr int value = (N <= 1) ? 0 : 1 + Log2<N / 2>::value;
};
template <>
struct Log2<1> {
  static constexpr int value = 0;
};

// In-register DFT of size N <= 32 (radix-2 decimation in frequency), natural order in and out.
template <int N, bool INV>
__device__ __forceinline__ void dft_regs(float2 (&v)[N]) {
  static_assert(N >= 2 && N <= 32 && (N & (N - 1)) == 0, "register DFT size");
#pragma unroll
  for (int span = N / 2; span >= 1; span >>= 1) {
#pragma unroll
    for (int start = 0; start < N; start += 2 * span) {
#pragma unroll
      for (int k = 0; k < span; ++k) {
        const float2 a = v[start + k];
        const float2 b = v[start + k + span];
        v[start + k] = c_add(a, b);
        v[start + k + span] = tw32_mul<INV>(c_sub(a, b), k * (32 / (2 * span)));
      }
    }
  }
  float2 t[N];
#pragma unroll
  for (int i = 0; i < N; ++i) t[i] = v[bitrev_const(i, Log2<N>::value)];
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = t[i];
}

// Four-step N = R*R complex FFT over a group of R lanes (see file header).
//   v     : lane's R elements, v[n2] = x[lane + R*n2] on entry, X[lane + R*k2] on exit
//   xbuf  : this group's R*(R+1) float2 shared scratch
//   tw    : shared [k1][n1] table of W_N^(n1*k1) (forward sign), R*R entries
// All lanes of the warp must call this together (uses __syncwarp()).
template <int R, bool INV>
__device__ __forceinline__ void group_fft(float2 (&v)[R], float2* xbuf, const float2* tw, int lane) {
  dft_regs<R, INV>(v);
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) {
    float2 w = tw[k1 * R + lane];
    if (INV) w.y = -w.y;
    v[k1] = c_mul(v[k1], w);
  }
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) xbuf[lane * (R + 1) + k1] = v[k1];
  __syncwarp();
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = xbuf[n1 * (R + 1) + lane];
  __syncwarp();
  dft_regs<R, INV>(v);
}

}  // namespace rk
