// Warp-resident complex FFT building blocks for sm_100a.
//
// An N-point transform with N = R*R is computed by a "group" of R lanes
// (R = 32: one warp; R = 16: half a warp) as a four-step FFT:
//   lane n1 holds x[n1 + R*n2] for n2 = 0..R-1 in registers,
//   (1) R-point DFT over n2 in registers (fully unrolled radix-2, constant twiddles),
//   (2) twiddle by W_N^(n1*k1) from a [k1][n1] table (bank-conflict free),
//   (3) transpose through an XOR-swizzled R x R shared buffer (conflict-free
//       for 64-bit accesses: half-warp phases hit 16 distinct bank pairs),
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

// Complex arithmetic on packed fp32 pairs.  sm_100a issues one FADD2 / FMUL2 /
// FFMA2 for both halves of a float2 and encodes scalar broadcast, half swap and
// partial negation as operand modifiers, so a complex add is one instruction and
// a complex multiply two (instead of two and four scalar ones).  -DRK_F32X2=0
// restores the scalar forms (identical results up to FMA contraction order).
#ifndef RK_F32X2
#define RK_F32X2 1
#endif
#ifndef RK_F32X2_MUL
#define RK_F32X2_MUL RK_F32X2
#endif
#if RK_F32X2
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 c_scale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
#else
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 c_scale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
#endif
#if RK_F32X2_MUL
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), b));
}
// a * conj(b) = b.x * a - b.y * (-a.y, a.x)
__device__ __forceinline__ float2 c_mulc(float2 a, float2 b) {
  return __ffma2_rn(make_float2(-b.y, -b.y), make_float2(-a.y, a.x), __fmul2_rn(make_float2(b.x, b.x), a));
}
#else
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 c_mulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
#endif
__device__ __forceinline__ float2 c_conj(float2 a) { return make_float2(a.x, -a.y); }

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

// (cos, sin)(2*pi*m/64) for m in [0, 32); m is a compile-time constant after unrolling.
__device__ __forceinline__ float2 unit64(int m) {
  switch (m) {
    case 1: return make_float2(9.951847267e-01f, 9.801714033e-02f);
    case 2: return make_float2(9.807852804e-01f, 1.950903220e-01f);
    case 3: return make_float2(9.569403357e-01f, 2.902846773e-01f);
    case 4: return make_float2(9.238795325e-01f, 3.826834324e-01f);
    case 5: return make_float2(8.819212643e-01f, 4.713967368e-01f);
    case 6: return make_float2(8.314696123e-01f, 5.555702330e-01f);
    case 7: return make_float2(7.730104534e-01f, 6.343932842e-01f);
    case 8: return make_float2(7.071067812e-01f, 7.071067812e-01f);
    case 9: return make_float2(6.343932842e-01f, 7.730104534e-01f);
    case 10: return make_float2(5.555702330e-01f, 8.314696123e-01f);
    case 11: return make_float2(4.713967368e-01f, 8.819212643e-01f);
    case 12: return make_float2(3.826834324e-01f, 9.238795325e-01f);
    case 13: return make_float2(2.902846773e-01f, 9.569403357e-01f);
    case 14: return make_float2(1.950903220e-01f, 9.807852804e-01f);
    case 15: return make_float2(9.801714033e-02f, 9.951847267e-01f);
    case 16: return make_float2(6.123233996e-17f, 1.000000000e+00f);
    case 17: return make_float2(-9.801714033e-02f, 9.951847267e-01f);
    case 18: return make_float2(-1.950903220e-01f, 9.807852804e-01f);
    case 19: return make_float2(-2.902846773e-01f, 9.569403357e-01f);
    case 20: return make_float2(-3.826834324e-01f, 9.238795325e-01f);
    case 21: return make_float2(-4.713967368e-01f, 8.819212643e-01f);
    case 22: return make_float2(-5.555702330e-01f, 8.314696123e-01f);
    case 23: return make_float2(-6.343932842e-01f, 7.730104534e-01f);
    case 24: return make_float2(-7.071067812e-01f, 7.071067812e-01f);
    case 25: return make_float2(-7.730104534e-01f, 6.343932842e-01f);
    case 26: return make_float2(-8.314696123e-01f, 5.555702330e-01f);
    case 27: return make_float2(-8.819212643e-01f, 4.713967368e-01f);
    case 28: return make_float2(-9.238795325e-01f, 3.826834324e-01f);
    case 29: return make_float2(-9.569403357e-01f, 2.902846773e-01f);
    case 30: return make_float2(-9.807852804e-01f, 1.950903220e-01f);
    case 31: return make_float2(-9.951847267e-01f, 9.801714033e-02f);
    default: return make_float2(1.0f, 0.0f);
  }
}

// Last radix-2 step of a 2M-point FFT (M = R*R, R = 32) from the M-point FFTs of
// its even (e) and odd (o) samples, both in group_fft's lane + R*k1 order:
//   X[k] = E[k] + W^k O[k],  X[k + M] = E[k] - W^k O[k],  W = exp(-+2*pi*i/2M),
// with W^k = W^lane * W_64^k1 (wl = W^lane, forward sign).  On exit e holds
// X[lane + R*k1] and o holds X[M + lane + R*k1].
template <bool INV>
__device__ __forceinline__ void radix2_last(float2 (&e)[32], float2 (&o)[32], float2 wl) {
  if (INV) wl.y = -wl.y;
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) {
    float2 w = unit64(k1);
    if (!INV) w.y = -w.y;
    const float2 t = c_mul(o[k1], k1 == 0 ? wl : c_mul(wl, w));
    o[k1] = c_sub(e[k1], t);
    e[k1] = c_add(e[k1], t);
  }
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

// Register DFT structure: decimation in time with fused FFMA2 butterflies (1,
// default with RK_F32X2) or the decimation-in-frequency form (0).
#ifndef RK_DIT
#define RK_DIT RK_F32X2
#endif
#if RK_DIT
// Radix-2 decimation-in-time butterfly with a compile-time twiddle W = W_32^m
// (W = exp(-+2*pi*i/32)):  a <- a + W b,  b <- a - W b.  W b is factored as
// c * (b + tau * i b) with |tau| <= 1 (tau = s/c, or the mirrored form when |s| > |c|),
// so a general butterfly is three FFMA2 and a trivial one (m = 0, 8) two FADD2.
template <bool INV>
__device__ __forceinline__ void bfly_dit(float2& a, float2& b, int m) {
  if (m == 0) {
    const float2 t = b;
    b = c_sub(a, t);
    a = c_add(a, t);
    return;
  }
  if (m == 8) {   // W = -i (forward) / +i (inverse)
    const float2 t = INV ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);
    b = c_sub(a, t);
    a = c_add(a, t);
    return;
  }
  float2 w = unit32(m);
  if (!INV) w.y = -w.y;
  const float2 ib = make_float2(-b.y, b.x);   // i * b
  float2 u;
  float sc;
  if (fabsf(w.x) >= fabsf(w.y)) {   // W b = c (b + (s/c) i b)
    const float tau = w.y / w.x;
    u = __ffma2_rn(make_float2(tau, tau), ib, b);
    sc = w.x;
  } else {                          // W b = s ((c/s) b + i b)
    const float kap = w.x / w.y;
    u = __ffma2_rn(make_float2(kap, kap), b, ib);
    sc = w.y;
  }
  b = __ffma2_rn(make_float2(-sc, -sc), u, a);
  a = __ffma2_rn(make_float2(sc, sc), u, a);
}

// In-register DFT of size N <= 32 (radix-2 decimation in time on the
// bit-reversed input; the permutations are register renames), natural order in and out.
template <int N, bool INV>
__device__ __forceinline__ void dft_regs(float2 (&v)[N]) {
  static_assert(N >= 2 && N <= 32 && (N & (N - 1)) == 0, "register DFT size");
  float2 t[N];
#pragma unroll
  for (int i = 0; i < N; ++i) t[i] = v[bitrev_const(i, Log2<N>::value)];
#pragma unroll
  for (int span = 1; span < N; span <<= 1) {
#pragma unroll
    for (int start = 0; start < N; start += 2 * span) {
#pragma unroll
      for (int k = 0; k < span; ++k) bfly_dit<INV>(t[start + k], t[start + k + span], k * (32 / (2 * span)));
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = t[i];
}
#else
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
#endif

// Four-step N = R*R complex FFT over a group of R lanes (see file header).
//   v     : lane's R elements, v[n2] = x[lane + R*n2] on entry, X[lane + R*k2] on exit
//   xbuf  : this group's R*R float2 shared scratch
//   tw    : [k1][n1] table of W_N^(n1*k1) (forward sign), R*R entries; shared
//           memory in the persistent kernels, global (L1-resident) elsewhere
// All lanes of the warp must call this together (uses __syncwarp()).
template <int R, bool INV>
__device__ __forceinline__ void group_fft(float2 (&v)[R], float2* xbuf, const float2* __restrict__ tw, int lane) {
  dft_regs<R, INV>(v);
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) {
    float2 w = tw[k1 * R + lane];
    if (INV) w.y = -w.y;
    v[k1] = c_mul(v[k1], w);
  }
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) xbuf[lane * R + (k1 ^ lane)] = v[k1];
  __syncwarp();
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = xbuf[n1 * R + (lane ^ n1)];
  __syncwarp();
  dft_regs<R, INV>(v);
}

// ---- Hopper/Blackwell bulk-copy (TMA 1D) + mbarrier helpers -------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_acq_rel_add_shared(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ unsigned atom_acq_rel_add(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// ---- L2 eviction-priority hints (createpolicy + .L2::cache_hint) -----------
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// read-only (non-coherent) 8-byte load with an L2 policy
__device__ __forceinline__ float2 ldg_nc_hint(const float2* a, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ldg_hint_f4(const void* a, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ float2 ldg_hint(const float2* a, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(a), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ void stg_hint_f4(float2* a, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_hint(float2* a, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(a), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ void prefetch_l1(const void* a) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
}

// Bulk prefetch of [a, a + bytes) into L2 (one thread; bytes multiple of 16).
__device__ __forceinline__ void prefetch_l2_bulk(const void* a, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
}

// ---- thread-block clusters -------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Full cluster barrier with release/acquire semantics (orders global and shared::cluster memory).
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of `p` (this CTA's shared memory) in the shared window of CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_st_f4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 dsmem_ld_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void dsmem_st_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void dsmem_add_f32(uint32_t addr, float v) {
  asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Same with an L2 eviction-priority policy (createpolicy) for the source lines.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

// Global -> shared bulk copy completing on `bar` (bytes multiple of 16, both ends 16-B aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Same with the lane's twiddles W_N^(lane*k1), k1 = 1..R-1, held in registers
// (they depend only on the lane): no shared-memory traffic for the twiddle step.
template <int R, bool INV>
__device__ __forceinline__ void group_fft_rt(float2 (&v)[R], float2* xbuf, const float2 (&w)[R], int lane) {
  dft_regs<R, INV>(v);
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) v[k1] = c_mul(v[k1], INV ? c_conj(w[k1]) : w[k1]);
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) xbuf[lane * R + (k1 ^ lane)] = v[k1];
  __syncwarp();
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = xbuf[n1 * R + (lane ^ n1)];
  __syncwarp();
  dft_regs<R, INV>(v);
}

// Same transform with a padded (stride R + 1) transpose buffer of R*(R+1) float2:
// every transpose address is the lane's base plus a compile-time offset, so the
// unrolled stores/loads carry no per-element address registers (the XOR swizzle
// above needs R of them, which spill under 255-register pressure).  Conflict-free
// for R = 32 (64-bit accesses are split into half-warp wavefronts).
template <int R, bool INV>
__device__ __forceinline__ void group_fft_pad(float2 (&v)[R], float2* xbuf, const float2* __restrict__ tw, int lane) {
  dft_regs<R, INV>(v);
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) {
    float2 w = tw[k1 * R + lane];
    if (INV) w.y = -w.y;
    v[k1] = c_mul(v[k1], w);
  }
  float2* wr = xbuf + lane * (R + 1);
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) wr[k1] = v[k1];
  __syncwarp();
  const float2* rd = xbuf + lane;
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = rd[n1 * (R + 1)];
  __syncwarp();
  dft_regs<R, INV>(v);
}

// group_fft_pad with the lane's twiddles W_N^(lane*k1) held in registers.
template <int R, bool INV>
__device__ __forceinline__ void group_fft_pad_rt(float2 (&v)[R], float2* xbuf, const float2 (&w)[R], int lane) {
  dft_regs<R, INV>(v);
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) v[k1] = c_mul(v[k1], INV ? c_conj(w[k1]) : w[k1]);
  float2* wr = xbuf + lane * (R + 1);
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) wr[k1] = v[k1];
  __syncwarp();
  const float2* rd = xbuf + lane;
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = rd[n1 * (R + 1)];
  __syncwarp();
  dft_regs<R, INV>(v);
}

}  // namespace rk
