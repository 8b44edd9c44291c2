// PRNU peak-to-correlation-energy (PCE) all-pairs compare for sm_100a.
//
// Item (preprocess, once per key):
//   x <- x - mean(x);  S = FFT2(x) / N   (real-to-complex half spectrum)
// stored in its slot as N/2 columns x N rows of complex64, column-major, with
// the real-valued DC (k_col = 0) and Nyquist (k_col = N/2) columns packed into
// column 0 as DC + i*Nyquist.  One slot is exactly N*N*4 bytes (4 MiB at 1024^2).
//
// Pair (compare):
//   C = IFFT2(S_i * conj(S_j))                     (circular cross-correlation)
//   p* = argmax C (first in row-major order on ties), peak = C[p*]
//   PCE = peak*|peak| / ( sum_{s not in A} C[s]^2 / (N*N - |A|) ),
//   A = the 11x11 wrap-around neighbourhood of p*.
// The oracle restating these definitions is oracle/pce.py (parity unpinned by
// the reference, which has no PCE: SURVEY.md section 8(c)).
//
// Compare kernel (pce_cluster<R, CL>, CL = 1 in production): persistent, one
// CTA = one SM per pair in flight (148 pairs); its 8 warps form two
// independent warp groups, each feeding itself through its own bulk-copy
// (TMA 1-D) + mbarrier pipeline (per-warp column slices; row blocks released by
// counted arrival); a grid round barrier keeps the in-flight pairs in step.  The 2-D inverse FFT needs one global
// transpose; its intermediate T (4 MiB per pair at 1024^2) goes to a per-CTA
// slot in HBM.  Per pair:
//   column phase  per 4-column slice of X and Y (refilled as soon as the products
//                 X*conj(Y) are in registers): inverse column FFTs -> T in 8-row blocks
//   CTA barrier   (+ fence.proxy.async: T's generic stores before the bulk reads)
//   row phase     per 8-row block (double-buffered bulk copies): inverse row C2R
//                 FFTs (two rows per complex FFT) with fused max/argmax/energy
//   reduction     fixed-order combine of the warp partials (deterministic)
//   window        6 warps recompute the 11 rows around the peak from staged
//                 blocks and sum the 11x11 energy; one thread writes PCE + flag.
// 256^2 runs the same kernel with a cluster of 2 CTAs per pair (DSMEM
// reductions); the measured-and-rejected variants of round 1 (clusters per pair at
// 1024^2, TMA tensor stores of T, a padded transpose, group-slice column staging,
// two 4-warp CTAs per SM, L2 policies) are recorded in DESIGN.md, not kept here.

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "fft.cuh"
#include "pce_common.cuh"
#include "internal.h"

namespace rk {

namespace {
using namespace pcek;

constexpr int kGroups = 8;              // FFT groups (row-pairs / columns) per preprocess CTA
constexpr int kRows = 2 * kGroups;      // rows per preprocess row-pass CTA
constexpr int kTileStride = kRows + 1;  // padded row stride of the [k][row] tile
// Warps per compare CTA: two independent warp groups of 4 lane groups each
// (8 warps at R = 32, 4 warps of two half-warp lane groups at R = 16).
__host__ __device__ constexpr int cta_warps(int R) { return 8 / (32 / R); }
__host__ __device__ constexpr int xpose_size(int R) { return R * R; }   // XOR-swizzled transpose buffer
// Row-phase buffer release by counted arrival (1) or a group barrier (0).
#ifndef PCE_ROW_ARRIVE
#define PCE_ROW_ARRIVE 1
#endif
template <int R>
__device__ __forceinline__ void compare_fft(float2 (&v)[R], float2* xbuf, const float2 (&w)[R], int lane) {
  group_fft_rt<R, true>(v, xbuf, w, lane);
}

// CTAs per pair: 1 at R = 32 (one SM per pair in flight, all 148 SMs; clusters of
// 2 / 4 / 8 measured slower), 2 at R = 16.
template <int R>
struct ClusterShape;
template <>
struct ClusterShape<32> {
  static constexpr int CL = 1;
};
template <>
struct ClusterShape<16> {
  static constexpr int CL = 2;
};

// ---------------------------------------------------------------------------
// Preprocess P0: per-item partial sums for the mean.
__global__ void __launch_bounds__(256) pce_mean_partial(const float* __restrict__ pix, size_t stride_f,
                                                        int nn, float* __restrict__ mean_part) {
  const int item = blockIdx.y;
  const float4* x = reinterpret_cast<const float4*>(pix + (size_t)item * stride_f);
  const int per = nn / 4 / kMeanParts;
  const float4* xs = x + (size_t)blockIdx.x * per;
  float acc = 0.f;
  for (int i = threadIdx.x; i < per; i += blockDim.x) {
    const float4 q = __ldg(xs + i);
    acc += (q.x + q.y) + (q.z + q.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    mean_part[item * kMeanParts + blockIdx.x] = t;
  }
}

// Preprocess P1: zero-mean, forward row FFTs (two real rows per complex FFT),
// unpack to half spectra, write U[item][k][row] with column 0 packed DC+i*Nyquist.
template <int R>
__global__ void __launch_bounds__(kGroups * R) pce_rows_fwd(const float* __restrict__ pix, size_t stride_f,
                                                           const float* __restrict__ mean_part,
                                                           float2* __restrict__ U,
                                                           const float2* __restrict__ tw_g) {
  constexpr int N = R * R;
  constexpr int NT = kGroups * R;
  extern __shared__ float2 smem[];
  float2* tile = smem;                               // (N/2) x kTileStride
  float2* xbufs = tile + (N / 2) * kTileStride;      // kGroups x R*R
  const float2* tw = tw_g;
  __shared__ float s_mean;
  const int tid = threadIdx.x;
  const int item = blockIdx.y;
  const int r0 = blockIdx.x * kRows;
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < kMeanParts; ++i) s += (double)mean_part[item * kMeanParts + i];
    s_mean = (float)(s / ((double)N * (double)N));
  }
  __syncthreads();
  const float mu = s_mean;
  const int g = tid / R, lane = tid % R;
  float2* xbuf = xbufs + g * R * R;
  const int ra = r0 + 2 * g;
  const float* xa = pix + (size_t)item * stride_f + (size_t)ra * N;
  const float* xb = xa + N;
  float2 v[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2)
    v[n2] = make_float2(__ldg(xa + lane + R * n2) - mu, __ldg(xb + lane + R * n2) - mu);
  group_fft<R, false>(v, xbuf, tw, lane);
  // natural-order Z in the (now free) transpose buffer
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) xbuf[lane + R * k2] = v[k2];
  __syncwarp();
#pragma unroll
  for (int n = 0; n < R / 2; ++n) {
    const int k = lane + R * n;
    const float2 z = xbuf[k];
    float2 a, b;
    if (k == 0) {
      const float2 zn = xbuf[N / 2];
      a = make_float2(z.x, zn.x);   // (A[0], A[N/2]) both real
      b = make_float2(z.y, zn.y);   // (B[0], B[N/2]) both real
    } else {
      const float2 zr = c_conj(xbuf[N - k]);
      a = c_scale(c_add(z, zr), 0.5f);
      const float2 d = c_sub(z, zr);
      b = make_float2(0.5f * d.y, -0.5f * d.x);   // d / (2i)
    }
    tile[k * kTileStride + 2 * g] = a;
    tile[k * kTileStride + 2 * g + 1] = b;
  }
  __syncthreads();
  float2* Ui = U + (size_t)item * (N / 2) * N;
  for (int idx = tid; idx < (N / 2) * kRows; idx += NT) {
    const int c = idx / kRows, rr = idx % kRows;
    Ui[(size_t)c * N + r0 + rr] = tile[c * kTileStride + rr];
  }
}

// Preprocess P2: forward column FFTs of U, scaled by 1/N, into the item's slot.
template <int R>
__global__ void __launch_bounds__(kGroups * R) pce_cols_fwd(const float2* __restrict__ U, char* __restrict__ slots,
                                                           size_t slot_stride, SlotList dst,
                                                           const float2* __restrict__ tw_g) {
  constexpr int N = R * R;
  extern __shared__ float2 smem[];
  const float2* tw = tw_g;
  const int tid = threadIdx.x;
  const int item = blockIdx.y;
  const int g = tid / R, lane = tid % R;
  float2* xbuf = smem + g * R * R;
  const int col = blockIdx.x * kGroups + g;
  const float2* Uc = U + (size_t)item * (N / 2) * N + (size_t)col * N;
  float2 v[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) v[n2] = Uc[lane + R * n2];
  group_fft<R, false>(v, xbuf, tw, lane);
  float2* S = reinterpret_cast<float2*>(slots + (size_t)dst.idx[item] * slot_stride) + (size_t)col * N;
  constexpr float kScale = 1.0f / (float)N;
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) S[lane + R * k2] = c_scale(v[k2], kScale);
}

// Optional phase timing (compile with -DPCE_PROBES): per (CTA, warp 0|last) and
// probe point, the summed clock64 of each phase boundary into a debug buffer.
#ifdef PCE_PROBES
__device__ unsigned long long g_pce_probe[148 * 2 * 8];
#define PCE_PROBE(k)                                                                                      \
  do {                                                                                                    \
    if (wl == 0 && (warp == 0 || warp == kCtaWarps - 1))                                                  \
      atomicAdd(&g_pce_probe[(blockIdx.x * 2 + (warp != 0)) * 8 + (k)], (unsigned long long)clock64()); \
  } while (0)
#else
#define PCE_PROBE(k) \
  do {               \
  } while (0)
#endif

template <int R, int CL>
__global__ void __launch_bounds__(cta_warps(R) * 32, 1) pce_cluster(
    const PairJob job, const char* __restrict__ slots, size_t slot_stride, float2* __restrict__ T, size_t t_stride,
    const float2* __restrict__ tw_g, double* __restrict__ out, uint8_t* __restrict__ flags, double threshold,
    const LedgerRef ledger, unsigned* __restrict__ rounds, int l2opts) {
  constexpr int N = R * R;
  constexpr int G = 32 / R;               // lane groups per warp
  constexpr int kCtaWarps = cta_warps(R);
  constexpr int NT = kCtaWarps * 32;
  constexpr int kNG = 2;                  // independent warp groups
  constexpr int kGW = kCtaWarps / kNG;    // warps per warp group
  constexpr int kGL = kGW * G;            // lane groups per warp group: 4 columns / 4 row pairs per round
  constexpr int NCOL = (N / 2) / CL;      // columns per CTA
  constexpr int NB8 = (N / 8) / CL;       // 8-row blocks per CTA
  constexpr int kPairsOfRows = (kWin + 1) / 2;
  constexpr int kHalf = 4 * N;            // float2: 4 columns of a slot == one 8-row block of T
  constexpr uint32_t kHalfBytes = kHalf * sizeof(float2);
  static_assert(kGL == 4, "a warp group owns 4 lane groups");
  static_assert(NCOL * CL == N / 2 && NCOL % 8 == 0 && NB8 * CL == N / 8 && NB8 % 2 == 0, "cluster split");
  extern __shared__ __align__(128) float2 smem[];
  float2* gbufs = smem;                   // kNG groups x 2 halves of 4N float2 (column slices / row blocks)
  float2* tw = smem + 2 * kNG * kHalf;    // R*R twiddles
  float2* xbufs = tw + R * R;             // one R*R transpose buffer per lane group
  __shared__ __align__(8) uint64_t s_bar[kNG][3];   // per group: column slices, row block 0 / 1
  __shared__ unsigned s_done[kNG][2];   // per group and row buffer: warps done reading (PCE_ROW_ARRIVE)
  __shared__ __align__(8) uint64_t s_wbar;
  __shared__ __align__(8) uint64_t s_cbar[kCtaWarps];   // per warp: its column slice
  __shared__ float4 s_part[CL];           // CTA partials, gathered in CTA 0
  __shared__ float s_wpart[8];            // window energy per row pair, gathered in CTA 0
  __shared__ float s_v[kCtaWarps];
  __shared__ int s_i[kCtaWarps];
  __shared__ float s_ss[kCtaWarps];
  __shared__ float s_peak;
  __shared__ int s_pidx;
  __shared__ double s_total;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, wl = tid & 31;
  const int g = wl / R, lane = wl % R;
  const int grp = warp * G + g;           // lane group in the CTA
  const int wg = warp / kGW;              // warp group 0 / 1
  const int gi = (warp % kGW) * G + g;    // lane group within the warp group, 0..3
  const bool leader = (tid % (kGW * 32)) == 0;
  const int q = (int)cluster_ctarank();
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  float2* xbuf = xbufs + grp * xpose_size(R);
  float2* gb = gbufs + wg * 2 * kHalf;    // this warp group's 2 x 4N float2
  float2* Tp = T + (size_t)cid * t_stride;
  for (int i = tid; i < R * R; i += NT) tw[i] = tw_g[i];
  if (tid == 0) {
    for (int w = 0; w < kNG; ++w)
      for (int b = 0; b < 3; ++b) mbar_init(&s_bar[w][b], 1);
    mbar_init(&s_wbar, 1);
    for (int w = 0; w < kCtaWarps; ++w) mbar_init(&s_cbar[w], 1);
    for (int w = 0; w < kNG; ++w) s_done[w][0] = s_done[w][1] = 0u;
  }
  uint32_t ph = 0;                        // parity bits of this group's three barriers (bit b)
  uint32_t wph = 0;
  uint32_t cph = 0;                       // parity of this warp's column-slice barrier
  __syncthreads();
  const uint32_t part0 = dsmem_addr(&s_part[0], 0);
  const uint32_t wpart0 = dsmem_addr(&s_wpart[0], 0);
  float2 twr[R];   // this lane's twiddles W_N^(lane*k1): no shared-memory traffic in the FFTs
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) twr[k1] = tw[k1 * R + lane];
  // L2 priority: with one pair per SM (148 T slots, 592 MiB) T cannot stay in L2,
  // so neither T nor the spectra (reused by the neighbouring pairs of a leaf) get a
  // special priority (evict_last / evict_first measured within 1 %); T blocks are
  // read once, evict_first.
  const uint64_t pol_first = l2_policy_evict_first();
  const uint64_t pol_T = (l2opts & 1) ? pol_first : l2_policy_evict_normal();
  const uint64_t pol_spec = (l2opts & 2) ? l2_policy_evict_last() : l2_policy_evict_normal();
  cluster_sync();

  for (int pi = cid; pi < job.npairs; pi += ncl) {
    if (CL == 1) round_wait(rounds, pi, ncl, tid, PCE_ROUND_SLACK_PCT);
    const DevPair pr = job.pairs[pi];
    float2 v[R];
    PCE_PROBE(0);

    // ---------------- column phase ----------------
    // Two warp groups run independently, each streaming 4-column
    // slices of X and Y (contiguous in the slots) through its own buffer; a slice
    // is refilled as soon as the group has formed its products, so the copy lands
    // while the FFTs run, and the two groups' smem-heavy and FMA-heavy steps interleave.
    const float2* Xs = reinterpret_cast<const float2*>(slots + (size_t)pr.slot_a * slot_stride);
    const float2* Ys = reinterpret_cast<const float2*>(slots + (size_t)pr.slot_b * slot_stride);
    {
      const int cbeg = q * NCOL + 4 * wg, cend = (q + 1) * NCOL;
      // Per-warp pipeline: each warp owns the G columns of X and Y its lane groups
      // transform, waits on its own mbarrier and refills its own slice as soon as its
      // products are in registers -- no group barrier couples the four warps.
      constexpr uint32_t kWarpBytes = (uint32_t)(G * N * sizeof(float2));
      const int wcol = (warp % kGW) * G;            // first column of this warp within a slice
      uint64_t* wbar = &s_cbar[warp];
      float2* wx = gb + wcol * N;
      float2* wy = gb + kHalf + wcol * N;
      if (wl == 0) {
        mbar_expect_tx(wbar, 2 * kWarpBytes);
        bulk_g2s_hint(wx, Xs + (size_t)(cbeg + wcol) * N, kWarpBytes, wbar, pol_spec);
        bulk_g2s_hint(wy, Ys + (size_t)(cbeg + wcol) * N, kWarpBytes, wbar, pol_spec);
      }
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 4 * kNG) {
        const int col = c0 + gi;
        mbar_wait(wbar, cph & 1u);
        cph ^= 1u;
        const float2* X = gb + gi * N;
        const float2* Y = gb + kHalf + gi * N;
        if (col != 0) {
#pragma unroll
          for (int n2 = 0; n2 < R; ++n2) v[n2] = c_mulc(X[lane + R * n2], Y[lane + R * n2]);
        } else {
          // packed DC/Nyquist column: split both sides into their Hermitian parts,
          // multiply separately, re-pack the (Hermitian) products
#pragma unroll
          for (int n2 = 0; n2 < R; ++n2) {
            const int m = lane + R * n2;
            const int mm = (N - m) & (N - 1);
            const float2 x = X[m], xr = c_conj(X[mm]);
            const float2 y = Y[m], yr = c_conj(Y[mm]);
            const float2 xa = c_scale(c_add(x, xr), 0.5f);
            const float2 dx = c_sub(x, xr);
            const float2 xb = make_float2(0.5f * dx.y, -0.5f * dx.x);
            const float2 ya = c_scale(c_add(y, yr), 0.5f);
            const float2 dy = c_sub(y, yr);
            const float2 yb = make_float2(0.5f * dy.y, -0.5f * dy.x);
            const float2 pa = c_mulc(xa, ya);
            const float2 pb = c_mulc(xb, yb);
            v[n2] = make_float2(pa.x - pb.y, pa.y + pb.x);
          }
        }
        __syncwarp();                  // this warp's columns are consumed
        if (wl == 0 && c0 + 4 * kNG < cend) {
          refill_fence();
          mbar_expect_tx(wbar, 2 * kWarpBytes);
          bulk_g2s_hint(wx, Xs + (size_t)(c0 + 4 * kNG + wcol) * N, kWarpBytes, wbar, pol_spec);
          bulk_g2s_hint(wy, Ys + (size_t)(c0 + 4 * kNG + wcol) * N, kWarpBytes, wbar, pol_spec);
        }
        compare_fft<R>(v, xbuf, twr, lane);
        // row lane + R*k2 -> 8-row block (lane>>3) + (R/8)*k2, row lane&7 (chunk-swizzled)
        const int rr = lane & 7;
        const int pos = (((rr >> 1) ^ ((col >> 1) & 3)) << 1) | (rr & 1);
        float2* dst = Tp + ((size_t)(lane >> 3) * (N / 2) + col) * 8 + pos;
        constexpr size_t kStep = (size_t)(R / 8) * (N / 2) * 8;
#pragma unroll
        for (int k2 = 0; k2 < R; ++k2) stg_hint(dst + k2 * kStep, v[k2], pol_T);
      }
    }
    PCE_PROBE(1);
    cluster_sync();
    PCE_PROBE(2);

    // ---------------- row phase ----------------
    // Each warp group streams its 8-row blocks (one row pair per lane group)
    // through a double buffer of bulk copies.
    float m = -INFINITY, ss = 0.f;
    int idx = 0x7fffffff;
    {
      const int bbeg = q * NB8 + wg, bend = (q + 1) * NB8;
      if (leader) {
        fence_proxy_async();     // T's generic-proxy stores (ordered by the cluster barrier) -> async proxy
        for (int b = 0; b < 2 && bbeg + kNG * b < bend; ++b) {
          mbar_expect_tx(&s_bar[wg][1 + b], kHalfBytes);
          bulk_g2s_hint(gb + b * kHalf, Tp + (size_t)(bbeg + kNG * b) * kHalf, kHalfBytes, &s_bar[wg][1 + b],
                        pol_first);
        }
      }
      int it = 0;
#pragma unroll 1
      for (int rb = bbeg; rb < bend; rb += kNG, ++it) {
        const int buf = it & 1;
        mbar_wait(&s_bar[wg][1 + buf], (ph >> (1 + buf)) & 1u);
        ph ^= 2u << buf;
        block8_rows_z<R>(v, gb + buf * kHalf, gi, lane);
#if PCE_ROW_ARRIVE
        // the block is consumed once all kGW warps have read their row pair: the
        // last warp to finish reading (acq_rel count) refills it, the others go
        // straight on to their FFT instead of waiting at a group barrier
        __syncwarp();
        if (wl == 0 && rb + 2 * kNG < bend &&
            atom_acq_rel_add_shared(&s_done[wg][buf], 1u) % kGW == (unsigned)(kGW - 1)) {
          refill_fence();
          mbar_expect_tx(&s_bar[wg][1 + buf], kHalfBytes);
          bulk_g2s_hint(gb + buf * kHalf, Tp + (size_t)(rb + 2 * kNG) * kHalf, kHalfBytes, &s_bar[wg][1 + buf],
                        pol_first);
        }
#else
        named_bar(1 + wg, kGW * 32);   // the block is consumed: refill it
        if (leader && rb + 2 * kNG < bend) {
          refill_fence();
          mbar_expect_tx(&s_bar[wg][1 + buf], kHalfBytes);
          bulk_g2s_hint(gb + buf * kHalf, Tp + (size_t)(rb + 2 * kNG) * kHalf, kHalfBytes, &s_bar[wg][1 + buf],
                        pol_first);
        }
#endif
        compare_fft<R>(v, xbuf, twr, lane);
        argmax_update<R>(v, 8 * rb + 2 * gi, lane, m, idx, ss);
      }
    }
    PCE_PROBE(3);
    {
      ArgMax best = warp_argmax(ArgMax{m, idx});
      ss = warp_sum(ss);
      if (wl == 0) {
        s_v[warp] = best.v;
        s_i[warp] = best.idx;
        s_ss[warp] = ss;
      }
      __syncthreads();
      if (tid == 0) {
        ArgMax bb{s_v[0], s_i[0]};
        float t = s_ss[0];
        for (int w = 1; w < kCtaWarps; ++w) {
          if (better(s_v[w], s_i[w], bb.v, bb.idx)) bb = ArgMax{s_v[w], s_i[w]};
          t += s_ss[w];
        }
        dsmem_st_f4(part0 + q * sizeof(float4), make_float4(bb.v, __int_as_float(bb.idx), t, 0.f));
      }
    }
    cluster_sync();
    PCE_PROBE(4);
    if (tid == 0) {
      ArgMax bb{-INFINITY, 0x7fffffff};
      double tt = 0.0;
      for (int c = 0; c < CL; ++c) {
        const float4 e = dsmem_ld_f4(part0 + c * sizeof(float4));
        const int ei = __float_as_int(e.y);
        if (better(e.x, ei, bb.v, bb.idx)) bb = ArgMax{e.x, ei};
        tt += (double)e.z;
      }
      s_peak = bb.v;
      s_pidx = bb.idx;
      s_total = tt;
    }
    __syncthreads();

    // ---------------- window: 11 rows around the peak ----------------
    // The 6 aligned row pairs covering rows peak-5 .. peak+5 lie in at most three
    // 8-row blocks: bulk-copy them into the (now free) group buffers, then six warps
    // (spread over the cluster) recompute one row pair each.
    {
      const int prow = s_pidx / N, pcol = s_pidx % N;
      const int rstart = (prow - kHalfWin + N) & (N - 1);
      const int e0 = rstart & ~1;                              // first aligned row of the 12-row span
      const int b0 = e0 >> 3;
      const int nblk = ((e0 + 2 * kPairsOfRows - 1) >> 3) - b0 + 1;   // 2 or 3 blocks
      constexpr int kStage = 2 * kNG;                          // staged blocks per pass (group buffers)
#pragma unroll 1
      for (int p0 = 0; p0 < nblk; p0 += kStage) {
        const int cnt = min(kStage, nblk - p0);
        if (tid == 0) {
          fence_proxy_async();
          mbar_expect_tx(&s_wbar, cnt * kHalfBytes);
          for (int j = 0; j < cnt; ++j)
            bulk_g2s_hint(gbufs + j * kHalf, Tp + (size_t)((b0 + p0 + j) & (N / 8 - 1)) * kHalf, kHalfBytes,
                          &s_wbar, pol_first);
        }
        mbar_wait(&s_wbar, wph & 1u);
        wph ^= 1u;
#pragma unroll 1
        for (int t = q + CL * warp; t < kPairsOfRows; t += CL * kCtaWarps) {   // row pair t of the span
          const int ra = (e0 + 2 * t) & (N - 1);                // even row: pair (ra, ra + 1)
          const int j = (((ra >> 3) - b0 + (N / 8)) & (N / 8 - 1)) - p0;   // staged slot of its block
          if (j < 0 || j >= cnt) continue;
          block8_rows_z<R>(v, gbufs + j * kHalf, (ra & 7) >> 1, lane);
          if (g != 0) {   // R = 16: the warp's second lane group has no row pair
#pragma unroll
            for (int n2 = 0; n2 < R; ++n2) v[n2] = make_float2(0.f, 0.f);
          }
          compare_fft<R>(v, xbuf, twr, lane);
          const bool va = ((ra - rstart + N) & (N - 1)) < kWin;
          const bool vb = ((ra + 1 - rstart + N) & (N - 1)) < kWin;
          float w = 0.f;
#pragma unroll
          for (int k2 = 0; k2 < R; ++k2) {
            const int s = lane + R * k2;
            if (((s - pcol + kHalfWin + N) & (N - 1)) < kWin) {
              if (va) w = fmaf(v[k2].x, v[k2].x, w);
              if (vb) w = fmaf(v[k2].y, v[k2].y, w);
            }
          }
          w = warp_sum(w);
          if (wl == 0) dsmem_st_f32(wpart0 + t * sizeof(float), w);   // fixed-order sum in CTA 0
        }
        if (p0 + kStage < nblk) cluster_sync();   // staged blocks consumed before the next pass
      }
    }
    PCE_PROBE(5);
    cluster_sync();
    PCE_PROBE(6);
    if (q == 0 && tid == 0) {
      const double peak = (double)s_peak;
      double wsum = 0.0;
      for (int t = 0; t < kPairsOfRows; ++t) wsum += (double)s_wpart[t];
      const double energy = (s_total - wsum) / ((double)N * (double)N - (double)(kWin * kWin));
      const double pce = peak * fabs(peak) / energy;
      out[pr.pid] = pce;
      ledger_mark(ledger, pr.pid);
      if (flags) flags[pr.pid] = isnan(threshold) ? 0 : (uint8_t)(1 | (pce >= threshold ? 2 : 0));
    }
    if (CL == 1) round_arrive(rounds, tid);
  }
}

template <int R>
size_t cols_fwd_smem() {
  return (size_t)(kGroups * R * R) * sizeof(float2);
}
template <int R>
size_t rows_fwd_smem() {
  constexpr int N = R * R;
  return (size_t)((N / 2) * kTileStride + kGroups * R * R) * sizeof(float2);
}
template <int R>
size_t cluster_smem() {
  constexpr int N = R * R;
  // 2 warp groups x 2 x 4N (column slices / 8-row blocks) + twiddles + one transpose per lane group
  return (size_t)(16 * N + R * R + cta_warps(R) * (32 / R) * xpose_size(R)) * sizeof(float2);
}

template <int R>
rk_status set_attrs() {
  constexpr int CL = ClusterShape<R>::CL;
  RK_CUDA(cudaFuncSetAttribute(pce_cluster<R, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cluster_smem<R>()));
  RK_CUDA(cudaFuncSetAttribute(pce_cols_fwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_fwd_smem<R>()));
  RK_CUDA(cudaFuncSetAttribute(pce_rows_fwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_fwd_smem<R>()));
  return RK_OK;
}

template <int R>
rk_status preprocess_impl(rk_app* app, const float* pix, size_t stride_f, int n_items, char* slots,
                          size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  constexpr int N = R * R;
  PceState& st = app->pce;
  for (int base = 0; base < n_items; base += st.batch) {
    const int m = (n_items - base < st.batch) ? n_items - base : st.batch;
    const float* px = pix + (size_t)base * stride_f;
    pce_mean_partial<<<dim3(kMeanParts, m), 256, 0, s>>>(px, stride_f, N * N, st.mean_part);
    pce_rows_fwd<R><<<dim3(N / kRows, m), kGroups * R, rows_fwd_smem<R>(), s>>>(px, stride_f, st.mean_part, st.U, st.tw);
    SlotList dst;
    dst.n = m;
    for (int k = 0; k < m; ++k) dst.idx[k] = h_slot_idx[base + k];
    pce_cols_fwd<R><<<dim3(N / 2 / kGroups, m), kGroups * R, cols_fwd_smem<R>(), s>>>(st.U, slots, slot_stride, dst, st.tw);
    app->launches += 3;
    RK_CUDA(cudaGetLastError());
  }
  return RK_OK;
}

template <int R>
cudaLaunchConfig_t cluster_config(int grid, cudaStream_t s, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(cta_warps(R) * 32);
  cfg.dynamicSmemBytes = cluster_smem<R>();
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ClusterShape<R>::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

template <int R>
rk_status compare_impl(rk_app* app, const char* slots, size_t slot_stride, const rk_pair* pairs, int n, double* d_out,
                       uint8_t* d_flags, cudaStream_t s) {
  constexpr int CL = ClusterShape<R>::CL;
  PceState& st = app->pce;
  PairJob& job = *st.job;
  job.npairs = n;
  job.depth = 0;
  for (int k = 0; k < n; ++k) {
    job.pairs[k].slot_a = pairs[k].slot_a;
    job.pairs[k].slot_b = pairs[k].slot_b;
    job.pairs[k].pid = pair_id(app->p.n, pairs[k].i, pairs[k].j);
  }
  const int clusters = std::min(st.clusters, n);
  unsigned* rounds = CL == 1 ? st.rounds : nullptr;
  if (rounds) RK_CUDA(cudaMemsetAsync(rounds, 0, sizeof(unsigned), s));
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = cluster_config<R>(clusters * CL, s, attr);
  RK_CUDA(cudaLaunchKernelEx(&cfg, pce_cluster<R, CL>, job, slots, slot_stride, st.T, st.t_stride, (const float2*)st.tw, d_out,
                             d_flags, threshold_or_nan(app), app->ledger, rounds, st.l2opts));
  app->launches += 1;
  return RK_OK;
}

template <int R>
rk_status cluster_init(rk_app* app) {
  PceState& st = app->pce;
  constexpr int N = R * R;
  constexpr int CL = ClusterShape<R>::CL;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = cluster_config<R>(CL * 64, nullptr, attr);
  int clusters = 0;
  RK_CUDA(cudaOccupancyMaxActiveClusters(&clusters, pce_cluster<R, CL>, &cfg));
  if (clusters < 1) return set_error(RK_ERR_DEVICE, "pce_cluster: no cluster of %d CTAs fits", CL);
  st.clusters = clusters;
  st.t_stride = (size_t)(N / 2) * N + stride_pad("RK_T_PAD", 0) / sizeof(float2);
  RK_CUDA(cudaMalloc(&st.T, sizeof(float2) * st.t_stride * clusters));
  st.job = new PairJob();
  return pce_round_init(st, 0);
}

}  // namespace

// Pairs per compare launch: whole rounds of the persistent grid (one pair per CTA
// per round), so no CTA idles in a launch's last round.
int pce_batch_limit(const rk_app* app) {
  const int g = app->pce.clusters > 0 ? app->pce.clusters : 1;
  const int rounds = kPipeMaxPairs / g;
  return rounds > 0 ? rounds * g : kPipeMaxPairs;
}

void pce_launch_mean(const float* pix, size_t stride_f, int nn, int n_items, float* mean_part, cudaStream_t s) {
  pce_mean_partial<<<dim3(kMeanParts, n_items), 256, 0, s>>>(pix, stride_f, nn, mean_part);
}

rk_status pce_compare_list(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* pairs, int n,
                           double* d_out, uint8_t* d_flags, cudaStream_t s) {
  const char* slots = static_cast<const char*>(d_slots);
  const int lim = pce_batch_limit(app);
  for (int base = 0; base < n; base += lim) {
    const int m = std::min(lim, n - base);
    if (app->pce.N == 2048) RK_TRY(pce2k_compare(app, slots, slot_stride, pairs + base, m, d_out, d_flags, s));
    else if (app->pce.R == 16) RK_TRY(compare_impl<16>(app, slots, slot_stride, pairs + base, m, d_out, d_flags, s));
    else RK_TRY(compare_impl<32>(app, slots, slot_stride, pairs + base, m, d_out, d_flags, s));
  }
  return RK_OK;
}

rk_status pce_init(rk_app* app) {
  const int h = app->p.height, w = app->p.width;
  if (h != w) return set_error(RK_ERR_UNSUPPORTED, "PCE patterns must be square (got %dx%d)", h, w);
  int R = 0;
  if (h == 256) R = 16;
  else if (h == 1024) R = 32;
  else if (h == 2048) R = 32;   // two 1024-point warp FFTs + a radix-2 step per line (pce2k.cu)
  else return set_error(RK_ERR_UNSUPPORTED, "PCE pattern side %d not built (256, 1024 or 2048)", h);
  PceState& st = app->pce;
  st.R = R;
  st.N = h;
  st.batch = app->p.batch_pairs > 0 ? app->p.batch_pairs : (h == 2048 ? 8 : R == 32 ? 16 : 64);
  if (st.batch > kMaxBatch) st.batch = kMaxBatch;
  const int N = st.N;
  app->slot_bytes = (size_t)N * N * sizeof(float);       // (N/2)*N complex64
  app->parsed_bytes = (size_t)N * N * sizeof(float);
  // twiddles W_N^(n1*k1), stored [k1][n1]
  std::vector<float2> tw((size_t)R * R);
  for (int k1 = 0; k1 < R; ++k1)
    for (int n1 = 0; n1 < R; ++n1) {
      const double ang = -2.0 * M_PI * (double)(n1 * k1) / (double)(R * R);
      tw[(size_t)k1 * R + n1] = make_float2((float)cos(ang), (float)sin(ang));
    }
  RK_CUDA(cudaMalloc(&st.tw, sizeof(float2) * R * R));
  RK_CUDA(cudaMemcpy(st.tw, tw.data(), sizeof(float2) * R * R, cudaMemcpyHostToDevice));
  RK_CUDA(cudaMalloc(&st.U, sizeof(float2) * (size_t)(N / 2) * N * st.batch));
  RK_CUDA(cudaMalloc(&st.mean_part, sizeof(float) * kMeanParts * st.batch));
  if (N == 2048) return pce2k_init(app);
  if (R == 16) {
    RK_TRY(set_attrs<16>());
    return cluster_init<16>(app);
  }
  RK_TRY(set_attrs<32>());
  return cluster_init<32>(app);
}

// Defaults measured on B200 (profiles/r2_ab_lockstep.json): the round
// barrier on at every size; at 2048^2 T stores evict_first + spectra evict_last
// (84.4k -> 104.9k pairs/s with the barrier), at 1024^2 no L2 hints (neutral).
rk_status pce_round_init(PceState& st, int l2opts_default) {
  const char* e = getenv("RK_PCE_LOCKSTEP");
  if (e == nullptr || atoi(e) != 0) RK_CUDA(cudaMalloc(&st.rounds, sizeof(unsigned)));
  const char* o = getenv("RK_PCE_L2OPTS");
  st.l2opts = o ? atoi(o) : l2opts_default;
  return RK_OK;
}

void pce_free(rk_app* app) {
  PceState& st = app->pce;
  cudaFree(st.rounds);
  cudaFree(st.tw);
  cudaFree(st.T);
  cudaFree(st.U);
  cudaFree(st.mean_part);
  delete st.job;
  st = PceState{};
}

rk_status pce_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                         size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  if (parsed_stride % 16 != 0) return set_error(RK_ERR_VALUE, "parsed_stride must be a multiple of 16 bytes");
  const float* pix = static_cast<const float*>(d_parsed);
  const size_t stride_f = parsed_stride / sizeof(float);
  if (app->pce.N == 2048)
    return pce2k_preprocess(app, pix, stride_f, n_items, static_cast<char*>(d_slots), slot_stride, h_slot_idx, s);
  if (app->pce.R == 16)
    return preprocess_impl<16>(app, pix, stride_f, n_items, static_cast<char*>(d_slots), slot_stride, h_slot_idx, s);
  return preprocess_impl<32>(app, pix, stride_f, n_items, static_cast<char*>(d_slots), slot_stride, h_slot_idx, s);
}

}  // namespace rk

#ifdef PCE_PROBES
extern "C" int rk_debug_pce_probes(unsigned long long* out, int n, int reset) {
  if (cudaMemcpyFromSymbol(out, rk::g_pce_probe, sizeof(unsigned long long) * n) != cudaSuccess) return 1;
  if (reset) {
    static unsigned long long zeros[148 * 2 * 8] = {};
    cudaMemcpyToSymbol(rk::g_pce_probe, zeros, sizeof(zeros));
  }
  return 0;
}
#endif
