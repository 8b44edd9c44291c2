// PRNU PCE at 2048 x 2048 (BASELINE config C3) for sm_100a.
//
// Same score as pce.cu (definitions there and in oracle/pce.py); what changes at
// 2048^2 is that one warp can no longer hold a whole line: every 2048-point FFT
// is two 1024-point warp FFTs (group_fft over the even and the odd samples, the
// four-step 32 x 32 transform of fft.cuh) plus one radix-2 step (radix2_last),
// so the data are laid out by sample parity wherever a line is loaded:
//
//   slot (S = FFT2(x - mean)/N, 16 MiB):  S[p][c][m] = S(row 2m + p, column c)
//       p = row parity, c in [0, 1024) half-spectrum columns (column 0 packs the
//       real DC and Nyquist columns as DC + i*Nyquist), m in [0, 1024).
//       A 4-column unit of one parity is 32 KiB contiguous (one bulk copy).
//   T (column-pass output, one 16 MiB slot per resident CTA):
//       T[rb][q][j][8]: 8-row block rb, column parity q, column j = c >> 1, the
//       block's 8 rows of column c in 64 B with pce.cu's chunk swizzle.  One half
//       block (512 columns x 8 rows) is 32 KiB contiguous and is exactly the
//       staged layout pce.cu's 1024-point row pass reads (block8_rows_z): the
//       even-column half IS a 1024-point half spectrum, DC/Nyquist packing and all.
//
// Compare kernel (pce2k_pair): persistent, one CTA (8 warps, 255 registers,
// 200 KiB shared memory) per SM and per pair in flight; two independent warp
// groups of 4 warps, each with its own bulk-copy (TMA 1-D) pipeline and named
// barrier, as in pce.cu.  Per pair:
//   column phase  per 4-column quartet: even rows -> product X*conj(Y), inverse
//                 1024-point FFT (E); odd rows -> product, FFT (O); radix-2 step;
//                 the 2048 outputs of each column go to T.
//   row phase     per 8-row block: even-column half -> Z_e, FFT (E); odd half ->
//                 Z_o, FFT (O); radix-2 step -> two real rows of C (C2R packing);
//                 fused max / first argmax / sum of squares.
//   window        6 warps recompute the row pairs covering the 11 rows around the
//                 peak (their blocks staged by TMA) and sum the 11 x 11 energy.

#include <math.h>
#include <stdio.h>

#include <algorithm>

// Complex arithmetic in this kernel: packed FADD2 adds and the decimation-in-time
// register DFT with FFMA2 butterflies, but scalar complex multiplies -- with two
// 32-value FFT operands (e, o) live at 255 registers, building the swapped
// operand of a packed multiply by a runtime twiddle costs more than it saves.
// Same-box A/B at N = 512: all scalar (DIF) 78.2k, packed multiplies too 61.5k,
// scalar + DIT 88.2k, packed adds + DIT 88.7k pairs/s (at a 110 MHz lower clock).
#ifndef PCE2K_F32X2
#define PCE2K_F32X2 1
#endif
#ifndef RK_F32X2
#define RK_F32X2 PCE2K_F32X2
#endif
#ifndef RK_F32X2_MUL
#define RK_F32X2_MUL 0
#endif
#ifndef RK_DIT
#define RK_DIT 1
#endif
#include "fft.cuh"
#include "pce_common.cuh"
#include "internal.h"

namespace rk {

namespace {
using namespace pcek;

constexpr int R = 32;
constexpr int N = 2048;            // pattern side
constexpr int H = 1024;            // half line: one warp FFT
constexpr int NC = N / 2;          // stored half-spectrum columns
constexpr int kWarps = 8;
constexpr int kUnitF2 = 4 * H;     // float2 per staged unit: 4 columns x 1024 rows == one T half block
constexpr uint32_t kUnitBytes = kUnitF2 * sizeof(float2);   // 32 KiB
constexpr int kQuartets = NC / 4;  // 256 column quartets, split over the two warp groups
constexpr int kBlocks = N / 8;     // 256 row blocks
constexpr int kP1Rows = 8;         // rows per row-pass preprocess CTA (4 warps)
constexpr int kP1Tile = kP1Rows + 1;
constexpr int kXbuf = R * (R + 1);   // padded transpose buffer (group_fft_pad)

// W_2048^lane, forward sign
__device__ __forceinline__ float2 lane_w2048(int lane) {
  float sn, cs;
  sincospif((float)lane / (float)H, &sn, &cs);
  return make_float2(cs, -sn);
}

// ---------------------------------------------------------------------------
// Preprocess P1: zero-mean, forward 2048-point row FFTs (two real rows per
// complex FFT), unpack to half spectra, U[item][c][row] (column 0 packed).
__global__ void __launch_bounds__(128) pce2k_rows_fwd(const float* __restrict__ pix, size_t stride_f,
                                                      const float* __restrict__ mean_part, float2* __restrict__ U,
                                                      const float2* __restrict__ tw) {
  extern __shared__ float2 smem[];
  float2* tile = smem;                       // NC x kP1Tile
  float2* nat = tile + NC * kP1Tile;         // 4 warps x N: natural-order Z (first R*R = FFT transpose buffer)
  __shared__ float s_mean;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = blockIdx.y;
  const int r0 = blockIdx.x * kP1Rows;
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < kMeanParts; ++i) s += (double)mean_part[item * kMeanParts + i];
    s_mean = (float)(s / ((double)N * (double)N));
  }
  __syncthreads();
  const float mu = s_mean;
  float2* nb = nat + warp * N;
  const int ra = r0 + 2 * warp;
  const float2* xa = reinterpret_cast<const float2*>(pix + (size_t)item * stride_f + (size_t)ra * N);
  const float2* xb = xa + N / 2;
  float2 e[R], o[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    const float2 a = __ldg(xa + lane + R * n2), b = __ldg(xb + lane + R * n2);   // samples 2j, 2j+1
    e[n2] = make_float2(a.x - mu, b.x - mu);
    o[n2] = make_float2(a.y - mu, b.y - mu);
  }
  group_fft_pad<R, false>(e, nb, tw, lane);
  group_fft_pad<R, false>(o, nb, tw, lane);
  radix2_last<false>(e, o, lane_w2048(lane));
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) {
    nb[lane + R * k1] = e[k1];
    nb[H + lane + R * k1] = o[k1];
  }
  __syncwarp();
#pragma unroll 4
  for (int n = 0; n < R; ++n) {
    const int k = lane + R * n;
    const float2 z = nb[k];
    float2 a, b;
    if (k == 0) {
      const float2 zn = nb[H];
      a = make_float2(z.x, zn.x);   // (A[0], A[N/2]) both real
      b = make_float2(z.y, zn.y);
    } else {
      const float2 zr = c_conj(nb[N - k]);
      a = c_scale(c_add(z, zr), 0.5f);
      const float2 d = c_sub(z, zr);
      b = make_float2(0.5f * d.y, -0.5f * d.x);   // d / (2i)
    }
    tile[k * kP1Tile + 2 * warp] = a;
    tile[k * kP1Tile + 2 * warp + 1] = b;
  }
  __syncthreads();
  float2* Ui = U + (size_t)item * NC * N;
  for (int idx = tid; idx < NC * kP1Rows; idx += 128) {
    const int c = idx / kP1Rows, rr = idx % kP1Rows;
    Ui[(size_t)c * N + r0 + rr] = tile[c * kP1Tile + rr];
  }
}

// Preprocess P2: forward 2048-point column FFTs of U (one warp per column),
// scaled by 1/N, into the slot's parity-split layout S[p][c][m].
__global__ void __launch_bounds__(kWarps * 32) pce2k_cols_fwd(const float2* __restrict__ U, char* __restrict__ slots,
                                                              size_t slot_stride, SlotList dst,
                                                              const float2* __restrict__ tw) {
  extern __shared__ float2 smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = blockIdx.y;
  const int col = blockIdx.x * kWarps + warp;
  float2* xbuf = smem + warp * kXbuf;
  const float4* Uc = reinterpret_cast<const float4*>(U + (size_t)item * NC * N + (size_t)col * N);
  float2 e[R], o[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    const float4 q = Uc[lane + R * n2];   // rows 2j, 2j+1
    e[n2] = make_float2(q.x, q.y);
    o[n2] = make_float2(q.z, q.w);
  }
  group_fft_pad<R, false>(e, xbuf, tw, lane);
  group_fft_pad<R, false>(o, xbuf, tw, lane);
  radix2_last<false>(e, o, lane_w2048(lane));
  float2* S = reinterpret_cast<float2*>(slots + (size_t)dst.idx[item] * slot_stride);
  constexpr float kScale = 1.0f / (float)N;
  // output row k = lane + R*k1 (and k + H): parity lane & 1, m = k >> 1
  float2* Sp = S + ((size_t)(lane & 1) * NC + col) * H + (lane >> 1);
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) {
    Sp[16 * k1] = c_scale(e[k1], kScale);
    Sp[H / 2 + 16 * k1] = c_scale(o[k1], kScale);
  }
}

// ---------------------------------------------------------------------------
// Z_o[m] = Z[2m + 1] for row pair rp of a staged odd-column half block:
// column j = m for m < 512, the Hermitian mirror j = 1023 - m (conjugated) above.
__device__ __forceinline__ void half_rows_zodd(float2 (&v)[R], const float2* blk, int rp, int lane) {
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    const int m = lane + R * n2;
    const int j = (n2 < R / 2) ? m : (H - 1 - m);
    const float4 q = *reinterpret_cast<const float4*>(blk + j * 8 + 2 * (rp ^ ((j >> 1) & 3)));
    float2 a = make_float2(q.x, q.y), c = make_float2(q.z, q.w);
    if (n2 >= R / 2) {
      a.y = -a.y;
      c.y = -c.y;
    }
    v[n2] = make_float2(a.x - c.y, a.y + c.x);
  }
}

// Running (max, first index, sum of squares) over one row pair: e holds columns
// lane + R*k1, o columns H + lane + R*k1; .x = row ra, .y = row ra + 1.
__device__ __forceinline__ void argmax2k_update(const float2 (&e)[R], const float2 (&o)[R], int ra, int lane,
                                                float& m, int& idx, double& ss) {
  float lm = -INFINITY, bs = 0.f;
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) {
    bs = fmaf(e[k1].x, e[k1].x, bs);
    bs = fmaf(e[k1].y, e[k1].y, bs);
    bs = fmaf(o[k1].x, o[k1].x, bs);
    bs = fmaf(o[k1].y, o[k1].y, bs);
    lm = fmaxf(lm, fmaxf(fmaxf(e[k1].x, e[k1].y), fmaxf(o[k1].x, o[k1].y)));
  }
  ss += (double)bs;
  if (lm >= m) {
    // first occurrence in row-major order: row ra before ra + 1, then column
    int li = 0x7fffffff;
#pragma unroll
    for (int k1 = R - 1; k1 >= 0; --k1)
      if (o[k1].x == lm) li = ra * N + H + lane + R * k1;
#pragma unroll
    for (int k1 = R - 1; k1 >= 0; --k1)
      if (e[k1].x == lm) li = ra * N + lane + R * k1;
    if (li == 0x7fffffff) {
#pragma unroll
      for (int k1 = R - 1; k1 >= 0; --k1)
        if (o[k1].y == lm) li = (ra + 1) * N + H + lane + R * k1;
#pragma unroll
      for (int k1 = R - 1; k1 >= 0; --k1)
        if (e[k1].y == lm) li = (ra + 1) * N + lane + R * k1;
    }
    if (lm > m || li < idx) {
      m = lm;
      idx = li;
    }
  }
}

// Two real rows (ra, ra + 1) of C from a staged 8-row block (even half at blk,
// odd half at blk + kUnitF2): e <- columns lane + R*k1, o <- columns H + lane + R*k1.
__device__ __forceinline__ void block_rows_c2r(float2 (&e)[R], float2 (&o)[R], const float2* even_half,
                                               const float2* odd_half, int rp, float2* xbuf, const float2* tw,
                                               float2 wl, int lane) {
  block8_rows_z<R>(e, even_half, rp, lane);
  group_fft_pad<R, true>(e, xbuf, tw, lane);
  half_rows_zodd(o, odd_half, rp, lane);
  group_fft_pad<R, true>(o, xbuf, tw, lane);
  radix2_last<true>(e, o, wl);
}

// Window energy of row pair (ra, ra + 1) from its staged 8-row block: the sum of
// C^2 over the rows within [rstart, rstart + 11) and the 11 columns around pcol.
// Kept out of line so the cold window path does not raise the register
// allocation (and spills) of the hot column and row passes.
__device__ __noinline__ float window_rows(const float2* blk, int ra, int rstart, int pcol, float2* xbuf,
                                          const float2* tw, float2 wl, int lane) {
  float2 e[R], o[R];
  block_rows_c2r(e, o, blk, blk + kUnitF2, (ra & 7) >> 1, xbuf, tw, wl, lane);
  const bool va = ((ra - rstart + N) & (N - 1)) < kWin;
  const bool vb = ((ra + 1 - rstart + N) & (N - 1)) < kWin;
  float w = 0.f;
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) {
    const int s0 = lane + R * k1, s1 = s0 + H;
    if (((s0 - pcol + kHalfWin + N) & (N - 1)) < kWin) {
      if (va) w = fmaf(e[k1].x, e[k1].x, w);
      if (vb) w = fmaf(e[k1].y, e[k1].y, w);
    }
    if (((s1 - pcol + kHalfWin + N) & (N - 1)) < kWin) {
      if (va) w = fmaf(o[k1].x, o[k1].x, w);
      if (vb) w = fmaf(o[k1].y, o[k1].y, w);
    }
  }
  return warp_sum(w);
}

// Column-phase staging: per-warp columns and mbarriers (1, default) or one 4-column
// unit per warp group refilled after a group barrier (0).  Same box at N = 512:
// with the scalar DIF FFT the group form won (80.2k vs 74.4k pairs/s); with the
// DIT FFMA2 butterflies the per-warp form wins (90.1k vs 89.0k at a 75 MHz lower clock).
// Row-phase half release by counted arrival (1) or a group barrier (0).
#ifndef PCE2K_ROW_ARRIVE
#define PCE2K_ROW_ARRIVE 1
#endif
#ifndef PCE2K_WARP_COLS
#define PCE2K_WARP_COLS 1
#endif

__global__ void __launch_bounds__(kWarps * 32, 1) pce2k_pair(const PairJob job, const char* __restrict__ slots,
                                                            size_t slot_stride, float2* __restrict__ T, size_t t_stride,
                                                            const float2* __restrict__ tw_g, double* __restrict__ out,
                                                            uint8_t* __restrict__ flags, double threshold,
                                                            const LedgerRef ledger, unsigned* __restrict__ rounds,
                                                            int l2opts) {
  constexpr int kGW = kWarps / 2;                        // warps per warp group
  constexpr int kPairsOfRows = (kWin + 1) / 2;
  extern __shared__ __align__(128) float2 smem[];
  float2* gbufs = smem;                                  // 2 groups x 2 units
  float2* tw = smem + 4 * kUnitF2;                       // R*R twiddles (W_1024)
  float2* xbufs = tw + R * R;                            // one padded transpose buffer per warp
  __shared__ __align__(8) uint64_t s_bar[2][3];          // per group: column units, row halves even / odd
  __shared__ unsigned s_done[2][2];                      // per group and row half: warps done reading
  __shared__ __align__(8) uint64_t s_wbar;
  __shared__ __align__(8) uint64_t s_cbar[kWarps];        // per warp: its column (PCE2K_WARP_COLS)
  __shared__ float s_v[kWarps];
  __shared__ int s_i[kWarps];
  __shared__ double s_ss[kWarps];
  __shared__ float s_wpart[kPairsOfRows];
  __shared__ float s_peak;
  __shared__ int s_pidx;
  __shared__ double s_total;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wg = warp / kGW;
  const int gi = warp % kGW;
  const bool leader = (tid % (kGW * 32)) == 0;
  float2* xbuf = xbufs + warp * kXbuf;
  float2* gb = gbufs + wg * 2 * kUnitF2;
  float2* Tp = T + (size_t)blockIdx.x * t_stride;
  for (int i = tid; i < R * R; i += kWarps * 32) tw[i] = tw_g[i];
  if (tid == 0) {
    for (int w = 0; w < 2; ++w)
      for (int b = 0; b < 3; ++b) mbar_init(&s_bar[w][b], 1);
    mbar_init(&s_wbar, 1);
    for (int w = 0; w < kWarps; ++w) mbar_init(&s_cbar[w], 1);
    s_done[0][0] = s_done[0][1] = s_done[1][0] = s_done[1][1] = 0u;
  }
  uint32_t ph = 0, wph = 0;
#if PCE2K_WARP_COLS
  uint32_t cph = 0;
#endif
  __syncthreads();
  // hot-loop FFTs: lane twiddles in registers (default) or from the shared table
#ifndef PCE2K_SMEM_TW
  float2 twr[R];
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) twr[k1] = tw[k1 * R + lane];
#define PCE2K_FFT(v) group_fft_pad_rt<R, true>(v, xbuf, twr, lane)
#else
#define PCE2K_FFT(v) group_fft_pad<R, true>(v, xbuf, tw, lane)
#endif
  const float2 wl = lane_w2048(lane);
  const uint64_t pol_first = l2_policy_evict_first();
  const uint64_t pol = (l2opts & 2) ? l2_policy_evict_last() : l2_policy_evict_normal();   // spectra
  const uint64_t pol_T = (l2opts & 1) ? pol_first : l2_policy_evict_normal();

  for (int pi = blockIdx.x; pi < job.npairs; pi += gridDim.x) {
    round_wait(rounds, pi, gridDim.x, tid, PCE2K_ROUND_SLACK_PCT);
    const DevPair pr = job.pairs[pi];
    const float2* Xs = reinterpret_cast<const float2*>(slots + (size_t)pr.slot_a * slot_stride);
    const float2* Ys = reinterpret_cast<const float2*>(slots + (size_t)pr.slot_b * slot_stride);

    // ---------------- column phase ----------------
    // unit u of this group: quartet wg + 2*(u >> 1), row parity u & 1
    {
      constexpr int kUnits = 2 * (kQuartets / 2);
#if PCE2K_WARP_COLS
      // per-warp pipeline: lane 0 copies this warp's own X and Y column of unit u
      uint64_t* wbar = &s_cbar[warp];
      auto issue = [&](int u) {
        const int col = 4 * (wg + 2 * (u >> 1)) + gi, p = u & 1;
        const size_t off = ((size_t)p * NC + col) * H;
        constexpr uint32_t kColBytes = (uint32_t)(H * sizeof(float2));
        refill_fence();
        mbar_expect_tx(wbar, 2 * kColBytes);
        bulk_g2s_hint(gb + gi * H, Xs + off, kColBytes, wbar, pol);
        bulk_g2s_hint(gb + kUnitF2 + gi * H, Ys + off, kColBytes, wbar, pol);
      };
#else
      uint64_t* bar = &s_bar[wg][0];
      auto issue = [&](int u) {
        const int cq = wg + 2 * (u >> 1), p = u & 1;
        const size_t off = ((size_t)p * NC + 4 * cq) * H;
        fence_proxy_async();   // measured: dropping it here is not faster at 2048^2
        mbar_expect_tx(bar, 2 * kUnitBytes);
        bulk_g2s_hint(gb, Xs + off, kUnitBytes, bar, pol);
        bulk_g2s_hint(gb + kUnitF2, Ys + off, kUnitBytes, bar, pol);
      };
#endif
      // product X * conj(Y) of this warp's column for unit u, then refill the buffers
      auto product = [&](int u, float2 (&v)[R]) {
        const int col = 4 * (wg + 2 * (u >> 1)) + gi;
        const int p = u & 1;
#if PCE2K_WARP_COLS
        mbar_wait(wbar, cph & 1u);
        cph ^= 1u;
#else
        mbar_wait(bar, ph & 1u);
        ph ^= 1u;
#endif
        const float2* X = gb + gi * H;
        const float2* Y = gb + kUnitF2 + gi * H;
        if (col != 0) {
#pragma unroll
          for (int n2 = 0; n2 < R; ++n2) v[n2] = c_mulc(X[lane + R * n2], Y[lane + R * n2]);
        } else {
          // packed DC/Nyquist column: Hermitian split (row r <-> N - r keeps parity:
          // even m <-> (H - m) mod H, odd m <-> H - 1 - m), separate products, re-pack
#pragma unroll
          for (int n2 = 0; n2 < R; ++n2) {
            const int m = lane + R * n2;
            const int mm = p == 0 ? ((H - m) & (H - 1)) : (H - 1 - m);
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
#if PCE2K_WARP_COLS
        __syncwarp();
        if (lane == 0 && u + 1 < kUnits) issue(u + 1);
      };
      if (lane == 0) issue(0);
#else
        named_bar(1 + wg, kGW * 32);
        if (leader && u + 1 < kUnits) issue(u + 1);
      };
      if (leader) issue(0);
#endif
#pragma unroll 1
      for (int u = 0; u < kUnits; u += 2) {
        const int col = 4 * (wg + 2 * (u >> 1)) + gi;
        float2 e[R], o[R];
        product(u, e);
        PCE2K_FFT(e);
        product(u + 1, o);
        PCE2K_FFT(o);
        radix2_last<true>(e, o, wl);
        // row n = lane + R*k1 -> block (lane >> 3) + 4*k1, row lane & 7; row n + H -> block + 128
        const int j = col >> 1;
        const int rr = lane & 7;
        const int pos = (((rr >> 1) ^ ((j >> 1) & 3)) << 1) | (rr & 1);
        float2* dst = Tp + (((size_t)(lane >> 3) * 2 + (col & 1)) * (NC / 2) + j) * 8 + pos;
        constexpr size_t kStep = (size_t)4 * 2 * (NC / 2) * 8;
        constexpr size_t kHalfRows = (size_t)(H / 8) * 2 * (NC / 2) * 8;
#pragma unroll
        for (int k1 = 0; k1 < R; ++k1) {
          stg_hint(dst + k1 * kStep, e[k1], pol_T);
          stg_hint(dst + kHalfRows + k1 * kStep, o[k1], pol_T);
        }
      }
    }
    __syncthreads();   // T complete (both groups) before any row block is read

    // ---------------- row phase ----------------
    float m = -INFINITY;
    int idx = 0x7fffffff;
    double ss = 0.0;
    {
      auto issue = [&](int rb, int half) {
        mbar_expect_tx(&s_bar[wg][1 + half], kUnitBytes);
        bulk_g2s_hint(gb + half * kUnitF2, Tp + ((size_t)rb * 2 + half) * kUnitF2, kUnitBytes,
                      &s_bar[wg][1 + half], pol_first);
      };
      // a half is consumed once the group's kGW warps have read their row pair: the
      // last reader (acq_rel count, PCE2K_ROW_ARRIVE) or the group leader after a
      // group barrier refills it, behind the generic -> async proxy fence
      auto release_half = [&](int rb, int half) {
#if PCE2K_ROW_ARRIVE
        __syncwarp();
        if (lane == 0 && rb + 2 < kBlocks &&
            atom_acq_rel_add_shared(&s_done[wg][half], 1u) % kGW == (unsigned)(kGW - 1)) {
          refill_fence();
          issue(rb + 2, half);
        }
#else
        named_bar(1 + wg, kGW * 32);
        if (leader && rb + 2 < kBlocks) {
          refill_fence();
          issue(rb + 2, half);
        }
#endif
      };
      if (leader) {
        fence_proxy_async();   // T's generic-proxy stores (ordered by the barrier) -> async proxy
        issue(wg, 0);
        issue(wg, 1);
      }
#pragma unroll 1
      for (int rb = wg; rb < kBlocks; rb += 2) {
        float2 e[R], o[R];
        mbar_wait(&s_bar[wg][1], (ph >> 1) & 1u);
        ph ^= 2u;
        block8_rows_z<R>(e, gb, gi, lane);
        release_half(rb, 0);
        PCE2K_FFT(e);
        mbar_wait(&s_bar[wg][2], (ph >> 2) & 1u);
        ph ^= 4u;
        half_rows_zodd(o, gb + kUnitF2, gi, lane);
        release_half(rb, 1);
        PCE2K_FFT(o);
        radix2_last<true>(e, o, wl);
        argmax2k_update(e, o, 8 * rb + 2 * gi, lane, m, idx, ss);
      }
    }
    {
      ArgMax best = warp_argmax(ArgMax{m, idx});
      ss = warp_sum(ss);
      if (lane == 0) {
        s_v[warp] = best.v;
        s_i[warp] = best.idx;
        s_ss[warp] = ss;
      }
      __syncthreads();
      if (tid == 0) {
        ArgMax bb{s_v[0], s_i[0]};
        double t = s_ss[0];
        for (int w = 1; w < kWarps; ++w) {
          if (better(s_v[w], s_i[w], bb.v, bb.idx)) bb = ArgMax{s_v[w], s_i[w]};
          t += s_ss[w];
        }
        s_peak = bb.v;
        s_pidx = bb.idx;
        s_total = t;
      }
      __syncthreads();
    }

    // ---------------- window: 11 rows around the peak ----------------
    // The 6 aligned row pairs covering rows peak-5 .. peak+5 lie in at most three
    // 8-row blocks; each block is staged whole (both halves, 64 KiB) and the warps
    // owning a row pair in it recompute that pair.
    {
      const int prow = s_pidx / N, pcol = s_pidx % N;
      const int rstart = (prow - kHalfWin + N) & (N - 1);
      const int e0 = rstart & ~1;
      const int b0 = e0 >> 3;
      const int ra = (e0 + 2 * warp) & (N - 1);   // warp t < 6 owns row pair (ra, ra + 1)
#pragma unroll 1
      for (int jb = 0; jb < 3; ++jb) {
        const int blk = (b0 + jb) & (kBlocks - 1);
        bool any = false;
        for (int t = 0; t < kPairsOfRows; ++t) any |= (((e0 + 2 * t) & (N - 1)) >> 3) == blk;
        if (!any) continue;
        if (tid == 0) {
          fence_proxy_async();
          mbar_expect_tx(&s_wbar, 2 * kUnitBytes);
          bulk_g2s_hint(gbufs, Tp + (size_t)blk * 2 * kUnitF2, 2 * kUnitBytes, &s_wbar, pol_first);
        }
        mbar_wait(&s_wbar, wph & 1u);
        wph ^= 1u;
        if (warp < kPairsOfRows && (ra >> 3) == blk) {
          const float w = window_rows(gbufs, ra, rstart, pcol, xbuf, tw, wl, lane);
          if (lane == 0) s_wpart[warp] = w;
        }
        __syncthreads();   // staged block consumed before the next one lands
      }
    }
    if (tid == 0) {
      const double peak = (double)s_peak;
      double wsum = 0.0;
      for (int t = 0; t < kPairsOfRows; ++t) wsum += (double)s_wpart[t];
      const double energy = (s_total - wsum) / ((double)N * (double)N - (double)(kWin * kWin));
      const double pce = peak * fabs(peak) / energy;
      out[pr.pid] = pce;
      ledger_mark(ledger, pr.pid);
      if (flags) flags[pr.pid] = isnan(threshold) ? 0 : (uint8_t)(1 | (pce >= threshold ? 2 : 0));
    }
    round_arrive(rounds, tid);
    __syncthreads();   // shared state and buffers free for the next pair
  }
}

constexpr size_t kRowsFwdSmem = (size_t)(NC * kP1Tile + 4 * N) * sizeof(float2);
constexpr size_t kColsFwdSmem = (size_t)(kWarps * kXbuf) * sizeof(float2);
constexpr size_t kPairSmem = (size_t)(4 * kUnitF2 + R * R + kWarps * kXbuf) * sizeof(float2);

}  // namespace

rk_status pce2k_init(rk_app* app) {
  PceState& st = app->pce;
  RK_CUDA(cudaFuncSetAttribute(pce2k_rows_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowsFwdSmem));
  RK_CUDA(cudaFuncSetAttribute(pce2k_cols_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kColsFwdSmem));
  RK_CUDA(cudaFuncSetAttribute(pce2k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPairSmem));
  int per_sm = 0, sms = 0, dev = 0;
  RK_CUDA(cudaGetDevice(&dev));
  RK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pce2k_pair, kWarps * 32, kPairSmem));
  if (per_sm < 1) return set_error(RK_ERR_DEVICE, "pce2k_pair: does not fit on an SM");
  st.clusters = per_sm * sms;
  st.t_stride = (size_t)NC * N + stride_pad("RK_T_PAD", 0) / sizeof(float2);
  RK_CUDA(cudaMalloc(&st.T, sizeof(float2) * st.t_stride * st.clusters));
  st.job = new PairJob();
  return pce_round_init(st, 3);
}

rk_status pce2k_preprocess(rk_app* app, const float* pix, size_t stride_f, int n_items, char* slots,
                           size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  PceState& st = app->pce;
  for (int base = 0; base < n_items; base += st.batch) {
    const int m = std::min(st.batch, n_items - base);
    const float* px = pix + (size_t)base * stride_f;
    pce_launch_mean(px, stride_f, N * N, m, st.mean_part, s);
    pce2k_rows_fwd<<<dim3(N / kP1Rows, m), 128, kRowsFwdSmem, s>>>(px, stride_f, st.mean_part, st.U, st.tw);
    SlotList dst;
    dst.n = m;
    for (int k = 0; k < m; ++k) dst.idx[k] = h_slot_idx[base + k];
    pce2k_cols_fwd<<<dim3(NC / kWarps, m), kWarps * 32, kColsFwdSmem, s>>>(st.U, slots, slot_stride, dst, st.tw);
    app->launches += 3;
    RK_CUDA(cudaGetLastError());
  }
  return RK_OK;
}

rk_status pce2k_compare(rk_app* app, const char* slots, size_t slot_stride, const rk_pair* pairs, int n,
                        double* d_out, uint8_t* d_flags, cudaStream_t s) {
  PceState& st = app->pce;
  PairJob& job = *st.job;
  job.npairs = n;
  job.depth = 0;
  for (int k = 0; k < n; ++k) {
    job.pairs[k].slot_a = pairs[k].slot_a;
    job.pairs[k].slot_b = pairs[k].slot_b;
    job.pairs[k].pid = pair_id(app->p.n, pairs[k].i, pairs[k].j);
  }
  const int grid = std::min(st.clusters, n);
  if (st.rounds) RK_CUDA(cudaMemsetAsync(st.rounds, 0, sizeof(unsigned), s));
  pce2k_pair<<<grid, kWarps * 32, kPairSmem, s>>>(job, slots, slot_stride, st.T, st.t_stride, st.tw, d_out, d_flags,
                                                   threshold_or_nan(app), app->ledger, st.rounds, st.l2opts);
  app->launches += 1;
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

}  // namespace rk
