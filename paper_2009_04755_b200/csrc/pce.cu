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
// Kernels per batch of pairs (all launched on one stream):
//   K1 pce_corr_cols  : product + inverse column FFTs  -> T (column-major, per pair)
//   K2 pce_rows_reduce: inverse row C2R FFTs (two rows per complex FFT), fused
//                       max/argmax/energy reduction; the last CTA of each pair
//                       recomputes the 11 peak rows and writes the PCE score.
// T stays L2-resident between K1 and K2 when batch * 4 MiB fits in L2.
#include <math.h>
#include <stdio.h>

#include "fft.cuh"
#include "internal.h"

namespace rk {

namespace {

constexpr int kGroups = 8;              // FFT groups (columns or row-pairs) per CTA
constexpr int kRows = 2 * kGroups;      // rows per row-pass CTA
constexpr int kTileStride = kRows + 1;  // padded row stride of the [k][row] tile
constexpr int kMeanParts = 64;          // CTAs per item in the mean reduction
constexpr int kWin = 11;                // PCE exclusion neighbourhood side
constexpr int kHalfWin = kWin / 2;

__device__ __forceinline__ bool better(float v, int idx, float bv, int bidx) {
  return v > bv || (v == bv && idx < bidx);
}

template <int R>
__device__ __forceinline__ void load_tw(float2* tw, const float2* __restrict__ tw_g, int tid, int nt) {
  for (int i = tid; i < R * R; i += nt) tw[i] = tw_g[i];
}

// Half-spectrum row value A[k] of row `rr` of a [k][row] tile (k in [0, N)),
// Hermitian-extended; column 0 holds (A[0], A[N/2]) packed, both real.
template <int N>
__device__ __forceinline__ float2 tile_row_value(const float2* tile, int ts, int k, int rr) {
  if (k == 0) return make_float2(tile[rr].x, 0.f);
  if (k == N / 2) return make_float2(tile[rr].y, 0.f);
  if (k < N / 2) return tile[k * ts + rr];
  return c_conj(tile[(N - k) * ts + rr]);
}

// Same from global memory: T is column-major, column k holds N rows.
template <int N>
__device__ __forceinline__ float2 global_row_value(const float2* __restrict__ Tp, int k, int row) {
  if (k == 0) return make_float2(Tp[row].x, 0.f);
  if (k == N / 2) return make_float2(Tp[row].y, 0.f);
  if (k < N / 2) return Tp[(size_t)k * N + row];
  return c_conj(Tp[(size_t)(N - k) * N + row]);
}

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
  float2* tw = smem;
  float2* tile = smem + R * R;                       // (N/2) x kTileStride
  float2* xbufs = tile + (N / 2) * kTileStride;      // kGroups x R*(R+1)
  __shared__ float s_mean;
  const int tid = threadIdx.x;
  const int item = blockIdx.y;
  const int r0 = blockIdx.x * kRows;
  load_tw<R>(tw, tw_g, tid, NT);
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < kMeanParts; ++i) s += (double)mean_part[item * kMeanParts + i];
    s_mean = (float)(s / ((double)N * (double)N));
  }
  __syncthreads();
  const float mu = s_mean;
  const int g = tid / R, lane = tid % R;
  float2* xbuf = xbufs + g * R * (R + 1);
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
  float2* tw = smem;
  const int tid = threadIdx.x;
  load_tw<R>(tw, tw_g, tid, kGroups * R);
  __syncthreads();
  const int item = blockIdx.y;
  const int g = tid / R, lane = tid % R;
  float2* xbuf = smem + R * R + g * R * (R + 1);
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

// ---------------------------------------------------------------------------
// Compare K1: P = S_a * conj(S_b) on one column group, inverse column FFT -> T.
template <int R>
__global__ void __launch_bounds__(kGroups * R) pce_corr_cols(PairBatch b, const char* __restrict__ slots,
                                                            size_t slot_stride, float2* __restrict__ T,
                                                            const float2* __restrict__ tw_g) {
  constexpr int N = R * R;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  const int tid = threadIdx.x;
  load_tw<R>(tw, tw_g, tid, kGroups * R);
  __syncthreads();
  const int p = blockIdx.y;
  const int g = tid / R, lane = tid % R;
  float2* xbuf = smem + R * R + g * R * (R + 1);
  const int col = blockIdx.x * kGroups + g;
  const float2* X = reinterpret_cast<const float2*>(slots + (size_t)b.slot_a[p] * slot_stride) + (size_t)col * N;
  const float2* Y = reinterpret_cast<const float2*>(slots + (size_t)b.slot_b[p] * slot_stride) + (size_t)col * N;
  float2 v[R];
  if (col != 0) {
#pragma unroll
    for (int n2 = 0; n2 < R; ++n2) v[n2] = c_mulc(__ldg(X + lane + R * n2), __ldg(Y + lane + R * n2));
  } else {
    // Packed DC/Nyquist column: split each side into its two Hermitian parts,
    // multiply separately, re-pack the (Hermitian) products.
#pragma unroll
    for (int n2 = 0; n2 < R; ++n2) {
      const int m = lane + R * n2;
      const int mm = (N - m) & (N - 1);
      const float2 x = __ldg(X + m), xr = c_conj(__ldg(X + mm));
      const float2 y = __ldg(Y + m), yr = c_conj(__ldg(Y + mm));
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
  group_fft<R, true>(v, xbuf, tw, lane);
  float2* Tp = T + (size_t)p * (N / 2) * N + (size_t)col * N;
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) Tp[lane + R * k2] = v[k2];
}

// Block-wide reductions for K2 (blockDim = kGroups * R threads).
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

// Compare K2: inverse row FFTs of 16 rows of T, fused reductions; the last CTA
// of each pair finalises the PCE score.
template <int R>
__global__ void __launch_bounds__(kGroups * R) pce_rows_reduce(PairBatch b, const float2* __restrict__ T,
                                                              float4* __restrict__ part,
                                                              unsigned* __restrict__ counters,
                                                              const float2* __restrict__ tw_g,
                                                              double* __restrict__ out,
                                                              uint8_t* __restrict__ flags, double threshold) {
  constexpr int N = R * R;
  constexpr int NT = kGroups * R;
  constexpr int NW = NT / 32;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* tile = smem + R * R;   // (N/2) x kTileStride; later the groups' transpose buffers
  __shared__ float s_v[NW];
  __shared__ int s_i[NW];
  __shared__ double s_d[NW];
  __shared__ int s_last;
  __shared__ float s_peak;
  __shared__ int s_pidx;
  __shared__ double s_total;

  const int tid = threadIdx.x;
  const int p = blockIdx.y;
  const int r0 = blockIdx.x * kRows;
  const int warp = tid >> 5;
  load_tw<R>(tw, tw_g, tid, NT);
  const float2* Tp = T + (size_t)p * (N / 2) * N;
  for (int idx = tid; idx < (N / 2) * kRows; idx += NT) {
    const int c = idx / kRows, rr = idx % kRows;
    tile[c * kTileStride + rr] = Tp[(size_t)c * N + r0 + rr];
  }
  __syncthreads();
  const int g = tid / R, lane = tid % R;
  float2 v[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) {
    const int k = lane + R * n2;
    const float2 a = tile_row_value<N>(tile, kTileStride, k, 2 * g);
    const float2 c = tile_row_value<N>(tile, kTileStride, k, 2 * g + 1);
    v[n2] = make_float2(a.x - c.y, a.y + c.x);
  }
  __syncthreads();  // tile becomes transpose scratch
  float2* xbuf = tile + g * R * (R + 1);
  group_fft<R, true>(v, xbuf, tw, lane);

  ArgMax best{-INFINITY, 0x7fffffff};
  float ss = 0.f;
  const int ra = r0 + 2 * g;
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) {
    const int s = lane + R * k2;
    const float ca = v[k2].x, cb = v[k2].y;
    ss = fmaf(ca, ca, ss);
    ss = fmaf(cb, cb, ss);
    const int ia = ra * N + s;
    if (better(ca, ia, best.v, best.idx)) best = ArgMax{ca, ia};
    const int ib = ia + N;
    if (better(cb, ib, best.v, best.idx)) best = ArgMax{cb, ib};
  }
  best = warp_argmax(best);
  ss = warp_sum(ss);
  if ((tid & 31) == 0) {
    s_v[warp] = best.v;
    s_i[warp] = best.idx;
    s_d[warp] = (double)ss;
  }
  __syncthreads();
  if (tid == 0) {
    ArgMax bb{s_v[0], s_i[0]};
    float t = (float)s_d[0];
    for (int w = 1; w < NW; ++w) {
      if (better(s_v[w], s_i[w], bb.v, bb.idx)) bb = ArgMax{s_v[w], s_i[w]};
      t += (float)s_d[w];
    }
    part[(size_t)p * gridDim.x + blockIdx.x] = make_float4(bb.v, __int_as_float(bb.idx), t, 0.f);
    __threadfence();
    s_last = (atomicAdd(&counters[p], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- finalize (last CTA of pair p) ----
  {
    ArgMax a{-INFINITY, 0x7fffffff};
    double t = 0.0;
    for (int q = tid; q < (int)gridDim.x; q += NT) {
      const float4 e = __ldcg(part + (size_t)p * gridDim.x + q);
      const int ei = __float_as_int(e.y);
      if (better(e.x, ei, a.v, a.idx)) a = ArgMax{e.x, ei};
      t += (double)e.z;
    }
    a = warp_argmax(a);
    t = warp_sum(t);
    if ((tid & 31) == 0) {
      s_v[warp] = a.v;
      s_i[warp] = a.idx;
      s_d[warp] = t;
    }
    __syncthreads();
    if (tid == 0) {
      ArgMax bb{s_v[0], s_i[0]};
      double tt = s_d[0];
      for (int w = 1; w < NW; ++w) {
        if (better(s_v[w], s_i[w], bb.v, bb.idx)) bb = ArgMax{s_v[w], s_i[w]};
        tt += s_d[w];
      }
      s_peak = bb.v;
      s_pidx = bb.idx;
      s_total = tt;
    }
    __syncthreads();
  }
  const int pr = s_pidx / N, pc = s_pidx % N;
  float wsum = 0.f;
  constexpr int kPairsOfRows = (kWin + 1) / 2;  // 6 groups recompute 11 rows
  if (g < kPairsOfRows) {
    const int t0 = 2 * g, t1 = 2 * g + 1;
    const bool has_b = t1 < kWin;
    const int rowa = (pr - kHalfWin + t0 + N) & (N - 1);
    const int rowb = (pr - kHalfWin + t1 + N) & (N - 1);
#pragma unroll
    for (int n2 = 0; n2 < R; ++n2) {
      const int k = lane + R * n2;
      const float2 a = global_row_value<N>(Tp, k, rowa);
      const float2 c = has_b ? global_row_value<N>(Tp, k, rowb) : make_float2(0.f, 0.f);
      v[n2] = make_float2(a.x - c.y, a.y + c.x);
    }
    group_fft<R, true>(v, xbuf, tw, lane);
#pragma unroll
    for (int k2 = 0; k2 < R; ++k2) {
      const int s = lane + R * k2;
      if (((s - pc + kHalfWin + N) & (N - 1)) < kWin) {
        wsum = fmaf(v[k2].x, v[k2].x, wsum);
        if (has_b) wsum = fmaf(v[k2].y, v[k2].y, wsum);
      }
    }
  }
  wsum = warp_sum(wsum);
  __syncthreads();
  if ((tid & 31) == 0) s_d[warp] = (double)wsum;
  __syncthreads();
  if (tid == 0) {
    double w = 0.0;
    for (int q = 0; q < NW; ++q) w += s_d[q];
    const double peak = (double)s_peak;
    const double energy = (s_total - w) / ((double)N * (double)N - (double)(kWin * kWin));
    const double pce = peak * fabs(peak) / energy;
    const int64_t pid = b.pid[p];
    out[pid] = pce;
    if (flags) flags[pid] = isnan(threshold) ? 0 : (uint8_t)(1 | (pce >= threshold ? 2 : 0));
    counters[p] = 0u;
  }
}

template <int R>
size_t cols_smem() {
  return (size_t)(R * R + kGroups * R * (R + 1)) * sizeof(float2);
}
template <int R>
size_t rows_smem() {
  constexpr int N = R * R;
  const size_t tile = (size_t)(N / 2) * kTileStride;
  const size_t xb = (size_t)kGroups * R * (R + 1);
  return (size_t)(R * R + (tile > xb ? tile : xb)) * sizeof(float2);
}
template <int R>
size_t rows_fwd_smem() {
  constexpr int N = R * R;
  return (size_t)(R * R + (N / 2) * kTileStride + kGroups * R * (R + 1)) * sizeof(float2);
}

template <int R>
rk_status set_attrs() {
  RK_CUDA(cudaFuncSetAttribute(pce_corr_cols<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem<R>()));
  RK_CUDA(cudaFuncSetAttribute(pce_cols_fwd<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem<R>()));
  RK_CUDA(cudaFuncSetAttribute(pce_rows_reduce<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_smem<R>()));
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
    pce_cols_fwd<R><<<dim3(N / 2 / kGroups, m), kGroups * R, cols_smem<R>(), s>>>(st.U, slots, slot_stride, dst, st.tw);
    app->launches += 3;
    RK_CUDA(cudaGetLastError());
  }
  return RK_OK;
}

template <int R>
rk_status compare_impl(rk_app* app, const char* slots, size_t slot_stride, const PairBatch& b, double* d_out,
                       uint8_t* d_flags, cudaStream_t s) {
  constexpr int N = R * R;
  PceState& st = app->pce;
  if (b.npairs > st.batch) return set_error(RK_ERR_VALUE, "PCE batch of %d pairs exceeds workspace (%d)", b.npairs, st.batch);
  pce_corr_cols<R><<<dim3(N / 2 / kGroups, b.npairs), kGroups * R, cols_smem<R>(), s>>>(b, slots, slot_stride, st.T, st.tw);
  pce_rows_reduce<R><<<dim3(N / kRows, b.npairs), kGroups * R, rows_smem<R>(), s>>>(
      b, st.T, reinterpret_cast<float4*>(st.part), st.counters, st.tw, d_out, d_flags, threshold_or_nan(app));
  app->launches += 2;
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

}  // namespace

rk_status pce_init(rk_app* app) {
  const int h = app->p.height, w = app->p.width;
  if (h != w) return set_error(RK_ERR_UNSUPPORTED, "PCE patterns must be square (got %dx%d)", h, w);
  int R = 0;
  if (h == 256) R = 16;
  else if (h == 1024) R = 32;
  else return set_error(RK_ERR_UNSUPPORTED, "PCE pattern side %d not built (256 or 1024)", h);
  PceState& st = app->pce;
  st.R = R;
  st.N = h;
  st.batch = app->p.batch_pairs > 0 ? app->p.batch_pairs : (R == 32 ? 16 : 64);
  if (st.batch > kMaxBatch) st.batch = kMaxBatch;
  const int N = st.N;
  app->slot_bytes = (size_t)N * N * sizeof(float);       // (N/2)*N complex64
  app->parsed_bytes = (size_t)N * N * sizeof(float);
  // twiddles W_N^(n1*k1), stored [k1][n1]
  std::vector<float2> tw((size_t)R * R);
  for (int k1 = 0; k1 < R; ++k1)
    for (int n1 = 0; n1 < R; ++n1) {
      const double ang = -2.0 * M_PI * (double)(n1 * k1) / (double)N;
      tw[(size_t)k1 * R + n1] = make_float2((float)cos(ang), (float)sin(ang));
    }
  RK_CUDA(cudaMalloc(&st.tw, sizeof(float2) * R * R));
  RK_CUDA(cudaMemcpy(st.tw, tw.data(), sizeof(float2) * R * R, cudaMemcpyHostToDevice));
  const size_t per = (size_t)(N / 2) * N;
  RK_CUDA(cudaMalloc(&st.T, sizeof(float2) * per * st.batch));
  st.U = st.T;  // preprocess and compare never overlap on one app (one stream per app)
  const int row_ctas = N / kRows;
  RK_CUDA(cudaMalloc(&st.part, sizeof(float4) * (size_t)row_ctas * st.batch));
  RK_CUDA(cudaMalloc(&st.counters, sizeof(unsigned) * 2 * st.batch));
  RK_CUDA(cudaMemset(st.counters, 0, sizeof(unsigned) * 2 * st.batch));
  RK_CUDA(cudaMalloc(&st.mean_part, sizeof(float) * kMeanParts * st.batch));
  if (R == 16) return set_attrs<16>();
  return set_attrs<32>();
}

void pce_free(rk_app* app) {
  PceState& st = app->pce;
  cudaFree(st.tw);
  cudaFree(st.T);
  cudaFree(st.part);
  cudaFree(st.counters);
  cudaFree(st.mean_part);
  st = PceState{};
}

rk_status pce_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                         size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  if (parsed_stride % 16 != 0) return set_error(RK_ERR_VALUE, "parsed_stride must be a multiple of 16 bytes");
  const float* pix = static_cast<const float*>(d_parsed);
  const size_t stride_f = parsed_stride / sizeof(float);
  if (app->pce.R == 16)
    return preprocess_impl<16>(app, pix, stride_f, n_items, static_cast<char*>(d_slots), slot_stride, h_slot_idx, s);
  return preprocess_impl<32>(app, pix, stride_f, n_items, static_cast<char*>(d_slots), slot_stride, h_slot_idx, s);
}

rk_status pce_compare(rk_app* app, const void* d_slots, size_t slot_stride, const PairBatch& b, double* d_out,
                      uint8_t* d_flags, cudaStream_t s) {
  const char* slots = static_cast<const char*>(d_slots);
  if (app->pce.R == 16) return compare_impl<16>(app, slots, slot_stride, b, d_out, d_flags, s);
  return compare_impl<32>(app, slots, slot_stride, b, d_out, d_flags, s);
}

}  // namespace rk
