// Localization-microscopy particle registration cost (GMM / Bhattacharyya) for sm_100a.
//
// Item: a particle of m localizations (x, y, sigma) fp32.
// Parsed layout (host):  u32 m | u32 pad | m x {f32 x, f32 y, f32 sigma}
// Slot layout (device):  u32 m | u32 pad | m x {f32 x - cx, f32 y - cy, f32 sigma^2}   (centroid removed)
//
// Pair cost over a fixed rotation grid theta_k = 2*pi*k/K (translation fixed by
// the centroids; Heydarian et al., with the transform search
// fixed so the result is deterministic):
//   E_k    = sum_a sum_b exp( -|R(theta_k) p_a - q_b|^2 / (s_a^2 + s_b^2 + s0) )
//   value  = max_k E_k / (m_i * m_j)
// One CTA per pair (gmm_pair_kernel below), up to 1,024 pairs per launch.
// Oracle: oracle/gmm.py (parity unpinned by the reference; 1e-4 relative).
#include <math.h>

#include "internal.h"

namespace rk {

namespace {


__global__ void gmm_preprocess_kernel(const uint8_t* __restrict__ parsed, size_t parsed_stride, SlotList dst,
                                      uint8_t* __restrict__ slots, size_t slot_stride, int cap,
                                      int* __restrict__ status) {
  const int item = blockIdx.x;
  const uint8_t* src = parsed + (size_t)item * parsed_stride;
  const uint32_t m = *reinterpret_cast<const uint32_t*>(src);
  if (m == 0 || (int)m > cap) {
    if (threadIdx.x == 0) atomicMax(status, m == 0 ? (int)RK_ERR_MALFORMED : (int)RK_ERR_SLOT_OVERFLOW);
    return;
  }
  const float* pts = reinterpret_cast<const float*>(src + 8);
  __shared__ double s_cx, s_cy;
  if (threadIdx.x == 0) {
    double cx = 0.0, cy = 0.0;   // fixed order: deterministic centroid
    for (uint32_t a = 0; a < m; ++a) {
      cx += pts[3 * a];
      cy += pts[3 * a + 1];
    }
    s_cx = cx / m;
    s_cy = cy / m;
  }
  __syncthreads();
  uint8_t* slot = slots + (size_t)dst.idx[item] * slot_stride;
  float* out = reinterpret_cast<float*>(slot + 8);
  const float cx = (float)s_cx, cy = (float)s_cy;
  for (uint32_t a = threadIdx.x; a < m; a += blockDim.x) {
    out[3 * a] = pts[3 * a] - cx;
    out[3 * a + 1] = pts[3 * a + 1] - cy;
    out[3 * a + 2] = pts[3 * a + 2] * pts[3 * a + 2];
  }
  if (threadIdx.x == 0) {
    *reinterpret_cast<uint32_t*>(slot) = m;
    *reinterpret_cast<uint32_t*>(slot + 4) = 0u;
  }
}

// One CTA (8 warps) per pair.  Work units = (32-point chunk of particle i) x
// (quarter of particle j), dealt round-robin to the warps; particle j sits in
// shared memory as (x, y, s^2 + s0, |q|^2) and is read by broadcast.  The
// rotation leaves |p| unchanged, so per (a, b, k)
//   -|R_k p - q|^2 w = (2 (R_k p).q - |p|^2 - |q|^2) w,   w = log2(e) / (s_a^2 + s_b^2)
// costs one FMUL + two FFMA + one MUFU.EX2 (+ the add), done for two angles at a
// time as packed fp32 pairs (FMUL2 / FFMA2 / FADD2); the reciprocal is shared by
// the 12 angles of a block, so the kernel is bound by the SFU's ex2 rate (moving
// 2 or 3 of the 12 exponentials to an FMA-pipe polynomial measured slower).
constexpr int kPairWarps = 8;
constexpr int kAngBlock = 12;

// 1/x for x > 0 on the FMA pipe (the SFU is the kernel's bottleneck): a bit-trick
// seed and three Newton steps, relative error < 1e-7 over the normal range.
__device__ __forceinline__ float rcp_fma(float x) {
  float y = __int_as_float(0x7EF311C7 - __float_as_int(x));
  y = y * fmaf(-x, y, 2.0f);
  y = y * fmaf(-x, y, 2.0f);
  y = y * fmaf(-x, y, 2.0f);
  return y;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// grid = pairs x angle blocks: CTA (p, ab) evaluates angles 12ab .. 12ab+11 of
// pair p and stores its best E_k in blk_best[p * nblk + ab]; gmm_finalize takes
// the max over the blocks (order-independent: deterministic).  Splitting the
// angle grid over CTAs gives ~7 waves per 1,024-pair launch instead of 2.3.
__global__ void __launch_bounds__(kPairWarps * 32) gmm_pair_kernel(const PairJob job, const uint8_t* __restrict__ slots,
                                                                   size_t slot_stride, int angles, float s0,
                                                                   double* __restrict__ blk_best) {
  extern __shared__ float4 Q[];                       // particle j (m_j entries)
  __shared__ float2 s_cs[kAngBlock];                  // (cos, sin) of this CTA's angles
  __shared__ float s_part[kPairWarps][kAngBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = (angles + kAngBlock - 1) / kAngBlock;
  const int ab = blockIdx.x % nblk;
  const DevPair pr = job.pairs[blockIdx.x / nblk];
  const uint8_t* si = slots + (size_t)pr.slot_a * slot_stride;
  const uint8_t* sj = slots + (size_t)pr.slot_b * slot_stride;
  const int mi = (int)*reinterpret_cast<const uint32_t*>(si);
  const int mj = (int)*reinterpret_cast<const uint32_t*>(sj);
  const float* pi = reinterpret_cast<const float*>(si + 8);
  const float* pj = reinterpret_cast<const float*>(sj + 8);
  for (int c = threadIdx.x; c < mj; c += blockDim.x) {
    const float x = pj[3 * c], y = pj[3 * c + 1];
    Q[c] = make_float4(x, y, pj[3 * c + 2] + s0, fmaf(x, x, y * y));
  }
  for (int t = threadIdx.x; t < kAngBlock; t += blockDim.x) {
    const int k = min(ab * kAngBlock + t, angles - 1);   // pad the last block with a repeated angle
    float sn, cs;
    sincospif(2.0f * (float)k / (float)angles, &sn, &cs);
    s_cs[t] = make_float2(cs, sn);
  }
  __syncthreads();
  constexpr float kLog2e = 1.4426950408889634f;
  const int n_chunks = (mi + 31) / 32;
  const int units = n_chunks * 4;
  const int qlen = (mj + 3) / 4;
  {
    // per angle pair: the two angles' running sums (fp32 lanes of one FADD2)
    float2 acc2[kAngBlock / 2];
#pragma unroll
    for (int t = 0; t < kAngBlock / 2; ++t) acc2[t] = make_float2(0.f, 0.f);
    for (int u = warp; u < units; u += kPairWarps) {
      const int a = (u >> 2) * 32 + lane;
      const int c0 = (u & 3) * qlen, c1 = min(mj, c0 + qlen);
      if (a < mi) {
        const float px = pi[3 * a], py = pi[3 * a + 1], sa = pi[3 * a + 2];
        const float pp = fmaf(px, px, py * py);
        // the rotated point for two angles at a time as packed fp32 pairs: the
        // FMUL2 / FFMA2 / FADD2 forms give the scalar results bit for bit with half
        // the issue slots, leaving the MUFU.EX2 pipe as the only limit
        float2 rx[kAngBlock / 2], ry[kAngBlock / 2];
#pragma unroll
        for (int t = 0; t < kAngBlock; t += 2) {
          const float2 wa = s_cs[t], wb = s_cs[t + 1];
          rx[t / 2] = make_float2(wa.x * px - wa.y * py, wb.x * px - wb.y * py);
          ry[t / 2] = make_float2(wa.y * px + wa.x * py, wb.y * px + wb.x * py);
        }
        for (int c = c0; c < c1; ++c) {
          const float4 q = Q[c];
          const float w = kLog2e * rcp_fma(sa + q.z);   // no MUFU.RCP: 12 ex2 per 12 terms
          const float w2 = 2.0f * w;
          const float base = -(pp + q.w) * w;
#pragma unroll
          for (int t = 0; t < kAngBlock / 2; ++t) {
            const float2 dot = __ffma2_rn(rx[t], make_float2(q.x, q.x), __fmul2_rn(ry[t], make_float2(q.y, q.y)));
            const float2 arg = __ffma2_rn(dot, make_float2(w2, w2), make_float2(base, base));
            acc2[t] = __fadd2_rn(acc2[t], make_float2(ex2_approx(arg.x), ex2_approx(arg.y)));
          }
        }
      }
    }
    // warp sums, then a fixed-order sum over the warps
#pragma unroll
    for (int t = 0; t < kAngBlock; ++t) {
      float v = (t & 1) ? acc2[t / 2].y : acc2[t / 2].x;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) s_part[warp][t] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double best = -1.0;
      for (int t = 0; t < kAngBlock; ++t) {
        double e = 0.0;
        for (int w = 0; w < kPairWarps; ++w) e += (double)s_part[w][t];
        best = fmax(best, e);
      }
      blk_best[blockIdx.x] = best / ((double)mi * (double)mj);
    }
  }
}

__global__ void gmm_finalize(const PairJob job, int nblk, const double* __restrict__ blk_best,
                             double* __restrict__ out, uint8_t* __restrict__ flags, double threshold,
                             const LedgerRef ledger) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= job.npairs) return;
  double v = -1.0;
  for (int b = 0; b < nblk; ++b) v = fmax(v, blk_best[(size_t)p * nblk + b]);
  const int64_t pid = job.pairs[p].pid;
  out[pid] = v;
  ledger_mark(ledger, pid);
  if (flags) flags[pid] = isnan(threshold) ? 0 : (uint8_t)(1 | (v >= threshold ? 2 : 0));
}

}  // namespace

rk_status gmm_init(rk_app* app) {
  const int cap = app->p.max_entries;
  if (cap <= 0) return set_error(RK_ERR_VALUE, "GMM app needs max_entries (max localizations) > 0");
  if (app->p.gmm_angles <= 0) app->p.gmm_angles = 36;
  app->slot_bytes = 8 + 12 * (size_t)cap;
  app->parsed_bytes = 8 + 12 * (size_t)cap;
  if (app->p.gmm_angles > 256) return set_error(RK_ERR_UNSUPPORTED, "GMM angle grid > 256");
  const size_t smem = (size_t)cap * sizeof(float4);
  if (smem > 200 * 1024) return set_error(RK_ERR_UNSUPPORTED, "GMM max_entries %d too large for shared memory", cap);
  RK_CUDA(cudaFuncSetAttribute(gmm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (!app->job) app->job = new PairJob();
  const int nblk = (app->p.gmm_angles + kAngBlock - 1) / kAngBlock;
  RK_CUDA(cudaMalloc(&app->gmm_scratch, sizeof(double) * kListPairs * nblk));
  return RK_OK;
}

rk_status gmm_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                         size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  int* d_status = nullptr;
  RK_TRY(status_begin(app, s, &d_status));
  for (int base = 0; base < n_items; base += kMaxBatch) {
    const int m = n_items - base < kMaxBatch ? n_items - base : kMaxBatch;
    SlotList dst;
    dst.n = m;
    for (int k = 0; k < m; ++k) dst.idx[k] = h_slot_idx[base + k];
    gmm_preprocess_kernel<<<m, 128, 0, s>>>(static_cast<const uint8_t*>(d_parsed) + (size_t)base * parsed_stride,
                                            parsed_stride, dst, static_cast<uint8_t*>(d_slots), slot_stride,
                                            app->p.max_entries, d_status);
    app->launches += 1;
    RK_CUDA(cudaGetLastError());
  }
  int h_status = 0;
  RK_TRY(status_end(app, s, &h_status));
  if (h_status == RK_ERR_SLOT_OVERFLOW)
    return set_error(RK_ERR_SLOT_OVERFLOW, "particle exceeds %d localizations", app->p.max_entries);
  if (h_status == RK_ERR_MALFORMED) return set_error(RK_ERR_MALFORMED, "particle has no localizations");
  return RK_OK;
}

rk_status gmm_compare_list(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* pairs, int n,
                          double* d_out, uint8_t* d_flags, cudaStream_t s) {
  const size_t smem = (size_t)app->p.max_entries * sizeof(float4);
  PairJob& job = *app->job;
  for (int base = 0; base < n; base += kListPairs) {
    const int m = n - base < kListPairs ? n - base : kListPairs;
    job.npairs = m;
    for (int k = 0; k < m; ++k) {
      const rk_pair& q = pairs[base + k];
      job.pairs[k] = DevPair{q.slot_a, q.slot_b, pair_id(app->p.n, q.i, q.j)};
    }
    const int nblk = (app->p.gmm_angles + kAngBlock - 1) / kAngBlock;
    gmm_pair_kernel<<<m * nblk, kPairWarps * 32, smem, s>>>(job, static_cast<const uint8_t*>(d_slots), slot_stride,
                                                            app->p.gmm_angles, app->p.gmm_scale, app->gmm_scratch);
    gmm_finalize<<<(m + 127) / 128, 128, 0, s>>>(job, nblk, app->gmm_scratch, d_out, d_flags, threshold_or_nan(app), app->ledger);
    app->launches += 2;
    RK_CUDA(cudaGetLastError());
  }
  return RK_OK;
}

}  // namespace rk
