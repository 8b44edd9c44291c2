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
// One warp per pair: both particles staged in the warp's shared memory, lane
// stripes over a, sequential over b (fixed order), warp tree reduction per k.
// Oracle: oracle/gmm.py (parity unpinned by the reference; 1e-4 relative).
#include <math.h>

#include "internal.h"

namespace rk {

namespace {

constexpr int kWarps = 4;   // pairs per CTA

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

__global__ void __launch_bounds__(kWarps * 32) gmm_compare_kernel(PairBatch b, const uint8_t* __restrict__ slots,
                                                                  size_t slot_stride, int cap, int angles, float s0,
                                                                  double* __restrict__ out,
                                                                  uint8_t* __restrict__ flags, double threshold) {
  extern __shared__ float4 gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * kWarps + warp;
  if (p >= b.npairs) return;
  float4* P = gsm + (size_t)warp * 2 * cap;   // particle i: (x, y, s^2)
  float4* Q = P + cap;                        // particle j
  const uint8_t* si = slots + (size_t)b.slot_a[p] * slot_stride;
  const uint8_t* sj = slots + (size_t)b.slot_b[p] * slot_stride;
  const int mi = (int)*reinterpret_cast<const uint32_t*>(si);
  const int mj = (int)*reinterpret_cast<const uint32_t*>(sj);
  const float* pi = reinterpret_cast<const float*>(si + 8);
  const float* pj = reinterpret_cast<const float*>(sj + 8);
  for (int a = lane; a < mi; a += 32) P[a] = make_float4(pi[3 * a], pi[3 * a + 1], pi[3 * a + 2], 0.f);
  for (int c = lane; c < mj; c += 32) Q[c] = make_float4(pj[3 * c], pj[3 * c + 1], pj[3 * c + 2] + s0, 0.f);
  __syncwarp();
  constexpr float kLog2e = 1.4426950408889634f;
  double best = -1.0;
  for (int k = 0; k < angles; ++k) {
    float sn, cs;
    sincospif(2.0f * (float)k / (float)angles, &sn, &cs);
    float acc = 0.f;
    for (int a = lane; a < mi; a += 32) {
      const float4 u = P[a];
      const float rx = cs * u.x - sn * u.y, ry = sn * u.x + cs * u.y;
      float part = 0.f;
      for (int c = 0; c < mj; ++c) {
        const float4 v = Q[c];
        const float dx = rx - v.x, dy = ry - v.y;
        const float d2 = fmaf(dx, dx, dy * dy);
        part += exp2f(-kLog2e * d2 / (u.z + v.z));
      }
      acc += part;
    }
    double e = (double)acc;
#pragma unroll
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    best = fmax(best, e);
  }
  if (lane == 0) {
    const double v = best / ((double)mi * (double)mj);
    out[b.pid[p]] = v;
    if (flags) flags[b.pid[p]] = isnan(threshold) ? 0 : (uint8_t)(1 | (v >= threshold ? 2 : 0));
  }
}

}  // namespace

rk_status gmm_init(rk_app* app) {
  const int cap = app->p.max_entries;
  if (cap <= 0) return set_error(RK_ERR_VALUE, "GMM app needs max_entries (max localizations) > 0");
  if (app->p.gmm_angles <= 0) app->p.gmm_angles = 36;
  app->slot_bytes = 8 + 12 * (size_t)cap;
  app->parsed_bytes = 8 + 12 * (size_t)cap;
  const size_t smem = (size_t)kWarps * 2 * cap * sizeof(float4);
  if (smem > 200 * 1024) return set_error(RK_ERR_UNSUPPORTED, "GMM max_entries %d too large for shared memory", cap);
  RK_CUDA(cudaFuncSetAttribute(gmm_compare_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return RK_OK;
}

rk_status gmm_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                         size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  int* d_status = nullptr;
  RK_CUDA(cudaMallocAsync(&d_status, sizeof(int), s));
  RK_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int), s));
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
  RK_CUDA(cudaMemcpyAsync(&h_status, d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
  RK_CUDA(cudaFreeAsync(d_status, s));
  RK_CUDA(cudaStreamSynchronize(s));
  if (h_status == RK_ERR_SLOT_OVERFLOW)
    return set_error(RK_ERR_SLOT_OVERFLOW, "particle exceeds %d localizations", app->p.max_entries);
  if (h_status == RK_ERR_MALFORMED) return set_error(RK_ERR_MALFORMED, "particle has no localizations");
  return RK_OK;
}

rk_status gmm_compare(rk_app* app, const void* d_slots, size_t slot_stride, const PairBatch& b, double* d_out,
                      uint8_t* d_flags, cudaStream_t s) {
  const size_t smem = (size_t)kWarps * 2 * app->p.max_entries * sizeof(float4);
  gmm_compare_kernel<<<(b.npairs + kWarps - 1) / kWarps, kWarps * 32, smem, s>>>(
      b, static_cast<const uint8_t*>(d_slots), slot_stride, app->p.max_entries, app->p.gmm_angles, app->p.gmm_scale,
      d_out, d_flags, threshold_or_nan(app));
  app->launches += 1;
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

}  // namespace rk
