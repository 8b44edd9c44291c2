// Microbenchmark: warp-FFT compute ceiling (no global traffic in the loop).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2009_04755_b200/csrc/fft.cuh"
using namespace rk;

template <int R, int WARPS, bool REG_TW>
__global__ void __launch_bounds__(WARPS * 32) fft_loop(const float2* __restrict__ tw_g, float2* out, int iters) {
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* xbuf = smem + R * R + (threadIdx.x / R) * R * R;
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) tw[i] = tw_g[i];
  __syncthreads();
  const int lane = threadIdx.x % R;
  float2 v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = make_float2(lane * 0.001f + i, i * 0.5f);
  float2 twr[R];
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) twr[k1] = tw[k1 * R + lane];
  for (int it = 0; it < iters; ++it) {
    if constexpr (REG_TW) group_fft_rt<R, true>(v, xbuf, twr, lane);   // the compare kernel's form
    else group_fft<R, true>(v, xbuf, tw, lane);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = c_scale(v[i], 1.0f / 1024.f);
  }
  float2 acc = make_float2(0, 0);
#pragma unroll
  for (int i = 0; i < R; ++i) acc = c_add(acc, v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int WARPS, bool REG_TW>
void run(int ctas_per_sm) {
  constexpr int R = 32;
  std::vector<float2> tw(R * R);
  for (int k = 0; k < R; ++k) for (int n = 0; n < R; ++n) { double a = -2 * M_PI * n * k / 1024.0; tw[k * R + n] = make_float2(cos(a), sin(a)); }
  float2 *dtw, *dout;
  cudaMalloc(&dtw, sizeof(float2) * R * R);
  cudaMemcpy(dtw, tw.data(), sizeof(float2) * R * R, cudaMemcpyHostToDevice);
  int grid = 148 * ctas_per_sm;
  cudaMalloc(&dout, sizeof(float2) * grid * WARPS * 32);
  size_t smem = (R * R + WARPS * R * R) * sizeof(float2);
  cudaFuncSetAttribute(fft_loop<R, WARPS, REG_TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int iters = 200;
  fft_loop<R, WARPS, REG_TW><<<grid, WARPS * 32, smem>>>(dtw, dout, 10);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  fft_loop<R, WARPS, REG_TW><<<grid, WARPS * 32, smem>>>(dtw, dout, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ffts = (double)grid * WARPS * iters;
  printf("%s warps/cta=%d ctas/sm=%d: %.3f ms, %.2f ns/FFT (chip), %.3f us per 1024 FFTs (=1 pair), err=%s\n", REG_TW ? "reg-tw" : "smem-tw", WARPS, ctas_per_sm, ms,
         ms * 1e6 / ffts, ms * 1e3 / ffts * 1024, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  // warps per SM: 8 (the compare kernel), 12, 16, 24 -- is the FFT issue-latency bound?
  run<8, true>(1); run<8, false>(1); run<4, true>(3); run<4, false>(3); run<8, false>(2); run<16, false>(1);
  run<4, false>(6);
  return 0;
}
