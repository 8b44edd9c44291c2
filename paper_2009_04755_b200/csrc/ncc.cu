// Zero-lag normalised cross-correlation (NCC) for sm_100a.
//
//   preprocess   x^ = (x - mean x) / ||x - mean x||        (fp32, one slot = D floats)
//   compare      ncc(i, j) = x^_i . x^_j                   (the forensics NCC)
//
// Two compare paths:
//   * rk_ncc_gram  -- the all-pairs path: the Gram matrix X^ X^T over the slot
//     arena as a tcgen05 tensor-core GEMM (kind::tf32, 128x128 tiles, TMEM
//     accumulators, TMA-fed 4-stage mbarrier pipeline, warp-specialised
//     producer / MMA issuer / epilogue).  Only upper-triangle tiles are launched;
//     the epilogue writes pair_id-indexed results for i < j.  TF32 rounds the
//     operands to 10 mantissa bits: |error| <= 2e-4 * ||x^_i|| ||x^_j|| = 2e-4
//     absolute for normalised items (stated looser bound, tests/test_ncc_gpu.py).
//   * rk_compare_pairs -- arbitrary pairs, one warp per pair, fp32 CUDA-core dot
//     (the reference-style per-pair Application path).
// Oracle: oracle/ncc.py (parity unpinned by the reference, which has no NCC).
#include <cuda.h>
#include <math.h>

#include <algorithm>

#include "fft.cuh"
#include "internal.h"

namespace rk {

namespace {

constexpr int kTile = 128;          // items per Gram tile side (UMMA M = N = 128)
constexpr int kBK = 32;             // fp32 elements per 128-B swizzled smem row (one TMA box row)
#ifndef NCC_STAGES
#define NCC_STAGES 6
#endif
constexpr int kStages = NCC_STAGES;  // 6 x 32 KiB in flight per SM (K = 1M streams: latency-bound at 4)
constexpr int kStageBytes = 2 * kTile * kBK * 4;   // A + B tiles: 32 KiB
constexpr int kGramThreads = 128;   // 4 warps: TMA producer, MMA issuer, all four in the epilogue
constexpr int kGroup = 128;         // slots per interleaved group (rk_app_slot_group)
constexpr int kKC = 1024;           // interleave run (floats) when D % 1024 == 0

// Byte offset of element e of slot s.  Group g = s / 128 owns the region
// [g*128*stride, (g+1)*128*stride) laid out as [D/kc][128][kc] floats, so the
// 128 items of a Gram tile row block at one k sit within 128*kc*4 bytes (one
// 512 KiB span) instead of 128 different pages: the TMA loads stop missing the
// TLB once the arena outgrows its reach (measured: 16 GiB arena -> 250 TF/s).
__host__ __device__ __forceinline__ size_t ncc_off(int64_t s, int64_t e, int64_t kc, size_t stride) {
  return (size_t)(s / kGroup) * kGroup * stride +
         (size_t)(((e / kc) * kGroup + (s % kGroup)) * kc + e % kc) * sizeof(float);
}

// ---------------------------------------------------------------------------
// preprocess: per item two passes -- (sum, sum of squares) then normalise
__global__ void __launch_bounds__(256) ncc_moments(const float* __restrict__ pix, size_t stride_f, int64_t d,
                                                   double* __restrict__ part) {
  const int item = blockIdx.y;
  const float4* x = reinterpret_cast<const float4*>(pix + (size_t)item * stride_f);
  const int64_t n4 = d / 4;
  double s = 0.0, q = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(x + i);
    s += (double)v.x + (double)v.y + (double)v.z + (double)v.w;
    q += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  __shared__ double rs[8], rq[8];
  if ((threadIdx.x & 31) == 0) {
    rs[threadIdx.x >> 5] = s;
    rq[threadIdx.x >> 5] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tq = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      ts += rs[w];
      tq += rq[w];
    }
    part[((size_t)item * gridDim.x + blockIdx.x) * 2 + 0] = ts;
    part[((size_t)item * gridDim.x + blockIdx.x) * 2 + 1] = tq;
  }
}

__global__ void __launch_bounds__(256) ncc_normalise(const float* __restrict__ pix, size_t stride_f, int64_t d,
                                                     int64_t kc, const double* __restrict__ part, int nparts,
                                                     char* slots, size_t slot_stride, SlotList dst,
                                                     int* __restrict__ status) {
  const int item = blockIdx.y;
  __shared__ float s_mu, s_inv;
  if (threadIdx.x == 0) {
    double s = 0.0, q = 0.0;
    for (int k = 0; k < nparts; ++k) {
      s += part[((size_t)item * nparts + k) * 2 + 0];
      q += part[((size_t)item * nparts + k) * 2 + 1];
    }
    const double mu = s / (double)d;
    const double var = q - (double)d * mu * mu;   // sum of squared deviations
    s_mu = (float)mu;
    s_inv = var > 0.0 ? (float)(1.0 / sqrt(var)) : 0.f;
    if (!(var > 0.0) && blockIdx.x == 0) atomicMax(status, (int)RK_ERR_MALFORMED);   // constant item
  }
  __syncthreads();
  const float mu = s_mu, inv = s_inv;
  const float4* x = reinterpret_cast<const float4*>(pix + (size_t)item * stride_f);
  const int64_t sl = dst.idx[item];
  // runs of kc floats: the first run's address plus the run stride (128 * kc floats)
  float4* y0 = reinterpret_cast<float4*>(slots + ncc_off(sl, 0, kc, slot_stride));
  const int64_t run4 = kc / 4, jump4 = (int64_t)kGroup * kc / 4;
  const int64_t n4 = d / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(x + i);
    y0[(i / run4) * jump4 + i % run4] = make_float4((v.x - mu) * inv, (v.y - mu) * inv, (v.z - mu) * inv, (v.w - mu) * inv);
  }
}

// ---------------------------------------------------------------------------
// per-pair path: one warp per pair, fp32 dot with float4 loads
__global__ void __launch_bounds__(256) ncc_pairs_kernel(PairBatch b, const char* __restrict__ slots, size_t slot_stride,
                                                        int64_t d, int64_t kc, double* __restrict__ out,
                                                        uint8_t* __restrict__ flags, double threshold,
                                                        const LedgerRef ledger) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * 8 + warp;
  if (p >= b.npairs) return;
  const float4* x = reinterpret_cast<const float4*>(slots + ncc_off(b.slot_a[p], 0, kc, slot_stride));
  const float4* y = reinterpret_cast<const float4*>(slots + ncc_off(b.slot_b[p], 0, kc, slot_stride));
  float acc0 = 0.f, acc1 = 0.f;
  const int64_t run4 = kc / 4, jump4 = (int64_t)kGroup * kc / 4;
  for (int64_t r = 0; r < d / kc; ++r) {      // runs of kc floats, 128*kc apart
    const float4* xr = x + r * jump4;
    const float4* yr = y + r * jump4;
    for (int64_t i = lane; i < run4; i += 32) {
      const float4 u = __ldg(xr + i), v = __ldg(yr + i);
      acc0 = fmaf(u.x, v.x, fmaf(u.y, v.y, acc0));
      acc1 = fmaf(u.z, v.z, fmaf(u.w, v.w, acc1));
    }
  }
  double acc = (double)acc0 + (double)acc1;
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    out[b.pid[p]] = acc;
    ledger_mark(ledger, b.pid[p]);
    if (flags) flags[b.pid[p]] = isnan(threshold) ? 0 : (uint8_t)(1 | (acc >= threshold ? 2 : 0));
  }
}

// ---------------------------------------------------------------------------
// tcgen05 Gram kernel
__device__ __forceinline__ uint64_t umma_smem_desc_sw128(uint32_t smem_addr) {
  // K-major, 128-byte swizzle: rows of 128 B, 8-row (1 KiB) swizzle atoms.
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);   // start address
  d |= (uint64_t)1 << 16;                         // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;               // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                         // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                         // layout: SWIZZLE_128B
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = N = 128
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// 128 rows (items row0 .. row0+127, row0 % 128 == 0) x 32 floats at element e of
// the interleaved slot tensor (see ncc_off): coordinates (e % kc, 0, e / kc, row0 / 128)
__device__ __forceinline__ void tma_load_rows(void* dst, const CUtensorMap* map, int64_t e, int64_t kc, int row0,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(map), "r"((int)(e % kc)), "r"(0), "r"((int)(e / kc)), "r"(row0 / kGroup),
        "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&r)[32]) {
  uint32_t u[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
        "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
        "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) r[k] = __uint_as_float(u[k]);
}


// ---- CTA-pair (cta_group::2) variants: UMMA M = N = 256 over two SMs ----------
// Each CTA of the pair stages 128 rows of A and 128 rows of B (the same smem
// offsets in both); the leader's single thread issues the MMA, which reads both
// CTAs' tiles, and each CTA's TMEM receives its 128 accumulator rows x 256
// columns.  Operand bytes per SM per MMA flop are half of the 128x128 kernel's.
__device__ __forceinline__ void tma_load_rows_pair(void* dst, const CUtensorMap* map, int64_t e, int64_t kc, int row0,
                                                   uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(map), "r"((int)(e % kc)), "r"(0), "r"((int)(e / kc)), "r"(row0 / kGroup),
        "r"(bar_cluster) : "memory");
}

__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// arrive on `bar` (same smem offset) in both CTAs of the pair once the issued MMAs retire
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      ::"r"(smem_u32(bar)), "h"((uint16_t)0x3) : "memory");
}

// One CTA per upper-triangle 128x128 tile of items (tiles dealt to ranks).
__global__ void __launch_bounds__(kGramThreads, 1) ncc_gram_kernel(const __grid_constant__ CUtensorMap tmap, int n,
                                                                   int64_t d, int64_t kc, int tiles_per_side, int rank, int world,
                                                                   double* __restrict__ out,
                                                                   uint8_t* __restrict__ flags, double threshold,
                                                                   const LedgerRef ledger) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], done_bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // tile index -> (ti, tj), ti <= tj, row-major over the upper triangle
  int t = blockIdx.x * world + rank;
  int ti = 0;
  while (t >= tiles_per_side - ti) {
    t -= tiles_per_side - ti;
    ++ti;
  }
  const int tj = ti + t;
  const int row0 = ti * kTile, col0 = tj * kTile;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(kTile));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int kblocks = (int)(d / kBK);

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (uint32_t)(kb / kStages) & 1u;
      mbar_wait(&empty_bar[s], ph ^ 1u);
      uint8_t* a = smem + (size_t)s * kStageBytes;
      uint8_t* b = a + kTile * kBK * 4;
      mbar_expect_tx(&full_bar[s], kStageBytes);
      tma_load_rows(a, &tmap, (int64_t)kb * kBK, kc, row0, &full_bar[s]);
      tma_load_rows(b, &tmap, (int64_t)kb * kBK, kc, col0, &full_bar[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread) ----
    constexpr uint32_t idesc = idesc_tf32(kTile, kTile);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (uint32_t)(kb / kStages) & 1u;
      mbar_wait(&full_bar[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a = smem_u32(smem + (size_t)s * kStageBytes);
      const uint32_t b = a + kTile * kBK * 4;
#pragma unroll
      for (int k = 0; k < kBK / 8; ++k) {   // UMMA K = 8 for tf32: 32 B along the swizzled row
        umma_tf32(tmem, umma_smem_desc_sw128(a + k * 32), umma_smem_desc_sw128(b + k * 32), idesc,
                  (kb | k) != 0);
      }
      umma_commit(&empty_bar[s]);   // smem stage free once these MMAs retire
    }
    umma_commit(&done_bar);         // accumulator complete
  }

  // ---- epilogue: all four warps; warp w owns TMEM lanes (tile rows) 32w..32w+31 ----
  __syncwarp();
  mbar_wait(&done_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int i = row0 + warp * 32 + lane;
  const int64_t nn = n;
#pragma unroll 1
  for (int c = 0; c < kTile; c += 32) {
    float r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, r);
    if (i < n) {
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int j = col0 + c + k;
        if (j > i && j < n) {
          const int64_t pid = (int64_t)i * (2 * nn - i - 1) / 2 + (j - i - 1);
          out[pid] = (double)r[k];
          if (flags) flags[pid] = isnan(threshold) ? 0 : (uint8_t)(1 | ((double)r[k] >= threshold ? 2 : 0));
        }
      }
      // the valid columns j of this run are contiguous, and so are their pair ids
      const int j0 = max(col0 + c, i + 1), j1 = min(col0 + c + 32, n);
      if (j1 > j0) ledger_mark_run(ledger, (int64_t)i * (2 * nn - i - 1) / 2 + (j0 - i - 1), j1 - j0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTile));
}


constexpr int kTile2 = 256;   // items per CTA-pair tile side
#ifndef NCC_KCHUNK
#define NCC_KCHUNK 4096   // k-blocks per launch; A/B (profiles/r1_ab_ncc_stages*.log): 1024 32.9 ms, 2048 29.1-29.6, 4096 26.8-29.0, 8192 27.6-28.4
#endif
constexpr int kChunkBlocks = NCC_KCHUNK;   // k-blocks (x 32 floats) per launch: 128K floats

// A Gram block: rows of A = slots a_row0 .. a_row0 + a_cnt - 1 holding items (keys)
// a_key0 .., the same for B; tri = A and B are the same block (upper-triangle
// tiles only).  Tiles t with t % world == rank are computed.  Slot rows must be
// multiples of 128 (the interleaved slot groups).  The all-resident Gram is the
// block (0, 0, n) x (0, 0, n).
// Block of the Gram: A = arena rows a_row0 .. a_row0+a_cnt-1 holding keys
// a_key0 + r*a_kstep (likewise B).  tri: A == B, pairs lc > lr; otherwise every
// (lr, lc) is a pair, stored at pair_id(min(i, j), max(i, j)).  kstep 1: contiguous
// key blocks; kstep = world: one rank's home items (key = rank + m*world, the
// peer tier's point of contact k mod world).
struct GramBlock {
  int a_row0, a_key0, a_cnt;
  int b_row0, b_key0, b_cnt;
  int tri, rank, world;
  int na, nb;   // 256-item tiles along A and B
  int a_kstep, b_kstep;
};

// One CTA pair (cluster of 2) per 256x256 tile of a Gram block.
// K is processed in chunks [kb0, kb1) of k-blocks, one launch each: every CTA of
// a launch streams the same K window, so the tiles sharing an operand row block
// read it while it is still in L2 (with K = 1M in one launch the CTAs drift
// apart and most operand reads miss L2).  Chunk 0 stores, later chunks add
// (fp64, fixed launch order: deterministic); the last chunk writes the flags.
__global__ void __launch_bounds__(kGramThreads, 1) ncc_gram2_kernel(const __grid_constant__ CUtensorMap tmap, int n,
                                                                    int64_t d, int64_t kc, int kb0, int kb1,
                                                                    const GramBlock blk, double* __restrict__ out,
                                                                    uint8_t* __restrict__ flags, double threshold,
                                                                    const LedgerRef ledger) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], done_bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;

  int t = (blockIdx.x >> 1) * blk.world + blk.rank;
  int ti = 0, tj = 0;
  if (blk.tri) {
    while (t >= blk.na - ti) {
      t -= blk.na - ti;
      ++ti;
    }
    tj = ti + t;
  } else {
    ti = t / blk.nb;
    tj = t % blk.nb;
  }
  const int lrow0 = ti * kTile2 + (int)cta * kTile, lcol0 = tj * kTile2;   // within the block
  const int row0 = blk.a_row0 + lrow0;                                      // slots

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(kTile2));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int kblocks = kb1 - kb0;
  const bool first = kb0 == 0;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer (both CTAs): own A and B halves, completion on the leader's barrier ----
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (uint32_t)(kb / kStages) & 1u;
      mbar_wait(&empty_bar[s], ph ^ 1u);
      uint8_t* a = smem + (size_t)s * kStageBytes;
      uint8_t* b = a + kTile * kBK * 4;
#ifdef NCC_PROBE_NOTMA   // diagnostic: MMA rate on stale tiles
      if (leader) mbar_expect_tx(&full_bar[s], 0);
      (void)a;
      (void)b;
#else
      if (leader) mbar_expect_tx(&full_bar[s], 2 * kStageBytes);   // both CTAs' bytes
      const uint32_t fb = dsmem_addr(&full_bar[s], 0);
      tma_load_rows_pair(a, &tmap, (int64_t)(kb0 + kb) * kBK, kc, row0, fb);
      tma_load_rows_pair(b, &tmap, (int64_t)(kb0 + kb) * kBK, kc, blk.b_row0 + lcol0 + (int)cta * kTile, fb);
#endif
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---- MMA issuer (leader CTA, single thread) ----
    constexpr uint32_t idesc = idesc_tf32(kTile2, kTile2);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (uint32_t)(kb / kStages) & 1u;
      mbar_wait(&full_bar[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a = smem_u32(smem + (size_t)s * kStageBytes);
      const uint32_t b = a + kTile * kBK * 4;
#ifndef NCC_PROBE_NOMMA   // diagnostic: operand feed rate without the MMAs
#pragma unroll
      for (int k = 0; k < kBK / 8; ++k)
        umma_tf32_pair(tmem, umma_smem_desc_sw128(a + k * 32), umma_smem_desc_sw128(b + k * 32), idesc,
                       (kb | k) != 0);
#else
      (void)a;
      (void)b;
#endif
      umma_commit_pair(&empty_bar[s]);   // stage free in both CTAs once these MMAs retire
    }
    umma_commit_pair(&done_bar);
  }

  // ---- epilogue: each CTA drains its 128 rows x 256 columns ----
  __syncwarp();
  mbar_wait(&done_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int lr = lrow0 + warp * 32 + lane;
  const int i = blk.a_key0 + lr * blk.a_kstep;
  const int64_t nn = n;
#pragma unroll 1
  for (int c = 0; c < kTile2; c += 32) {
    float r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, r);
    if (lr < blk.a_cnt) {
      const bool last = (int64_t)kb1 * kBK >= d;   // the pairs complete with their last K chunk
      LedgerRun run{-1, 0u};
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int lc = lcol0 + c + k;
        if (lc < blk.b_cnt && (!blk.tri || lc > lr)) {
          const int j = blk.b_key0 + lc * blk.b_kstep;
          const int lo = min(i, j), hi = max(i, j);
          const int64_t pid = (int64_t)lo * (2 * nn - lo - 1) / 2 + (hi - lo - 1);
          const double v = first ? (double)r[k] : out[pid] + (double)r[k];
          out[pid] = v;
          if (last) {
            if (flags) flags[pid] = isnan(threshold) ? 0 : (uint8_t)(1 | (v >= threshold ? 2 : 0));
            ledger_run_add(ledger, run, pid);
          }
        }
      }
      ledger_run_flush(ledger, run);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTile2));
}

size_t gram_smem() { return (size_t)kStages * kStageBytes + 1024; }

}  // namespace

int ncc_gram_tile(int n) {
#ifndef NCC_GRAM_1CTA
  if (n > kTile) return kTile2;
#endif
  (void)n;
  return kTile;
}

rk_status tensor_map_encoder(EncodeTiledFn* fn) {
  static EncodeTiledFn cached = nullptr;
  if (!cached) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    RK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      return set_error(RK_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable from the driver");
    cached = reinterpret_cast<EncodeTiledFn>(p);
  }
  *fn = cached;
  return RK_OK;
}

rk_status ncc_init(rk_app* app) {
  const int64_t d = (int64_t)app->p.height * app->p.width;
  if (d <= 0 || d % kBK != 0)
    return set_error(RK_ERR_UNSUPPORTED, "NCC item size %lld must be a positive multiple of %d", (long long)d, kBK);
  app->slot_bytes = (size_t)d * sizeof(float);
  app->parsed_bytes = (size_t)d * sizeof(float);
  app->ncc.kc = (d % kKC == 0) ? kKC : d;
  app->slot_group = kGroup;
  RK_CUDA(cudaMalloc(&app->ncc.part, sizeof(double) * 2 * 64 * kMaxBatch));
  RK_CUDA(cudaFuncSetAttribute(ncc_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem()));
  RK_CUDA(cudaFuncSetAttribute(ncc_gram2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem()));
  return RK_OK;
}

void ncc_free(rk_app* app) {
  cudaFree(app->ncc.part);
  app->ncc.part = nullptr;
}

rk_status ncc_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                         size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  if (parsed_stride % 16 != 0 || slot_stride % 16 != 0)
    return set_error(RK_ERR_VALUE, "NCC strides must be multiples of 16 bytes");
  const int64_t d = (int64_t)app->p.height * app->p.width;
  int* d_status = nullptr;
  RK_TRY(status_begin(app, s, &d_status));
  const size_t stride_f = parsed_stride / sizeof(float);
  constexpr int kParts = 64;
  for (int base = 0; base < n_items; base += kMaxBatch) {
    const int m = std::min(kMaxBatch, n_items - base);
    const float* px = static_cast<const float*>(d_parsed) + (size_t)base * stride_f;
    ncc_moments<<<dim3(kParts, m), 256, 0, s>>>(px, stride_f, d, app->ncc.part);
    SlotList dst;
    dst.n = m;
    for (int k = 0; k < m; ++k) dst.idx[k] = h_slot_idx[base + k];
    ncc_normalise<<<dim3(kParts, m), 256, 0, s>>>(px, stride_f, d, app->ncc.kc, app->ncc.part, kParts,
                                                 static_cast<char*>(d_slots), slot_stride, dst, d_status);
    app->launches += 2;
    RK_CUDA(cudaGetLastError());
  }
  int h_status = 0;
  RK_TRY(status_end(app, s, &h_status));
  if (h_status == RK_ERR_MALFORMED) return set_error(RK_ERR_MALFORMED, "NCC item has zero variance");
  return RK_OK;
}

rk_status ncc_compare(rk_app* app, const void* d_slots, size_t slot_stride, const PairBatch& b, double* d_out,
                      uint8_t* d_flags, cudaStream_t s) {
  const int64_t d = (int64_t)app->p.height * app->p.width;
  ncc_pairs_kernel<<<(b.npairs + 7) / 8, 256, 0, s>>>(b, static_cast<const char*>(d_slots), slot_stride, d,
                                                       app->ncc.kc, d_out,
                                                       d_flags, threshold_or_nan(app), app->ledger);
  app->launches += 1;
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

// K-chunked launches of the CTA-pair kernel over one Gram block
rk_status gram_block_launch(rk_app* app, const CUtensorMap& map, const GramBlock& blk, double* d_out,
                            uint8_t* d_flags, cudaStream_t s) {
  const int64_t d = (int64_t)app->p.height * app->p.width;
  const int tiles = blk.tri ? blk.na * (blk.na + 1) / 2 : blk.na * blk.nb;
  const int mine = (tiles - blk.rank + blk.world - 1) / blk.world;
  if (mine <= 0) return RK_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * mine);
  cfg.blockDim = dim3(kGramThreads);
  cfg.dynamicSmemBytes = gram_smem();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int kblocks = (int)(d / kBK);
  for (int kb0 = 0; kb0 < kblocks; kb0 += kChunkBlocks) {
    const int kb1 = std::min(kblocks, kb0 + kChunkBlocks);
    RK_CUDA(cudaLaunchKernelEx(&cfg, ncc_gram2_kernel, map, app->p.n, d, app->ncc.kc, kb0, kb1, blk, d_out, d_flags,
                               threshold_or_nan(app), app->ledger));
    app->launches += 1;
  }
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

// the interleaved slot arena as a 4-D tensor map: (e % kc, slot % 128, e / kc, slot / 128)
rk_status gram_tensor_map(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, CUtensorMap* map) {
  const int64_t d = (int64_t)app->p.height * app->p.width;
  if (slot_stride % 16 != 0) return set_error(RK_ERR_VALUE, "slot stride must be a multiple of 16 bytes");
  if (n_rows % kGroup != 0)
    return set_error(RK_ERR_VALUE, "Gram arena must hold whole slot groups of %d (got %d slots)", kGroup, n_rows);
  EncodeTiledFn encode = nullptr;
  RK_TRY(tensor_map_encoder(&encode));
  const int64_t kc = app->ncc.kc;
  const cuuint64_t dims[4] = {(cuuint64_t)kc, (cuuint64_t)kGroup, (cuuint64_t)(d / kc), (cuuint64_t)(n_rows / kGroup)};
  const cuuint64_t strides[3] = {(cuuint64_t)kc * 4, (cuuint64_t)kGroup * kc * 4, (cuuint64_t)kGroup * slot_stride};
  const cuuint32_t box[4] = {(cuuint32_t)kBK, (cuuint32_t)kTile, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult cr = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(d_slots), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return set_error(RK_ERR_DEVICE, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
  return RK_OK;
}

rk_status ncc_gram_block(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t a_row0,
                         int32_t a_key0, int32_t a_cnt, int32_t b_row0, int32_t b_key0, int32_t b_cnt, double* d_out,
                         uint8_t* d_flags, cudaStream_t s) {
  if (a_row0 % kGroup || b_row0 % kGroup)
    return set_error(RK_ERR_VALUE, "Gram block rows must start on a slot group (%d)", kGroup);
  if (a_cnt <= 0 || b_cnt <= 0 || a_row0 + a_cnt > n_rows || b_row0 + b_cnt > n_rows)
    return set_error(RK_ERR_VALUE, "Gram block outside the arena");
  if (a_key0 < 0 || b_key0 < 0 || a_key0 + a_cnt > app->p.n || b_key0 + b_cnt > app->p.n)
    return set_error(RK_ERR_VALUE, "Gram block keys outside [0, n)");
  const bool tri = a_row0 == b_row0 && a_key0 == b_key0 && a_cnt == b_cnt;
  if (!tri && a_key0 + a_cnt > b_key0 && b_key0 + b_cnt > a_key0)
    return set_error(RK_ERR_VALUE, "distinct Gram blocks must not overlap in keys");
  if (!tri && a_key0 > b_key0)   // keep i < j: A is the lower key range
    return ncc_gram_block(app, d_slots, slot_stride, n_rows, b_row0, b_key0, b_cnt, a_row0, a_key0, a_cnt, d_out,
                          d_flags, s);
  CUtensorMap map;
  RK_TRY(gram_tensor_map(app, d_slots, slot_stride, n_rows, &map));
  GramBlock blk{a_row0, a_key0, a_cnt, b_row0, b_key0, b_cnt, tri ? 1 : 0, 0, 1,
                (a_cnt + kTile2 - 1) / kTile2, (b_cnt + kTile2 - 1) / kTile2, 1, 1};
  return gram_block_launch(app, map, blk, d_out, d_flags, s);
}

// Strided-key block (the engine's peer-tier NCC path): A = rows a_row0.. holding
// keys a_key0 + r*kstep, B likewise; tri = A is B.  The caller guarantees
// disjoint key sets for distinct blocks.
rk_status ncc_gram_block_strided(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t a_row0,
                                 int32_t a_key0, int32_t a_cnt, int32_t b_row0, int32_t b_key0, int32_t b_cnt,
                                 int32_t kstep, bool tri, double* d_out, uint8_t* d_flags, cudaStream_t s) {
  if (a_row0 % kGroup || b_row0 % kGroup)
    return set_error(RK_ERR_VALUE, "Gram block rows must start on a slot group (%d)", kGroup);
  if (a_cnt <= 0 || b_cnt <= 0 || a_row0 + a_cnt > n_rows || b_row0 + b_cnt > n_rows || kstep < 1)
    return set_error(RK_ERR_VALUE, "Gram block outside the arena");
  if (a_key0 + (int64_t)(a_cnt - 1) * kstep >= app->p.n || b_key0 + (int64_t)(b_cnt - 1) * kstep >= app->p.n)
    return set_error(RK_ERR_VALUE, "Gram block keys outside [0, n)");
  CUtensorMap map;
  RK_TRY(gram_tensor_map(app, d_slots, slot_stride, n_rows, &map));
  GramBlock blk{a_row0, a_key0, a_cnt, b_row0, b_key0, b_cnt, tri ? 1 : 0, 0, 1,
                (a_cnt + kTile2 - 1) / kTile2, (b_cnt + kTile2 - 1) / kTile2, kstep, kstep};
  return gram_block_launch(app, map, blk, d_out, d_flags, s);
}

rk_status ncc_gram(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t rank, int32_t world,
                   double* d_out, uint8_t* d_flags, cudaStream_t s) {
  const int64_t d = (int64_t)app->p.height * app->p.width;
  const int n = app->p.n;
  if (n_rows < n) return set_error(RK_ERR_VALUE, "Gram path needs every item resident: %d slots < n = %d", n_rows, n);
  if (slot_stride % 16 != 0) return set_error(RK_ERR_VALUE, "slot stride must be a multiple of 16 bytes");
  if (world < 1 || rank < 0 || rank >= world) return set_error(RK_ERR_VALUE, "bad rank/world");
  EncodeTiledFn encode = nullptr;
  RK_TRY(tensor_map_encoder(&encode));
  if (n_rows % kGroup != 0)
    return set_error(RK_ERR_VALUE, "Gram arena must hold whole slot groups of %d (got %d slots)", kGroup, n_rows);
  // the interleaved slot layout as a 4-D tensor: (e % kc, slot % 128, e / kc, slot / 128)
  const int64_t kc = app->ncc.kc;
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)kc, (cuuint64_t)kGroup, (cuuint64_t)(d / kc), (cuuint64_t)(n_rows / kGroup)};
  const cuuint64_t strides[3] = {(cuuint64_t)kc * 4, (cuuint64_t)kGroup * kc * 4, (cuuint64_t)kGroup * slot_stride};
  const cuuint32_t box[4] = {(cuuint32_t)kBK, (cuuint32_t)kTile, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(d_slots), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return set_error(RK_ERR_DEVICE, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
#ifndef NCC_GRAM_1CTA
  if (ncc_gram_tile(n) == kTile2) {
    const int side = (n + kTile2 - 1) / kTile2;
    GramBlock blk{0, 0, n, 0, 0, n, 1, rank, world, side, side, 1, 1};
    return gram_block_launch(app, map, blk, d_out, d_flags, s);
  }
#endif
  const int side = (n + kTile - 1) / kTile;
  const int tiles = side * (side + 1) / 2;
  const int mine = (tiles - rank + world - 1) / world;
  if (mine <= 0) return RK_OK;
  ncc_gram_kernel<<<mine, kGramThreads, gram_smem(), s>>>(map, n, d, kc, side, rank, world, d_out, d_flags,
                                                          threshold_or_nan(app), app->ledger);
  app->launches += 1;
  RK_CUDA(cudaGetLastError());
  return RK_OK;
}

}  // namespace rk
