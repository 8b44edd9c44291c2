// CompositionVectorApp on sm_100a: preprocess (count -> frequency) and the
// sparse k-mer cosine as a warp-per-pair merge-path kernel.
//
// Restates /root/reference/pkg/src/allpairs/apps.py:
//   preprocess  :304-318  freq = count / total   (bit-exact: both ints < 2^53)
//   compare     :331-354  sorted merge dot / (norm_a * norm_b), 0 if a norm is 0
//   postprocess :356-358  match = value >= threshold
// Norms are computed once at preprocess instead of per compare (SURVEY.md
// appendix: changes only the fp64 summation order, inside the 1e-9 tests).
//
// Parsed item (reference byte format, apps.py:299-302): <I dim> + dim x <Q token><I count>.
// Slot layout (device):  u32 dim | u32 pad | f64 norm | u64 token[cap] | f64 freq[cap]
#include <math.h>

#include <algorithm>

#include "internal.h"

namespace rk {

namespace {

// Preprocess, three kernels per batch of items (grid = kPrepParts chunks x items,
// so a load group keeps the whole GPU busy):
//   cvp_sum    integer sum of the counts (exact, order-free atomics)
//   cvp_write  tokens and freq = count / total into the slot, per-chunk sum of freq^2
//   cvp_final  fixed-order sum of the chunks -> norm, slot header, status
// The parsed records (<Q token><I count>, 12 B) are 4-byte aligned: three u32 loads.
constexpr int kPrepParts = 32;

__device__ __forceinline__ bool cv_item_ok(uint32_t dim, int cap) { return dim != 0 && (int64_t)dim <= cap; }

__global__ void __launch_bounds__(256) cvp_sum(const uint8_t* __restrict__ parsed, size_t parsed_stride, int cap,
                                               unsigned long long* __restrict__ totals) {
  const int item = blockIdx.y;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(parsed + (size_t)item * parsed_stride);
  const uint32_t dim = src[0];
  if (!cv_item_ok(dim, cap)) return;
  unsigned long long t = 0;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < dim; k += gridDim.x * blockDim.x)
    t += __ldg(src + 1 + 3 * (size_t)k + 2);
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0 && t) atomicAdd(&totals[item], t);
}

__global__ void __launch_bounds__(256) cvp_write(const uint8_t* __restrict__ parsed, size_t parsed_stride,
                                                 SlotList dst, uint8_t* __restrict__ slots, size_t slot_stride, int cap,
                                                 const unsigned long long* __restrict__ totals,
                                                 double* __restrict__ part) {
  const int item = blockIdx.y;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(parsed + (size_t)item * parsed_stride);
  const uint32_t dim = src[0];
  if (!cv_item_ok(dim, cap)) return;
  const double total = (double)totals[item];
  uint8_t* slot = slots + (size_t)dst.idx[item] * slot_stride;
  uint64_t* tok = reinterpret_cast<uint64_t*>(slot + 16);
  double* freq = reinterpret_cast<double*>(slot + 16 + 8 * (size_t)cap);
  double sq = 0.0;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < dim; k += gridDim.x * blockDim.x) {
    const uint32_t* e = src + 1 + 3 * (size_t)k;
    const double f = (double)__ldg(e + 2) / total;
    tok[k] = (uint64_t)__ldg(e) | ((uint64_t)__ldg(e + 1) << 32);
    freq[k] = f;
    sq = fma(f, f, sq);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  __shared__ double s_sq[8];
  if ((threadIdx.x & 31) == 0) s_sq[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_sq[w];
    part[(size_t)item * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void cvp_final(const uint8_t* __restrict__ parsed, size_t parsed_stride, int n_items, SlotList dst,
                          uint8_t* __restrict__ slots, size_t slot_stride, int cap, const double* __restrict__ part,
                          int* __restrict__ status) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= n_items) return;
  const uint32_t dim = *reinterpret_cast<const uint32_t*>(parsed + (size_t)item * parsed_stride);
  if (!cv_item_ok(dim, cap)) {
    atomicMax(status, dim == 0 ? (int)RK_ERR_MALFORMED : (int)RK_ERR_SLOT_OVERFLOW);
    return;
  }
  double sq = 0.0;
  for (int c = 0; c < kPrepParts; ++c) sq += part[(size_t)item * kPrepParts + c];
  uint8_t* slot = slots + (size_t)dst.idx[item] * slot_stride;
  *reinterpret_cast<uint32_t*>(slot) = dim;
  *reinterpret_cast<uint32_t*>(slot + 4) = 0u;
  *reinterpret_cast<double*>(slot + 8) = sqrt(sq);
}

// Merge-path split: number of A elements among the first `diag` merged
// elements, where ties go to A first (A[i] <= B[j] takes A).
__device__ __forceinline__ int merge_path(const uint64_t* a, int na, const uint64_t* b, int nb, int diag) {
  int lo = max(0, diag - nb), hi = min(diag, na);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    // take mid A elements and diag-mid B elements: valid if A[mid] > B[diag-mid-1]
    if (a[mid] <= b[diag - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Work is split into units of ~kUnit merged tokens: pair p gets Q_p =
// ceil((na + nb) / kUnit) units (diagonals of its merge path), so the skewed
// sizes of C5 (1e5 .. 1.8e6 tokens) cost proportionally and the launch has no
// per-pair tail.  cv_units sizes and scans them, persistent warps of cv_work
// grab units from an atomic counter, cv_finalize sums each pair's unit partials
// in unit order (deterministic) and writes the cosine.
//
// Inside a unit the warp walks both lists in coalesced 32-token windows: every
// lane binary-searches its A token in the B window (register shuffles), matches
// add fa*fb (fp64, in order), and the window whose last token is smaller is
// consumed whole while the other advances by the ballot count of tokens below
// it; the next windows are loaded one step ahead.  A match is always counted
// from the A side, so a B token just past the unit (equal to the unit's last A
// token, ties go to A) is still found: the B window may read beyond the unit.
constexpr int kCvWarps = 8;
constexpr int kUnit = 32768;
constexpr int kMaxUnits = 64;      // per pair (larger pairs get larger units)

struct CvPairRef {
  const uint64_t* ta;
  const uint64_t* tb;
  const double* fa;
  const double* fb;
  int na, nb;
};

__device__ __forceinline__ CvPairRef cv_pair_ref(const DevPair& pr, const uint8_t* slots, size_t slot_stride, int cap) {
  const uint8_t* sa = slots + (size_t)pr.slot_a * slot_stride;
  const uint8_t* sb = slots + (size_t)pr.slot_b * slot_stride;
  CvPairRef r;
  r.na = (int)*reinterpret_cast<const uint32_t*>(sa);
  r.nb = (int)*reinterpret_cast<const uint32_t*>(sb);
  r.ta = reinterpret_cast<const uint64_t*>(sa + 16);
  r.tb = reinterpret_cast<const uint64_t*>(sb + 16);
  r.fa = reinterpret_cast<const double*>(sa + 16 + 8 * (size_t)cap);
  r.fb = reinterpret_cast<const double*>(sb + 16 + 8 * (size_t)cap);
  return r;
}

__device__ __forceinline__ int cv_units_of(int na, int nb) {
  const int64_t t = (int64_t)na + nb;
  const int64_t q = (t + kUnit - 1) / kUnit;
  return q < 1 ? 1 : (q > kMaxUnits ? kMaxUnits : (int)q);
}

// one CTA of 1024 threads: unit offsets (exclusive scan), total, counter reset
__global__ void __launch_bounds__(1024) cv_units(const PairJob job, const uint8_t* __restrict__ slots,
                                                 size_t slot_stride, int* __restrict__ offsets,
                                                 int* __restrict__ ctl) {
  __shared__ int s_scan[1024];
  const int p = threadIdx.x;
  int q = 0;
  if (p < job.npairs) {
    const uint8_t* sa = slots + (size_t)job.pairs[p].slot_a * slot_stride;
    const uint8_t* sb = slots + (size_t)job.pairs[p].slot_b * slot_stride;
    q = cv_units_of((int)*reinterpret_cast<const uint32_t*>(sa), (int)*reinterpret_cast<const uint32_t*>(sb));
  }
  s_scan[p] = q;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {   // Hillis-Steele inclusive scan
    const int v = p >= o ? s_scan[p - o] : 0;
    __syncthreads();
    s_scan[p] += v;
    __syncthreads();
  }
  offsets[p + 1] = s_scan[p];
  if (p == 0) {
    offsets[0] = 0;
    ctl[0] = 0;                 // work counter
    ctl[1] = s_scan[1023];      // total units
  }
}

__global__ void __launch_bounds__(kCvWarps * 32) cv_work(const PairJob job, const uint8_t* __restrict__ slots,
                                                         size_t slot_stride, int cap, const int* __restrict__ offsets,
                                                         int* __restrict__ ctl, double* __restrict__ partial) {
  __shared__ int s_off[1025];
  for (int k = threadIdx.x; k <= job.npairs; k += blockDim.x) s_off[k] = offsets[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int total_units = ctl[1];
  for (;;) {
    int u = 0;
    if (lane == 0) u = atomicAdd(&ctl[0], 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= total_units) break;
    int lo = 0, hi = job.npairs;            // pair p: s_off[p] <= u < s_off[p + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= u) lo = mid;
      else hi = mid;
    }
    const int p = lo, q = u - s_off[p], nq = s_off[p + 1] - s_off[p];
    const CvPairRef r = cv_pair_ref(job.pairs[p], slots, slot_stride, cap);
    const uint64_t* ta = r.ta;
    const uint64_t* tb = r.tb;
    const double* fa = r.fa;
    const double* fb = r.fb;
    const int na = r.na, nb = r.nb;
    const int64_t tot = (int64_t)na + nb;
    const int d0 = (int)(tot * q / nq), d1 = (int)(tot * (q + 1) / nq);
    int i = merge_path(ta, na, tb, nb, d0);
    int j = d0 - i;
    const int i_end = merge_path(ta, na, tb, nb, d1);
  constexpr uint64_t kInf = ~0ull;   // sentinel: k-mer ids of UTF-8 text never reach 2^64 - 1
    auto lda = [&](int idx) { return idx < i_end ? __ldg(ta + idx) : kInf; };
    auto ldb = [&](int idx) { return idx < nb ? __ldg(tb + idx) : kInf; };
    // current windows (a, b) and the next ones (an, bn), loaded one iteration ahead
    uint64_t a = lda(i + lane), an = lda(i + 32 + lane);
    uint64_t b = ldb(j + lane), bn = ldb(j + 32 + lane);
    double dot = 0.0;
    while (i < i_end && j < nb) {
      const int na_w = min(32, i_end - i);
      const int nb_w = min(32, nb - j);
      const uint64_t amax = __shfl_sync(0xffffffffu, a, na_w - 1);
      const uint64_t bmax = __shfl_sync(0xffffffffu, b, nb_w - 1);
      // lower_bound of a in the B window (lanes >= nb_w hold +inf)
      int pos = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint64_t probe = __shfl_sync(0xffffffffu, b, pos + step - 1);
        if (probe < a) pos += step;
      }
      const uint64_t at = __shfl_sync(0xffffffffu, b, pos & 31);
      if (a != kInf && pos < nb_w && at == a) dot = fma(__ldg(fa + i + lane), __ldg(fb + j + pos), dot);
      int adv_a, adv_b;
      if (amax < bmax) {          // A window done; B tokens <= amax done too
        adv_a = na_w;
        adv_b = __popc(__ballot_sync(0xffffffffu, b <= amax));
      } else if (bmax < amax) {   // B window done; A tokens <= bmax were checked against it
        adv_b = nb_w;
        adv_a = __popc(__ballot_sync(0xffffffffu, a <= bmax));
      } else {
        adv_a = na_w;
        adv_b = nb_w;
      }
      if (adv_a) {   // slide the A window from (a, an), prefetch the next one
        const int src = lane + adv_a;
        const uint64_t x0 = __shfl_sync(0xffffffffu, a, src & 31), x1 = __shfl_sync(0xffffffffu, an, src & 31);
        a = src < 32 ? x0 : x1;
        i += adv_a;
        an = lda(i + 32 + lane);
      }
      if (adv_b) {
        const int src = lane + adv_b;
        const uint64_t x0 = __shfl_sync(0xffffffffu, b, src & 31), x1 = __shfl_sync(0xffffffffu, bn, src & 31);
        b = src < 32 ? x0 : x1;
        j += adv_b;
        bn = ldb(j + 32 + lane);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) partial[u] = dot;
  }
}

__global__ void cv_finalize(const PairJob job, const uint8_t* __restrict__ slots, size_t slot_stride,
                            const int* __restrict__ offsets, const double* __restrict__ partial,
                            double* __restrict__ out, uint8_t* __restrict__ flags, double threshold,
                            const LedgerRef ledger) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= job.npairs) return;
  double t = 0.0;
  for (int u = offsets[p]; u < offsets[p + 1]; ++u) t += partial[u];
  const double norm_a = *reinterpret_cast<const double*>(slots + (size_t)job.pairs[p].slot_a * slot_stride + 8);
  const double norm_b = *reinterpret_cast<const double*>(slots + (size_t)job.pairs[p].slot_b * slot_stride + 8);
  const double v = (norm_a > 0.0 && norm_b > 0.0) ? t / (norm_a * norm_b) : 0.0;
  out[job.pairs[p].pid] = v;
  ledger_mark(ledger, job.pairs[p].pid);
  if (flags) flags[job.pairs[p].pid] = isnan(threshold) ? 0 : (uint8_t)(1 | (v >= threshold ? 2 : 0));
}

}  // namespace

rk_status cv_init(rk_app* app) {
  const int cap = app->p.max_entries;
  if (cap <= 0) return set_error(RK_ERR_VALUE, "CV app needs max_entries > 0");
  app->slot_bytes = 16 + 16 * (size_t)cap;
  app->parsed_bytes = 4 + 12 * (size_t)cap;
  return RK_OK;
}

rk_status cv_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                        size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s) {
  if (parsed_stride % 4 != 0) return set_error(RK_ERR_VALUE, "CV parsed_stride must be a multiple of 4 bytes");
  if (!app->cv_prep) {   // totals [kMaxBatch] u64 | partials [kMaxBatch * kPrepParts] f64
    RK_CUDA(cudaMalloc(&app->cv_prep, sizeof(unsigned long long) * kMaxBatch +
                                          sizeof(double) * kMaxBatch * kPrepParts));
  }
  unsigned long long* totals = static_cast<unsigned long long*>(app->cv_prep);
  double* part = reinterpret_cast<double*>(totals + kMaxBatch);
  int* d_status = nullptr;
  RK_TRY(status_begin(app, s, &d_status));
  const uint8_t* parsed = static_cast<const uint8_t*>(d_parsed);
  uint8_t* slots = static_cast<uint8_t*>(d_slots);
  for (int base = 0; base < n_items; base += kMaxBatch) {
    const int m = n_items - base < kMaxBatch ? n_items - base : kMaxBatch;
    SlotList dst;
    dst.n = m;
    for (int k = 0; k < m; ++k) dst.idx[k] = h_slot_idx[base + k];
    const uint8_t* px = parsed + (size_t)base * parsed_stride;
    RK_CUDA(cudaMemsetAsync(totals, 0, sizeof(unsigned long long) * m, s));
    cvp_sum<<<dim3(kPrepParts, m), 256, 0, s>>>(px, parsed_stride, app->p.max_entries, totals);
    cvp_write<<<dim3(kPrepParts, m), 256, 0, s>>>(px, parsed_stride, dst, slots, slot_stride, app->p.max_entries,
                                                   totals, part);
    cvp_final<<<(m + 63) / 64, 64, 0, s>>>(px, parsed_stride, m, dst, slots, slot_stride, app->p.max_entries, part,
                                           d_status);
    app->launches += 3;
    RK_CUDA(cudaGetLastError());
  }
  int h_status = 0;
  RK_TRY(status_end(app, s, &h_status));
  if (h_status == RK_ERR_SLOT_OVERFLOW)
    return set_error(RK_ERR_SLOT_OVERFLOW, "preprocessed item exceeds slot capacity of %d entries", app->p.max_entries);
  if (h_status == RK_ERR_MALFORMED) return set_error(RK_ERR_MALFORMED, "parsed item has no k-mers");
  return RK_OK;
}

rk_status cv_compare_list(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* pairs, int n,
                         double* d_out, uint8_t* d_flags, cudaStream_t s) {
  if (!app->job) app->job = new PairJob();
  if (!app->cv_scratch) {
    // offsets [1025] | ctl [2] | partials [1024 * kMaxUnits]
    RK_CUDA(cudaMalloc(&app->cv_scratch, sizeof(int) * 1028 + sizeof(double) * kListPairs * kMaxUnits));
    int dev = 0, sms = 0, per_sm = 0;
    RK_CUDA(cudaGetDevice(&dev));
    RK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cv_work, kCvWarps * 32, 0));
    app->cv_grid = sms * std::max(1, per_sm);
  }
  int* offsets = static_cast<int*>(app->cv_scratch);
  int* ctl = offsets + 1025;
  double* partial = reinterpret_cast<double*>(static_cast<char*>(app->cv_scratch) + sizeof(int) * 1028);
  const uint8_t* slots = static_cast<const uint8_t*>(d_slots);
  PairJob& job = *app->job;
  for (int base = 0; base < n; base += kListPairs) {
    const int m = n - base < kListPairs ? n - base : kListPairs;
    job.npairs = m;
    for (int k = 0; k < m; ++k) {
      const rk_pair& q = pairs[base + k];
      job.pairs[k] = DevPair{q.slot_a, q.slot_b, pair_id(app->p.n, q.i, q.j)};
    }
    cv_units<<<1, 1024, 0, s>>>(job, slots, slot_stride, offsets, ctl);
    cv_work<<<app->cv_grid, kCvWarps * 32, 0, s>>>(job, slots, slot_stride, app->p.max_entries, offsets, ctl,
                                                   partial);
    cv_finalize<<<(m + 127) / 128, 128, 0, s>>>(job, slots, slot_stride, offsets, partial, d_out, d_flags,
                                                threshold_or_nan(app), app->ledger);
    app->launches += 3;
    RK_CUDA(cudaGetLastError());
  }
  return RK_OK;
}

}  // namespace rk
