// Internal state shared by the librocket translation units (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/rocket.h"

namespace rk {

// Thread-local last-error message; set_error returns the status for chaining.
rk_status set_error(rk_status st, const char* fmt, ...);
rk_status check_cuda(cudaError_t err, const char* what);
#define RK_CUDA(call)                                  \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return rk::check_cuda(_e, #call); \
  } while (0)
#define RK_TRY(call)                                   \
  do {                                                 \
    rk_status _s = (call);                             \
    if (_s != RK_OK) return _s;                        \
  } while (0)

__host__ __device__ inline int64_t pair_id(int64_t n, int64_t i, int64_t j) {
  return i * (2 * n - i - 1) / 2 + (j - i - 1);
}

// Pairs per kernel launch are passed by value in the launch parameters, so a
// batch needs no host->device copy and is capture-safe for CUDA graphs.
constexpr int kMaxBatch = 64;
struct PairBatch {
  int32_t npairs;
  int32_t slot_a[kMaxBatch];
  int32_t slot_b[kMaxBatch];
  int32_t key_i[kMaxBatch];
  int32_t key_j[kMaxBatch];
  int64_t pid[kMaxBatch];
};

// Exactly-once ledger (PairLedger, scheduler.py:218-246) on the device: one bit
// per pair id, set with a system-scope atomicOr in every compare epilogue (the
// bitmap may live on another GPU of the box: the shared ledger of a multi-GPU
// job sits on rank 0 and is marked over NVLink).  A bit that was already set is
// a duplicate completion -- the reference's AssertionError: ctr[0] counts them,
// ctr[1] holds the first duplicate pair id + 1.  bits == nullptr: no ledger.
struct LedgerRef {
  uint32_t* bits;
  unsigned long long* ctr;   // [0] duplicate marks, [1] first duplicate pid + 1, [2] scratch (popcount)
};
#ifdef __CUDACC__
__device__ __forceinline__ void ledger_mark(const LedgerRef& L, int64_t pid) {
  if (L.bits == nullptr) return;
  const uint32_t bit = 1u << (uint32_t)(pid & 31);
  const uint32_t old = atomicOr_system(L.bits + (pid >> 5), bit);
  if (old & bit) {
    atomicAdd_system(L.ctr, 1ull);
    atomicCAS_system(L.ctr + 1, 0ull, (unsigned long long)pid + 1ull);
  }
}
// Marks of a thread's pair ids in ascending order (a tile row's columns), one
// atomicOr per 32-bit word of the bitmap touched: add() each id, flush() at the end.
struct LedgerRun {
  int64_t word;
  uint32_t mask;
};
__device__ __forceinline__ void ledger_run_flush(const LedgerRef& L, LedgerRun& r) {
  if (L.bits != nullptr && r.mask != 0u) {
    const uint32_t dup = atomicOr_system(L.bits + r.word, r.mask) & r.mask;
    if (dup) {
      atomicAdd_system(L.ctr, (unsigned long long)__popc(dup));
      atomicCAS_system(L.ctr + 1, 0ull, (unsigned long long)(r.word * 32 + __ffs(dup) - 1) + 1ull);
    }
  }
  r.mask = 0u;
}
__device__ __forceinline__ void ledger_run_add(const LedgerRef& L, LedgerRun& r, int64_t pid) {
  if ((pid >> 5) != r.word) {
    ledger_run_flush(L, r);
    r.word = pid >> 5;
  }
  r.mask |= 1u << (uint32_t)(pid & 31);
}
// `cnt` consecutive pair ids from pid0 (a tile row's run of columns): one
// atomicOr per 32-bit word instead of one per pair.
__device__ __forceinline__ void ledger_mark_run(const LedgerRef& L, int64_t pid0, int cnt) {
  if (L.bits == nullptr) return;
  int64_t p = pid0;
  while (cnt > 0) {
    const int off = (int)(p & 31);
    const int take = cnt < 32 - off ? cnt : 32 - off;
    const uint32_t mask = (take == 32 ? 0xffffffffu : ((1u << take) - 1u)) << off;
    const uint32_t dup = atomicOr_system(L.bits + (p >> 5), mask) & mask;
    if (dup) {
      atomicAdd_system(L.ctr, (unsigned long long)__popc(dup));
      atomicCAS_system(L.ctr + 1, 0ull, (unsigned long long)((p & ~(int64_t)31) + __ffs(dup) - 1) + 1ull);
    }
    p += take;
    cnt -= take;
  }
}
#endif

struct SlotList {
  int32_t n;
  int32_t idx[kMaxBatch];
};

// Pair lists of up to 1,024 pairs (PCE, GMM, CV launches), also passed by value
// (16 KiB of kernel parameters): slot indices and the packed-triangle pair id.
constexpr int kPipeMaxPairs = 1924;   // 13 x 148: whole rounds of the persistent PCE grid
constexpr int kListPairs = 1024;      // GMM / CV launches (their scans assume <= 1024 pairs)
int pce_batch_limit(const rk_app* app);
struct DevPair {
  int32_t slot_a;
  int32_t slot_b;
  int64_t pid;
};
struct PairJob {
  int32_t npairs;
  int32_t depth;   // unused (kept for layout stability)
  DevPair pairs[kPipeMaxPairs];
};
struct PceState {
  int R = 0;               // group width; N = R*R (R = 32 and N = 2048: two warp FFTs per line)
  int N = 0;               // pattern side
  int batch = 0;           // items per preprocess launch
  float2* tw = nullptr;    // [k1][n1] W_N^(n1*k1), R*R entries
  float2* U = nullptr;     // batch * (N/2) * N: preprocess row-pass output
  float* mean_part = nullptr;    // batch * 64 partial sums
  int clusters = 0;        // co-resident compare clusters (= pairs in flight)
  float2* T = nullptr;     // clusters * t_stride: column-pass output, one slot per cluster
  size_t t_stride = 0;     // float2 between T slots: (N/2)*N + padding (breaks the power-of-two stride)
  PairJob* job = nullptr;   // host staging of the launch parameters
  unsigned* rounds = nullptr;   // round-barrier counter of the compare grid (RK_PCE_LOCKSTEP), else null
  int l2opts = 0;           // RK_PCE_L2OPTS: bit 0 T stores evict_first, bit 1 spectra evict_last
};

struct CvState {};
struct NccState {
  double* part = nullptr;   // per-CTA (sum, sum of squares) partials of the preprocess
  int64_t kc = 0;           // interleave run (floats): 1024 when D % 1024 == 0, else D (contiguous slots)
};
struct GmmState {};

}  // namespace rk

struct rk_app {
  rk_app_params p{};
  int device = 0;
  size_t slot_bytes = 0;
  size_t parsed_bytes = 0;
  int64_t launches = 0;    // kernels launched through this app (for bench accounting)
  int32_t slot_group = 1;  // slots interleaved in groups of this many (rk_app_slot_group)
  rk::PairJob* job = nullptr;   // host staging of by-value pair lists (GMM, CV launches)
  double* gmm_scratch = nullptr;   // per (pair, angle block) best of one GMM launch
  int* d_status = nullptr;          // preprocess status word (device) and its pinned host mirror
  int* h_status = nullptr;
  void* cv_scratch = nullptr;       // CV unit offsets, work counter and unit partials
  void* cv_prep = nullptr;          // CV preprocess totals and norm partials
  int cv_grid = 0;                  // persistent CV work grid (SMs x resident CTAs)
  rk::PceState pce;
  rk::NccState ncc;
  rk::LedgerRef ledger{nullptr, nullptr};   // marked by every compare epilogue (null: off)
};

namespace rk {
// Per-kind implementations (each in its own .cu).
rk_status pce_init(rk_app* app);
void pce_free(rk_app* app);
rk_status pce_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items,
                         void* d_slots, size_t slot_stride, const int32_t* h_slot_idx,
                         cudaStream_t s);

// 2048^2 variant (pce2k.cu) and the shared mean-reduction launch (pce.cu)
rk_status pce2k_init(rk_app* app);
// Compare-grid round barrier + L2 options of the PCE kernels (env RK_PCE_LOCKSTEP,
// RK_PCE_L2OPTS), set up at app creation (pce.cu).
rk_status pce_round_init(PceState& st, int l2opts_default);
rk_status pce2k_preprocess(rk_app* app, const float* pix, size_t stride_f, int n_items, char* slots,
                           size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s);
rk_status pce2k_compare(rk_app* app, const char* slots, size_t slot_stride, const rk_pair* pairs, int n,
                        double* d_out, uint8_t* d_flags, cudaStream_t s);
void pce_launch_mean(const float* pix, size_t stride_f, int nn, int n_items, float* mean_part, cudaStream_t s);

// NCC Gram tile side for n items (256: CTA-pair kernel, 128: single-CTA kernel)
int ncc_gram_tile(int n);
rk_status ncc_gram_block(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t a_row0,
                         int32_t a_key0, int32_t a_cnt, int32_t b_row0, int32_t b_key0, int32_t b_cnt, double* d_out,
                         uint8_t* d_flags, cudaStream_t s);

rk_status ncc_gram_block_strided(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t a_row0,
                                 int32_t a_key0, int32_t a_cnt, int32_t b_row0, int32_t b_key0, int32_t b_cnt,
                                 int32_t kstep, bool tri, double* d_out, uint8_t* d_flags, cudaStream_t s);

rk_status pce_compare_list(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* pairs, int n,
                           double* d_out, uint8_t* d_flags, cudaStream_t s);

rk_status synth_compare(rk_app* app, const PairBatch& b, double* d_out, uint8_t* d_flags,
                        cudaStream_t s);

rk_status gmm_init(rk_app* app);
rk_status gmm_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                         size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s);
rk_status gmm_compare_list(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* pairs, int n,
                          double* d_out, uint8_t* d_flags, cudaStream_t s);
rk_status ncc_init(rk_app* app);
void ncc_free(rk_app* app);
rk_status ncc_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                         size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s);
rk_status ncc_compare(rk_app* app, const void* d_slots, size_t slot_stride, const PairBatch& b, double* d_out,
                      uint8_t* d_flags, cudaStream_t s);
rk_status ncc_gram(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t rank, int32_t world,
                   double* d_out, uint8_t* d_flags, cudaStream_t s);

double threshold_or_nan(const rk_app* app);
// Preprocess status word: reset on `s` (allocated once per app; no per-call
// cudaMallocAsync, whose pool trimming stalled the load stream for ~0.5 s), then
// read back after the kernels (synchronous on `s`).
rk_status status_begin(rk_app* app, cudaStream_t s, int** d_status);
rk_status status_end(rk_app* app, cudaStream_t s, int* h_status);
// Padding (bytes) added to power-of-two per-item / per-CTA strides (env RK_SLOT_PAD / RK_T_PAD)
size_t stride_pad(const char* env, size_t dflt);

// cuTensorMapEncodeTiled, fetched from the driver through the runtime (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
rk_status tensor_map_encoder(EncodeTiledFn* fn);

// Quadtree leaf [r0, r1) x [c0, c1) (Region, scheduler.py:20-71).
struct Leaf {
  int32_t r0, r1, c0, c1;
};
int64_t region_pairs(int64_t r0, int64_t r1, int64_t c0, int64_t c1);
std::vector<Leaf> quadtree_leaves(int32_t n, int leaf_block);
std::vector<Leaf> rank_share(const std::vector<Leaf>& leaves, int rank, int world);

// Device-tier slot table: the CacheTier policy (slotcache.py:139-282) for a
// single-threaded, stream-ordered driver.  Slot payloads live in the HBM arena.
enum SlotState : uint8_t { kEmpty = 0, kWrite = 1, kRead = 2 };
enum TierKind { kHit = 0, kMustWait = 1, kMiss = 2, kNoEvictable = 3 };
struct TierResult {
  int kind;
  int slot;
};
struct SlotTier {
  explicit SlotTier(int cap);
  TierResult acquire(int32_t key);
  void publish(int slot, bool retain);
  void abort(int slot);
  void release(int slot);
  int find(int32_t key) const;
  int capacity;
  std::vector<int32_t> key;
  std::vector<uint8_t> state;
  std::vector<int32_t> readers;
  std::vector<uint64_t> stamp;
  std::vector<int> free_list;
  std::unordered_map<int32_t, int> index;
  uint64_t clock = 0;
  int64_t hits = 0, misses = 0, waits = 0, evictions = 0;
  int last_evicted = -1;
};
}  // namespace rk
