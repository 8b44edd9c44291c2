// All-pairs engine: quadtree leaves (scheduler.py:20-117) over a device slot
// tier (slotcache.py:139-282) fed by the load pipeline (engine.py:436-508).
//
// The driver is one host thread per GPU that enqueues everything on CUDA
// streams, so the tier's WRITE state never blocks: a slot is published as
// soon as its load is enqueued.  Loads (H2D + preprocess, peer fetches) run on
// a load stream and compares on the engine stream; events order them: a
// compare batch waits for the loads issued before it, a load into an evicted
// slot waits for every compare launched before the eviction -- the reference's
// lease rule (engine.py:530-534) in stream order.
//
// Multi-GPU (one engine per rank): the peer-GPU tier (home GPU k mod world,
// CUDA IPC mappings of the other ranks' arenas) and the cross-GPU work queue
// (hierarchical stealing with system-scope atomics on per-rank queue words).
// NCC runs as a tcgen05 Gram instead of per-pair launches: all items resident,
// or key blocks of half the arena when the slots are fewer than the items.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <vector>

#include "internal.h"

namespace rk {

rk_status compare_pairs(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* h_pairs, int n_pairs,
                        double* d_out, uint8_t* d_flags, cudaStream_t s);
int batch_limit(const rk_app* app);

// ---------------------------------------------------------------------------
// Quadtree (Region.split / iter_leaves, scheduler.py:33-86)
int64_t region_pairs(int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
  int64_t full_rows = std::max<int64_t>(0, std::min(r1, c0) - r0);
  int64_t total = full_rows * (c1 - c0);
  const int64_t a = std::max(r0, c0);
  const int64_t b = std::min(r1, c1 - 1);
  if (b > a) total += (c1 - 1 - a + c1 - b) * (b - a) / 2;
  return total;
}

static void leaves_rec(int32_t r0, int32_t r1, int32_t c0, int32_t c1, int leaf, std::vector<Leaf>& out) {
  if (region_pairs(r0, r1, c0, c1) == 0) return;
  if (r1 - r0 <= leaf && c1 - c0 <= leaf) {
    out.push_back(Leaf{r0, r1, c0, c1});
    return;
  }
  const int32_t rm = (r0 + r1) / 2, cm = (c0 + c1) / 2;
  leaves_rec(r0, rm, c0, cm, leaf, out);
  leaves_rec(r0, rm, cm, c1, leaf, out);
  leaves_rec(rm, r1, c0, cm, leaf, out);
  leaves_rec(rm, r1, cm, c1, leaf, out);
}

std::vector<Leaf> quadtree_leaves(int32_t n, int leaf_block) {
  std::vector<Leaf> out;
  if (n >= 2) leaves_rec(0, n, 0, n, leaf_block, out);
  return out;
}

// Contiguous DFS blocks of leaves balanced by pair count (locality per rank).
std::vector<Leaf> rank_share(const std::vector<Leaf>& leaves, int rank, int world) {
  if (world <= 1) return leaves;
  int64_t total = 0;
  for (const Leaf& l : leaves) total += region_pairs(l.r0, l.r1, l.c0, l.c1);
  std::vector<Leaf> mine;
  int64_t prefix = 0;
  for (const Leaf& l : leaves) {
    const int64_t pc = region_pairs(l.r0, l.r1, l.c0, l.c1);
    // owner = rank whose share contains the leaf's midpoint
    const int64_t mid = prefix + pc / 2;
    const int owner = (int)std::min<int64_t>(world - 1, (mid * world) / std::max<int64_t>(total, 1));
    if (owner == rank) mine.push_back(l);
    prefix += pc;
  }
  return mine;
}

// The same share as an index range [lo, hi) of the DFS leaf list (owners are
// non-decreasing along the list, so every share is contiguous).
std::pair<int, int> rank_range(const std::vector<Leaf>& leaves, int rank, int world) {
  if (world <= 1) return {0, (int)leaves.size()};
  int64_t total = 0;
  for (const Leaf& l : leaves) total += region_pairs(l.r0, l.r1, l.c0, l.c1);
  int lo = -1, hi = -1;
  int64_t prefix = 0;
  for (int q = 0; q < (int)leaves.size(); ++q) {
    const Leaf& l = leaves[q];
    const int64_t pc = region_pairs(l.r0, l.r1, l.c0, l.c1);
    const int owner = (int)std::min<int64_t>(world - 1, ((prefix + pc / 2) * world) / std::max<int64_t>(total, 1));
    if (owner == rank) {
      if (lo < 0) lo = q;
      hi = q + 1;
    }
    prefix += pc;
  }
  if (lo < 0) return {0, 0};
  return {lo, hi};
}

// ---------------------------------------------------------------------------
// Cross-GPU work queue (hierarchical stealing, engine.py:274-309 and
// scheduler.py:126-157 restated for one box): every rank owns a 64-bit word
// (head << 32 | tail) over the global DFS leaf list, initialised to its
// rank_range.  The owner takes chunks from the head (depth-first order, the
// reference's pop at the back of its deque); a thief CASes away the back half of
// the victim with the most remaining leaves (the largest task, like stealing at
// the front) and publishes it as its own range, so it can be re-stolen.  The
// words live in device memory and peers update them with system-scope atomics
// over NVLink (CUDA IPC mappings); the host reads the result from mapped memory.
// One queue transition on a word value: op 0 = the owner takes up to `arg` leaves
// from the head, op 1 = a thief takes the back half if at least `arg` leaves
// remain on each side.  False when there is nothing to take.  Shared by the device
// CAS loop and the host test hook rk_queue_step.
__host__ __device__ inline bool queue_step(unsigned long long old, int op, unsigned long long arg,
                                           unsigned long long* nw, unsigned long long* got) {
  const unsigned h = (unsigned)(old >> 32), t = (unsigned)old;
  const unsigned rem = t > h ? t - h : 0u;
  if (op == 0) {
    if (rem == 0) return false;
    const unsigned take = rem < arg ? rem : (unsigned)arg;
    *nw = ((unsigned long long)(h + take) << 32) | t;
    *got = ((unsigned long long)h << 32) | (h + take);
    return true;
  }
  if (rem < 2 * arg) return false;
  const unsigned k = rem / 2;
  *nw = ((unsigned long long)h << 32) | (t - k);
  *got = ((unsigned long long)(t - k) << 32) | t;
  return true;
}

__global__ void queue_op_kernel(unsigned long long* word, int op, unsigned long long arg,
                                unsigned long long* res) {
  unsigned long long old = atomicAdd_system(word, 0ull);
  if (op == 2) {            // read
    *res = old;
    return;
  }
  if (op == 3) {            // set (own word, when it is empty or at reset)
    atomicExch_system(word, arg);
    *res = arg;
    return;
  }
  for (;;) {
    unsigned long long nw, got;
    if (!queue_step(old, op, arg, &nw, &got)) {
      *res = ~0ull;
      return;
    }
    const unsigned long long prev = atomicCAS_system(word, old, nw);
    if (prev == old) {
      *res = got;
      return;
    }
    old = prev;
  }
}

// ---------------------------------------------------------------------------
// Exactly-once ledger region: C(n,2) bits (rounded up to 256 B), then 256 B of
// counters (LedgerRef.ctr).  Lives in the engine's arena allocation so that the
// same IPC handle that maps the home region maps it for the other ranks.
size_t ledger_bits_bytes(int64_t n) {
  const int64_t total = n > 1 ? n * (n - 1) / 2 : 0;
  return (size_t)((total + 31) / 32 * 4 + 255) / 256 * 256;
}
size_t ledger_region_bytes(int64_t n) { return ledger_bits_bytes(n) + 256; }
LedgerRef ledger_at(void* region, int64_t n) {
  char* r = static_cast<char*>(region);
  return LedgerRef{reinterpret_cast<uint32_t*>(r), reinterpret_cast<unsigned long long*>(r + ledger_bits_bytes(n))};
}

__global__ void ledger_count_kernel(const uint32_t* __restrict__ bits, int64_t words, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
    c += (unsigned long long)__popc(bits[w]);
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd_system(out, c);
}

// completed = popcount of the bitmap, plus the duplicate counters (synchronous on s)
rk_status ledger_read(void* region, int64_t n, cudaStream_t s, rk_ledger_stats* out) {
  const int64_t total = n > 1 ? n * (n - 1) / 2 : 0;
  const LedgerRef L = ledger_at(region, n);
  RK_CUDA(cudaMemsetAsync(L.ctr + 2, 0, sizeof(unsigned long long), s));
  const int64_t words = (total + 31) / 32;
  if (words > 0) {
    const int blocks = (int)std::min<int64_t>(1184, (words + 255) / 256);
    ledger_count_kernel<<<blocks, 256, 0, s>>>(L.bits, words, L.ctr + 2);
    RK_CUDA(cudaGetLastError());
  }
  unsigned long long h[3] = {0, 0, 0};
  RK_CUDA(cudaMemcpyAsync(h, L.ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
  RK_CUDA(cudaStreamSynchronize(s));
  out->total = total;
  out->completed = (int64_t)h[2];
  out->dup_marks = (int64_t)h[0];
  out->first_dup_pid = h[1] ? (int64_t)h[1] - 1 : -1;
  out->full = out->completed == total && out->dup_marks == 0;
  out->shared = 0;
  return RK_OK;
}

// Peer-tier block copies over NVLink: the copy engine (cudaMemcpyAsync) or an
// SM-driven copy (RK_PEER_COPY_CTAS > 0 CTAs of 512 threads, four 16-byte peer
// loads in flight per thread through the IPC mapping, local stores).
__global__ void __launch_bounds__(512) peer_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                        size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

int peer_copy_ctas() {
  const char* v = getenv("RK_PEER_COPY_CTAS");
  return v && *v ? atoi(v) : 0;
}

rk_status peer_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  const int ctas = peer_copy_ctas();
  if (ctas > 0 && bytes % 16 == 0 && ((uintptr_t)dst | (uintptr_t)src) % 16 == 0) {
    peer_copy_kernel<<<ctas, 512, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), bytes / 16);
    RK_CUDA(cudaGetLastError());
    return RK_OK;
  }
  RK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
  return RK_OK;
}

rk_status duplicate_error(int64_t n, const rk_ledger_stats& ls) {
  int64_t i = 0, j = 0, pid = ls.first_dup_pid;
  while (pid >= n - 1 - i) {
    pid -= n - 1 - i;
    ++i;
  }
  j = i + 1 + pid;
  return set_error(RK_ERR_DUPLICATE, "pair (%lld, %lld) completed twice (%lld duplicate marks)", (long long)i,
                   (long long)j, (long long)ls.dup_marks);
}

// ---------------------------------------------------------------------------
// Slot tier (CacheTier restated, slotcache.py:139-282)
SlotTier::SlotTier(int cap) : capacity(cap) {
  key.assign(cap, -1);
  state.assign(cap, kEmpty);
  readers.assign(cap, 0);
  stamp.assign(cap, 0);
  for (int s = cap - 1; s >= 0; --s) free_list.push_back(s);  // slot 0 handed out first (slotcache.py:150)
}

int SlotTier::find(int32_t k) const {
  auto it = index.find(k);
  return it == index.end() ? -1 : it->second;
}

TierResult SlotTier::acquire(int32_t k) {
  const int s = find(k);
  if (s >= 0) {
    if (state[s] == kRead) {
      ++hits;
      ++readers[s];
      stamp[s] = ++clock;
      return TierResult{kHit, s};
    }
    ++waits;
    return TierResult{kMustWait, s};
  }
  int slot = -1;
  if (!free_list.empty()) {
    slot = free_list.back();
    free_list.pop_back();
  } else {
    uint64_t best = 0;
    for (int c = 0; c < capacity; ++c) {
      if (state[c] == kRead && readers[c] == 0 && (slot < 0 || stamp[c] < best)) {
        slot = c;
        best = stamp[c];
      }
    }
    if (slot < 0) return TierResult{kNoEvictable, -1};
    index.erase(key[slot]);
    key[slot] = -1;
    state[slot] = kEmpty;
    ++evictions;
    last_evicted = slot;
  }
  ++misses;
  key[slot] = k;
  state[slot] = kWrite;
  readers[slot] = 0;
  stamp[slot] = ++clock;
  index[k] = slot;
  return TierResult{kMiss, slot};
}

void SlotTier::publish(int s, bool retain) {
  state[s] = kRead;
  readers[s] = retain ? 1 : 0;
}

void SlotTier::abort(int s) {
  index.erase(key[s]);
  key[s] = -1;
  state[s] = kEmpty;
  free_list.push_back(s);
}

void SlotTier::release(int s) {
  --readers[s];
  stamp[s] = ++clock;
}

}  // namespace rk

struct rk_engine {
  rk_app_params app_params{};
  rk_engine_params p{};
  int device = 0;
  rk_app* app = nullptr;
  cudaStream_t stream = nullptr;    // compare stream (rk_engine_stream)
  // Load pipeline (engine.py:436-487 on a stream of its own): H2D + preprocess and
  // peer fetches of the next leaves run on `lstream` while the compare stream
  // executes the current batch.  Ordering: a compare batch waits for `ev_loaded`
  // (the last load issued before it); a load into an evicted slot waits for
  // `ev_compared` (every compare launched before the eviction).
  cudaStream_t lstream = nullptr;
  cudaEvent_t ev_loaded = nullptr;
  cudaEvent_t ev_compared = nullptr;
  bool loads_unsynced = false;      // loads issued since the compare stream last waited
  // cross-GPU work queue (queue_op_kernel): own word at the arena's tail, peers' via IPC
  unsigned long long* qword = nullptr;
  std::vector<unsigned long long*> peer_q;
  bool queues_ready = false;
  cudaStream_t cstream = nullptr;   // control stream for the queue operations
  unsigned long long* h_qres = nullptr;   // mapped pinned result word
  unsigned long long* d_qres = nullptr;
  cudaEvent_t ev_chunk[2] = {nullptr, nullptr};
  int64_t steals = 0;
  bool queue_armed = false;         // rk_engine_queue_reset since the last run
  void* arena = nullptr;
  size_t slot_stride = 0;
  size_t arena_slots = 0;           // device_slots rounded up to the app's slot group
  void* staging = nullptr;
  int staging_items = 0;
  rk::SlotTier* tier = nullptr;
  // host (L2) tier of preprocessed items: the reference's host CacheTier
  // (slotcache.py:139-282) over pinned host slots, written through on every fresh
  // load (engine.py:482-508) and read back H2D on a device miss (engine.py:375-394)
  rk::SlotTier* htier = nullptr;
  char* harena = nullptr;
  rk_engine_stats stats{};
  // peer-GPU tier (distcache.py owner_of: home(k) = k mod world): this rank's home
  // items live at arena slots [arena_slots, arena_slots + home_slots), item k at
  // arena_slots + k / world; other ranks' home regions are IPC-mapped
  int home_slots = 0;
  std::vector<const char*> peer_home;   // per rank: base of its home region (own entry = local)
  bool peers_ready = false;
  // sampled kernel timing of the compare batches
  // trace events (metrics.py TraceEvent): one per compare batch / load group / fetch group
  struct TraceRec {
    int32_t lane, i, j, count;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> tr_pool;
  std::vector<TraceRec> tr;
  cudaEvent_t tr_t0 = nullptr;
  int tr_max = 0;
  std::vector<rk_trace_event> tr_done;
  int profile_every = 0;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_pairs;
  int ev_used = 0;
  // exactly-once ledger: own region in the arena allocation; marks go to `ledger_target`
  // (own, or rank 0's region mapped over IPC when the job shares one ledger)
  // NCC Gram over the peer tier: one compute stream per home sub-block, fetch events
  std::vector<cudaStream_t> gstreams;
  std::vector<cudaEvent_t> gevents;
  size_t ledger_off = 0;
  size_t ledger_bytes = 0;
  void* ledger_own = nullptr;
  void* ledger_target = nullptr;
  bool ledger_shared = false;
};

using namespace rk;

namespace {

struct LoadReq {
  int32_t key;
  int32_t slot;
  int32_t hslot = -1;   // host-tier slot: write-through target (fresh load) or source (host hit)
};

// Device timestamps of the finished run's trace records, relative to its start.
rk_status trace_collect(rk_engine* e) {
  for (const auto& r : e->tr) {
    float a = 0.f, b = 0.f;
    RK_CUDA(cudaEventElapsedTime(&a, e->tr_t0, r.a));
    RK_CUDA(cudaEventElapsedTime(&b, e->tr_t0, r.b));
    rk_trace_event ev{};
    ev.lane = r.lane;
    ev.i = r.i;
    ev.j = r.j;
    ev.count = r.count;
    ev.start_ns = (int64_t)((double)a * 1e6);
    ev.end_ns = (int64_t)((double)b * 1e6);
    e->tr_done.push_back(ev);
  }
  e->tr.clear();
  return RK_OK;
}

// One queue operation on `word` (own or a peer's), synchronous.
rk_status queue_call(rk_engine* e, unsigned long long* word, int op, unsigned long long arg, unsigned long long* res) {
  queue_op_kernel<<<1, 1, 0, e->cstream>>>(word, op, arg, e->d_qres);
  RK_CUDA(cudaGetLastError());
  RK_CUDA(cudaStreamSynchronize(e->cstream));
  *res = *(volatile unsigned long long*)e->h_qres;
  return RK_OK;
}

// Trace record around work on `st` (no-op unless rk_engine_set_trace is on)
int trace_begin(rk_engine* e, int lane, int i, int j, int count, cudaStream_t st) {
  if (e->tr_max == 0 || (int)e->tr.size() >= e->tr_max) return -1;
  const size_t k = e->tr.size();
  e->tr.push_back(rk_engine::TraceRec{lane, i, j, count, e->tr_pool[2 * k], e->tr_pool[2 * k + 1]});
  cudaEventRecord(e->tr.back().a, st);
  return (int)k;
}
void trace_end(rk_engine* e, int k, cudaStream_t st) {
  if (k >= 0) cudaEventRecord(e->tr[k].b, st);
}

rk_status flush_pairs(rk_engine* e, std::vector<rk_pair>& pend, double* d_out, uint8_t* d_flags) {
  if (pend.empty()) return RK_OK;
  if (e->loads_unsynced) {   // the batch reads slots loaded on the load stream
    RK_CUDA(cudaStreamWaitEvent(e->stream, e->ev_loaded, 0));
    e->loads_unsynced = false;
  }
  const int lim = batch_limit(e->app);
  for (size_t base = 0; base < pend.size(); base += lim) {
    const int m = (int)std::min<size_t>(lim, pend.size() - base);
    const bool timed = e->profile_every > 0 && (e->stats.tiles % e->profile_every) == 0 &&
                       e->ev_used + 2 <= (int)e->ev.size();
    if (timed) RK_CUDA(cudaEventRecord(e->ev[e->ev_used], e->stream));
    const int tk = trace_begin(e, 0, pend[base].i, pend[base].j, m, e->stream);
    RK_TRY(compare_pairs(e->app, e->arena, e->slot_stride, pend.data() + base, m, d_out, d_flags, e->stream));
    trace_end(e, tk, e->stream);
    if (timed) {
      RK_CUDA(cudaEventRecord(e->ev[e->ev_used + 1], e->stream));
      e->ev_pairs[e->ev_used / 2] = m;
      e->ev_used += 2;
    }
    e->stats.pairs_done += m;
    e->stats.tiles += 1;
  }
  pend.clear();
  return RK_OK;
}

rk_status flush_loads(rk_engine* e, std::vector<LoadReq>& loads, const void* h_parsed, const void* d_parsed,
                      size_t parsed_stride) {
  if (loads.empty()) return RK_OK;
  const size_t pbytes = e->app->parsed_bytes;
  for (size_t base = 0; base < loads.size(); base += e->staging_items) {
    const int m = (int)std::min<size_t>(e->staging_items, loads.size() - base);
    std::vector<int32_t> slots(m);
    for (int k = 0; k < m; ++k) slots[k] = loads[base + k].slot;
    const int tk = trace_begin(e, 1, loads[base].key, -1, m, e->lstream);
    if (h_parsed) {
      for (int k = 0; k < m; ++k) {
        const char* src = static_cast<const char*>(h_parsed) + (size_t)loads[base + k].key * parsed_stride;
        RK_CUDA(cudaMemcpyAsync(static_cast<char*>(e->staging) + (size_t)k * pbytes, src, pbytes,
                                cudaMemcpyHostToDevice, e->lstream));
        e->stats.h2d_bytes += (int64_t)pbytes;
      }
      RK_TRY(rk_preprocess(e->app, e->staging, pbytes, m, e->arena, e->slot_stride, slots.data(), e->lstream));
    } else {
      // device-resident parsed items: preprocess runs of consecutive keys in place
      int k = 0;
      while (k < m) {
        int run = 1;
        while (k + run < m && loads[base + k + run].key == loads[base + k].key + run) ++run;
        const char* src = static_cast<const char*>(d_parsed) + (size_t)loads[base + k].key * parsed_stride;
        RK_TRY(rk_preprocess(e->app, src, parsed_stride, run, e->arena, e->slot_stride, slots.data() + k, e->lstream));
        k += run;
      }
    }
    trace_end(e, tk, e->lstream);
    e->stats.loads += m;
  }
  for (const LoadReq& l : loads) {
    e->tier->publish(l.slot, true);  // retained lease (slotcache.py:188-213)
    if (l.hslot >= 0) {
      // write-through: the host copy is published with (here: right after) the device
      // copy (engine.py:482-487, assert :503); stream order on the load stream keeps a
      // later reuse of this host slot behind the copy
      RK_CUDA(cudaMemcpyAsync(e->harena + (size_t)l.hslot * e->slot_stride,
                              static_cast<char*>(e->arena) + (size_t)l.slot * e->slot_stride, e->app->slot_bytes,
                              cudaMemcpyDeviceToHost, e->lstream));
      e->stats.d2h_bytes += (int64_t)e->app->slot_bytes;
      e->htier->publish(l.hslot, false);
    }
  }
  loads.clear();
  RK_CUDA(cudaEventRecord(e->ev_loaded, e->lstream));
  e->loads_unsynced = true;
  return RK_OK;
}

// Device misses served by the host tier: H2D of the preprocessed slot, no parse /
// preprocess (not a load, engine.py:443-448); the host lease ends once the copy
// is enqueued (later host-slot reuse is ordered behind it on the load stream).
rk_status flush_host_hits(rk_engine* e, std::vector<LoadReq>& hits) {
  if (hits.empty()) return RK_OK;
  const int tk = trace_begin(e, 1, hits[0].key, -1, (int)hits.size(), e->lstream);
  for (const LoadReq& h : hits) {
    RK_CUDA(cudaMemcpyAsync(static_cast<char*>(e->arena) + (size_t)h.slot * e->slot_stride,
                            e->harena + (size_t)h.hslot * e->slot_stride, e->app->slot_bytes, cudaMemcpyHostToDevice,
                            e->lstream));
    e->stats.h2d_bytes += (int64_t)e->app->slot_bytes;
    e->htier->release(h.hslot);
    e->tier->publish(h.slot, true);
  }
  trace_end(e, tk, e->lstream);
  hits.clear();
  RK_CUDA(cudaEventRecord(e->ev_loaded, e->lstream));
  e->loads_unsynced = true;
  return RK_OK;
}

}  // namespace

// NCC with fewer device slots than items: key blocks of B items (B = half the
// arena, a multiple of the 256-item tile), block I in rows [0, B), block J in
// rows [B, 2B); for every block pair I <= J dealt to this rank, the triangle of I
// (J == I) or the I x J rectangle through rk_ncc_gram_block.  Block I is loaded
// once per row of blocks, J once per pair (R ~ blocks / 2).
rk_status ncc_blocked_run(rk_engine* e, const void* h_parsed, const void* d_parsed, size_t parsed_stride,
                          double* d_out, uint8_t* d_flags, int64_t launches0) {
  const int32_t n = e->app->p.n;
  const int32_t B = (int32_t)(e->arena_slots / 2) / 256 * 256;
  if (B < 256)
    return set_error(RK_ERR_NO_EVICTABLE, "blocked NCC Gram needs >= 512 device slots (have %zu)", e->arena_slots);
  const int32_t nb = (n + B - 1) / B;
  const size_t pbytes = e->app->parsed_bytes;
  auto load_block = [&](int32_t blk, int32_t row0) -> rk_status {
    const int32_t k0 = blk * B, cnt = std::min(n, k0 + B) - k0;
    for (int32_t base = 0; base < cnt; base += e->staging_items) {
      const int m = std::min(e->staging_items, cnt - base);
      std::vector<int32_t> slots(m);
      for (int q = 0; q < m; ++q) slots[q] = row0 + base + q;
      if (h_parsed) {
        for (int q = 0; q < m; ++q) {
          RK_CUDA(cudaMemcpyAsync(static_cast<char*>(e->staging) + (size_t)q * pbytes,
                                  static_cast<const char*>(h_parsed) + (size_t)(k0 + base + q) * parsed_stride, pbytes,
                                  cudaMemcpyHostToDevice, e->stream));
          e->stats.h2d_bytes += (int64_t)pbytes;
        }
        RK_TRY(rk_preprocess(e->app, e->staging, pbytes, m, e->arena, e->slot_stride, slots.data(), e->stream));
      } else {
        RK_TRY(rk_preprocess(e->app, static_cast<const char*>(d_parsed) + (size_t)(k0 + base) * parsed_stride,
                             parsed_stride, m, e->arena, e->slot_stride, slots.data(), e->stream));
      }
      e->stats.loads += m;
      e->stats.misses += m;
    }
    return RK_OK;
  };
  int64_t t = 0;
  for (int32_t bi = 0; bi < nb; ++bi) {
    bool loaded_i = false;
    for (int32_t bj = bi; bj < nb; ++bj, ++t) {
      if (t % e->p.world != e->p.rank) continue;
      if (!loaded_i) {
        RK_TRY(load_block(bi, 0));
        loaded_i = true;
      }
      const int32_t ki = bi * B, ci = std::min(n, ki + B) - ki;
      const int32_t kj = bj * B, cj = std::min(n, kj + B) - kj;
      if (bj == bi) {
        RK_TRY(rk_ncc_gram_block(e->app, e->arena, e->slot_stride, (int32_t)e->arena_slots, 0, ki, ci, 0, ki, ci, d_out,
                                 d_flags, e->stream));
        e->stats.pairs_done += (int64_t)ci * (ci - 1) / 2;
      } else {
        RK_TRY(load_block(bj, B));
        RK_TRY(rk_ncc_gram_block(e->app, e->arena, e->slot_stride, (int32_t)e->arena_slots, 0, ki, ci, B, kj, cj, d_out,
                                 d_flags, e->stream));
        e->stats.pairs_done += (int64_t)ci * cj;
      }
      e->stats.tiles += 1;
    }
  }
  RK_CUDA(cudaStreamSynchronize(e->stream));
  RK_TRY(trace_collect(e));
  e->stats.kernel_launches += e->app->launches - launches0;
  return RK_OK;
}

// NCC Gram over the peer tier (distcache.py owner_of(k) = k mod p for the Gram's
// key blocks).  Rank s's home items (keys s + m*world, home slots m) are cut into
// sub-blocks of B items, B = half the cache arena; all M sub-blocks of the job in
// (t, s) order.  Every unordered pair of sub-blocks {a, b} (a = b included) is one
// Gram block, computed by the owner of a when b lies in the circulant half after a
// (b - a mod M in [1, M/2), the diametric pair by the lower index), so every rank
// gets the same number of blocks.  A rank walks its partner sub-blocks b: a home
// b is read in place, any other is copied from its owner's home region over
// NVLink (CUDA IPC) into one of two fetch buffers on the load stream while the
// previous partner's blocks multiply -- the blocks of one partner run on one
// stream per home sub-block so together they fill the SMs.
rk_status ncc_peer_run(rk_engine* e, double* d_out, uint8_t* d_flags, int64_t launches0) {
  const int32_t n = e->app->p.n, w = e->p.world, r = e->p.rank;
  const int grp = std::max(1, e->app->slot_group);
  const int32_t Bmax = (int32_t)(e->arena_slots / 2) / grp * grp;
  if (Bmax < grp)
    return set_error(RK_ERR_NO_EVICTABLE, "NCC over the peer tier needs >= %d device slots (have %zu)", 2 * grp,
                     e->arena_slots);
  auto home_cnt = [&](int32_t s) { return n > s ? (n - s + w - 1) / w : 0; };
  // an even number T of sub-blocks per rank (at least 2): with the (t, s) order the
  // diametric block pairs then split evenly over the ranks
  int32_t T = std::max<int32_t>(2, (home_cnt(0) + Bmax - 1) / Bmax);
  T += T & 1;
  const int32_t tile = grp * 2;   // 256-item Gram tiles
  const int32_t B = std::min(Bmax, std::max(grp, ((home_cnt(0) + T - 1) / T + tile - 1) / tile * tile));
  struct Sub {
    int32_t s, m0, cnt;
  };
  std::vector<Sub> subs;
  int32_t tmax = 0;
  for (int32_t s = 0; s < w; ++s) tmax = std::max(tmax, (home_cnt(s) + B - 1) / B);
  for (int32_t t = 0; t < tmax; ++t)
    for (int32_t s = 0; s < w; ++s)
      if (t * B < home_cnt(s)) subs.push_back(Sub{s, t * B, std::min(B, home_cnt(s) - t * B)});
  const int M = (int)subs.size();
  std::vector<int> mine;
  for (int a = 0; a < M; ++a)
    if (subs[a].s == r) mine.push_back(a);
  // partner b -> the home sub-blocks a that pair with it on this rank
  std::vector<std::vector<int>> with(M);
  for (int a : mine) {
    with[a].push_back(a);
    for (int dd = 1; 2 * dd <= M; ++dd) {
      const int b = (a + dd) % M;
      if (2 * dd < M || a < b) with[b].push_back(a);
    }
  }
  // partners: home ones first (no copy), then the fetched ones in circulant order
  std::vector<int> order;
  for (int b = 0; b < M; ++b)
    if (!with[b].empty() && subs[b].s == r) order.push_back(b);
  const int a0 = mine.empty() ? 0 : mine[0];
  for (int dd = 1; dd < M; ++dd) {
    const int b = (a0 + dd) % M;
    if (!with[b].empty() && subs[b].s != r) order.push_back(b);
  }
  const size_t stride = e->slot_stride;
  while ((int)e->gstreams.size() < (int)mine.size()) {
    cudaStream_t st;
    RK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    e->gstreams.push_back(st);
  }
  // events: 2 fetch-done + per buffer and stream one use-done
  const size_t need_ev = 2 + 2 * e->gstreams.size() + 1;
  while (e->gevents.size() < need_ev) {
    cudaEvent_t ev;
    RK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->gevents.push_back(ev);
  }
  cudaEvent_t* ev_fetched = &e->gevents[0];
  cudaEvent_t* ev_used = &e->gevents[2];            // [buf * S + stream]
  cudaEvent_t ev_start = e->gevents[need_ev - 1];
  const int S = (int)e->gstreams.size();
  RK_CUDA(cudaEventRecord(ev_start, e->stream));
  for (int q = 0; q < S; ++q) RK_CUDA(cudaStreamWaitEvent(e->gstreams[q], ev_start, 0));
  RK_CUDA(cudaStreamWaitEvent(e->lstream, ev_start, 0));
  std::vector<int> slot_stream(M, -1);
  for (int q = 0; q < (int)mine.size(); ++q) slot_stream[mine[q]] = q;
  int nf = 0;
  for (int b : order) {
    int32_t brow;
    if (subs[b].s == r) {
      brow = (int32_t)e->arena_slots + subs[b].m0;
    } else {
      const int f = nf % 2;
      if (nf >= 2)   // buffer f's previous partner is multiplied on every stream
        for (int q = 0; q < S; ++q) RK_CUDA(cudaStreamWaitEvent(e->lstream, ev_used[f * S + q], 0));
      const int tk = trace_begin(e, 2, subs[b].s + subs[b].m0 * w, -1, subs[b].cnt, e->lstream);
      // whole slot groups: the NCC layout interleaves each group's 128 items ([D/1024][128][1024]),
      // so a partial group is not a byte prefix (home regions are allocated in whole groups)
      const size_t rows = (size_t)(subs[b].cnt + grp - 1) / grp * grp;
      RK_TRY(peer_copy(static_cast<char*>(e->arena) + (size_t)f * B * stride,
                       e->peer_home[subs[b].s] + (size_t)subs[b].m0 * stride, rows * stride, e->lstream));
      trace_end(e, tk, e->lstream);
      RK_CUDA(cudaEventRecord(ev_fetched[f], e->lstream));
      for (int q = 0; q < S; ++q) RK_CUDA(cudaStreamWaitEvent(e->gstreams[q], ev_fetched[f], 0));
      e->stats.peer_fetches += subs[b].cnt;
      e->stats.peer_bytes += (int64_t)subs[b].cnt * (int64_t)stride;
      brow = f * B;
      ++nf;
    }
    for (int a : with[b]) {
      const int q = slot_stream[a];
      const int tk = trace_begin(e, 0, subs[a].s + subs[a].m0 * w, subs[b].s + subs[b].m0 * w,
                                 a == b ? subs[a].cnt * (subs[a].cnt - 1) / 2 : subs[a].cnt * subs[b].cnt,
                                 e->gstreams[q]);
      RK_TRY(ncc_gram_block_strided(e->app, e->arena, stride, (int32_t)(e->arena_slots + e->home_slots),
                                    (int32_t)e->arena_slots + subs[a].m0, subs[a].s + subs[a].m0 * w, subs[a].cnt,
                                    brow, subs[b].s + subs[b].m0 * w, subs[b].cnt, w, a == b, d_out, d_flags,
                                    e->gstreams[q]));
      trace_end(e, tk, e->gstreams[q]);
      e->stats.pairs_done += a == b ? (int64_t)subs[a].cnt * (subs[a].cnt - 1) / 2
                                    : (int64_t)subs[a].cnt * subs[b].cnt;
      e->stats.tiles += 1;
    }
    if (subs[b].s != r)
      for (int q = 0; q < S; ++q) RK_CUDA(cudaEventRecord(ev_used[((nf - 1) % 2) * S + q], e->gstreams[q]));
  }
  for (int q = 0; q < S; ++q) RK_CUDA(cudaStreamSynchronize(e->gstreams[q]));
  RK_CUDA(cudaStreamSynchronize(e->lstream));
  RK_CUDA(cudaStreamSynchronize(e->stream));
  RK_TRY(trace_collect(e));
  e->stats.kernel_launches += e->app->launches - launches0;
  return RK_OK;
}

extern "C" {

rk_status rk_engine_create(const rk_app_params* app_params, const rk_engine_params* params, int device,
                           rk_engine** out) {
  if (!app_params || !params || !out) return set_error(RK_ERR_VALUE, "null argument");
  *out = nullptr;
  if (params->leaf_block < 1) return set_error(RK_ERR_VALUE, "leaf_block must be >= 1");
  if (params->world < 1 || params->rank < 0 || params->rank >= params->world)
    return set_error(RK_ERR_VALUE, "bad rank/world %d/%d", params->rank, params->world);
  if (params->device_slots < 2) return set_error(RK_ERR_VALUE, "device tiers need >= 2 slots to hold a pair");
  RK_CUDA(cudaSetDevice(device));
  rk_engine* e = new rk_engine();
  e->app_params = *app_params;
  e->p = *params;
  e->device = device;
  rk_status st = rk_app_create(app_params, device, &e->app);
  if (st != RK_OK) {
    delete e;
    return st;
  }
  auto fail = [&](rk_status s) {
    rk_engine_destroy(e);
    return s;
  };
  e->slot_stride = (e->app->slot_bytes + 255) / 256 * 256 + stride_pad("RK_SLOT_PAD", 0);
  cudaError_t ce = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) return fail(check_cuda(ce, "cudaStreamCreate"));
  ce = cudaStreamCreateWithFlags(&e->lstream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) return fail(check_cuda(ce, "cudaStreamCreate(load)"));
  ce = cudaEventCreateWithFlags(&e->ev_loaded, cudaEventDisableTiming);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->ev_compared, cudaEventDisableTiming);
  if (ce != cudaSuccess) return fail(check_cuda(ce, "cudaEventCreate"));
  if (params->peer_tier && params->world > 1) {
    // whole slot groups, so the home region is a block of rows of the Gram's tensor map
    const int g = std::max(1, e->app->slot_group);
    e->home_slots = ((app_params->n + params->world - 1) / params->world + g - 1) / g * g;
  }
  // interleaved slot groups (rk_app_slot_group): whole groups only
  const size_t g = (size_t)std::max(1, e->app->slot_group);
  e->arena_slots = ((size_t)params->device_slots + g - 1) / g * g;
  const size_t arena_bytes = e->slot_stride * (e->arena_slots + e->home_slots);
  // + the work-queue word and the ledger region (shared with the home region over IPC)
  e->ledger_off = arena_bytes + 256;
  e->ledger_bytes = ledger_region_bytes(app_params->n);
  ce = cudaMalloc(&e->arena, arena_bytes + 256 + e->ledger_bytes);
  if (ce != cudaSuccess) return fail(check_cuda(ce, "cudaMalloc(slot arena)"));
  e->qword = reinterpret_cast<unsigned long long*>(static_cast<char*>(e->arena) + arena_bytes);
  e->ledger_own = static_cast<char*>(e->arena) + e->ledger_off;
  e->ledger_target = e->ledger_own;
  e->app->ledger = ledger_at(e->ledger_own, app_params->n);
  ce = cudaMemset(e->qword, 0, 256 + e->ledger_bytes);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&e->cstream, cudaStreamNonBlocking);
  if (ce == cudaSuccess) ce = cudaHostAlloc(&e->h_qres, 64, cudaHostAllocMapped);
  if (ce == cudaSuccess) ce = cudaHostGetDevicePointer(&e->d_qres, e->h_qres, 0);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->ev_chunk[0], cudaEventDisableTiming);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->ev_chunk[1], cudaEventDisableTiming);
  if (ce != cudaSuccess) return fail(check_cuda(ce, "work queue setup"));
  e->staging_items = std::max(1, batch_limit(e->app));
  if (e->app->p.kind == RK_APP_PCE) e->staging_items = e->app->pce.batch;
  ce = cudaMalloc(&e->staging, std::max<size_t>(e->app->parsed_bytes, 16) * e->staging_items);
  if (ce != cudaSuccess) return fail(check_cuda(ce, "cudaMalloc(staging)"));
  e->tier = new SlotTier(params->device_slots);
  if (params->host_slots > 0 && !(params->peer_tier && params->world > 1) && app_params->kind != RK_APP_NCC &&
      app_params->kind != RK_APP_SYNTHETIC) {
    if (params->host_slots < 2) return fail(set_error(RK_ERR_VALUE, "host tiers need >= 2 slots"));
    e->htier = new SlotTier(params->host_slots);
    ce = cudaHostAlloc(reinterpret_cast<void**>(&e->harena), (size_t)params->host_slots * e->slot_stride,
                       cudaHostAllocDefault);
    if (ce != cudaSuccess) return fail(check_cuda(ce, "cudaHostAlloc(host tier)"));
  }
  *out = e;
  return RK_OK;
}

void rk_engine_destroy(rk_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  for (cudaEvent_t ev : e->ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : e->tr_pool) cudaEventDestroy(ev);
  if (e->tr_t0) cudaEventDestroy(e->tr_t0);
  if (e->stream) cudaStreamDestroy(e->stream);
  if (e->lstream) cudaStreamDestroy(e->lstream);
  if (e->ev_loaded) cudaEventDestroy(e->ev_loaded);
  if (e->ev_compared) cudaEventDestroy(e->ev_compared);
  for (cudaEvent_t ev : e->ev_chunk)
    if (ev) cudaEventDestroy(ev);
  for (cudaStream_t st : e->gstreams) cudaStreamDestroy(st);
  for (cudaEvent_t ev : e->gevents) cudaEventDestroy(ev);
  if (e->cstream) cudaStreamDestroy(e->cstream);
  if (e->h_qres) cudaFreeHost(e->h_qres);
  cudaFree(e->arena);
  cudaFree(e->staging);
  if (e->harena) cudaFreeHost(e->harena);
  delete e->htier;
  delete e->tier;
  rk_app_destroy(e->app);
  delete e;
}

rk_status rk_engine_set_profiling(rk_engine* e, int every, int max_samples) {
  if (!e) return set_error(RK_ERR_VALUE, "null engine");
  RK_CUDA(cudaSetDevice(e->device));
  for (cudaEvent_t ev : e->ev) cudaEventDestroy(ev);
  e->ev.clear();
  e->profile_every = every;
  if (every > 0) {
    e->ev.resize((size_t)2 * std::max(1, max_samples));
    e->ev_pairs.assign((size_t)std::max(1, max_samples), 0);
    for (auto& ev : e->ev) RK_CUDA(cudaEventCreate(&ev));
  }
  e->ev_used = 0;
  return RK_OK;
}

static rk_status engine_run_impl(rk_engine* e, const void* h_parsed, const void* d_parsed, size_t parsed_stride,
                                 double* d_out, uint8_t* d_flags);

// Every run marks each completed pair in the ledger; a duplicate fails the run
// (PairLedger.mark's AssertionError).  A private ledger is cleared and checked
// here; a shared one (multi-GPU) by rank 0 around the job's barriers.
rk_status rk_engine_run(rk_engine* e, const void* h_parsed, const void* d_parsed, size_t parsed_stride, double* d_out,
                        uint8_t* d_flags) {
  if (!e) return set_error(RK_ERR_VALUE, "null engine");
  RK_CUDA(cudaSetDevice(e->device));
  if (!e->ledger_shared) RK_CUDA(cudaMemsetAsync(e->ledger_own, 0, e->ledger_bytes, e->stream));
  RK_TRY(engine_run_impl(e, h_parsed, d_parsed, parsed_stride, d_out, d_flags));
  if (e->ledger_shared) {
    e->stats.ledger_marked = -1;
    return RK_OK;
  }
  rk_ledger_stats ls{};
  RK_TRY(ledger_read(e->ledger_own, e->app->p.n, e->stream, &ls));
  e->stats.ledger_marked = ls.completed;
  e->stats.dup_marks += ls.dup_marks;
  if (ls.dup_marks) return duplicate_error(e->app->p.n, ls);
  return RK_OK;
}

static rk_status engine_run_impl(rk_engine* e, const void* h_parsed, const void* d_parsed, size_t parsed_stride,
                                 double* d_out, uint8_t* d_flags) {
  if (!h_parsed && !d_parsed && e->app->p.kind != RK_APP_SYNTHETIC && e->home_slots == 0)
    return set_error(RK_ERR_VALUE, "need host or device parsed items");
  RK_CUDA(cudaSetDevice(e->device));
  const int32_t n = e->app->p.n;
  e->ev_used = 0;
  // every run starts from a cold tier: parsed inputs may differ between runs
  {
    const int64_t h = e->tier->hits, m = e->tier->misses, ev = e->tier->evictions;
    *e->tier = SlotTier(e->tier->capacity);
    e->tier->hits = h;
    e->tier->misses = m;
    e->tier->evictions = ev;
    if (e->htier) {
      const int64_t hh = e->htier->hits, hm = e->htier->misses, he = e->htier->evictions;
      *e->htier = SlotTier(e->htier->capacity);
      e->htier->hits = hh;
      e->htier->misses = hm;
      e->htier->evictions = he;
    }
  }
  const int64_t launches0 = e->app->launches;
  e->tr.clear();
  e->tr_done.clear();
  if (e->tr_max > 0) RK_CUDA(cudaEventRecord(e->tr_t0, e->stream));
  // the load stream starts after everything already queued on the engine stream
  RK_CUDA(cudaEventRecord(e->ev_compared, e->stream));
  RK_CUDA(cudaStreamWaitEvent(e->lstream, e->ev_compared, 0));
  e->loads_unsynced = false;
  if (e->app->p.kind == RK_APP_NCC) {
    // Gram path over the peer tier: home items resident, others fetched over NVLink
    if (e->home_slots > 0) {
      if (!e->peers_ready)
        return set_error(RK_ERR_VALUE, "peer tier: call rk_engine_load_home and rk_engine_set_peer_homes first");
      return ncc_peer_run(e, d_out, d_flags, launches0);
    }
    // every item resident in slot == key, then one tcgen05 GEMM over this rank's
    // upper-triangle tiles
    if (e->tier->capacity < n) return ncc_blocked_run(e, h_parsed, d_parsed, parsed_stride, d_out, d_flags, launches0);
    std::vector<LoadReq> all;
    for (int32_t k = 0; k < n; ++k) {
      const TierResult r = e->tier->acquire(k);
      if (r.kind == kMiss) all.push_back(LoadReq{k, r.slot});
    }
    RK_TRY(flush_loads(e, all, h_parsed, d_parsed, parsed_stride));
    for (int32_t k = 0; k < n; ++k) e->tier->release(e->tier->find(k));
    if (e->loads_unsynced) RK_CUDA(cudaStreamWaitEvent(e->stream, e->ev_loaded, 0));
    e->loads_unsynced = false;
    RK_TRY(rk_ncc_gram(e->app, e->arena, e->slot_stride, (int32_t)e->arena_slots, e->p.rank, e->p.world, d_out,
                       d_flags, e->stream));
    const int tile = ncc_gram_tile(n);
    const int side = (n + tile - 1) / tile;
    int64_t mine = 0;
    for (int ti = 0, t = 0; ti < side; ++ti)
      for (int tj = ti; tj < side; ++tj, ++t)
        if (t % e->p.world == e->p.rank)
          mine += region_pairs(ti * tile, std::min(n, ti * tile + tile), tj * tile, std::min(n, tj * tile + tile));
    e->stats.pairs_done += mine;
    e->stats.tiles += 1;
    RK_CUDA(cudaStreamSynchronize(e->stream));
    RK_TRY(trace_collect(e));
    e->stats.hits = e->tier->hits;
    e->stats.misses = e->tier->misses;
    e->stats.evictions = e->tier->evictions;
    e->stats.kernel_launches += e->app->launches - launches0;
    return RK_OK;
  }
  const std::vector<Leaf> all_leaves = quadtree_leaves(n, e->p.leaf_block);
  const bool steal = e->p.steal && e->p.world > 1;
  if (steal && !e->queues_ready)
    return set_error(RK_ERR_VALUE, "work stealing: call rk_engine_queue_reset and rk_engine_set_peer_queues first");
  if (steal && !e->queue_armed)
    return set_error(RK_ERR_VALUE, "work stealing: rk_engine_queue_reset (and a barrier) must precede every run");
  e->queue_armed = false;
  const bool peer = e->home_slots > 0;
  if (peer && !e->peers_ready)
    return set_error(RK_ERR_VALUE, "peer tier: call rk_engine_load_home and rk_engine_set_peer_homes first");
  const int world = e->p.world;
  std::vector<rk_pair> pend;
  std::vector<LoadReq> loads;
  std::vector<LoadReq> fetches;
  std::vector<LoadReq> host_hits;
  std::vector<int32_t> keys;
  std::vector<int32_t> pinned;
  std::vector<int32_t> slot_of(peer ? n : 0, -1);
  const int lim = batch_limit(e->app);
  std::function<rk_status(const Leaf&)> do_leaf = [&](const Leaf& l) -> rk_status {
    if (e->app->p.kind == RK_APP_SYNTHETIC) {
      // no item state: the hash needs only the keys (apps.py:201-208)
      RK_TRY(rk_compare_tile(e->app, nullptr, 0, l.r0, l.r1, l.c0, l.c1, nullptr, d_out, d_flags, e->stream));
      e->stats.pairs_done += region_pairs(l.r0, l.r1, l.c0, l.c1);
      e->stats.tiles += 1;
      return RK_OK;
    }
    // ascending key acquisition over the leaf's items (engine.py:510-516)
    keys.clear();
    for (int32_t k = l.r0; k < l.r1; ++k) keys.push_back(k);
    for (int32_t k = l.c0; k < l.c1; ++k) keys.push_back(k);
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    {
      // tight tier (test_engine.py:88-93 "tight tier completes"): a leaf whose items do
      // not fit the device slots is split into its quadrants (Region.split,
      // scheduler.py:56-68) until they do; a 1 x 1 region needs 2 slots
      int64_t need = 0;
      for (int32_t k : keys) need += !(peer && k % world == e->p.rank);
      if (need > e->tier->capacity && (l.r1 - l.r0 > 1 || l.c1 - l.c0 > 1)) {
        const int32_t rm = (l.r0 + l.r1 + 1) / 2, cm = (l.c0 + l.c1 + 1) / 2;
        const Leaf q[4] = {{l.r0, rm, l.c0, cm}, {l.r0, rm, cm, l.c1}, {rm, l.r1, l.c0, cm}, {rm, l.r1, cm, l.c1}};
        for (const Leaf& sub : q)
          if (sub.r0 < sub.r1 && sub.c0 < sub.c1 && region_pairs(sub.r0, sub.r1, sub.c0, sub.c1) > 0)
            RK_TRY(do_leaf(sub));
        return RK_OK;
      }
    }
    pinned.clear();
    for (int32_t k : keys) {
      if (peer && k % world == e->p.rank) {
        slot_of[k] = (int32_t)e->arena_slots + k / world;   // home item: resident for the whole run
        continue;
      }
      const int64_t evictions_before = e->tier->evictions;
      TierResult r = e->tier->acquire(k);
      if (r.kind == kNoEvictable) {
        for (int s : pinned) e->tier->release(s);
        for (const LoadReq& q : loads) {
          e->tier->abort(q.slot);
          if (q.hslot >= 0) e->htier->abort(q.hslot);
        }
        for (const LoadReq& q : host_hits) {
          e->tier->abort(q.slot);
          e->htier->release(q.hslot);
        }
        loads.clear();
        host_hits.clear();
        return set_error(RK_ERR_NO_EVICTABLE, "all %d device slots are pinned (leaf needs %zu)", e->tier->capacity,
                         keys.size());
      }
      if (r.kind == kMiss) {
        // the victim may still be read by pairs not yet launched, or launched and
        // still running on the compare stream: the load into it waits for them
        if (e->tier->evictions != evictions_before) {
          RK_TRY(flush_pairs(e, pend, d_out, d_flags));
          RK_CUDA(cudaEventRecord(e->ev_compared, e->stream));
          RK_CUDA(cudaStreamWaitEvent(e->lstream, e->ev_compared, 0));
        }
        if (peer) {
          fetches.push_back(LoadReq{k, r.slot});
        } else if (e->htier) {
          // next level down: the host tier (engine.py:375-394)
          const TierResult hr = e->htier->acquire(k);
          if (hr.kind == kHit || hr.kind == kMustWait) host_hits.push_back(LoadReq{k, r.slot, hr.slot});
          else if (hr.kind == kMiss) loads.push_back(LoadReq{k, r.slot, hr.slot});
          else loads.push_back(LoadReq{k, r.slot});   // every host slot pinned: load without write-through
        } else {
          loads.push_back(LoadReq{k, r.slot});
        }
      }
      pinned.push_back(r.slot);
      if (peer) slot_of[k] = r.slot;
    }
    RK_TRY(flush_host_hits(e, host_hits));
    RK_TRY(flush_loads(e, loads, h_parsed, d_parsed, parsed_stride));
    if (!fetches.empty()) {
      // peer tier hit: copy the preprocessed item from its home GPU over NVLink
      const size_t sb = e->app->slot_bytes;
      const int tk = trace_begin(e, 2, fetches[0].key, -1, (int)fetches.size(), e->lstream);
      for (const LoadReq& f : fetches) {
        const char* src = e->peer_home[f.key % world] + (size_t)(f.key / world) * e->slot_stride;
        char* dst = static_cast<char*>(e->arena) + (size_t)f.slot * e->slot_stride;
        RK_CUDA(cudaMemcpyAsync(dst, src, sb, cudaMemcpyDeviceToDevice, e->lstream));
        e->tier->publish(f.slot, true);
        e->stats.peer_fetches += 1;
        e->stats.peer_bytes += (int64_t)sb;
      }
      trace_end(e, tk, e->lstream);
      fetches.clear();
      RK_CUDA(cudaEventRecord(e->ev_loaded, e->lstream));
      e->loads_unsynced = true;
    }
    for (int32_t i = l.r0; i < l.r1; ++i)
      for (int32_t j = std::max(l.c0, i + 1); j < l.c1; ++j) {
        pend.push_back(peer ? rk_pair{i, j, slot_of[i], slot_of[j]} : rk_pair{i, j, e->tier->find(i), e->tier->find(j)});
        if ((int)pend.size() >= lim) RK_TRY(flush_pairs(e, pend, d_out, d_flags));
      }
    for (int s : pinned) e->tier->release(s);
      return RK_OK;
  };
  if (!steal) {
    const auto rr = rank_range(all_leaves, e->p.rank, e->p.world);
    for (int q = rr.first; q < rr.second; ++q) RK_TRY(do_leaf(all_leaves[q]));
  } else {
    // dynamic: chunks from the own queue word, then steals; at most two chunks in
    // flight on the GPU so grabbing stays close to execution (balance at the tail)
    const int leaf_pairs = std::max(1, e->p.leaf_block * e->p.leaf_block);
    const unsigned long long chunk =
        e->p.steal_chunk > 0 ? (unsigned long long)e->p.steal_chunk : (unsigned long long)std::max(1, lim / leaf_pairs);
    int64_t c = 0;
    for (;;) {
      unsigned long long got = ~0ull;
      if (c >= 2) RK_CUDA(cudaEventSynchronize(e->ev_chunk[c & 1]));   // chunk c - 2 finished
      RK_TRY(queue_call(e, e->qword, 0, chunk, &got));
      while (got == ~0ull) {
        // own range exhausted: steal from the rank with the most remaining leaves
        int best = -1;
        unsigned best_rem = 0;
        for (int v = 0; v < world; ++v) {
          if (v == e->p.rank) continue;
          unsigned long long w = 0;
          RK_TRY(queue_call(e, e->peer_q[v], 2, 0, &w));
          const unsigned h = (unsigned)(w >> 32), t = (unsigned)w;
          const unsigned rem = t > h ? t - h : 0u;
          if (rem >= 2 * chunk && rem > best_rem) {
            best = v;
            best_rem = rem;
          }
        }
        if (best < 0) break;
        unsigned long long st = ~0ull;
        RK_TRY(queue_call(e, e->peer_q[best], 1, chunk, &st));
        if (st == ~0ull) continue;   // lost the race: look again
        e->steals += 1;
        unsigned long long tmp = 0;
        RK_TRY(queue_call(e, e->qword, 3, st, &tmp));   // the stolen range is now ours (and stealable)
        RK_TRY(queue_call(e, e->qword, 0, chunk, &got));
      }
      if (got == ~0ull) break;
      const int a = (int)(got >> 32), b = (int)(unsigned)got;
      for (int q = a; q < b; ++q) RK_TRY(do_leaf(all_leaves[q]));
      RK_TRY(flush_pairs(e, pend, d_out, d_flags));
      RK_CUDA(cudaEventRecord(e->ev_chunk[c & 1], e->stream));
      ++c;
    }
  }
  RK_TRY(flush_pairs(e, pend, d_out, d_flags));
  (void)world;
  RK_CUDA(cudaStreamSynchronize(e->lstream));
  RK_CUDA(cudaStreamSynchronize(e->stream));
  RK_TRY(trace_collect(e));
  e->stats.steals = e->steals;
  // lease hygiene at run end (test_engine.py:124-133): no reader, no slot in WRITE
  e->stats.pinned_at_end = 0;
  e->stats.writing_at_end = 0;
  for (int q = 0; q < e->tier->capacity; ++q) {
    e->stats.pinned_at_end += e->tier->readers[q] > 0;
    e->stats.writing_at_end += e->tier->state[q] == kWrite;
  }
  e->stats.hits = e->tier->hits;
  e->stats.misses = e->tier->misses;
  e->stats.evictions = e->tier->evictions;
  if (e->htier) {
    e->stats.host_hits = e->htier->hits;
    e->stats.host_misses = e->htier->misses;
    e->stats.host_evictions = e->htier->evictions;
  }
  e->stats.kernel_launches += e->app->launches - launches0;
  return RK_OK;
}

rk_status rk_engine_ledger_region(const rk_engine* e, size_t* offset, size_t* bytes) {
  if (!e || !offset || !bytes) return set_error(RK_ERR_VALUE, "null argument");
  *offset = e->ledger_off;
  *bytes = e->ledger_bytes;
  return RK_OK;
}

rk_status rk_engine_use_ledger(rk_engine* e, void* d_region) {
  if (!e || !d_region) return set_error(RK_ERR_VALUE, "null argument");
  e->ledger_target = d_region;
  e->ledger_shared = true;
  e->app->ledger = ledger_at(d_region, e->app->p.n);
  return RK_OK;
}

rk_status rk_engine_ledger_reset(rk_engine* e) {
  if (!e) return set_error(RK_ERR_VALUE, "null engine");
  if (e->ledger_target != e->ledger_own) return RK_OK;   // the owner (rank 0) clears a shared ledger
  RK_CUDA(cudaSetDevice(e->device));
  RK_CUDA(cudaMemsetAsync(e->ledger_own, 0, e->ledger_bytes, e->stream));
  RK_CUDA(cudaStreamSynchronize(e->stream));
  return RK_OK;
}

rk_status rk_engine_ledger(rk_engine* e, rk_ledger_stats* out) {
  if (!e || !out) return set_error(RK_ERR_VALUE, "null argument");
  RK_CUDA(cudaSetDevice(e->device));
  RK_TRY(ledger_read(e->ledger_target, e->app->p.n, e->cstream, out));
  out->shared = e->ledger_shared ? 1 : 0;
  return RK_OK;
}

size_t rk_ledger_bytes(int64_t n) { return ledger_region_bytes(n); }

rk_status rk_app_set_ledger(rk_app* app, void* d_region) {
  if (!app) return set_error(RK_ERR_VALUE, "null app");
  app->ledger = d_region ? ledger_at(d_region, app->p.n) : LedgerRef{nullptr, nullptr};
  return RK_OK;
}

rk_status rk_ledger_read(void* d_region, int64_t n, rk_ledger_stats* out) {
  if (!d_region || !out) return set_error(RK_ERR_VALUE, "null argument");
  return ledger_read(d_region, n, nullptr, out);
}

rk_status rk_engine_stats_get(const rk_engine* e, rk_engine_stats* out) {
  if (!e || !out) return set_error(RK_ERR_VALUE, "null argument");
  *out = e->stats;
  return RK_OK;
}

rk_status rk_engine_reset_stats(rk_engine* e) {
  if (!e) return set_error(RK_ERR_VALUE, "null engine");
  e->stats = rk_engine_stats{};
  e->steals = 0;
  e->tier->hits = e->tier->misses = e->tier->waits = e->tier->evictions = 0;
  if (e->htier) e->htier->hits = e->htier->misses = e->htier->waits = e->htier->evictions = 0;
  return RK_OK;
}

rk_status rk_engine_set_trace(rk_engine* e, int32_t max_events) {
  if (!e || max_events < 0) return set_error(RK_ERR_VALUE, "bad trace argument");
  RK_CUDA(cudaSetDevice(e->device));
  for (cudaEvent_t ev : e->tr_pool) cudaEventDestroy(ev);
  e->tr_pool.clear();
  e->tr.clear();
  e->tr_done.clear();
  e->tr_max = max_events;
  if (max_events > 0) {
    e->tr_pool.resize((size_t)2 * max_events);
    for (auto& ev : e->tr_pool) RK_CUDA(cudaEventCreate(&ev));
    if (!e->tr_t0) RK_CUDA(cudaEventCreate(&e->tr_t0));
  }
  return RK_OK;
}

int64_t rk_engine_trace_get(const rk_engine* e, rk_trace_event* out, int64_t cap) {
  if (!e) return -1;
  const int64_t n = (int64_t)e->tr_done.size();
  if (out)
    for (int64_t k = 0; k < std::min(n, cap); ++k) out[k] = e->tr_done[(size_t)k];
  return n;
}

rk_status rk_engine_kernel_time(const rk_engine* e, double* ms_total, int64_t* samples, int64_t* pairs) {
  if (!e || !ms_total || !samples || !pairs) return set_error(RK_ERR_VALUE, "null argument");
  double tot = 0.0;
  int64_t np = 0;
  for (int q = 0; q + 1 < e->ev_used; q += 2) {
    float ms = 0.f;
    RK_CUDA(cudaEventElapsedTime(&ms, e->ev[q], e->ev[q + 1]));
    tot += ms;
    np += e->ev_pairs[q / 2];
  }
  *ms_total = tot;
  *samples = e->ev_used / 2;
  *pairs = np;
  return RK_OK;
}

void* rk_engine_stream(const rk_engine* e) { return e ? (void*)e->stream : nullptr; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Peer-GPU tier: home-item preprocessing and IPC-mapped peer home regions.
extern "C" {

rk_status rk_engine_home_region(const rk_engine* e, void** d_base, size_t* bytes) {
  if (!e || !d_base || !bytes) return set_error(RK_ERR_VALUE, "null argument");
  *d_base = static_cast<char*>(e->arena) + e->arena_slots * e->slot_stride;
  *bytes = (size_t)e->home_slots * e->slot_stride;
  return RK_OK;
}

rk_status rk_engine_arena(const rk_engine* e, void** d_base, size_t* slot_stride) {
  if (!e || !d_base || !slot_stride) return set_error(RK_ERR_VALUE, "null argument");
  *d_base = e->arena;
  *slot_stride = e->slot_stride;
  return RK_OK;
}

rk_status rk_engine_load_home_range(rk_engine* e, const void* h_parsed, const void* d_parsed, size_t parsed_stride,
                                    int32_t m0, int32_t count) {
  if (!e) return set_error(RK_ERR_VALUE, "null engine");
  if (e->home_slots == 0) return set_error(RK_ERR_VALUE, "engine was created without the peer tier");
  if (!h_parsed && !d_parsed) return set_error(RK_ERR_VALUE, "need host or device parsed items");
  RK_CUDA(cudaSetDevice(e->device));
  const int32_t n = e->app->p.n;
  std::vector<LoadReq> home;
  for (int32_t m = m0; m < m0 + count; ++m) {
    const int32_t k = e->p.rank + m * e->p.world;
    if (m < 0 || k >= n) return set_error(RK_ERR_VALUE, "home item %d out of range", m);
    home.push_back(LoadReq{k, (int32_t)e->arena_slots + m});
  }
  // flush_loads publishes into the tier; home slots live outside it, so load directly
  const size_t pbytes = e->app->parsed_bytes;
  for (size_t base = 0; base < home.size(); base += e->staging_items) {
    const int m = (int)std::min<size_t>(e->staging_items, home.size() - base);
    std::vector<int32_t> slots(m);
    for (int k = 0; k < m; ++k) slots[k] = home[base + k].slot;
    // home item m0 + q (key rank + (m0 + q)*world) is at parsed + q * parsed_stride
    if (h_parsed) {
      for (int k = 0; k < m; ++k) {
        const char* src = static_cast<const char*>(h_parsed) + (base + k) * parsed_stride;
        RK_CUDA(cudaMemcpyAsync(static_cast<char*>(e->staging) + (size_t)k * pbytes, src, pbytes,
                                cudaMemcpyHostToDevice, e->stream));
        e->stats.h2d_bytes += (int64_t)pbytes;
      }
      RK_TRY(rk_preprocess(e->app, e->staging, pbytes, m, e->arena, e->slot_stride, slots.data(), e->stream));
    } else {
      const char* src = static_cast<const char*>(d_parsed) + base * parsed_stride;
      RK_TRY(rk_preprocess(e->app, src, parsed_stride, m, e->arena, e->slot_stride, slots.data(), e->stream));
    }
    e->stats.loads += m;
  }
  RK_CUDA(cudaStreamSynchronize(e->stream));
  return RK_OK;
}

rk_status rk_engine_load_home(rk_engine* e, const void* h_parsed, const void* d_parsed, size_t parsed_stride) {
  if (!e) return set_error(RK_ERR_VALUE, "null engine");
  const int32_t n = e->app->p.n;
  const int32_t count = n > e->p.rank ? (n - e->p.rank + e->p.world - 1) / e->p.world : 0;
  return rk_engine_load_home_range(e, h_parsed, d_parsed, parsed_stride, 0, count);
}

rk_status rk_engine_peer_bandwidth(rk_engine* e, int32_t src_rank, size_t bytes, double* gb_per_s) {
  if (!e || !gb_per_s) return set_error(RK_ERR_VALUE, "null argument");
  if (!e->peers_ready || src_rank < 0 || src_rank >= e->p.world) return set_error(RK_ERR_VALUE, "peer tier not connected");
  RK_CUDA(cudaSetDevice(e->device));
  const size_t cap = std::min((size_t)e->home_slots, (size_t)e->p.device_slots) * e->slot_stride;
  bytes = std::min(bytes, cap);
  cudaEvent_t a, b;
  RK_CUDA(cudaEventCreate(&a));
  RK_CUDA(cudaEventCreate(&b));
  RK_CUDA(cudaEventRecord(a, e->lstream));
  // the copies the run issues: slot-sized pieces (PCE / CV / GMM peer fetches), or
  // one block (the NCC Gram's sub-block fetch) when the app is NCC
  if (e->app->p.kind == RK_APP_NCC) {
    RK_TRY(peer_copy(e->arena, e->peer_home[src_rank], bytes, e->lstream));
  } else {
    for (size_t off = 0; off < bytes; off += e->slot_stride)
      RK_CUDA(cudaMemcpyAsync(static_cast<char*>(e->arena) + off, e->peer_home[src_rank] + off,
                              std::min(e->slot_stride, bytes - off), cudaMemcpyDeviceToDevice, e->lstream));
  }
  RK_CUDA(cudaEventRecord(b, e->lstream));
  RK_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  RK_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *gb_per_s = ms > 0.f ? (double)bytes / (ms * 1e-3) / 1e9 : 0.0;
  return RK_OK;
}

rk_status rk_engine_queue_word(const rk_engine* e, void** d_word) {
  if (!e || !d_word) return set_error(RK_ERR_VALUE, "null argument");
  *d_word = e->qword;
  return RK_OK;
}

rk_status rk_engine_queue_reset(rk_engine* e) {
  if (!e) return set_error(RK_ERR_VALUE, "null engine");
  RK_CUDA(cudaSetDevice(e->device));
  const auto rr = rank_range(quadtree_leaves(e->app->p.n, e->p.leaf_block), e->p.rank, e->p.world);
  unsigned long long tmp = 0;
  RK_TRY(queue_call(e, e->qword, 3, ((unsigned long long)rr.first << 32) | (unsigned)rr.second, &tmp));
  e->queue_armed = true;
  return RK_OK;
}

rk_status rk_engine_set_peer_queues(rk_engine* e, int32_t world, void* const* d_words) {
  if (!e || !d_words) return set_error(RK_ERR_VALUE, "null argument");
  if (world != e->p.world) return set_error(RK_ERR_VALUE, "work queue world mismatch");
  e->peer_q.assign(world, nullptr);
  for (int r = 0; r < world; ++r) e->peer_q[r] = static_cast<unsigned long long*>(d_words[r]);
  e->queues_ready = true;
  return RK_OK;
}

rk_status rk_engine_set_peer_homes(rk_engine* e, int32_t world, void* const* d_home_bases) {
  if (!e || !d_home_bases) return set_error(RK_ERR_VALUE, "null argument");
  if (world != e->p.world || e->home_slots == 0) return set_error(RK_ERR_VALUE, "peer tier world mismatch");
  e->peer_home.assign(world, nullptr);
  for (int r = 0; r < world; ++r) e->peer_home[r] = static_cast<const char*>(d_home_bases[r]);
  e->peers_ready = true;
  return RK_OK;
}

rk_status rk_ipc_handle(const void* d_ptr, uint8_t* out_handle64) {
  if (!d_ptr || !out_handle64) return set_error(RK_ERR_VALUE, "null argument");
  cudaIpcMemHandle_t h;
  RK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(out_handle64, &h, 64);
  return RK_OK;
}

rk_status rk_ipc_open(const uint8_t* handle64, int device, void** d_ptr) {
  if (!handle64 || !d_ptr) return set_error(RK_ERR_VALUE, "null argument");
  RK_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  RK_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RK_OK;
}

rk_status rk_ipc_close(void* d_ptr) {
  RK_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return RK_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Test/inspection surface of the runtime's host-side structures.
struct rk_tier {
  rk::SlotTier t;
  explicit rk_tier(int cap) : t(cap) {}
};

extern "C" {

rk_status rk_tier_create(int32_t capacity, rk_tier** out) {
  if (!out) return set_error(RK_ERR_VALUE, "null argument");
  if (capacity < 1) return set_error(RK_ERR_VALUE, "capacity must be >= 1 slot");
  *out = new rk_tier(capacity);
  return RK_OK;
}

void rk_tier_destroy(rk_tier* t) { delete t; }

rk_status rk_tier_acquire(rk_tier* t, int32_t key, int32_t* kind, int32_t* slot) {
  if (!t || !kind || !slot) return set_error(RK_ERR_VALUE, "null argument");
  const TierResult r = t->t.acquire(key);
  if (r.kind == kNoEvictable)
    return set_error(RK_ERR_NO_EVICTABLE, "all %d slots are pinned", t->t.capacity);
  *kind = r.kind;
  *slot = r.slot;
  return RK_OK;
}

static rk_status tier_slot_ok(const rk_tier* t, int32_t slot, uint8_t state) {
  if (!t) return set_error(RK_ERR_VALUE, "null tier");
  if (slot < 0 || slot >= t->t.capacity) return set_error(RK_ERR_VALUE, "slot %d out of range", slot);
  if (t->t.state[slot] != state) return set_error(RK_ERR_VALUE, "slot %d in wrong state", slot);
  return RK_OK;
}

rk_status rk_tier_publish(rk_tier* t, int32_t slot, int32_t retain) {
  RK_TRY(tier_slot_ok(t, slot, kWrite));
  t->t.publish(slot, retain != 0);
  return RK_OK;
}

rk_status rk_tier_abort(rk_tier* t, int32_t slot) {
  RK_TRY(tier_slot_ok(t, slot, kWrite));
  t->t.abort(slot);
  return RK_OK;
}

rk_status rk_tier_release(rk_tier* t, int32_t slot) {
  RK_TRY(tier_slot_ok(t, slot, kRead));
  if (t->t.readers[slot] <= 0) return set_error(RK_ERR_VALUE, "double release of slot %d", slot);
  t->t.release(slot);
  return RK_OK;
}

rk_status rk_tier_stats(const rk_tier* t, int64_t* out5) {
  if (!t || !out5) return set_error(RK_ERR_VALUE, "null argument");
  out5[0] = t->t.hits;
  out5[1] = t->t.misses;
  out5[2] = t->t.waits;
  out5[3] = t->t.evictions;
  out5[4] = (int64_t)t->t.index.size();
  return RK_OK;
}

int32_t rk_tier_slot_key(const rk_tier* t, int32_t slot) {
  if (!t || slot < 0 || slot >= t->t.capacity) return -1;
  return t->t.key[slot];
}

int32_t rk_queue_step(uint64_t old, int32_t op, uint64_t arg, uint64_t* nw, uint64_t* got) {
  if (!nw || !got || op < 0 || op > 1) return -1;
  unsigned long long a = 0, b = 0;
  if (!queue_step(old, op, arg, &a, &b)) return 0;
  *nw = a;
  *got = b;
  return 1;
}

int64_t rk_leaves(int32_t n, int32_t leaf_block, int32_t rank, int32_t world, int32_t* out4, int64_t cap) {
  if (leaf_block < 1 || world < 1 || rank < 0 || rank >= world) return -1;
  const std::vector<Leaf> v = rank_share(quadtree_leaves(n, leaf_block), rank, world);
  for (int64_t k = 0; k < (int64_t)v.size() && k < cap; ++k) {
    out4[4 * k + 0] = v[k].r0;
    out4[4 * k + 1] = v[k].r1;
    out4[4 * k + 2] = v[k].c0;
    out4[4 * k + 3] = v[k].c1;
  }
  return (int64_t)v.size();
}

}  // extern "C"
