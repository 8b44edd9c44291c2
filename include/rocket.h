/*
 * rocket.h -- C ABI of librocket, the B200-native all-pairs compare engine.
 *
 * This is the drop-in boundary for the reference's plugin path: the
 * `allpairs.apps.Application` contract
 *   /root/reference/pkg/src/allpairs/apps.py:74-125
 * (path_for_key / fetch_raw / parse / preprocess / compare / postprocess)
 * and the packed upper-triangle result layout of
 *   PairLedger.pair_id  /root/reference/pkg/src/allpairs/scheduler.py:228-231
 *   completion record   /root/reference/pkg/src/allpairs/wire.py:120, :163-181
 *
 * Plain pointers and sizes only.  Device pointers are named d_*, host
 * pointers h_*.  Streams are cudaStream_t passed as void* (NULL = legacy
 * default stream).  Every entry point returns an rk_status; the message of
 * the last failure on the calling thread is available from rk_last_error().
 *
 * Ownership: slot arenas and output buffers belong to the caller; an rk_app
 * owns only its constant tables and scratch workspace.  Kernels borrow slot
 * memory for the stream-ordered duration of a call (the reference's ReadLease
 * contract, slotcache.py:42-59).  One rk_app may be used by one stream at a
 * time; create one app per stream for concurrency.
 */
#ifndef ROCKET_H
#define ROCKET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RK_ABI_VERSION 1

/* Status codes map 1:1 onto the reference's exception taxonomy
 * (/root/reference/pkg/src/allpairs/errors.py). */
typedef enum {
  RK_OK = 0,
  RK_ERR_VALUE = 1,         /* ValueError: i >= j, stage/shape mismatch (apps.py:69-71, :205-206, :335-336) */
  RK_ERR_MALFORMED = 2,     /* MalformedInput (errors.py:8-9; apps.py:293-298) */
  RK_ERR_SLOT_OVERFLOW = 3, /* SlotOverflow (errors.py:12-13; apps.py:128-132) */
  RK_ERR_NO_EVICTABLE = 4,  /* NoEvictableSlot (errors.py:16-20; slotcache.py:276-277) */
  RK_ERR_DEVICE = 5,        /* AppError: a CUDA call or kernel failed (errors.py:4-5) */
  RK_ERR_UNSUPPORTED = 6,   /* parameter combination not built for sm_100a in this library */
  RK_ERR_DUPLICATE = 7      /* AssertionError: a pair completed twice (PairLedger.mark, scheduler.py:233-241) */
} rk_status;

/* Application kinds.  SYNTHETIC and CV restate the reference's two built-in
 * apps (apps.py:154-227, :251-363); PCE / NCC / GMM are the paper's
 * forensics and microscopy comparisons, absent from the
 * reference and pinned by the oracle in /root/repo/oracle. */
typedef enum {
  RK_APP_SYNTHETIC = 0,
  RK_APP_CV = 1,
  RK_APP_PCE = 2,
  RK_APP_NCC = 3,
  RK_APP_GMM = 4
} rk_app_kind;

typedef struct {
  int32_t kind;          /* rk_app_kind */
  int32_t n;             /* item count; pair ids are dense over C(n,2) */
  int32_t height;        /* PCE/NCC: pattern rows */
  int32_t width;         /* PCE/NCC: pattern columns */
  uint64_t seed;         /* SYNTHETIC: value = mix64(seed, 0xC0403A3E, i, j) / 2^64 (apps.py:207) */
  double threshold;      /* postprocess: match = value >= threshold; NaN => match is None */
  int32_t max_entries;   /* CV: slot capacity in (u64 token, f64 freq) entries; GMM: max localizations */
  int32_t batch_pairs;   /* pairs per launch (PCE workspace sizing); 0 = default */
  int32_t gmm_angles;    /* GMM: rotation grid size; 0 = default */
  float gmm_scale;       /* GMM: Gaussian scale added to per-point sigma^2; 0 = default */
} rk_app_params;

/* One pair job.  slot_a/slot_b index the caller's slot arena; i < j are the
 * item keys; the result lands at out[pair_id(i, j)]. */
typedef struct {
  int32_t i;
  int32_t j;
  int32_t slot_a;
  int32_t slot_b;
} rk_pair;

typedef struct rk_app rk_app;

int rk_abi_version(void);
const char* rk_last_error(void);
const char* rk_status_name(int status);

/* pair_id(i, j) = i*(2n-i-1)/2 + (j-i-1); -1 when !(0 <= i < j < n).
 * Restates PairLedger.pair_id (scheduler.py:228-231). */
int64_t rk_pair_id(int64_t n, int64_t i, int64_t j);
/* Inverse of rk_pair_id; returns RK_ERR_VALUE when pid is out of range. */
rk_status rk_pair_from_id(int64_t n, int64_t pid, int64_t* i, int64_t* j);

rk_status rk_app_create(const rk_app_params* params, int device, rk_app** out);
void rk_app_destroy(rk_app* app);
/* Bytes of one preprocessed item in its device slot (Application.slot_size). */
size_t rk_app_slot_bytes(const rk_app* app);
/* Bytes of one parsed item as handed to rk_preprocess. */
size_t rk_app_parsed_bytes(const rk_app* app);
/* Slots are interleaved in groups of this many (1 = every slot contiguous).  NCC
 * uses 128: group g's 128 slots share the region [g*128*stride, (g+1)*128*stride)
 * as [D/1024][128][1024] floats, so one TMA box (128 items x 32 floats) spans
 * 512 KiB instead of 128 pages.  Arenas must hold a multiple of this many slots. */
int32_t rk_app_slot_group(const rk_app* app);

/* Application.preprocess for a batch of items already resident on the device
 * (replaces apps.py:304-318 and the gpu-lane preprocess at engine.py:464-472).
 * d_parsed: n_items parsed items, parsed_stride bytes apart.
 * Item k is written to d_slots + h_slot_idx[k]*slot_stride. */
rk_status rk_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items,
                        void* d_slots, size_t slot_stride, const int32_t* h_slot_idx,
                        void* stream);

/* Application.compare + postprocess for a batch of pairs (replaces apps.py:201-208,
 * :331-358 and the compare dispatch at engine.py:519-548).  Writes
 * d_out[pair_id] (f64) and, if d_flags != NULL, d_flags[pair_id] with the wire
 * encoding of PairResult.match: 0 = None, 1 = False, 3 = True (wire.py:165-167). */
rk_status rk_compare_pairs(rk_app* app, const void* d_slots, size_t slot_stride,
                           const rk_pair* h_pairs, int n_pairs,
                           double* d_out, uint8_t* d_flags, void* stream);

/* Quadtree leaf: all pairs (i, j) with i in rows, j in cols and i < j, enumerated
 * row-major like Region.pairs (scheduler.py:45-48).  h_row_slots/h_col_slots give
 * the slot of each key. */
rk_status rk_compare_tile(rk_app* app, const void* d_slots, size_t slot_stride,
                          int32_t r0, int32_t r1, int32_t c0, int32_t c1,
                          const int32_t* h_slot_of_key,
                          double* d_out, uint8_t* d_flags, void* stream);

/* NCC all-pairs as a tcgen05 Gram GEMM (kind::tf32, 128x128 item tiles, TMEM
 * accumulators, TMA pipeline) over a slot arena where item k lives in slot k
 * (n_rows >= n slots).  Upper-triangle tiles t with t % world == rank are
 * computed; results go to d_out[pair_id].  TF32 bound: |error| <= 2e-4. */
rk_status rk_ncc_gram(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t rank,
                      int32_t world, double* d_out, uint8_t* d_flags, void* stream);

/* One block of the NCC Gram over an arena that holds only some items (C3-sized
 * jobs): A = slots a_row0 .. a_row0+a_cnt-1 holding keys a_key0 .., B likewise;
 * the same block twice computes its upper triangle, distinct blocks (disjoint
 * key ranges) all their pairs.  Rows start on slot groups (multiples of 128). */
rk_status rk_ncc_gram_block(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t a_row0,
                            int32_t a_key0, int32_t a_cnt, int32_t b_row0, int32_t b_key0, int32_t b_cnt,
                            double* d_out, uint8_t* d_flags, void* stream);

/* Deterministic synthetic inputs (test/bench data generators, not the hot path). */
/* PRNU-like patterns: item k = 0.2*K[k % cameras] + N(0,1), fp32, h*w each. */
rk_status rk_synth_prnu(int32_t h, int32_t w, int32_t first_key, int32_t n_items, int32_t cameras,
                        uint64_t seed, float* d_out, void* stream);

/* ---------------------------------------------------------------------------
 * All-pairs engine: quadtree tiling (scheduler.py:20-117) over a device slot
 * table with LRU eviction (slotcache.py:139-282), fed from a pinned host
 * tier of parsed items with async H2D + preprocess (engine.py:436-508).
 * ------------------------------------------------------------------------- */
typedef struct rk_engine rk_engine;

typedef struct {
  int32_t leaf_block;      /* quadtree leaf side (config.py:73 default 8) */
  int32_t device_slots;    /* device tier capacity in slots */
  int32_t streams;         /* compare streams (each owns an rk_app workspace) */
  int32_t rank;            /* this rank's share of the leaves ... */
  int32_t world;           /* ... out of world (contiguous, pair-balanced DFS blocks of leaves) */
  int32_t peer_tier;       /* world > 1: items live on their home GPU (k mod world), others fetch them over NVLink */
  int32_t steal;           /* world > 1: dynamic leaf chunks + cross-GPU stealing through device atomics */
  int32_t steal_chunk;     /* leaves per grab (0: one compare batch worth) */
  int32_t host_slots;      /* host (L2) tier of preprocessed items in pinned memory, write-through
                              (engine.py:375-394, :482-508); 0 = none.  Single-GPU runs only: with the
                              peer tier the home GPU is the next level (distcache.py owner_of) */
} rk_engine_params;

typedef struct {
  int64_t pairs_done;
  int64_t loads;           /* fresh preprocess executions (engine.py:443-448) */
  int64_t hits;            /* device tier hits   (slotcache.py:166-170) */
  int64_t misses;          /* device tier misses (slotcache.py:178-186) */
  int64_t evictions;
  int64_t tiles;
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int64_t kernel_launches;
  int64_t peer_fetches;    /* items copied from a peer GPU's home region (the remote tier, distcache.py) */
  int64_t peer_bytes;
  int64_t steals;          /* chunks this rank stole from other ranks' queues */
  int64_t pinned_at_end;   /* device slots still leased when the run returned (must be 0) */
  int64_t writing_at_end;  /* device slots still in WRITE when the run returned (must be 0) */
  int64_t ledger_marked;   /* pair ids set in the engine's own ledger after the run (-1: ledger shared, see rk_engine_ledger) */
  int64_t dup_marks;       /* duplicate completions seen by the engine's own ledger */
  int64_t host_hits;       /* host tier (slotcache.py:166-170): device misses served from pinned host slots */
  int64_t host_misses;     /* host tier misses (fresh loads, written through to the host tier) */
  int64_t host_evictions;
} rk_engine_stats;

rk_status rk_engine_create(const rk_app_params* app_params, const rk_engine_params* params,
                           int device, rk_engine** out);
void rk_engine_destroy(rk_engine* eng);
/* Run every pair assigned to this rank.  Parsed items come from host memory
 * (h_parsed, parsed_stride apart, pinned for async copies) or, when h_parsed is
 * NULL, from device memory d_parsed.  Results go to d_out/d_flags (device,
 * C(n,2) entries).  Synchronous on return. */
rk_status rk_engine_run(rk_engine* eng, const void* h_parsed, const void* d_parsed,
                        size_t parsed_stride, double* d_out, uint8_t* d_flags);
rk_status rk_engine_stats_get(const rk_engine* eng, rk_engine_stats* out);
rk_status rk_engine_reset_stats(rk_engine* eng);

/* Peer-GPU cache tier (the point-of-contact rule owner_of(k) = k mod p,
 * distcache.py:19-23, collapsed to one NVLink hop).  Each rank preprocesses its
 * home items (k % world == rank) into the home region of its slot arena
 * (item k at slot device_slots + k / world); the caller exchanges the home
 * regions with rk_ipc_handle / rk_ipc_open and a barrier, then
 * rk_engine_set_peer_homes; rk_engine_run copies every non-home item it needs
 * device-to-device from its home GPU instead of reloading it from the host. */
rk_status rk_engine_home_region(const rk_engine* eng, void** d_base, size_t* bytes);
rk_status rk_engine_arena(const rk_engine* eng, void** d_base, size_t* slot_stride);
/* Home item m (key = rank + m*world) is read at parsed + m*parsed_stride. */
rk_status rk_engine_load_home(rk_engine* eng, const void* h_parsed, const void* d_parsed, size_t parsed_stride);
/* The same for home items m0 .. m0+count-1 only (item m0 + q at parsed + q * parsed_stride),
 * so a home region larger than the free HBM can be filled chunk by chunk. */
rk_status rk_engine_load_home_range(rk_engine* eng, const void* h_parsed, const void* d_parsed, size_t parsed_stride,
                                    int32_t m0, int32_t count);
rk_status rk_engine_set_peer_homes(rk_engine* eng, int32_t world, void* const* d_home_bases);
/* CUDA IPC of a device allocation (64-byte handle) for the peer tier. */
/* Cross-GPU work queue (hierarchical stealing, engine.py:274-309 and
 * scheduler.py:126-157 for the GPUs of one box).  Each rank's 64-bit queue word
 * (head << 32 | tail over the global depth-first leaf list) lives in device
 * memory at the tail of its slot arena (rk_engine_arena's allocation, so the
 * home-region IPC handle maps it too).  Before every run with steal != 0:
 * rk_engine_queue_reset on every rank (own word <- its contiguous share), a
 * barrier, then rk_engine_run.  rk_engine_set_peer_queues takes every rank's
 * mapped word (own entry = local) once after the IPC exchange. */
/* Peer-tier copy bandwidth: `bytes` from rank src_rank's home region into this
 * rank's cache slots with the run's own D2D copies (NVLink), GB/s.  Clobbers
 * the cache slots: call between runs only. */
rk_status rk_engine_peer_bandwidth(rk_engine* eng, int32_t src_rank, size_t bytes, double* gb_per_s);
rk_status rk_engine_queue_word(const rk_engine* eng, void** d_word);
rk_status rk_engine_queue_reset(rk_engine* eng);
rk_status rk_engine_set_peer_queues(rk_engine* eng, int32_t world, void* const* d_words);

/* Plain device buffers for arenas shared over CUDA IPC (the handle of a cudaMalloc
 * base pointer) and a stream-ordered device-to-device (or peer, over NVLink) copy. */
rk_status rk_device_alloc(size_t bytes, int device, void** d_ptr);
rk_status rk_device_free(void* d_ptr);
rk_status rk_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);

rk_status rk_ipc_handle(const void* d_ptr, uint8_t* out_handle64);
rk_status rk_ipc_open(const uint8_t* handle64, int device, void** d_ptr);
rk_status rk_ipc_close(void* d_ptr);
/* Exactly-once ledger (PairLedger, scheduler.py:218-246): a C(n,2)-bit bitmap in
 * device memory, set by every compare epilogue with a system-scope atomicOr.  A
 * bit found already set counts a duplicate, and the run fails with
 * RK_ERR_DUPLICATE (the reference's AssertionError "pair (i, j) completed
 * twice"); `completed == total` is the reference's `full`.
 * Single GPU: the engine's own ledger, cleared at the start of every run.
 * Multi-GPU: rank 0's ledger is the job's (its region of the IPC-shared arena);
 * every rank passes rank 0's mapped region to rk_engine_use_ledger once, rank 0
 * calls rk_engine_ledger_reset before the pre-run barrier and reads
 * rk_engine_ledger after the post-run barrier. */
typedef struct {
  int64_t total;           /* C(n,2) */
  int64_t completed;       /* bits set */
  int64_t dup_marks;       /* duplicate completions */
  int64_t first_dup_pid;   /* first duplicate pair id, -1 if none */
  int32_t full;            /* completed == total && dup_marks == 0 */
  int32_t shared;          /* marks go to a (possibly remote) shared ledger */
} rk_ledger_stats;
/* Offset and size of this engine's ledger region inside its arena allocation
 * (the allocation rk_engine_arena returns and rk_ipc_handle exports). */
rk_status rk_engine_ledger_region(const rk_engine* eng, size_t* offset, size_t* bytes);
/* Mark into the ledger region at d_region (own or a peer's mapped one) from now on. */
rk_status rk_engine_use_ledger(rk_engine* eng, void* d_region);
rk_status rk_engine_ledger_reset(rk_engine* eng);
rk_status rk_engine_ledger(rk_engine* eng, rk_ledger_stats* out);
/* Ledger for callers of rk_compare_pairs / rk_compare_tile without an engine:
 * d_region of rk_ledger_bytes(n) bytes, zeroed by the caller; NULL turns it off. */
size_t rk_ledger_bytes(int64_t n);
rk_status rk_app_set_ledger(rk_app* app, void* d_region);
rk_status rk_ledger_read(void* d_region, int64_t n, rk_ledger_stats* out);

/* Sample CUDA-event timing of every `every`-th compare batch (0 = off), at most
 * max_samples per run, on the engine's stream. */
rk_status rk_engine_set_profiling(rk_engine* eng, int every, int max_samples);

/* Trace events of the last run (the reference's metrics.py TraceEvent, one per
 * compare batch on the gpu lane and per load / peer-fetch group on the up lane),
 * device timestamps in ns from the start of the run.  max_events = 0 disables. */
typedef struct {
  int32_t lane;      /* 0: compare batch, 1: load (H2D + preprocess), 2: peer fetch */
  int32_t i;         /* first pair's i (compare) or first key loaded */
  int32_t j;         /* first pair's j, or -1 */
  int32_t count;     /* pairs in the batch, or items */
  int64_t start_ns;
  int64_t end_ns;
} rk_trace_event;
rk_status rk_engine_set_trace(rk_engine* eng, int32_t max_events);
/* Copies up to cap events to out (may be NULL) and returns how many were recorded. */
int64_t rk_engine_trace_get(const rk_engine* eng, rk_trace_event* out, int64_t cap);
/* Summed device time, count and pair total of the sampled compare launches of the last run. */
rk_status rk_engine_kernel_time(const rk_engine* eng, double* ms_total, int64_t* samples, int64_t* pairs);
/* The engine's cudaStream_t (for callers that order their own work after a run). */
void* rk_engine_stream(const rk_engine* eng);

/* ---------------------------------------------------------------------------
 * Host-side runtime structures, exported for inspection and parity tests.
 * ------------------------------------------------------------------------- */
/* Slot tier: the CacheTier policy (slotcache.py:139-282) the engine runs on its
 * device slot arena.  acquire -> *kind 0 = Hit (reader pinned), 1 = MustWait,
 * 2 = Miss (slot claimed for writing, LRU victim evicted if needed);
 * RK_ERR_NO_EVICTABLE when every slot is pinned. */
typedef struct rk_tier rk_tier;
rk_status rk_tier_create(int32_t capacity, rk_tier** out);
void rk_tier_destroy(rk_tier* tier);
rk_status rk_tier_acquire(rk_tier* tier, int32_t key, int32_t* kind, int32_t* slot);
rk_status rk_tier_publish(rk_tier* tier, int32_t slot, int32_t retain);
rk_status rk_tier_abort(rk_tier* tier, int32_t slot);
rk_status rk_tier_release(rk_tier* tier, int32_t slot);
/* out5 = {hits, misses, waits, evictions, occupancy} (snapshot_stats, slotcache.py:252-260) */
rk_status rk_tier_stats(const rk_tier* tier, int64_t* out5);
int32_t rk_tier_slot_key(const rk_tier* tier, int32_t slot);
/* One work-queue transition on a word value (head << 32 | tail): op 0 = the owner
 * takes up to `arg` leaves from the head, op 1 = a thief takes the back half when
 * at least `arg` leaves remain on each side.  Returns 1 with the new word and the
 * taken range (same encoding), 0 when nothing can be taken, -1 on bad arguments.
 * The device queue applies exactly this transition under atomicCAS_system. */
int32_t rk_queue_step(uint64_t old_word, int32_t op, uint64_t arg, uint64_t* new_word, uint64_t* taken);
/* Depth-first quadtree leaves (iter_leaves, scheduler.py:78-86) of this rank's
 * share; writes min(count, cap) leaves as (r0, r1, c0, c1) and returns count. */
int64_t rk_leaves(int32_t n, int32_t leaf_block, int32_t rank, int32_t world, int32_t* out4, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* ROCKET_H */
