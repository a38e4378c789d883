/*
 * tangram.h — C-ABI of the B200-native Tangram model-loading hot path.
 *
 * Drop-in boundary for the reference's C++ pool / loader API
 * (/root/reference/proj/include/warmsim).  Every entry point names the
 * reference member it replaces; argument meaning, ordering rules and error
 * behaviour are the reference's.  Plain pointers and sizes only; the library
 * is libtangram.so (paper_2512_01357_b200/libtangram.so), no torch types.
 *
 * Return codes: 0 = ok; 1..10 = warmsim::Error ordinal + 1
 * (types.hpp:155-166: InsufficientMemory=1, PoolExhausted=2, Infeasible=3,
 * Pinned=4, NotFound=5, OverlapMove=6, DestinationOccupied=7,
 * OrderingError=8, InstanceTooLarge=9, InvalidArgument=10); >= 100 are
 * runtime errors of this implementation (TG_ERR_*).  A tg_load_model that
 * fails with a domain error (1..10) or for want of a byte source
 * (TG_ERR_NO_SOURCE: no registered source, a missing or short checkpoint
 * file) leaves the pool unchanged (reuse_store.hpp:117-119).  A runtime
 * failure once bytes move (TG_ERR_CUDA, a short read of a file that shrank,
 * TG_ERR_VERIFY: bytes that fail their fingerprint with nothing to repair
 * them) keeps the reference's decision in the pool — the outcome is still
 * written, with suspect_tensors > 0 — and leaves every tensor whose bytes it
 * could not verify *suspect*: never exported to peers or used as a source,
 * verified and re-sent from its source on its next reuse.  A failed batch
 * KV allocation leaves engine and pool unchanged (kv_engine.hpp:104-106).
 * Thread-safety: single writer per pool, like the reference
 * (reuse_store.hpp:4-6).
 */
#ifndef TANGRAM_H
#define TANGRAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_OK 0
#define TG_ERR_CUDA 100
#define TG_ERR_NO_DEVICE 101      /* data-plane call on a control-plane-only pool / no GPU */
#define TG_ERR_NO_SOURCE 102      /* a miss has no registered host (or peer) source */
#define TG_ERR_BUFFER 103         /* caller buffer too small; *needed says how big */
#define TG_ERR_BAD_ARG 104        /* null handle / malformed argument */
#define TG_ERR_VERIFY 105         /* reused bytes fail their fingerprint and cannot be repaired */
#define TG_ERR_INTERNAL 106
#define TG_ERR_KV_ARMED 107       /* pool layout / host KV call while an engine is armed (tg_kv_device_sync first) */
#define TG_ERR_KV_LOG 108         /* the device batch log overflowed between arm and sync: batches were dropped */

#define TG_POOL_NO_DEVICE (-1)    /* device argument: control plane only, moves no bytes */

/* tg_load_policy.flags */
#define TG_LOAD_VERIFY_REUSE 1u    /* fingerprint reused tensors, compare to the recorded digest */
#define TG_LOAD_FINGERPRINT_NEW 2u /* fingerprint placed tensors, record the digest */
#define TG_LOAD_PEER 4u            /* pull misses resident on a peer pool over NVLink */
#define TG_LOAD_FUSED 8u           /* one load-kernel launch (move + fingerprint in one pass) instead of K3 waves then K1 */
#define TG_LOAD_ASYNC 16u           /* return once the decision is committed and the data plane enqueued;
                                       the wait and the digest bookkeeping run at the pool's next operation
                                       (or tg_pool_sync), so loads on different pools / GPUs overlap */
#define TG_LOAD_DEFAULT 11u
/* flags carrying this bit are taken literally: TG_LOAD_EXPLICIT alone asks for
 * no optional work (flags == 0 without it means TG_LOAD_DEFAULT) */
#define TG_LOAD_EXPLICIT 0x80000000u

typedef struct tg_pool tg_pool;
typedef struct tg_stats tg_stats;
typedef struct tg_kv tg_kv;
typedef struct tg_rng tg_rng;
typedef struct tg_model tg_model;
typedef struct tg_snapshot tg_snapshot;

typedef struct { uint64_t hi, lo; } tg_tensor_id; /* warmsim::TensorId (types.hpp:46-60) */
typedef struct { uint64_t hi, lo; } tg_digest;    /* tgfp1 content fingerprint */

/* warmsim::GpuSpec (model.hpp:39-45) */
typedef struct {
    const char* gpu_id;
    uint64_t pool_size;
    double pcie_bandwidth;
    double intra_copy_bandwidth;
    double store_bandwidth;
} tg_gpu_spec;

/* warmsim::TensorSpec (model.hpp:17-22); model_id defaults to the model's */
typedef struct {
    tg_tensor_id id;
    const char* name;
    uint64_t size;
    const char* model_id; /* nullable */
} tg_tensor_spec;

/* warmsim::ModelSpec (model.hpp:30-37); tensors ordered by name */
typedef struct {
    const char* model_id;
    const tg_tensor_spec* tensors;
    uint32_t n_tensors;
    uint64_t total_size;
    double latency_sensitivity;
    int32_t location; /* 0 model_cache, 1 model_store */
    uint64_t bytes_per_token;
} tg_model_spec;

/* warmsim::LoadPolicy (reuse_store.hpp:43-48) + data-plane flags */
typedef struct {
    int32_t merge;          /* 0 PartitionedGain, 1 GlobalMerge (packing.hpp:125) */
    int32_t strictness;     /* 0 Functional, 1 LiteralGuard (packing.hpp:92) */
    int32_t random_eviction;
    tg_rng* rng;            /* required for random eviction (or the callback below) */
    uint32_t flags;         /* TG_LOAD_* ; 0 means TG_LOAD_DEFAULT */
    /* alternative to rng: the caller's own stream, uniform in [0, n) */
    uint64_t (*uniform_below)(void* ctx, uint64_t n);
    void* rng_ctx;
} tg_load_policy;

/* warmsim::LoadOutcome (reuse_store.hpp:34-41) summary + measured data plane */
typedef struct {
    uint32_t n_hits, n_misses, n_evictions, n_relocations, n_placements, n_waves;
    uint64_t fallback_evictions;
    uint64_t bytes_transferred, bytes_merged;
    double eviction_cost_total;
    uint64_t total_merge_cost, pgp_merge_cost, initial_merge_cost;
    double total_eviction_cost;
    /* data plane (device pools) */
    uint64_t pcie_bytes, peer_bytes, device_src_bytes, fingerprint_bytes, repaired_bytes;
    uint32_t verify_mismatches, expected_mismatches;
    /* relocate_ms: fused, the load kernel's span — with the verification split (at most three waves), from the
     * first start to the last end of the load kernel and its concurrent K1 launch; unfused, the K3 waves */
    double plan_us, total_ms, relocate_ms, h2d_ms, peer_ms, fp_kernel_ms, fp_reuse_ms, fp_reuse_max_ms;
    /* host side of the call: entry -> all device work enqueued, waiting for it, entry -> return */
    double host_issue_us, host_wait_us, host_total_us;
    /* tensors of the model left suspect (bytes unverified); 0 after a successful load */
    uint32_t suspect_tensors, reserved0;
    /* device timeline from entry: the load kernel / last relocation wave ends; the first H2D placement
     * gated on a relocation wave may start (0 when there is none) */
    double kernel_end_ms, gated_h2d_start_ms;
} tg_load_outcome;

/* warmsim::EvictionCandidate (packing.hpp:32-38); model_id valid until the next call on the pool */
typedef struct {
    tg_tensor_id tensor;
    uint64_t size;
    double cost;
    double last_access;
    const char* model_id;
} tg_eviction;

/* warmsim::Relocation (packing.hpp:216-221) + its WAR wave */
typedef struct {
    tg_tensor_id tensor;
    uint64_t from, to, size;
    uint32_t wave;
} tg_relocation;

/* warmsim::Placement (packing.hpp:223-226) + byte source */
typedef struct {
    tg_tensor_id tensor;
    uint64_t offset, size;
    uint32_t source; /* 0 host/PCIe, 1 peer pool/NVLink, 2 device-resident source (HBM),
                        3 re-shard: assembled over NVLink from peer shards of another layout */
} tg_placement;

/* warmsim::Region (region_pool.hpp:22-28) */
typedef struct {
    uint64_t offset, size;
    int32_t kind; /* 0 free, 1 tensor, 2 kv_block */
    tg_tensor_id tensor;
    uint64_t block_id;
} tg_region;

/* ReuseStore accessors (reuse_store.hpp:56-74) */
typedef struct {
    uint64_t pool_size, free_bytes, kv_bytes, pinned_tensor_bytes, pinned_bytes, reusable_bytes;
    uint64_t bytes_merged_total, bytes_transferred_total, evictions_total;
    uint64_t region_count, extent_count, tensor_count, largest_free;
    int32_t device;
    void* arena;
    /* data plane totals since creation (device pools) */
    uint64_t loads;
    double data_plane_ms;
    uint64_t pcie_bytes, peer_bytes, device_src_bytes, fingerprint_bytes, relocated_bytes;
    uint64_t epoch; /* changes whenever the tensor map does (unique process-wide) */
    /* integrity totals: reused / peer bytes that failed their fingerprint, bytes
     * re-sent to repair them, loads that ended with a runtime error */
    uint64_t verify_mismatches, repaired_bytes, failed_loads;
} tg_pool_info;

/* ReuseStore::tensor_map() entry (reuse_store.hpp:26-32); model_id valid while the pool is unchanged */
typedef struct {
    tg_tensor_id id;
    uint64_t offset, size;
    double last_access;
    int32_t pinned, suspect;
    const char* model_id;
} tg_tensor_entry;

typedef struct {
    uint64_t offset, size;
    double last_access;
    int32_t pinned, has_digest; /* has_digest: `digest` is the content truth (source / manifest / peer digest) */
    tg_digest digest;
    void* device_ptr;
    int32_t suspect, reserved0; /* resident bytes not known to equal the content (see tg_load_model) */
} tg_tensor_info;

/* warmsim::KvAllocStats (kv_engine.hpp:33-39) + engine state */
typedef struct {
    uint64_t pool_invocations, alloc_batches, blocks_from_free_list, blocks_from_pool, reclaim_events;
    uint64_t free_list_size, active_requests, next_pbn, block_bytes;
} tg_kv_stats;

/* ---- library ------------------------------------------------------------- */
int tg_version(void);
const char* tg_error_string(int code);
const char* tg_last_error_detail(void); /* thread-local detail of the last failure */
int tg_device_count(int* n);
uint64_t tg_kernel_launches(void); /* kernels launched by this library so far */

/* ---- ids, catalog (types.hpp:131-146, catalog.hpp:37-90) ------------------- */
int tg_murmur3_x64_128(const void* data, uint64_t len, uint64_t seed, tg_digest* out);
int tg_tensor_key(const char* model_id, const char* name, const int64_t* shape, int32_t ndim, int32_t dtype,
                  tg_tensor_id* out);
int tg_model_make(const char* model_id, uint64_t total_size, int32_t layers, uint64_t bytes_per_token,
                  int32_t location, double latency_sensitivity, tg_model** out);
int tg_model_default_catalog(uint32_t index, tg_model** out); /* index < tg_model_catalog_size() */
uint32_t tg_model_catalog_size(void);
void tg_model_destroy(tg_model* m);
int tg_model_view(const tg_model* m, tg_model_spec* out); /* pointers valid while m lives */
int tg_model_shard(const tg_model* m, uint32_t rank, uint32_t world, tg_model** out); /* §8(e) tensor shards */

/* ---- request shares (ModelStatsTable, model.hpp:70-133) -------------------- */
int tg_stats_create(double decay, tg_stats** out);
/* Statistics owned by the caller (e.g. the reference's ModelStatsTable behind
 * the C++ facade): p_m and b_m are read through callbacks when eviction costs
 * are computed (reuse_store.hpp:104-105).  record_* calls do not apply. */
int tg_stats_create_external(void* ctx, double (*miss_probability)(void* ctx, const char* model_id),
                             double (*load_bandwidth_or)(void* ctx, const char* model_id, double fallback),
                             tg_stats** out);
void tg_stats_destroy(tg_stats* s);
int tg_stats_record_request(tg_stats* s, const char* model_id, double t);
int tg_stats_record_eviction(tg_stats* s, const char* model_id, double t);
int tg_stats_set_load_bandwidth(tg_stats* s, const char* model_id, double bw);
double tg_stats_miss_probability(const tg_stats* s, const char* model_id);

int tg_rng_create(uint64_t seed, tg_rng** out); /* warmsim::Rng (rng.hpp:18-73) */
void tg_rng_destroy(tg_rng* r);
uint64_t tg_rng_uniform_below(tg_rng* r, uint64_t n);

/* ---- pool (ReuseStore, reuse_store.hpp:50-345) ------------------------------ */
int tg_pool_create(const tg_gpu_spec* gpu, int32_t device, tg_pool** out); /* ReuseStore(GpuSpec) :54 */
void tg_pool_destroy(tg_pool* p);
/* Value semantics (reuse_store.hpp:336-344; the reference copies stores for
 * rollback, kv_engine.hpp:146-158).  tg_pool_clone: an independent
 * control-plane pool with p's metadata (decisions identical, no arena).
 * tg_pool_assign: dst takes src's metadata; dst keeps its arena, and a tensor
 * keeps its verified bytes only where dst already held it at the same offset,
 * otherwise it is suspect in dst (re-sent on its next reuse). */
int tg_pool_clone(const tg_pool* p, tg_pool** out);
int tg_pool_assign(tg_pool* dst, const tg_pool* src);
int tg_pool_tensors(const tg_pool* p, tg_tensor_entry* buf, uint64_t cap, uint64_t* n); /* tensor_map() */
int tg_pool_info_get(const tg_pool* p, tg_pool_info* out);
int tg_pool_stream(const tg_pool* p, void** cuda_stream); /* stream every pool operation is ordered on */
int tg_set_model_alpha(tg_pool* p, const char* model_id, double alpha); /* :76 */

/* load_model (:120-174).  On success the plan arrays of this load can be read
 * with tg_last_* until the next mutating call on the pool. */
int tg_load_model(tg_pool* p, const tg_model_spec* m, const tg_stats* s, double clock, const tg_load_policy* pol,
                  tg_load_outcome* out);
uint32_t tg_last_hits(const tg_pool* p, tg_tensor_id* buf, uint32_t cap);
uint32_t tg_last_misses(const tg_pool* p, tg_tensor_id* buf, uint32_t cap);
uint32_t tg_last_evictions(const tg_pool* p, tg_eviction* buf, uint32_t cap);
uint32_t tg_last_relocations(const tg_pool* p, tg_relocation* buf, uint32_t cap);
uint32_t tg_last_placements(const tg_pool* p, tg_placement* buf, uint32_t cap);
uint32_t tg_last_digests(const tg_pool* p, tg_digest* buf, uint32_t cap); /* model order */

int tg_end_instance(tg_pool* p, const char* model_id);                     /* :177 */
int tg_evict_tensor(tg_pool* p, tg_tensor_id id);                          /* :186 */
int tg_evict_model(tg_pool* p, const char* model_id);                      /* :197 */
int tg_move_tensor(tg_pool* p, tg_tensor_id id, uint64_t new_offset);      /* :212 (+ K3 bytes) */
int tg_alloc_kv_region(tg_pool* p, uint64_t size, uint64_t block_id, uint64_t* offset); /* :224 */
int tg_free_kv_region(tg_pool* p, uint64_t offset);                        /* :230 */
int tg_lookup(const tg_pool* p, const tg_model_spec* m, uint8_t* hit_mask, uint64_t* reuse_size); /* :81 */
int tg_reuse_size(const tg_pool* p, const tg_model_spec* m, uint64_t* out); /* :92 */
int tg_peer_reuse_size(const tg_pool* p, const tg_model_spec* m, uint64_t* out); /* §8(e) extension */
int tg_eviction_candidates(tg_pool* p, const tg_stats* s, const char* exclude, tg_eviction* buf, uint32_t cap,
                           uint32_t* n); /* :99 */
int tg_validate(const tg_pool* p);                                         /* :238 */
int tg_dump(const tg_pool* p, char* buf, uint64_t cap, uint64_t* needed);  /* :270 (JSON) */
int tg_regions(const tg_pool* p, tg_region* buf, uint64_t cap, uint64_t* n); /* RegionList::snapshot */
int tg_tensor_info_get(const tg_pool* p, tg_tensor_id id, tg_tensor_info* out);
/* ---- device tensor index -------------------------------------
 * The pool's tensor map (ReuseStore::tensors_ reuse_store.hpp:338, TensorEntry
 * :26-32) mirrored in HBM as an open-addressing table for device-side
 * consumers: capacity a power of two >= 2 x entries (>= 1024), home slot
 * key.lo & (capacity - 1), linear probing, one 64-byte slot per probe.  Every
 * mutating call (load_model, end_instance, evict_*, move_tensor, restore)
 * re-publishes it on the pool stream; include/tangram_index.cuh probes it. */
typedef struct {
    uint64_t key_hi, key_lo;
    uint64_t offset, size;
    double last_access;
    uint64_t model; /* murmur3_x64_128(model id, seed 0).lo of the owning model */
    uint32_t flags; /* TG_INDEX_OCCUPIED | TG_INDEX_PINNED */
    uint32_t reserved0;
    uint64_t reserved1;
} tg_index_slot;
#define TG_INDEX_OCCUPIED 1u
#define TG_INDEX_PINNED 2u
typedef struct {
    uint64_t offset, size;
    uint32_t found, flags;
} tg_index_hit;
/* Host image of the table (any pool, device or not): writes min(capacity,
 * cap_slots) slots to buf (nullable) and the capacity to *capacity. */
int tg_pool_index_image(const tg_pool* p, tg_index_slot* buf, uint64_t cap_slots, uint64_t* capacity);
/* The published device table (device pools). */
int tg_pool_device_index(tg_pool* p, const tg_index_slot** table, uint64_t* capacity);
/* Batch lookup through the device table (one thread per key, K6), results to host. */
int tg_index_lookup(tg_pool* p, const tg_tensor_id* ids, uint32_t n, tg_index_hit* out);
int tg_fingerprint_tensor(tg_pool* p, tg_tensor_id id, tg_digest* out);    /* K1 over resident bytes */
int tg_pool_add_peer(tg_pool* p, tg_pool* peer);                           /* NVLink peer pool (K5) */
/* Peers in other processes (one process per GPU): export the
 * arena as a CUDA IPC handle plus the index of fingerprinted residents; a
 * peer attaches both and then pulls misses over NVLink (TG_LOAD_PEER).  The
 * pulled bytes are fingerprinted and checked against the index's digest; a
 * stale index falls back to the host source. */
typedef struct {
    tg_tensor_id id;
    uint64_t offset, size;
    tg_digest digest;
} tg_index_entry;
#define TG_IPC_HANDLE_BYTES 64
int tg_pool_export_ipc(const tg_pool* p, void* handle /* TG_IPC_HANDLE_BYTES */);
int tg_pool_index(const tg_pool* p, tg_index_entry* buf, uint64_t cap, uint64_t* n);
int tg_pool_attach_remote(tg_pool* p, const void* handle, const tg_index_entry* idx, uint64_t n, int32_t* peer_id);
int tg_pool_update_remote(tg_pool* p, int32_t peer_id, const tg_index_entry* idx, uint64_t n);
int tg_pool_snapshot(tg_pool* p, tg_snapshot** out);
int tg_pool_restore(tg_pool* p, const tg_snapshot* s);
void tg_snapshot_destroy(tg_snapshot* s);

/* ---- shard lineage (re-shard pulls) -----------------
 * tg_model_shard records, for every shard tensor, the byte range of its
 * parent tensor it holds.  A load with TG_LOAD_PEER whose miss has no exact
 * copy on a peer assembles it from resident shards of the same parent in any
 * other layout on peer pools (in-process peers or attached remote pools):
 * one NVLink piece per overlapping shard, then a fingerprint of the assembled
 * tensor (placement source 3).  tg_lineage_register declares the relation
 * for shards made elsewhere; tg_lineage_get reads it. */
int tg_lineage_register(tg_tensor_id child, tg_tensor_id parent, uint64_t begin, uint64_t size);
int tg_lineage_get(tg_tensor_id child, tg_tensor_id* parent, uint64_t* begin, uint64_t* size);

/* ---- host checkpoint sources (data side-channel) --------------
 * ptr may be pinned host memory (placed over PCIe by the copy engine) or
 * device memory, e.g. an HBM-resident model cache (placed by the K3 copy
 * kernel; source kind 2 in tg_placement). */
int tg_host_register(tg_tensor_id id, const void* ptr, uint64_t size, const tg_digest* expected /*nullable*/);
/* Model Store source (ModelLocation::ModelStore, model.hpp:24): the tensor's
 * bytes are `size` bytes at `file_offset` of a checkpoint file; loads stream
 * them file → pinned ring (reader threads) → HBM, overlapping storage reads
 * with PCIe. */
int tg_file_register(tg_tensor_id id, const char* path, uint64_t file_offset, uint64_t size,
                     const tg_digest* expected /*nullable*/);
int tg_host_unregister(tg_tensor_id id);
int tg_host_clear(void);
int tg_host_alloc(uint64_t size, void** out); /* pinned */
int tg_host_free(void* p);

/* ---- test failpoints ----------------------------------------------------------
 * Arm a named fault so that its nth hit from now fails the way the real fault
 * would; nth <= 0 disarms.  "file_read": a checkpoint-file chunk reads short;
 * "h2d": the host->device copy of a placement fails with TG_ERR_CUDA.
 * One-shot; process-wide. */
/* Finish an asynchronous load (TG_LOAD_ASYNC) still in flight on p: wait for its
 * data plane, record / verify its digests.  out (nullable) receives that load's
 * completed outcome (all zero when none was pending).  Returns 0, or the
 * runtime error the load ended with (its unverified tensors are then suspect
 * and re-sent on their next reuse, as after a failed synchronous load).  Every
 * call that mutates p or reads digests finishes a pending load first; reads of
 * the committed decisions (tg_reuse_size, tg_lookup, tg_dump, tg_pool_info_get
 * ...) do not wait. */
int tg_pool_sync(tg_pool* p, tg_load_outcome* out);
int tg_failpoint(const char* name, int64_t nth);

/* ---- raw device helpers ------------------------------------------------------ */
int tg_fingerprint_device(const void* dptr, uint64_t n, int32_t device, tg_digest* out); /* K1 */
int tg_synth_fill_device(tg_tensor_id id, uint64_t begin, uint64_t len, void* dptr, int32_t device);
/* Kernel-only timing: one K1 launch over n_bufs device buffers / one K3 wave
 * of n_moves (src, dst, len) moves, `reps` back-to-back launches bracketed by
 * CUDA events on the launching stream (after a warm-up launch). */
int tg_bench_fingerprint(const void* const* dptrs, const uint64_t* ns, uint32_t n_bufs, int32_t device, int32_t reps,
                         double* ms_per_launch, tg_digest* out /* n_bufs, nullable */);
int tg_bench_relocate(const uint64_t* moves /* src,dst,len triples (device addresses) */, uint32_t n_moves,
                      int32_t device, int32_t reps, double* ms_per_launch);
/* K3F (the load kernel): move n_moves hazard-free (src, dst, len) byte ranges
 * and return each one's tgfp1 digest from the same pass (one launch, then
 * `reps` timed ones); dst == 0 fingerprints the range in place. */
int tg_copy_fingerprint(const uint64_t* moves, uint32_t n_moves, int32_t device, int32_t reps, double* ms_per_launch,
                        tg_digest* digests /* n_moves */);
int tg_synth_fill_host(tg_tensor_id id, uint64_t begin, uint64_t len, void* dst, int32_t threads);
int tg_device_alloc(int32_t device, uint64_t size, void** out);
int tg_device_free(int32_t device, void* p);
int tg_memcpy(void* dst, const void* src, uint64_t n); /* cudaMemcpy default kind, synchronous */

/* ---- KV engine (KvEngine, kv_engine.hpp:43-239) ------------------------------- */
int tg_kv_create(const char* model_id, uint64_t block_size_tokens, uint64_t bytes_per_token, tg_kv** out); /* :47 */
void tg_kv_destroy(tg_kv* kv);
int tg_kv_clone(const tg_kv* kv, tg_kv** out);
/* ensure_capacity (:75-102): granted PBNs into buf (nullable) */
int tg_kv_ensure_capacity(tg_kv* kv, tg_pool* p, const tg_stats* s, uint64_t request_id, uint64_t tokens,
                          uint64_t* granted, uint64_t cap, uint64_t* n_granted);
/* batch_allocate (:107-161): counts[i] = blocks granted to request i;
 * pbns (nullable, cap entries) receives all granted PBNs in order. */
int tg_kv_batch_allocate(tg_kv* kv, tg_pool* p, const tg_stats* s, const uint64_t* request_ids,
                         const uint64_t* tokens, uint64_t n, uint64_t* counts, uint64_t* pbns, uint64_t cap,
                         uint64_t* total);
int tg_kv_release_request(tg_kv* kv, uint64_t request_id);              /* :165 */
int tg_kv_teardown(tg_kv* kv, tg_pool* p);                              /* :174 */
int tg_kv_urgent_reclaim(tg_kv* kv, tg_pool* p, const tg_stats* s, uint64_t blocks); /* :183 */
int tg_kv_table(const tg_kv* kv, uint64_t request_id, uint64_t* pbns, uint64_t cap, uint64_t* n,
                uint64_t* token_count);                                 /* table() :55 (reads HBM) */
int tg_kv_address_table(const tg_kv* kv, uint64_t* triples /*pbn,off,size*/, uint64_t cap, uint64_t* n); /* :63 */
int tg_kv_stats_get(const tg_kv* kv, tg_kv_stats* out);
/* Device tables for a paged-attention engine: tables[slot * stride + lbn] = PBN
 * (0 = not granted), addr[pbn] = arena offset.  They are updated on the
 * engine's own stream: a consumer on another stream first calls
 * tg_kv_wait_tables(kv, its_stream).  Growth (more request slots, longer
 * tables, more PBNs than reserved) moves them to new arrays, so re-query
 * after any allocating call — or size them once with tg_kv_reserve, after
 * which they never move.  Old arrays stay allocated until the engine is
 * destroyed: a stale pointer reads stale tables, never freed memory. */
int tg_kv_device_tables(const tg_kv* kv, void** tables, uint64_t* stride, void** addr);
int tg_kv_wait_tables(tg_kv* kv, void* cuda_stream); /* cuda_stream waits for the table updates enqueued so far */
int tg_kv_reserve(tg_kv* kv, tg_pool* p, uint32_t max_requests, uint64_t max_blocks_per_request,
                  uint64_t max_blocks); /* pre-size the device tables (binds kv to p's device) */
/* Block-table consumers (the cache write / gather of a paged-attention engine,
 * PAPER.md:807 reshape_and_cache_segment): token i of the request in table
 * slot d_slots[i] at token position d_positions[i] lives at
 *   arena + addr[tables[slot][pos / block_tokens]] + (pos % block_tokens) * bytes_per_token.
 * write_tokens copies d_buf[i] (bytes_per_token each) there; read_tokens
 * gathers it into d_buf[i].  Device pointers.  The copy is ordered after every
 * table update enqueued before the call, on any stream (`cuda_stream` null =
 * the engine's stream).  A token outside the granted blocks (unknown slot, LBN
 * past the table, PBN 0, a block outside the arena) moves nothing and counts a
 * fault: tg_kv_token_faults waits for the consumers launched so far and
 * returns the running count. */
int tg_kv_write_tokens(tg_kv* kv, tg_pool* p, const uint64_t* d_slots, const uint64_t* d_positions, const void* d_buf,
                       uint32_t n, void* cuda_stream);
int tg_kv_read_tokens(tg_kv* kv, tg_pool* p, const uint64_t* d_slots, const uint64_t* d_positions, void* d_buf,
                      uint32_t n, void* cuda_stream);
int tg_kv_token_faults(tg_kv* kv, uint64_t* faults);

/* ---- device-decided KV batches (K4D; new, no reference counterpart) ------------
 * The allocator decision of batch_allocate (:107-161) taken by a kernel, for
 * requests the engine already knows, with no host round trip per batch:
 *   tg_kv_request_slot     table row of a request (ensure_capacity(rid, 0)
 *                          makes a new request known, as in the reference);
 *   tg_kv_device_arm       upload the allocator state and the pool's free runs;
 *                          from here until sync the pool layout is frozen
 *                          (layout-changing pool calls and host KV calls on any
 *                          engine of that pool return TG_ERR_KV_ARMED);
 *   tg_kv_batch_allocate_device
 *                          enqueue one batch on `stream` (null: the engine's
 *                          stream): request table slots and token counts in
 *                          DEVICE memory, n <= max_requests; capturable in a
 *                          CUDA graph (every pointer is read at run time;
 *                          the engine must outlive the graph); batches of
 *                          one session must be stream-ordered;
 *   tg_kv_device_sync      wait, fold the device decisions into the host state,
 *                          replay on the reference path every batch the device
 *                          left to it (contended pool, unknown slot, shrinking
 *                          token count, duplicate request, ...), and disarm.
 * After sync, tables, address table, counters and pool regions equal running
 * the same batches through tg_kv_batch_allocate.  Sync must name the pool the
 * engine was armed on (TG_ERR_BAD_ARG otherwise, the engine stays armed).  Errors of replayed batches
 * are reported by sync (the first one); TG_ERR_KV_LOG if more than
 * max_batches batches were enqueued. */
int tg_kv_request_slot(const tg_kv* kv, uint64_t request_id, uint32_t* slot);
int tg_kv_device_arm(tg_kv* kv, tg_pool* p, uint64_t max_blocks_per_request, uint32_t max_requests,
                     uint32_t max_batches);
int tg_kv_batch_allocate_device(tg_kv* kv, const uint64_t* d_slots, const uint64_t* d_tokens, uint32_t n,
                                void* cuda_stream);
int tg_kv_device_sync(tg_kv* kv, tg_pool* p, const tg_stats* s, uint64_t* applied_batches,
                      uint64_t* replayed_batches);

/* ---- planner (plan_allocation, packing.hpp:311-483) ----------------------------
 * Pure two-stage plan over an address-ordered region tiling.  new_tensors are
 * placed in the given order after a stable size-descending sort; candidates
 * are sorted by (cost, -size, last_access, id) unless keep_candidate_order. */
typedef struct tg_plan tg_plan;
int tg_plan_allocation(const tg_region* regions, uint64_t n_regions, const tg_tensor_spec* new_tensors,
                       uint32_t n_new, const tg_eviction* candidates, uint32_t n_candidates,
                       const tg_tensor_id* immovable, uint32_t n_immovable, int32_t strictness, int32_t merge,
                       int32_t keep_candidate_order, tg_plan** out);
uint32_t tg_plan_evictions(const tg_plan* p, tg_eviction* buf, uint32_t cap);
uint32_t tg_plan_relocations(const tg_plan* p, tg_relocation* buf, uint32_t cap);
uint32_t tg_plan_placements(const tg_plan* p, tg_placement* buf, uint32_t cap);
int tg_plan_costs(const tg_plan* p, double* total_eviction_cost, uint64_t* total_merge_cost, uint64_t* pgp_merge_cost,
                  uint64_t* initial_merge_cost, uint64_t* fallback_evictions);
void tg_plan_destroy(tg_plan* p);

/* ---- scheduler (scheduler.hpp:41-120) ------------------------------------------ */
typedef struct {
    const char* gpu_id;
    int32_t available;
    uint64_t pool_size;
    uint64_t free_bytes;
    double pcie_bandwidth;
    double store_bandwidth;
    double nvlink_bandwidth; /* peer term; 0 disables it (reference behaviour) */
} tg_gpu_snapshot;
/* reuse[g * n_models + m] = S' of model m on GPU g; peer_reuse likewise (nullable).
 * request_models[i] indexes models; assignment[i] = chosen GPU index or -1;
 * estimates[i * n_gpus + g] = estimate or -1 when infeasible (nullable). */
int tg_schedule(const uint32_t* request_models, uint32_t n_requests, const tg_gpu_snapshot* gpus, uint32_t n_gpus,
                const tg_model_spec* models, uint32_t n_models, const uint64_t* reuse, const uint64_t* peer_reuse,
                uint32_t batch_size, uint64_t block_size_tokens, int32_t* assignment, double* estimates);
double tg_estimate_load_time(const tg_model_spec* m, uint64_t reuse_size, const tg_gpu_snapshot* g,
                             uint64_t peer_reuse_size);

#ifdef __cplusplus
}
#endif
#endif /* TANGRAM_H */
