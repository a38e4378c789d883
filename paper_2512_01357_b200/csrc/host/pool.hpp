// One GPU's Tangram pool: the control plane (Store) bound to its B200 data
// plane — a device-resident arena of pool_size bytes, a copy stream for
// host→device placement, a compute stream for relocation waves and reuse
// verification, and a fingerprint stream that trails the copies tensor by
// tensor.  load_model() keeps ReuseStore::load_model's decisions
// (reuse_store.hpp:120-174) and adds the bytes: relocations as WAR-ordered
// waves of the K3 kernel, misses as H2D (or NVLink peer pulls through the
// same kernel), and K1 content fingerprints of every placed and every reused
// tensor.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../device/kernels.hpp"
#include "kv.hpp"
#include "store.hpp"

namespace tg {

constexpr int kErrNoDevice = 101;
constexpr int kErrNoSource = 102;
constexpr int kErrVerify = 105;

// Host-side checkpoint bytes per tensor key, with an optional expected
// content fingerprint (e.g. from a checkpoint manifest).
struct HostSource {
    const void* ptr = nullptr;
    u64 size = 0;
    bool has_expected = false;
    Digest expected;
    bool on_device = false;  // HBM-resident source: placed by the K3 copy kernel
    int device = -1;         // ... on this device (another pool's device reads it over NVLink)
    // Model Store source (model.hpp:24 ModelLocation::ModelStore): bytes live
    // in a checkpoint file and stream file → pinned ring → HBM
    std::string path;
    u64 file_off = 0;
    bool is_file() const { return !path.empty(); }
};

// Pinned staging ring for file-backed placements (Model Store → GPU).  A
// load hands the stager every file range it will place, in issue order
// (begin); reader threads then pread fixed-size chunks into the ring ahead
// of the caller — each slot reused once the H2D that drained it completed —
// while the caller issues the H2D of each range in turn (issue), so storage
// reads, PCIe copies and the fingerprint kernels trailing them all overlap
// across tensors.  One per pool, created on first use; the ring stays
// allocated, the reader threads live for one load (end / destructor join
// them).
class FileStager {
public:
    FileStager(int device, std::size_t chunk, int slots, int threads);
    ~FileStager();
    struct Range {
        std::string path;
        u64 off = 0, size = 0;
    };
    // Start reading `ranges` (in the order they will be issued).
    void begin(std::vector<Range> ranges);
    // Enqueue range i's H2D into dst on stream s, chunk by chunk as the
    // readers fill them (ranges must be issued in order).  Throws
    // DeviceError(kErrNoSource) on a short read / missing file.
    void issue(std::size_t i, std::uint8_t* dst, cudaStream_t s);
    void end() noexcept;  // stop and join the readers (idempotent)
    // begin + issue + end of one range
    void stage(const std::string& path, u64 off, u64 size, std::uint8_t* dst, cudaStream_t s);
    u64 bytes_read() const { return bytes_read_; }

private:
    struct Chunk {
        std::size_t range;
        u64 at, n;  // within the range
    };
    void reader();
    int device_;
    std::size_t chunk_;
    std::vector<std::uint8_t*> slot_;
    std::vector<cudaEvent_t> free_;  // recorded after the H2D that drained the slot
    int threads_;
    u64 bytes_read_ = 0;
    // one load's session
    std::vector<Range> ranges_;
    std::vector<int> fd_;  // per range (shared per path)
    std::vector<Chunk> chunks_;
    std::vector<std::size_t> first_chunk_;  // per range
    std::vector<std::uint8_t> state_;       // per chunk: 0 pending, 1 ready, 2 failed
    std::size_t next_read_ = 0, issued_ = 0;
    bool stop_ = false;
    std::mutex mu_;
    std::condition_variable cv_;
    std::vector<std::thread> pool_;
};

// Test failpoints (tg_failpoint, include/tangram.h): arm a named point so that
// its n-th hit from now fails the way the real fault would (a short file
// read, a CUDA error in the middle of a load).  Disarmed points cost one
// relaxed atomic load.
class Failpoints {
public:
    static void arm(const std::string& name, long long nth);  // nth <= 0 disarms
    static bool hit(const char* name);                         // true: fail here
};

class SourceRegistry {
public:
    static SourceRegistry& get();
    void put(const Key& k, const HostSource& s);
    bool find(const Key& k, HostSource* out) const;
    void erase(const Key& k);
    void clear();

private:
    mutable std::mutex mu_;
    std::unordered_map<Key, HostSource, KeyHash> map_;
};

// Shard lineage (process-wide): tensor `child` holds bytes [begin, begin +
// size) of tensor `parent` — what tg_model_shard produces for every shard.
// A load may then assemble a missing shard from the resident shards of the
// same parent in another layout on peer pools (re-shard pull, SURVEY §8(d)
// C4 "shards resident on peers in a previous TP layout").
struct ShardOf {
    Key parent;
    u64 begin = 0;
    u64 size = 0;
};
class ShardLineage {
public:
    static ShardLineage& get();
    void put(const Key& child, const ShardOf& s);
    bool find(const Key& child, ShardOf* out) const;
    // children of `parent` as (child, lineage)
    std::vector<std::pair<Key, ShardOf>> children(const Key& parent) const;

private:
    mutable std::mutex mu_;
    std::unordered_map<Key, ShardOf, KeyHash> of_;
    std::unordered_map<Key, std::vector<Key>, KeyHash> kids_;
};

// A resident, fingerprinted tensor of a peer pool (what peers exchange).
struct RemoteEntry {
    Key id;
    u64 off = 0;
    u64 size = 0;
    Digest digest;
};

// load flags (tg_load_policy.flags)
constexpr u32 kLoadVerifyReuse = 1u;     // fingerprint reused tensors, compare to the recorded digest
constexpr u32 kLoadFingerprintNew = 2u;  // fingerprint placed tensors and record the digest
constexpr u32 kLoadPeer = 4u;            // pull misses from peer pools that hold them
// Default: the whole device side of a load is one load-kernel launch —
// relocation waves, device-source placements and in-place verification, each
// moved tensor fingerprinted from the copy's own read (C2 step: 8.8 ms, vs
// 9.4 ms for the separate K3 waves + K1 passes, which remain available by
// leaving this flag out).
constexpr u32 kLoadFused = 8u;
// Return once the decision is committed and the data plane is enqueued; the
// wait and the digest bookkeeping run before the next operation on the pool
// (Pool::complete_pending), so loads on different pools — different GPUs —
// overlap while the caller carries on (trace replay, §8(f) row 1).
constexpr u32 kLoadAsync = 16u;
constexpr u32 kLoadDefault = kLoadVerifyReuse | kLoadFingerprintNew | kLoadFused;
// tg_load_policy.flags with this bit are taken literally (0 | explicit = no
// optional work); without it, 0 means kLoadDefault.
constexpr u32 kLoadExplicit = 0x80000000u;

struct LoadTimings {
    double plan_us = 0;          // host planning (decide)
    double total_ms = 0;         // device span: entry .. all bytes placed and verified
    double relocate_ms = 0;      // relocation waves (K3)
    double h2d_ms = 0;           // first .. last host→device copy
    double peer_ms = 0;          // peer pulls
    double fp_kernel_ms = 0;     // Σ K1 launch durations
    double fp_reuse_ms = 0;      // Σ K1 launch durations over reused tensors (≤ 2 launches)
    double fp_reuse_max_ms = 0;  // the longer of the two
    double host_issue_us = 0;    // host: entry .. all device work enqueued
    double host_wait_us = 0;     // host: waiting for the device work
    double host_total_us = 0;    // host: entry .. return
    double kernel_end_ms = 0;        // device: entry .. the load kernel (or the last K3 wave) ends
    double gated_h2d_start_ms = 0;   // device: entry .. the first wave-gated H2D may start (0: none)
};

struct LoadReport {
    LoadDecision decision;           // hits / misses / plan (placements index miss_desc)
    std::vector<u32> reloc_wave;     // WAR wave of each relocation
    std::vector<std::uint8_t> placement_src;  // 0 host (PCIe), 1 peer (NVLink), 2 HBM source, 3 re-shard pieces
    u32 waves = 0;
    u64 pcie_bytes = 0, peer_bytes = 0, device_src_bytes = 0, fingerprint_bytes = 0, repaired_bytes = 0;
    u32 verify_mismatches = 0, expected_mismatches = 0;
    std::vector<Digest> digests;     // per model tensor (model order), when fingerprinted
    LoadTimings t;
    // The decision was committed to the store (a runtime error after this
    // point leaves the reference's decision in place, with every tensor the
    // load could not verify marked suspect; see Pool::load_model).
    bool committed = false;
    u32 suspect_after = 0;           // tensors of this load left suspect (0 on success)
};

// A load whose data plane is still running (kLoadAsync).
struct PendingLoad {
    LoadReport report;
    ModelDesc model;
    std::function<int(LoadReport*, const ModelDesc&)> finish;
};

class Pool {
public:
    // device < 0: control plane only (no arena; moves no bytes).
    Pool(GpuDesc gpu, int device);
    ~Pool();
    Pool(const Pool&) = delete;
    Pool& operator=(const Pool&) = delete;

    Store& store() { return store_; }
    const Store& store() const { return store_; }
    int device() const { return device_; }
    bool has_device() const { return device_ >= 0; }
    std::uint8_t* arena() const { return arena_; }
    cudaStream_t stream() const { return s_main_; }
    int sm_count() const { return sm_count_; }

    struct Totals {
        u64 loads = 0;
        double data_plane_ms = 0;
        u64 pcie_bytes = 0, peer_bytes = 0, device_src_bytes = 0, fingerprint_bytes = 0, relocated_bytes = 0;
        u64 verify_mismatches = 0, repaired_bytes = 0, failed_loads = 0;
    };
    const Totals& totals() const { return totals_; }

    St load_model(const ModelDesc& m, const StatsView& stats, double clock, const LoadOptions& opt, u32 flags,
                  LoadReport* rep);
    St move_tensor(const Key& k, u64 to);  // metadata + bytes
    // Finish an asynchronous load (kLoadAsync): wait for its data plane, then
    // record / verify its digests.  Returns 0 or the runtime error the load
    // ended with (its tensors are then suspect, as after a failed synchronous
    // load).  Every mutating operation calls it first.
    int complete_pending();
    bool has_pending() const { return pending_ != nullptr; }
    bool pending_shares(const std::vector<Key>& keys) const;
    const LoadReport& last_completed() const { return last_async_; }
    int last_completed_rc() const { return last_async_rc_; }
    const std::string& last_completed_error() const { return last_async_err_; }

    Digest fingerprint_resident(const Key& k);  // K1 over the resident bytes
    void add_peer(Pool* p);
    // Peers in other processes: export this arena (CUDA IPC), publish the
    // index of fingerprinted residents, attach a remote arena + its index.
    void export_handle(cudaIpcMemHandle_t* h) const;
    std::vector<RemoteEntry> index() const;
    int attach_remote(const cudaIpcMemHandle_t& h, const std::vector<RemoteEntry>& idx);
    void update_remote(int id, const std::vector<RemoteEntry>& idx);
    u64 peer_reuse_size(const ModelDesc& m) const;  // bytes of m's misses resident on a peer

    // Whole-pool checkpoint (metadata + arena bytes) for rollback / benchmarks.
    struct Snapshot;
    Snapshot* snapshot();
    void restore(const Snapshot* s);
    static void drop(Snapshot* s);

    std::unique_ptr<KvDevice> make_kv_device();

    // Value semantics of the reference store (reuse_store.hpp:336-344; copied
    // for rollback, kv_engine.hpp:146-158): adopt another store's metadata.
    // Bytes do not travel: a tensor keeps its verified state only where this
    // arena already holds it (same offset and size, not suspect); every other
    // tensor of the adopted map is suspect here (its next reuse re-sends it).
    void adopt_store(const Store& src);

    // Device tensor index: republish the store's tensor map to
    // HBM on the pool stream when it changed since the last publish (no-op on
    // control-plane pools).  device_index() is the published table.
    void publish_index(cudaStream_t stream = nullptr);  // upload stream (null: the pool stream)
    const void* device_index(u64* capacity) const {
        *capacity = index_cap_;
        return d_index_;
    }
    // One device lookup per key (K6); out: 3 u64 per key (offset, size, found | flags << 32).
    void index_lookup(const std::vector<Key>& keys, std::vector<u64>* out);

private:
    void ensure_events(std::size_t n);
    void sync_all_streams() noexcept;  // best effort, after a failure mid-load
    St load_model_impl(const ModelDesc& m, const StatsView& stats, double clock, const LoadOptions& opt, u32 flags,
                       LoadReport* rep);
    void fetch(const HostSource& hs, std::uint8_t* dst, u64 size, cudaStream_t s);
    cudaEvent_t ev(std::size_t i) { return events_[i]; }

    Store store_;
    int device_ = -1;
    int sm_count_ = 148;
    std::uint8_t* arena_ = nullptr;
    cudaStream_t s_main_ = nullptr, s_copy_ = nullptr, s_fp_ = nullptr, s_peer_ = nullptr, s_verify_ = nullptr;
    std::vector<cudaEvent_t> events_;
    bool assemble_shard(const TensorDesc& t, std::vector<MoveDesc>* pieces, const Plan* plan, u64* local_bytes) const;
    std::vector<Pool*> peers_;
    std::vector<Pool*> peer_of_;  // pools that have this one as a peer
    std::vector<int> peer_devices_;  // devices whose HBM this pool's kernels may access
    void enable_peer_access(int other);
    // Events of in-process pools that read this arena (peer pulls), recorded
    // after their loads; this pool's next data plane waits on them, so bytes
    // a peer is still reading are never overwritten.
    std::unordered_map<const Pool*, cudaEvent_t> reader_events_;
    cudaEvent_t ev_reader_ = nullptr;
    void note_readers();
    void wait_readers();
    // descriptors of the last upload still on the device, and whether the
    // stage's sums / counters are zero (a lone load kernel cleaned them)
    std::vector<std::uint8_t> resident_desc_;
    std::pair<std::size_t, std::size_t> resident_layout_{0, 0};
    bool resident_clean_ = false;
    std::unique_ptr<PendingLoad> pending_;
    LoadReport last_async_;
    int last_async_rc_ = 0;
    std::string last_async_err_;
    struct RemotePeer {
        std::uint8_t* base = nullptr;  // IPC-mapped peer arena
        std::unordered_map<Key, RemoteEntry, KeyHash> index;
    };
    std::vector<RemotePeer> remotes_;
    std::unique_ptr<FileStager> stager_;
    Totals totals_;
    // staging
    void* h_stage_ = nullptr;
    void* d_stage_ = nullptr;
    void* h_stage_dev_ = nullptr;  // device alias of h_stage_ (mapped pinned memory)
    std::size_t stage_cap_ = 0;
    void ensure_stage(std::size_t bytes);
    // device index
    void* d_index_ = nullptr;
    u64 index_cap_ = 0;
    void* h_index_ = nullptr;  // pinned image being uploaded
    u64 h_index_cap_ = 0;
    cudaEvent_t ev_index_ = nullptr;
    u64 published_epoch_ = ~u64{0};
};

std::unique_ptr<KvDevice> make_kv_device(int device, cudaStream_t stream);
void fingerprint_device(const void* ptr, u64 n, int device, Digest* out);
void synth_fill_device(const Key& k, u64 begin, u64 len, void* dst, int device);
double bench_fingerprint(const std::vector<std::pair<const void*, u64>>& bufs, int device, int reps,
                         std::vector<Digest>* out);
double bench_relocate(const std::vector<MoveDesc>& moves, int device, int reps);
double bench_copy_fp(const std::vector<MoveDesc>& moves, int device, int reps, std::vector<Digest>* out);

}  // namespace tg
