#include "pool.hpp"

#include <algorithm>
#include <chrono>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>

#include <cstdlib>
#include <cstring>
#include <thread>
#include <unordered_set>

#include <cuda.h>  // stream memory-op types only; the entry point is resolved at run time

#include "../device/common.cuh"
#include "../device/kernels.hpp"
#include "index.hpp"
#include "murmur_mix.hpp"

namespace tg {


namespace {
// cuStreamWaitValue64 through the runtime's driver entry point (no -lcuda):
// lets a copy stream wait on a counter the load kernel bumps, so a placement
// gated on relocation wave w starts when that wave's tiles are done instead
// of when the whole launch ends.  Null when the driver lacks it.
using WaitValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WaitValue64Fn wait_value64() {
    static const WaitValue64Fn fn = []() -> WaitValue64Fn {
        if (const char* e = std::getenv("TANGRAM_WAIT_VALUE"); e && std::strcmp(e, "0") == 0) return nullptr;  // A/B
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue64", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p) {
            cudaGetLastError();
            return nullptr;
        }
        return reinterpret_cast<WaitValue64Fn>(p);
    }();
    return fn;
}
}  // namespace

// ---- host source registry ----------------------------------------------------
SourceRegistry& SourceRegistry::get() {
    static SourceRegistry r;
    return r;
}
void SourceRegistry::put(const Key& k, const HostSource& s) {
    std::lock_guard<std::mutex> g(mu_);
    map_[k] = s;
}
bool SourceRegistry::find(const Key& k, HostSource* out) const {
    std::lock_guard<std::mutex> g(mu_);
    auto it = map_.find(k);
    if (it == map_.end()) return false;
    *out = it->second;
    return true;
}
void SourceRegistry::erase(const Key& k) {
    std::lock_guard<std::mutex> g(mu_);
    map_.erase(k);
}
ShardLineage& ShardLineage::get() {
    static ShardLineage r;
    return r;
}
void ShardLineage::put(const Key& child, const ShardOf& s) {
    std::lock_guard<std::mutex> g(mu_);
    if (of_.count(child)) return;
    of_[child] = s;
    kids_[s.parent].push_back(child);
}
bool ShardLineage::find(const Key& child, ShardOf* out) const {
    std::lock_guard<std::mutex> g(mu_);
    auto it = of_.find(child);
    if (it == of_.end()) return false;
    *out = it->second;
    return true;
}
std::vector<std::pair<Key, ShardOf>> ShardLineage::children(const Key& parent) const {
    std::lock_guard<std::mutex> g(mu_);
    std::vector<std::pair<Key, ShardOf>> out;
    auto it = kids_.find(parent);
    if (it == kids_.end()) return out;
    for (const Key& c : it->second) out.push_back({c, of_.at(c)});
    return out;
}

namespace {
std::mutex g_fp_mu;
std::unordered_map<std::string, long long> g_fp_armed;  // name -> hits left before the failing one
std::atomic<bool> g_fp_any{false};
}  // namespace

void Failpoints::arm(const std::string& name, long long nth) {
    std::lock_guard<std::mutex> g(g_fp_mu);
    if (nth <= 0) g_fp_armed.erase(name);
    else g_fp_armed[name] = nth;
    g_fp_any.store(!g_fp_armed.empty(), std::memory_order_relaxed);
}

bool Failpoints::hit(const char* name) {
    if (!g_fp_any.load(std::memory_order_relaxed)) return false;
    std::lock_guard<std::mutex> g(g_fp_mu);
    auto it = g_fp_armed.find(name);
    if (it == g_fp_armed.end() || --it->second > 0) return false;
    g_fp_armed.erase(it);  // one-shot
    g_fp_any.store(!g_fp_armed.empty(), std::memory_order_relaxed);
    return true;
}

// A file source must hold its whole range when the load is planned; a file
// that shrinks under a running load is a runtime failure (short read).
void check_file_source(const HostSource& s, const Key& id) {
    struct stat st {};
    if (::stat(s.path.c_str(), &st) != 0)
        throw DeviceError(kErrNoSource, "checkpoint file " + s.path + " of tensor " + id.hex() + " is missing");
    if (static_cast<u64>(st.st_size) < s.file_off + s.size)
        throw DeviceError(kErrNoSource, "checkpoint file " + s.path + " is too short for tensor " + id.hex());
}

void SourceRegistry::clear() {
    std::lock_guard<std::mutex> g(mu_);
    map_.clear();
}

// ---- file-backed sources (Model Store) ---------------------------------------
FileStager::FileStager(int device, std::size_t chunk, int slots, int threads)
    : device_(device), chunk_(chunk), threads_(threads) {
    DeviceScope ds(device_);
    for (int i = 0; i < slots; ++i) {
        void* p = nullptr;
        TG_CUDA(cudaMallocHost(&p, chunk_));
        slot_.push_back(static_cast<std::uint8_t*>(p));
        cudaEvent_t e;
        TG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        free_.push_back(e);
    }
}

FileStager::~FileStager() {
    end();
    DeviceScope ds(device_);
    for (cudaEvent_t e : free_) {
        cudaEventSynchronize(e);
        cudaEventDestroy(e);
    }
    for (std::uint8_t* p : slot_) cudaFreeHost(p);
}

void FileStager::begin(std::vector<Range> ranges) {
    end();
    ranges_ = std::move(ranges);
    chunks_.clear();
    first_chunk_.clear();
    fd_.assign(ranges_.size(), -1);
    std::unordered_map<std::string, int> fds;
    for (std::size_t r = 0; r < ranges_.size(); ++r) {
        auto it = fds.find(ranges_[r].path);
        if (it == fds.end()) it = fds.emplace(ranges_[r].path, ::open(ranges_[r].path.c_str(), O_RDONLY)).first;
        fd_[r] = it->second;  // -1: reported by issue() as a missing file
        first_chunk_.push_back(chunks_.size());
        for (u64 at = 0; at < ranges_[r].size; at += chunk_)
            chunks_.push_back(Chunk{r, at, std::min<u64>(chunk_, ranges_[r].size - at)});
    }
    first_chunk_.push_back(chunks_.size());
    state_.assign(chunks_.size(), 0);
    next_read_ = issued_ = 0;
    stop_ = false;
    const int n = static_cast<int>(std::min<std::size_t>(threads_, chunks_.size()));
    for (int t = 0; t < n; ++t) pool_.emplace_back([this] { reader(); });
}

// Reader thread: claim the next chunk, wait until its ring slot is free (the
// H2D of the chunk `slots` earlier was issued and has completed), pread it.
void FileStager::reader() {
    cudaSetDevice(device_);
    const std::size_t nslots = slot_.size();
    for (;;) {
        std::size_t k;
        {
            std::unique_lock<std::mutex> g(mu_);
            if (stop_ || next_read_ >= chunks_.size()) return;
            k = next_read_++;
            cv_.wait(g, [&] { return stop_ || k < issued_ + nslots; });
            if (stop_) return;
        }
        cudaEventSynchronize(free_[k % nslots]);  // the slot's previous H2D (this load's or an earlier one's) drained
        const Chunk& c = chunks_[k];
        const Range& r = ranges_[c.range];
        const int fd = fd_[c.range];
        std::uint8_t* buf = slot_[k % nslots];
        bool ok = fd >= 0 && !Failpoints::hit("file_read");  // injected short read
        for (u64 done = 0; ok && done < c.n;) {
            const ssize_t got = ::pread(fd, buf + done, c.n - done, static_cast<off_t>(r.off + c.at + done));
            if (got <= 0) ok = false;
            else done += static_cast<u64>(got);
        }
        {
            std::lock_guard<std::mutex> g(mu_);
            state_[k] = ok ? 1 : 2;
        }
        cv_.notify_all();
    }
}

void FileStager::issue(std::size_t i, std::uint8_t* dst, cudaStream_t s) {
    const std::size_t nslots = slot_.size();
    for (std::size_t k = first_chunk_[i]; k < first_chunk_[i + 1]; ++k) {
        {
            std::unique_lock<std::mutex> g(mu_);
            if (k != issued_) throw DeviceError(kErrCuda, "file stager: ranges issued out of order");
            cv_.wait(g, [&] { return state_[k] != 0; });
            if (state_[k] == 2) {
                const std::string what = (fd_[i] < 0 ? "cannot open " : "short read from ") + ranges_[i].path;
                g.unlock();
                end();
                throw DeviceError(kErrNoSource, what);
            }
        }
        const Chunk& c = chunks_[k];
        TG_CUDA(cudaMemcpyAsync(dst + c.at, slot_[k % nslots], c.n, cudaMemcpyHostToDevice, s));
        TG_CUDA(cudaEventRecord(free_[k % nslots], s));
        bytes_read_ += c.n;
        {
            std::lock_guard<std::mutex> g(mu_);
            ++issued_;
        }
        cv_.notify_all();
    }
    if (issued_ == chunks_.size()) end();
}

void FileStager::end() noexcept {
    {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (std::thread& t : pool_) t.join();
    pool_.clear();
    std::vector<int> closed;
    for (int fd : fd_)
        if (fd >= 0 && std::find(closed.begin(), closed.end(), fd) == closed.end()) {
            ::close(fd);
            closed.push_back(fd);
        }
    fd_.clear();
}

void FileStager::stage(const std::string& path, u64 off, u64 size, std::uint8_t* dst, cudaStream_t s) {
    begin({Range{path, off, size}});
    issue(0, dst, s);
    end();
}

// A load kernel with writing tasks and at most kSplitMaxWaves relocation
// waves leaves the in-place verification of the untouched hits to a K1
// launch on the verify stream.  The K1 CTAs take the SM slots the load
// kernel's CTAs release, so the verification runs on K1's own (faster) ring
// and fills the load kernel's tail.  With more serial waves the gate waits
// dominate, and verification tiles inside the load kernel fill them better
// (same-box A/B: C2, 3 waves, split 1-2.6 % faster; C2 under GlobalMerge,
// 11 waves, split 3-4 % slower).  TANGRAM_VERIFY_SPLIT=0 / =1 forces either.
constexpr unsigned kSplitMaxWaves = 3;
bool verify_split(unsigned waves) {
    static const int mode = [] {
        const char* e = std::getenv("TANGRAM_VERIFY_SPLIT");
        return !e ? -1 : std::strcmp(e, "0") == 0 ? 0 : 1;
    }();
    return mode < 0 ? waves <= kSplitMaxWaves : mode == 1;
}

bool split_candidate(bool fused, bool fp_reuse, bool kernel_writes, std::size_t n_still, unsigned waves) {
    return fused && fp_reuse && kernel_writes && n_still > 0 && verify_split(waves);
}

// Resident-warp rounds of verification tiles behind each gate of the load
// kernel (TANGRAM_VERIFY_ROUNDS; split loads: TANGRAM_SPLIT_ROUNDS).
unsigned long long verify_rounds(bool split) {
    static const unsigned long long in_kernel = [] {
        const char* e = std::getenv("TANGRAM_VERIFY_ROUNDS");
        return e ? std::strtoull(e, nullptr, 10) : 8ull;
    }();
    static const unsigned long long with_split = [] {
        const char* e = std::getenv("TANGRAM_SPLIT_ROUNDS");
        return e ? std::strtoull(e, nullptr, 10) : 0ull;
    }();
    return split ? with_split : in_kernel;
}

// 8 MiB chunks, a 256 MiB ring, 3/4 of the host threads reading (4..16;
// TANGRAM_STAGER_THREADS overrides): page-cache preads run ~6 GB/s a thread,
// so a dozen saturate the PCIe link.
int stager_threads() {
    if (const char* e = std::getenv("TANGRAM_STAGER_THREADS")) return std::max(1, std::atoi(e));
    return std::clamp(static_cast<int>(std::thread::hardware_concurrency() * 3 / 4), 4, 16);
}
std::unique_ptr<FileStager> make_stager(int device) {
    const int threads = stager_threads();
    return std::make_unique<FileStager>(device, 8u << 20, 32, threads);
}

// ---- pool --------------------------------------------------------------------
Pool::Pool(GpuDesc gpu, int device) : store_(std::move(gpu)), device_(device) {
    if (device_ < 0) return;
    DeviceScope ds(device_);
    TG_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device_));
    // +256 B slack: aligned 16-byte word reads at a tensor's last byte may
    // touch the following word.
    TG_CUDA(cudaMalloc(reinterpret_cast<void**>(&arena_), store_.pool_size() + 256));
    for (cudaStream_t* s : {&s_main_, &s_copy_, &s_fp_, &s_peer_, &s_verify_})
        TG_CUDA(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
    // One-time setup here, not inside the first load's latency: the pinned /
    // device descriptor stage (a pinned allocation costs milliseconds) and
    // the events a load of up to ~100 tensors records.
    ensure_stage(1 << 20);
    ensure_events(256);
}

Pool::~Pool() {
    if (device_ < 0) return;
    DeviceScope ds(device_);
    try {
        complete_pending();
    } catch (...) {
    }
    cudaDeviceSynchronize();
    for (Pool* p : peers_) {
        p->peer_of_.erase(std::remove(p->peer_of_.begin(), p->peer_of_.end(), this), p->peer_of_.end());
        p->reader_events_.erase(this);
    }
    for (Pool* q : peer_of_) q->peers_.erase(std::remove(q->peers_.begin(), q->peers_.end(), this), q->peers_.end());
    if (ev_reader_) cudaEventDestroy(ev_reader_);
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
    for (cudaStream_t s : {s_main_, s_copy_, s_fp_, s_peer_, s_verify_})
        if (s) cudaStreamDestroy(s);
    for (RemotePeer& r : remotes_)
        if (r.base) cudaIpcCloseMemHandle(r.base);
    if (arena_) cudaFree(arena_);
    if (d_stage_) cudaFree(d_stage_);
    if (h_stage_) cudaFreeHost(h_stage_);
    if (d_index_) cudaFree(d_index_);
    if (h_index_) cudaFreeHost(h_index_);
    if (ev_index_) cudaEventDestroy(ev_index_);
}

void Pool::publish_index(cudaStream_t stream) {
    if (!has_device() || store_.epoch() == published_epoch_) return;
    cudaStream_t st = stream ? stream : s_main_;
    DeviceScope ds(device_);
    const std::vector<IndexSlot> img = build_index_image(store_);
    const u64 cap = img.size(), bytes = cap * sizeof(IndexSlot);
    if (ev_index_) TG_CUDA(cudaEventSynchronize(ev_index_));  // the previous image has been read
    else TG_CUDA(cudaEventCreateWithFlags(&ev_index_, cudaEventDisableTiming));
    if (cap > h_index_cap_) {
        if (h_index_) TG_CUDA(cudaFreeHost(h_index_));
        TG_CUDA(cudaHostAlloc(&h_index_, bytes, cudaHostAllocDefault));
        h_index_cap_ = cap;
    }
    if (cap != index_cap_) {  // the table grew: consumers re-query tg_pool_device_index
        if (d_index_) {
            TG_CUDA(cudaStreamSynchronize(s_main_));
            TG_CUDA(cudaFree(d_index_));
        }
        TG_CUDA(cudaMalloc(&d_index_, bytes));
        index_cap_ = cap;
    }
    std::memcpy(h_index_, img.data(), bytes);
    TG_CUDA(cudaMemcpyAsync(d_index_, h_index_, bytes, cudaMemcpyHostToDevice, st));
    TG_CUDA(cudaEventRecord(ev_index_, st));
    if (st != s_main_) TG_CUDA(cudaStreamWaitEvent(s_main_, ev_index_));  // ordered for the pool stream's users
    published_epoch_ = store_.epoch();
}

void Pool::index_lookup(const std::vector<Key>& keys, std::vector<u64>* out) {
    if (!has_device()) throw DeviceError(kErrNoDevice, "index lookup on a control-plane pool");
    publish_index();
    DeviceScope ds(device_);
    const std::size_t n = keys.size();
    out->assign(3 * n, 0);
    if (!n) return;
    ensure_stage(n * 5 * sizeof(u64) + 64);
    resident_clean_ = false;  // the stage now holds keys, not a load's descriptors
    auto* h = static_cast<u64*>(h_stage_);
    auto* d = static_cast<u64*>(d_stage_);
    for (std::size_t i = 0; i < n; ++i) {
        h[2 * i] = keys[i].hi;
        h[2 * i + 1] = keys[i].lo;
    }
    TG_CUDA(cudaMemcpyAsync(d, h, 2 * n * sizeof(u64), cudaMemcpyHostToDevice, s_main_));
    index_lookup_launch(d_index_, index_cap_, d, static_cast<u32>(n), d + 2 * n, s_main_);
    TG_CUDA(cudaGetLastError());
    TG_CUDA(cudaMemcpyAsync(h + 2 * n, d + 2 * n, 3 * n * sizeof(u64), cudaMemcpyDeviceToHost, s_main_));
    TG_CUDA(cudaStreamSynchronize(s_main_));
    std::memcpy(out->data(), h + 2 * n, 3 * n * sizeof(u64));
}

void Pool::ensure_events(std::size_t n) {
    while (events_.size() < n) {
        cudaEvent_t e;
        TG_CUDA(cudaEventCreate(&e));
        events_.push_back(e);
    }
}

void Pool::ensure_stage(std::size_t bytes) {
    if (bytes <= stage_cap_) return;
    std::size_t n = stage_cap_ ? stage_cap_ : 1 << 16;
    while (n < bytes) n *= 2;
    if (h_stage_) {
        TG_CUDA(cudaStreamSynchronize(s_main_));
        cudaFreeHost(h_stage_);
        cudaFree(d_stage_);
    }
    TG_CUDA(cudaMallocHost(&h_stage_, n));
    TG_CUDA(cudaMalloc(&d_stage_, n));
    resident_clean_ = false;
    // pinned memory is mapped (UVA): the load kernel's last warp writes the
    // digests straight into it, no D2H copy after the launch
    TG_CUDA(cudaHostGetDevicePointer(&h_stage_dev_, h_stage_, 0));
    stage_cap_ = n;
}

namespace {

bool overlaps(u64 a, u64 alen, u64 b, u64 blen) { return a < b + blen && b < a + alen; }

double ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    TG_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

// Tile prefix for a list of (ptr, n) tasks; returns total tiles.
u64 build_tasks(std::vector<FpTask>& tasks) {
    u64 tiles = 0;
    for (auto& t : tasks) {
        t.tile0 = tiles;
        const u64 leaves = (t.n + kLeafBytes - 1) / kLeafBytes;
        tiles += (leaves + kLeavesPerTile - 1) / kLeavesPerTile;
    }
    return tiles;
}

}  // namespace

void Pool::sync_all_streams() noexcept {
    if (!has_device()) return;
    cudaSetDevice(device_);
    for (cudaStream_t s : {s_main_, s_copy_, s_fp_, s_peer_, s_verify_})
        if (s) cudaStreamSynchronize(s);
    cudaGetLastError();
}

// Failure semantics (reuse_store.hpp:117-119 for what the reference can fail
// on): planning errors and missing byte sources are found before anything
// changes, so those failures leave the pool unchanged.  Runtime failures
// after the commit (a short checkpoint read, a CUDA error, bytes that fail
// their fingerprint with no source to repair them) keep the reference's
// decision — the store is what ReuseStore::load_model would have made it —
// but every tensor whose bytes the load wrote is marked suspect before the
// first byte moves and cleared only once verified (or landed, when the
// caller asked for no fingerprints).  A suspect tensor is never exported or
// used as a source, and its next reuse verifies it and re-sends it from its
// registered source: no unverified bytes are ever reused.
St Pool::load_model(const ModelDesc& m, const StatsView& stats, double clock, const LoadOptions& opt, u32 flags,
                    LoadReport* rep) {
    complete_pending();  // a deferred failure stays reported by tg_pool_sync; its tensors are suspect
    try {
        return load_model_impl(m, stats, clock, opt, flags, rep);
    } catch (...) {
        ++totals_.failed_loads;
        if (stager_) stager_->end();  // readers still ahead of a failed issue loop
        if (rep->committed && has_device()) {
            sync_all_streams();  // nothing of this load may still be writing when we return
            rep->suspect_after = 0;
            for (const auto& t : m.tensors)
                if (const Entry* e = store_.entry(t.id); e && e->suspect) ++rep->suspect_after;
        }
        throw;
    }
}

St Pool::load_model_impl(const ModelDesc& m, const StatsView& stats, double clock, const LoadOptions& opt,
                         u32 flags, LoadReport* rep) {
    using clk = std::chrono::steady_clock;
    NvtxRange nvtx_load("tg.load_model");
    *rep = LoadReport{};
    std::unique_ptr<DeviceScope> ds;
    if (has_device()) {
        ds = std::make_unique<DeviceScope>(device_);
        ensure_events(9);
        wait_readers();
        TG_CUDA(cudaEventRecord(ev(0), s_main_));  // t0: entry
    }
    const auto h0 = clk::now();
    auto dec = [&] {
        NvtxRange r("tg.plan");
        return store_.decide(m, stats, opt);
    }();
    rep->t.plan_us = std::chrono::duration<double, std::micro>(clk::now() - h0).count();
    if (!dec) return dec.error();
    LoadDecision& d = dec.value();

    // Resolve a byte source for every miss before anything changes, so a
    // missing source leaves the store untouched (like a failed plan).
    const std::size_t np = d.plan.placements.size();
    std::vector<HostSource> src(np);
    std::vector<const std::uint8_t*> peer_src(np, nullptr);
    std::vector<Digest> peer_digest(np);  // what the peer's index says the bytes fingerprint to
    std::vector<std::vector<MoveDesc>> pieces(np);  // re-shard pulls: src, dst offset in the tensor, len
    std::vector<u64> local_piece_bytes(np, 0);       // ... of which sourced from this pool (HBM)
    // The content truth each placement is checked against, when one is known
    // before the bytes land: the peer's recorded digest, or the source's
    // expected (manifest) digest.  Without one, the landed bytes' digest is
    // recorded as the truth.
    std::vector<Digest> truth(np);
    std::vector<char> has_truth(np, 0);
    rep->placement_src.assign(np, 0);
    if (has_device() && (flags & kLoadPeer) && np) {
        // A peer whose asynchronous load is still placing tensors we miss
        // lands first: its digests are the truth our pulls are checked
        // against.  Peers busy with unrelated models keep running.
        std::vector<Key> want;
        for (const Place& pl : d.plan.placements) want.push_back(d.miss_desc[pl.tensor].id);
        for (Pool* p : peers_)
            if (p->pending_shares(want)) p->complete_pending();
    }
    if (has_device()) {
        for (std::size_t i = 0; i < np; ++i) {
            const TensorDesc& t = d.miss_desc[d.plan.placements[i].tensor];
            if (flags & kLoadPeer) {
                for (Pool* p : peers_) {
                    const Entry* e = p->store_.entry(t.id);
                    if (e && e->size == t.size && e->has_digest && !e->suspect) {
                        peer_src[i] = p->arena_ + e->off;
                        peer_digest[i] = e->digest;
                        rep->placement_src[i] = 1;
                        break;
                    }
                }
                for (std::size_t r = 0; !peer_src[i] && r < remotes_.size(); ++r) {
                    auto it = remotes_[r].index.find(t.id);
                    if (it != remotes_[r].index.end() && it->second.size == t.size) {
                        peer_src[i] = remotes_[r].base + it->second.off;
                        peer_digest[i] = it->second.digest;
                        rep->placement_src[i] = 1;
                    }
                }
            }
            if (peer_src[i]) {
                truth[i] = peer_digest[i];
                has_truth[i] = 1;
                continue;
            }
            if ((flags & kLoadPeer) && assemble_shard(t, &pieces[i], &d.plan, &local_piece_bytes[i])) {
                rep->placement_src[i] = 3;
                continue;
            }
            if (!SourceRegistry::get().find(t.id, &src[i]) || src[i].size != t.size)
                throw DeviceError(kErrNoSource, "no host source registered for tensor " + t.id.hex() + " (" +
                                                    t.model_id + "/" + t.name + ")");
            if (src[i].is_file()) check_file_source(src[i], t.id);
            if (src[i].has_expected) {
                truth[i] = src[i].expected;
                has_truth[i] = 1;
            }
            if (src[i].on_device) {  // HBM-resident model cache: SM copy, not the PCIe engine
                if (src[i].device >= 0 && src[i].device != device_) enable_peer_access(src[i].device);
                peer_src[i] = static_cast<const std::uint8_t*>(src[i].ptr);
                rep->placement_src[i] = 2;
            }
        }
    }

    // Relocation waves: wave(k) = 1 + max wave(j), j < k, dst_k ∩ src_j ≠ ∅.
    // The planner moves each tensor at most once and only into free space
    // (packing.hpp:412-456), so write-after-read is the only hazard it
    // produces.  Read-after-write / write-after-write edges (a tensor moved
    // twice) also raise the wave, and route the load through the separately
    // launched waves: the load kernel prefetches a gated tile's sources
    // before its gate opens, which is only safe for WAR.
    // (copy: the decision is moved into the report below)
    const std::vector<Move> rel = d.plan.relocations;
    rep->reloc_wave.assign(rel.size(), 0);
    u32 waves = 0;
    bool raw_edges = false;
    for (std::size_t k = 0; k < rel.size(); ++k) {
        u32 w = 0;
        for (std::size_t j = 0; j < k; ++j) {
            const bool war = overlaps(rel[k].to, rel[k].size, rel[j].from, rel[j].size);
            const bool raw = overlaps(rel[k].from, rel[k].size, rel[j].to, rel[j].size) ||
                             overlaps(rel[k].to, rel[k].size, rel[j].to, rel[j].size);
            raw_edges = raw_edges || raw;
            if (war || raw) w = std::max(w, rep->reloc_wave[j] + 1);
        }
        rep->reloc_wave[k] = w;
        waves = std::max(waves, w + 1);
    }
    rep->waves = waves;
    // A placement must wait for the last wave that reads bytes it overwrites.
    std::vector<int> dep(np, -1);
    for (std::size_t i = 0; i < np; ++i) {
        const auto& pl = d.plan.placements[i];
        const u64 sz = d.miss_desc[pl.tensor].size;
        for (std::size_t j = 0; j < rel.size(); ++j)
            if (overlaps(pl.off, sz, rel[j].from, rel[j].size)) dep[i] = std::max(dep[i], static_cast<int>(rep->reloc_wave[j]));
    }

    // Reused tensors to verify: all of them with kLoadVerifyReuse, and the
    // suspect ones (left unverified by an earlier failed load) in any case.
    // A suspect tensor without a recorded digest can only be re-sent, so its
    // source must exist now, before anything changes.
    std::vector<Key> hit_keys;
    std::vector<u32> hit_pos;  // position in m.tensors, parallel to hit_keys
    for (u32 i : d.hits) {
        const Key& k = m.tensors[i].id;
        const Entry* e = store_.entry(k);
        if (!(flags & kLoadVerifyReuse) && !e->suspect) continue;
        if (has_device() && e->suspect && !e->has_digest) {
            HostSource hs;
            if (!SourceRegistry::get().find(k, &hs) || hs.size != e->size)
                throw DeviceError(kErrNoSource, "suspect tensor " + k.hex() + " has no source to re-send it from");
            if (hs.is_file()) check_file_source(hs, k);
        }
        hit_keys.push_back(k);
        hit_pos.push_back(i);
    }
    store_.commit(m, d, clock);
    rep->committed = true;
    rep->decision = std::move(d);
    LoadDecision& D = rep->decision;
    if (!has_device()) return ok();

    // Write-ahead: every tensor whose bytes this load writes is suspect from
    // here until verified (placements start without a digest unless a truth
    // is known; a relocated tensor keeps its digest, the content does not
    // change by moving).
    std::vector<char> prior_suspect;  // relocated tensors' state before this load, by relocation
    for (std::size_t i = 0; i < np; ++i) {
        Entry* e = store_.entry(D.miss_desc[D.plan.placements[i].tensor].id);
        e->suspect = true;
        if (has_truth[i]) {
            e->digest = truth[i];
            e->has_digest = true;
        }
    }
    for (std::size_t j = 0; j < D.plan.relocations.size(); ++j) {
        Entry* e = store_.entry(D.plan.relocations[j].tensor);
        char was = e->suspect;  // a tensor moved twice keeps its state from before the first move
        for (std::size_t i = 0; i < j; ++i)
            if (D.plan.relocations[i].tensor == D.plan.relocations[j].tensor) was = prior_suspect[i];
        prior_suspect.push_back(was);
        e->suspect = true;
    }

    for (std::size_t i = 0; i < np; ++i) {
        const u64 sz = D.miss_desc[D.plan.placements[i].tensor].size;
        const std::uint8_t k = rep->placement_src[i];
        if (k == 3) {  // re-shard pieces: NVLink from peers, HBM from this pool
            rep->peer_bytes += sz - local_piece_bytes[i];
            rep->device_src_bytes += local_piece_bytes[i];
            continue;
        }
        (k == 0 ? rep->pcie_bytes : k == 1 ? rep->peer_bytes : rep->device_src_bytes) += sz;
    }

    // ---- event layout -----------------------------------------------------------
    // 0 t0 | 1 reloc start | 2 reloc end | 3 end | 4 h2d start | 5 h2d end | 6 peer start | 7 peer end
    // 8 verify joined | 9.. wave ends (waves) | then per placement "bytes landed" | then fp start/end pairs
    const bool fused = (flags & kLoadFused) != 0 && !raw_edges;
    const std::size_t ev_wave = 9, ev_land = ev_wave + waves, ev_fp = ev_land + np;
    const bool fp_new = flags & kLoadFingerprintNew, fp_reuse = !hit_keys.empty();
    // Reused tensors no relocation touches are verified right away on the
    // verify stream, in parallel with the waves.  Relocated ones are verified
    // by the copy+fingerprint (K3F) of their wave — or, unfused, by a K1
    // launch after the waves.  hit_keys is reordered [untouched..., relocated...].
    // (tens of tensors and relocations per load: linear scans, no hashing)
    constexpr std::size_t kNone = ~std::size_t{0};
    constexpr std::size_t kPostTask = std::size_t{1} << 62;  // provisional index of a post-kernel task
    auto reloc_index = [&](const Key& k) {
        for (std::size_t j = 0; j < rel.size(); ++j)
            if (rel[j].tensor == k) return j;
        return kNone;
    };
    std::vector<std::size_t> hit_rel;  // relocation of each hit (kNone: untouched), parallel to hit_keys
    std::size_t n_still = hit_keys.size();
    if (fp_reuse) {
        std::vector<std::size_t> idx(hit_keys.size());
        for (std::size_t h = 0; h < idx.size(); ++h) idx[h] = h;
        std::vector<std::size_t> rel_of(hit_keys.size());
        for (std::size_t h = 0; h < idx.size(); ++h) rel_of[h] = rel.empty() ? kNone : reloc_index(hit_keys[h]);
        auto mid = std::stable_partition(idx.begin(), idx.end(), [&](std::size_t h) { return rel_of[h] == kNone; });
        n_still = static_cast<std::size_t>(mid - idx.begin());
        std::vector<Key> hk(idx.size());
        std::vector<u32> hp(idx.size());
        hit_rel.resize(idx.size());
        for (std::size_t h = 0; h < idx.size(); ++h) {
            hk[h] = hit_keys[idx[h]];
            hp[h] = hit_pos[idx[h]];
            hit_rel[h] = rel_of[idx[h]];
        }
        hit_keys.swap(hk);
        hit_pos.swap(hp);
    }
    // K1 after landing: host-sourced placements always; device-sourced ones
    // only when unfused (fused: K3F hashes them while it copies)
    // (re-shard pulls, kind 3, are assembled from several pieces: K1 after the last lands)
    // (bytes pulled from a peer — kinds 1 and 3 — are always fingerprinted:
    // that check is what makes a stale peer index safe)
    // Re-shard pulls into free space (no wave gate) are assembled by the load
    // kernel itself: each piece's leaf-aligned interior is a copy task hashed
    // from its own read (seeds from the piece's leaf index, raw sums added on
    // the host), and the few leaves that straddle a piece boundary are
    // pre-copied by K3 and verified in place — two HBM passes instead of
    // three (K3 pieces, then K1 over the assembled tensor).  A pull into bytes
    // a relocation wave has yet to read takes the wave's gate for its piece
    // tasks and copies its straddle fragments inside the load kernel too (a
    // K3 pre-copy would overwrite them before the wave); its straddle leaves
    // are then verified by a second, small launch after the load kernel.
    auto fuse_reshard = [&](std::size_t i) { return fused && rep->placement_src[i] == 3; };
    auto k1_placement = [&](std::size_t i) {
        const std::uint8_t k = rep->placement_src[i];
        if (k == 3 && fuse_reshard(i)) return false;
        return (fp_new || k == 1 || k == 3) && (!fused || k == 0 || k == 3);
    };
    auto tiles_of = [](u64 n) { return ((n + kLeafBytes - 1) / kLeafBytes + kLeavesPerTile - 1) / kLeavesPerTile; };

    // ---- descriptor tables (one H2D) ---------------------------------------------
    // FpTask (K1): [K1 placements...][unfused: untouched hits..., relocated hits...]
    // CopyFpTask (fused: one load-kernel launch), in tile order, for g = 0..waves:
    //   [wave g moves, gate g-1][device-source placements gated on wave g-1]
    //   [a share of the in-place verifications of untouched hits]
    // The verification share behind each gate keeps the warps that run out of
    // gated work streaming while the wave's last tiles finish; the rest of the
    // verifications follow the last group.
    std::vector<FpTask> tasks;
    std::vector<std::size_t> fp_of_placement(np, kNone);
    std::vector<u64> new_tiles;
    for (std::size_t i = 0; i < np; ++i) {
        if (!k1_placement(i)) continue;
        const auto& pl = D.plan.placements[i];
        fp_of_placement[i] = tasks.size();
        tasks.push_back(FpTask{arena_ + pl.off, D.miss_desc[pl.tensor].size, 0});
        new_tiles.push_back(tiles_of(tasks.back().n));
    }
    const std::size_t hit_base = tasks.size();
    u64 still_tiles = 0, moved_tiles = 0;
    // A fused load whose load kernel writes verifies its untouched hits in a
    // concurrent K1 launch (verify_split); a load kernel that would only
    // verify (a warm reload) stays one lone launch.
    bool kernel_writes = !rel.empty();
    for (std::size_t i = 0; i < np; ++i) kernel_writes = kernel_writes || rep->placement_src[i] != 0;
    // Verification tiles per gate inside the load kernel: `rounds` resident-
    // warp rounds behind each wave's tasks (they fill the gate waits).  Split,
    // the share behind the last group (the bulk) goes to the K1 launch
    // instead: hits [0, k_in) are verified in the load kernel, [k_in, n_still)
    // by K1.
    const u64 share = (fused ? verify_rounds(split_candidate(fused, fp_reuse, kernel_writes, n_still, waves)) : 0) *
                      copy_fp_resident_warps(sm_count_);
    std::size_t k_in = 0;
    for (u32 g = 0; g < waves && split_candidate(fused, fp_reuse, kernel_writes, n_still, waves); ++g)
        for (u64 got = 0; k_in < n_still && got < share; ++k_in) got += tiles_of(store_.entry(hit_keys[k_in])->size);
    const bool split = split_candidate(fused, fp_reuse, kernel_writes, n_still, waves) && k_in < n_still;
    if (fp_reuse && (!fused || split)) {
        std::vector<FpTask> still, moved_hits;
        for (std::size_t h = split ? k_in : 0; h < (split ? n_still : hit_keys.size()); ++h) {
            const Entry* e = store_.entry(hit_keys[h]);
            (h < n_still ? still : moved_hits).push_back(FpTask{arena_ + e->off, e->size, 0});
        }
        still_tiles = build_tasks(still);
        moved_tiles = build_tasks(moved_hits);
        tasks.insert(tasks.end(), still.begin(), still.end());
        tasks.insert(tasks.end(), moved_hits.begin(), moved_hits.end());
    }
    std::vector<CopyFpTask> ctasks;
    std::vector<std::size_t> ctask_of_reloc(rel.size(), kNone), ctask_of_placement(np, kNone),
        ctask_of_still(hit_keys.size(), kNone);
    std::vector<u64> need(waves, 0);
    u64 ctiles = 0;
    std::vector<std::vector<std::size_t>> ctasks_of_reshard(np);  // fused re-shard: its piece / straddle tasks
    std::vector<MoveDesc> reshard_pre;                            // straddle fragments, K3 before the kernel
    std::vector<CopyFpTask> post;  // straddle leaves of gated re-shard pulls: verified after the load kernel
    u64 post_tiles = 0;
    if (fused) {
        auto push = [&](const std::uint8_t* from, std::uint8_t* to, u64 n, int gate, int wave, u64 leaf_base = 0) {
            ctasks.push_back(CopyFpTask{from, to, n, ctiles, gate, wave, leaf_base});
            ctiles += tiles_of(n);
            if (wave >= 0) need[static_cast<std::size_t>(wave)] += tiles_of(n);
        };
        auto push_reshard = [&](std::size_t i) {
            std::uint8_t* dst = arena_ + D.plan.placements[i].off;
            const u64 n = D.miss_desc[D.plan.placements[i].tensor].size;
            const int gate = dep[i];  // >= 0: the wave whose reads this pull must follow
            std::vector<u64> straddle;  // leaves touched by a fragment
            auto fragment = [&](const std::uint8_t* from, u64 a, u64 b) {
                if (a >= b) return;
                if (gate < 0) reshard_pre.push_back(MoveDesc{reinterpret_cast<u64>(from), reinterpret_cast<u64>(dst + a), b - a});
                else push(from, dst + a, b - a, gate, -1);  // copied in the kernel after the wave (sums unused)
                for (u64 l = a / kLeafBytes; l * kLeafBytes < b; ++l) straddle.push_back(l);
            };
            for (const MoveDesc& pc : pieces[i]) {  // pc: src pointer, offset in the tensor, length
                const auto* src = reinterpret_cast<const std::uint8_t*>(pc.src);
                const u64 a = pc.dst, b = pc.dst + pc.len;
                const u64 A = (a + kLeafBytes - 1) / kLeafBytes * kLeafBytes;
                const u64 B = b == n ? n : b / kLeafBytes * kLeafBytes;
                if (A < B) {
                    ctasks_of_reshard[i].push_back(ctasks.size());
                    push(src + (A - a), dst + A, B - A, gate, -1, (A / kLeafBytes) | kRawSums);
                    fragment(src, a, A);
                    fragment(src + (B - a), B, b);
                } else {
                    fragment(src, a, b);
                }
            }
            std::sort(straddle.begin(), straddle.end());
            straddle.erase(std::unique(straddle.begin(), straddle.end()), straddle.end());
            for (u64 l : straddle) {
                const u64 len = std::min<u64>(kLeafBytes, n - l * kLeafBytes);
                if (gate >= 0) {  // index in ctasks once `post` is appended behind the load kernel's tasks
                    ctasks_of_reshard[i].push_back(kPostTask + post.size());
                    post.push_back(CopyFpTask{dst + l * kLeafBytes, nullptr, len, post_tiles, -1, -1, l | kRawSums});
                    post_tiles += tiles_of(len);
                    continue;
                }
                ctasks_of_reshard[i].push_back(ctasks.size());
                push(dst + l * kLeafBytes, nullptr, len, -1, -1, l | kRawSums);
            }
        };
        for (std::size_t i = 0; i < np; ++i)
            if (fuse_reshard(i) && dep[i] < 0) push_reshard(i);
        const std::size_t n_verify = fp_reuse ? (split ? k_in : n_still) : 0;
        std::size_t next_verify = 0;
        for (u32 g = 0; g <= waves; ++g) {
            const int gate = static_cast<int>(g) - 1;
            for (std::size_t j = 0; g < waves && j < rel.size(); ++j) {
                if (rep->reloc_wave[j] != g) continue;
                ctask_of_reloc[j] = ctasks.size();
                push(arena_ + rel[j].from, arena_ + rel[j].to, rel[j].size, gate, static_cast<int>(g));
            }
            for (std::size_t i = 0; i < np; ++i) {
                if (rep->placement_src[i] == 0 || dep[i] != gate || (gate < 0 && rep->placement_src[i] == 3)) continue;
                if (rep->placement_src[i] == 3) {  // gated re-shard pull: its pieces follow the wave
                    push_reshard(i);
                    continue;
                }
                ctask_of_placement[i] = ctasks.size();
                push(peer_src[i], arena_ + D.plan.placements[i].off, D.miss_desc[D.plan.placements[i].tensor].size,
                     gate, -1);
            }
            for (u64 got = 0; next_verify < n_verify && (g == waves || got < share); ++next_verify) {
                const Entry* e = store_.entry(hit_keys[next_verify]);
                ctask_of_still[next_verify] = ctasks.size();
                push(arena_ + e->off, nullptr, e->size, -1, -1);
                got += tiles_of(e->size);
            }
        }
    }
    // the post-kernel straddle verifications go behind the load kernel's tasks
    // (their tile numbers restart at 0: a launch of their own)
    const std::size_t nc_main = ctasks.size();
    for (auto& v : ctasks_of_reshard)
        for (std::size_t& k : v)
            if (k >= kPostTask) k = nc_main + (k - kPostTask);
    ctasks.insert(ctasks.end(), post.begin(), post.end());
    const std::size_t nf = tasks.size(), nc = ctasks.size();
    std::size_t n_fp_launch = 2 + (post.empty() ? 0 : 1);
    for (std::size_t i = 0; i < np; ++i) n_fp_launch += fp_of_placement[i] != kNone;
    const std::size_t ev_gate = ev_fp + 2 * n_fp_launch;  // copy stream: first gated H2D may start
    ensure_events(ev_gate + 1);
    // stage: [FpTask...][CopyFpTask...][need...] (H2D) | sums | digests | sync
    const std::size_t fdesc = nf * sizeof(FpTask), cdesc = nc * sizeof(CopyFpTask), ndesc = waves * sizeof(u64);
    const std::size_t desc_bytes = (fdesc + cdesc + ndesc + 15) & ~std::size_t{15};
    const std::size_t sums_bytes = (nf + nc) * 2 * sizeof(u64);
    // stage: [descriptors][sums = 0][sync counters = 0][digests]; the first
    // three go up in one H2D, so no memset precedes the kernels
    const std::size_t sync_bytes = (2 + waves + 2 * n_fp_launch) * sizeof(u64);
    ensure_stage(desc_bytes + 2 * sums_bytes + sync_bytes + 64);
    auto* h = static_cast<std::uint8_t*>(h_stage_);
    auto* dptr = static_cast<std::uint8_t*>(d_stage_);
    if (nf) std::memcpy(h, tasks.data(), fdesc);
    if (nc) std::memcpy(h + fdesc, ctasks.data(), cdesc);
    if (waves) std::memcpy(h + fdesc + cdesc, need.data(), ndesc);
    std::memset(h + desc_bytes, 0, sums_bytes + sync_bytes);
    // A load kernel with verification tasks only (a warm reload) runs as K1:
    // the same tiles as fingerprint-only tasks, whose smaller descriptor
    // keeps the tile loop leaner (K1 6.36-6.46 TB/s vs 6.31-6.34 for the
    // verification tasks of a writing launch, misaligned, same box).
    bool verify_only = fused && nc && waves == 0;
    for (const CopyFpTask& t : ctasks) verify_only = verify_only && t.dst == nullptr && t.leaf_base == 0;
    if (verify_only) {
        auto* ft = reinterpret_cast<FpTask*>(h + fdesc);
        for (std::size_t k = 0; k < nc; ++k) ft[k] = FpTask{ctasks[k].src, ctasks[k].n, ctasks[k].tile0};
        std::memset(h + fdesc + nc * sizeof(FpTask), 0, cdesc - nc * sizeof(FpTask));
    }
    const auto* d_tasks = reinterpret_cast<const FpTask*>(dptr);
    const auto* d_ctasks = reinterpret_cast<const CopyFpTask*>(dptr + fdesc);
    const auto* d_need = reinterpret_cast<const u64*>(dptr + fdesc + cdesc);
    auto* d_sums = reinterpret_cast<u64*>(dptr + desc_bytes);
    auto* d_sync = reinterpret_cast<u64*>(dptr + desc_bytes + sums_bytes);
    // digests: written by the kernels into mapped pinned memory (read after
    // the stream synchronises; no D2H)
    auto* d_dig = reinterpret_cast<u64*>(static_cast<std::uint8_t*>(h_stage_dev_) + desc_bytes + sums_bytes + sync_bytes);
    u64* d_fp_sync = d_sync + 2 + waves;  // two counters (tiles, finished CTAs) per K1 launch
    // the load kernel's globaltimer stamps (start, end), mapped like the digests
    const std::size_t stamp_off = desc_bytes + 2 * sums_bytes + sync_bytes;
    auto* h_stamps = reinterpret_cast<u64*>(h + stamp_off);
    auto* d_stamps = reinterpret_cast<u64*>(static_cast<std::uint8_t*>(h_stage_dev_) + stamp_off);
    h_stamps[0] = h_stamps[1] = h_stamps[2] = h_stamps[3] = 0;  // load kernel, split K1
    // Side streams join only when they carry work: a load with neither host
    // nor peer-stream placements (a warm reload) is the load kernel alone on
    // the pool stream, with no cross-stream dependency to resolve at its end
    // and no events around the kernel (its span comes from its stamps).
    bool copy_used = false, peer_used = false, fp_used = false;
    for (std::size_t i = 0; i < np; ++i) {
        copy_used = copy_used || rep->placement_src[i] == 0;
        peer_used = peer_used || (rep->placement_src[i] == 3 && !fuse_reshard(i)) ||
                    (rep->placement_src[i] != 0 && !fused);
        fp_used = fp_used || fp_of_placement[i] != kNone;
    }
    const bool lone = fused && ctiles && !copy_used && !peer_used && !fp_used && !split && post.empty();
    // Resident descriptors: a lone load kernel leaves its sums and counters
    // zeroed (it cleans up after its digests), so a load whose descriptors
    // equal the ones already on the device (a reload of an unchanged model)
    // launches with no upload in front of the kernel.
    const bool resident = lone && resident_clean_ && resident_desc_.size() == desc_bytes &&
                          resident_layout_ == std::make_pair(sums_bytes, sync_bytes) &&
                          std::memcmp(resident_desc_.data(), h, desc_bytes) == 0;
    resident_clean_ = false;  // until this load's kernel has cleaned up
    if (nf + nc && !resident) {
        TG_CUDA(cudaMemcpyAsync(dptr, h, desc_bytes + sums_bytes + sync_bytes, cudaMemcpyHostToDevice, s_main_));
        resident_desc_.assign(h, h + desc_bytes);
        resident_layout_ = {sums_bytes, sync_bytes};
    }

    // ---- device work on the main stream: the load kernel (fused) or the K3
    // relocation waves (unfused) ----------------------------------------------------
    if (!lone) TG_CUDA(cudaEventRecord(ev(1), s_main_));
    if (fused && !reshard_pre.empty()) {  // straddle leaves of fused re-shard pulls, verified by the kernel
        relocate_launch(reshard_pre.data(), static_cast<int>(reshard_pre.size()), sm_count_, s_main_);
        TG_CUDA(cudaGetLastError());
    }
    if (fused) {
        if (verify_only)
            fp_launch(reinterpret_cast<const FpTask*>(d_ctasks), static_cast<u32>(nc), ctiles, d_sums + 2 * nf,
                      d_dig + 2 * nf, d_sync, sm_count_, s_main_, /*sync_zeroed=*/true, d_stamps, /*clean=*/lone);
        else
            copy_fp_launch(d_ctasks, static_cast<u32>(nc_main), ctiles, d_sums + 2 * nf, d_dig + 2 * nf, d_sync, d_need,
                           waves, sm_count_, s_main_, /*sync_zeroed=*/true, d_stamps, /*clean=*/lone);
        TG_CUDA(cudaGetLastError());
        for (u32 w = 0; w < waves; ++w) TG_CUDA(cudaEventRecord(ev(ev_wave + w), s_main_));
        for (std::size_t i = 0; i < np; ++i)
            if (ctask_of_placement[i] != kNone) TG_CUDA(cudaEventRecord(ev(ev_land + i), s_main_));
        if (!post.empty()) {  // straddle leaves of gated re-shard pulls, written by the load kernel above
            copy_fp_launch(d_ctasks + nc_main, static_cast<u32>(post.size()), post_tiles, d_sums + 2 * (nf + nc_main),
                           d_dig + 2 * (nf + nc_main), d_fp_sync + 2 * (n_fp_launch - 1), nullptr, 0, sm_count_, s_main_,
                           /*sync_zeroed=*/true, nullptr, /*clean=*/false);
            TG_CUDA(cudaGetLastError());
        }
    }
    for (u32 w = 0; !fused && w < waves; ++w) {
        std::vector<MoveDesc> mv;
        for (std::size_t j = 0; j < rel.size(); ++j)
            if (rep->reloc_wave[j] == w)
                mv.push_back(MoveDesc{reinterpret_cast<u64>(arena_ + rel[j].from), reinterpret_cast<u64>(arena_ + rel[j].to),
                                      rel[j].size});
        relocate_launch(mv.data(), static_cast<int>(mv.size()), sm_count_, s_main_);
        TG_CUDA(cudaGetLastError());
        TG_CUDA(cudaEventRecord(ev(ev_wave + w), s_main_));
    }
    if (!lone) TG_CUDA(cudaEventRecord(ev(2), s_main_));

    // ---- placements: host→device on the copy stream, device sources (peer pool,
    // HBM cache) on the peer stream.  Independent placements first, then those
    // gated on a relocation wave.
    std::vector<std::size_t> order(np);
    for (std::size_t i = 0; i < np; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return dep[a] < dep[b]; });
    if (copy_used) {
        TG_CUDA(cudaStreamWaitEvent(s_copy_, ev(0)));
        TG_CUDA(cudaEventRecord(ev(4), s_copy_));
    }
    if (peer_used) {
        TG_CUDA(cudaStreamWaitEvent(s_peer_, ev(1)));  // K3F reads its descriptors
        TG_CUDA(cudaEventRecord(ev(6), s_peer_));
    }
    // Gates: unfused, the event after wave w's K3 launch.  Fused, the load
    // kernel's own counter of wave w's finished tiles (each bumped with a
    // release after the tile's last read of its source): the stream waits
    // for done[w] >= need[w] (cuStreamWaitValue64), once the counters of this
    // load are zeroed (ev 1), so the H2D overlaps the rest of the launch.
    int waited_copy = -1, waited_peer = -1;
    bool zeroed_copy = false, zeroed_peer = false, gate_recorded = false;
    const WaitValue64Fn wv = fused ? wait_value64() : nullptr;
    auto gate = [&](cudaStream_t s, bool& zeroed, int w) {
        if (wv) {
            if (!zeroed) {
                TG_CUDA(cudaStreamWaitEvent(s, ev(1)));
                zeroed = true;
            }
            const CUresult r = wv(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(d_sync + 1 + w),
                                  need[static_cast<std::size_t>(w)], CU_STREAM_WAIT_VALUE_GEQ);
            if (r == CUDA_SUCCESS) return;
        }
        TG_CUDA(cudaStreamWaitEvent(s, ev(ev_wave + w)));
    };
    // Device-sourced placements (peer pool, HBM cache, re-shard pieces), whole,
    // in gate order on the peer stream (fused: inside the load kernel).
    std::vector<std::size_t> land_order;  // placements in the order their last byte is enqueued
    for (std::size_t i : order) {
        const auto& pl = D.plan.placements[i];
        const u64 sz = D.miss_desc[pl.tensor].size;
        if (rep->placement_src[i] == 0) continue;
        if (fused && (rep->placement_src[i] != 3 || fuse_reshard(i))) continue;  // in the load kernel
        if (dep[i] > waited_peer) {
            gate(s_peer_, zeroed_peer, dep[i]);
            waited_peer = dep[i];
        }
        if (rep->placement_src[i] == 3) {
            std::vector<MoveDesc> mv = pieces[i];
            for (MoveDesc& md : mv) md.dst += reinterpret_cast<u64>(arena_ + pl.off);
            for (std::size_t at = 0; at < mv.size(); at += kMaxMovesPerLaunch) {
                relocate_launch(mv.data() + at, static_cast<int>(std::min<std::size_t>(kMaxMovesPerLaunch, mv.size() - at)),
                                sm_count_, s_peer_);
                TG_CUDA(cudaGetLastError());
            }
        } else {
            MoveDesc md{reinterpret_cast<u64>(peer_src[i]), reinterpret_cast<u64>(arena_ + pl.off), sz};
            relocate_launch(&md, 1, sm_count_, s_peer_);
            TG_CUDA(cudaGetLastError());
        }
        TG_CUDA(cudaEventRecord(ev(ev_land + i), s_peer_));
        land_order.push_back(i);
    }
    // Host-sourced placements on the copy stream, split where relocation
    // sources end: each piece waits only for the last wave that reads the
    // bytes it overwrites (a placement usually overlaps a moved tensor's old
    // range only in part), so the link starts at t = 0 with every ungated
    // piece and the gated ones follow their waves.
    struct Piece {
        std::size_t pl;
        u64 at, len;  // within the tensor
        int dep;
    };
    std::vector<Piece> hp;
    for (std::size_t i = 0; i < np; ++i) {
        if (rep->placement_src[i] != 0) continue;
        const u64 off = D.plan.placements[i].off, sz = D.miss_desc[D.plan.placements[i].tensor].size;
        std::vector<u64> cuts{0, sz};
        for (const Move& r : rel)
            for (u64 c : {r.from, r.from + r.size})
                if (c > off && c < off + sz) cuts.push_back(c - off);
        std::sort(cuts.begin(), cuts.end());
        cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
        for (std::size_t c = 0; c + 1 < cuts.size(); ++c) {
            int w = -1;
            for (std::size_t j = 0; j < rel.size(); ++j)
                if (overlaps(off + cuts[c], cuts[c + 1] - cuts[c], rel[j].from, rel[j].size))
                    w = std::max(w, static_cast<int>(rep->reloc_wave[j]));
            if (!hp.empty() && hp.back().pl == i && hp.back().dep == w) hp.back().len += cuts[c + 1] - cuts[c];
            else hp.push_back(Piece{i, cuts[c], cuts[c + 1] - cuts[c], w});
        }
        if (sz == 0) hp.push_back(Piece{i, 0, 0, -1});
    }
    std::stable_sort(hp.begin(), hp.end(), [](const Piece& a, const Piece& b) { return a.dep < b.dep; });
    // Model Store pieces: the stager's readers start on all of them now and
    // run ahead of the issue loop below.
    std::vector<std::size_t> file_range(hp.size(), kNone);
    {
        std::vector<FileStager::Range> ranges;
        for (std::size_t k = 0; k < hp.size(); ++k)
            if (hp[k].len && src[hp[k].pl].is_file()) {
                file_range[k] = ranges.size();
                ranges.push_back(FileStager::Range{src[hp[k].pl].path, src[hp[k].pl].file_off + hp[k].at, hp[k].len});
            }
        if (!ranges.empty()) {
            if (!stager_) stager_ = make_stager(device_);
            stager_->begin(std::move(ranges));
        }
    }
    std::vector<std::size_t> last_piece(np, kNone);
    for (std::size_t k = 0; k < hp.size(); ++k) last_piece[hp[k].pl] = k;
    for (std::size_t k = 0; k < hp.size(); ++k) {
        const Piece& pc = hp[k];
        if (pc.dep > waited_copy) {
            gate(s_copy_, zeroed_copy, pc.dep);
            waited_copy = pc.dep;
            if (!gate_recorded) {
                TG_CUDA(cudaEventRecord(ev(ev_gate), s_copy_));
                gate_recorded = true;
            }
        }
        std::uint8_t* dst = arena_ + D.plan.placements[pc.pl].off + pc.at;
        const HostSource& hs = src[pc.pl];
        if (pc.len) {
            if (hs.is_file()) {
                stager_->issue(file_range[k], dst, s_copy_);
            } else {
                if (Failpoints::hit("h2d")) throw DeviceError(kErrCuda, "failpoint h2d: injected copy failure");
                TG_CUDA(cudaMemcpyAsync(dst, static_cast<const std::uint8_t*>(hs.ptr) + pc.at, pc.len,
                                        cudaMemcpyHostToDevice, s_copy_));
            }
        }
        if (last_piece[pc.pl] == k) {
            TG_CUDA(cudaEventRecord(ev(ev_land + pc.pl), s_copy_));
            land_order.push_back(pc.pl);
        }
    }
    if (copy_used) TG_CUDA(cudaEventRecord(ev(5), s_copy_));
    if (peer_used) TG_CUDA(cudaEventRecord(ev(7), s_peer_));

    // ---- K1 over placed tensors, trailing the copies ------------------------------
    std::size_t fp_i = 0;
    bool fp_stream_used = false;
    for (std::size_t i : land_order) {
        const std::size_t k = fp_of_placement[i];
        if (k == kNone) continue;
        if (!fp_stream_used) TG_CUDA(cudaStreamWaitEvent(s_fp_, ev(1)));  // descriptors uploaded, sums zeroed
        TG_CUDA(cudaStreamWaitEvent(s_fp_, ev(ev_land + i)));
        TG_CUDA(cudaEventRecord(ev(ev_fp + 2 * fp_i), s_fp_));
        fp_launch(d_tasks + k, 1, new_tiles[k], d_sums + 2 * k, d_dig + 2 * k, d_fp_sync + 2 * fp_i, sm_count_, s_fp_,
                  /*sync_zeroed=*/true);
        TG_CUDA(cudaGetLastError());
        TG_CUDA(cudaEventRecord(ev(ev_fp + 2 * fp_i + 1), s_fp_));
        ++fp_i;
        fp_stream_used = true;
    }
    // ---- K1 over reused tensors: untouched ones now (verify stream); relocated
    // ones after the waves (main stream) unless K3F already hashed them --------
    std::size_t fp_reuse_slot = fp_i, fp_reuse_launches = 0;
    if (fp_reuse && (!fused || split)) {  // fused: the load kernel verifies them
        auto launch = [&](cudaStream_t s, std::size_t first, std::size_t count, u64 tiles) {
            if (!count) return;
            TG_CUDA(cudaEventRecord(ev(ev_fp + 2 * fp_i), s));
            fp_launch(d_tasks + first, static_cast<u32>(count), tiles, d_sums + 2 * first, d_dig + 2 * first,
                      d_fp_sync + 2 * fp_i, sm_count_, s, /*sync_zeroed=*/true, split ? d_stamps + 2 : nullptr);
            TG_CUDA(cudaGetLastError());
            TG_CUDA(cudaEventRecord(ev(ev_fp + 2 * fp_i + 1), s));
            ++fp_i;
            ++fp_reuse_launches;
        };
        TG_CUDA(cudaStreamWaitEvent(s_verify_, ev(1)));
        launch(s_verify_, hit_base, split ? n_still - k_in : n_still, still_tiles);
        if (!fused) launch(s_main_, hit_base + n_still, hit_keys.size() - n_still, moved_tiles);
        TG_CUDA(cudaEventRecord(ev(8), s_verify_));
        TG_CUDA(cudaStreamWaitEvent(s_main_, ev(8)));
    }
    // ---- device index: the committed map, uploaded on a side stream while the
    // data plane runs (the pool stream joins it: valid for work ordered after
    // the load on the pool stream) ---------------------------------------------
    if (store_.epoch() != published_epoch_) {
        TG_CUDA(cudaStreamWaitEvent(s_verify_, ev(0)));
        publish_index(s_verify_);
    }
    // ---- join, read digests, end ------------------------------------------------
    if (copy_used) TG_CUDA(cudaStreamWaitEvent(s_main_, ev(5)));
    if (peer_used) TG_CUDA(cudaStreamWaitEvent(s_main_, ev(7)));
    if (fp_stream_used) {
        TG_CUDA(cudaEventRecord(ev(3), s_fp_));
        TG_CUDA(cudaStreamWaitEvent(s_main_, ev(3)));
    }
    TG_CUDA(cudaEventRecord(ev(3), s_main_));
    auto* h_dig = reinterpret_cast<u64*>(h + desc_bytes + sums_bytes + sync_bytes);
    // Peers this load reads from must not overwrite those bytes before the
    // reads are done: each records our end-of-load event and waits on it
    // before its own next data plane (cross-device stream wait, no host sync).
    for (std::size_t i = 0; i < np; ++i)
        if (!peers_.empty() && (rep->placement_src[i] == 1 || rep->placement_src[i] == 3)) {
            note_readers();
            break;
        }
    const auto h_issued = clk::now();
    rep->t.host_issue_us = std::chrono::duration<double, std::micro>(h_issued - h0).count();

    // ---- completion: wait for the data plane, then record / verify digests.
    // Runs now, or — with kLoadAsync — before the next operation on this pool
    // (complete_pending), so loads on different pools overlap.
    auto finish = [this, h_dig, h_stamps, ctiles, lone, split, k_in, np, nf, fused,
                   ctasks_of_reshard = std::move(ctasks_of_reshard), copy_used, peer_used, hit_base, n_still, fp_reuse, waves, nc, gate_recorded, ev_gate, ev_fp,
                   fp_i, fp_reuse_slot, fp_reuse_launches, h0, h_issued, fp_of_placement = std::move(fp_of_placement),
                   ctask_of_placement = std::move(ctask_of_placement), has_truth = std::move(has_truth),
                   truth = std::move(truth), hit_keys = std::move(hit_keys), hit_pos = std::move(hit_pos),
                   hit_rel = std::move(hit_rel), ctask_of_still = std::move(ctask_of_still),
                   ctask_of_reloc = std::move(ctask_of_reloc), rel = std::move(rel),
                   prior_suspect = std::move(prior_suspect)](LoadReport* rep, const ModelDesc& m) -> int {
    LoadDecision& D = rep->decision;
    {
        NvtxRange r("tg.wait_data_plane");
        // A load that is the load kernel alone: poll its end stamp in mapped
        // memory (written after the digests) — the host sees the end a few
        // microseconds before a stream synchronize would return; the
        // synchronize that follows then finds the stream (nearly) drained.
        if (lone) {
            const volatile u64* end = h_stamps + 1;
            for (std::uint32_t spin = 0; *end == 0 && spin < (1u << 26); ++spin) {
            }
        }
        TG_CUDA(cudaStreamSynchronize(s_main_));
    }
    rep->t.host_wait_us = std::chrono::duration<double, std::micro>(clk::now() - h_issued).count();
    NvtxRange nvtx_verify("tg.record_verify_digests");

    // (each event query costs ~3 us of host time: the load kernel's span comes
    // from its own globaltimer stamps, and a load that is that kernel alone
    // on the pool stream ends with it)
    rep->t.total_ms = ms_between(ev(0), ev(3));
    bool stamped = fused && ctiles && h_stamps[1] > h_stamps[0] && h_stamps[0];
    u64 t_start = h_stamps[0], t_end = h_stamps[1];
    if (split && stamped) {  // and its concurrent verification launch (both stamped)
        stamped = h_stamps[3] > h_stamps[2] && h_stamps[2];
        t_start = std::min(t_start, h_stamps[2]);
        t_end = std::max(t_end, h_stamps[3]);
    }
    // fused: the whole load kernel (waves, device-source placements,
    // verification — split: up to the end of the concurrent K1)
    rep->t.relocate_ms = stamped ? (t_end - t_start) * 1e-6
                                 : (!lone && (waves || (fused && nc))) ? ms_between(ev(1), ev(2)) : 0.0;
    rep->t.kernel_end_ms = lone ? rep->t.total_ms : ms_between(ev(0), ev(2));
    rep->t.gated_h2d_start_ms = gate_recorded ? ms_between(ev(0), ev(ev_gate)) : 0.0;
    rep->t.h2d_ms = copy_used && rep->pcie_bytes ? ms_between(ev(4), ev(5)) : 0.0;
    rep->t.peer_ms = peer_used ? ms_between(ev(6), ev(7)) : 0.0;
    for (std::size_t f = 0; f < fp_i; ++f) {
        const double t = ms_between(ev(ev_fp + 2 * f), ev(ev_fp + 2 * f + 1));
        rep->t.fp_kernel_ms += t;
        if (fp_reuse && f >= fp_reuse_slot && f < fp_reuse_slot + fp_reuse_launches) {
            rep->t.fp_reuse_ms += t;
            rep->t.fp_reuse_max_ms = std::max(rep->t.fp_reuse_max_ms, t);
        }
    }

    // ---- record / verify digests ----------------------------------------------
    // Every tensor is settled before a failure is reported, so one bad tensor
    // does not leave the others of the load suspect.
    auto digest_at = [&](std::size_t slot) { return Digest{h_dig[2 * slot], h_dig[2 * slot + 1]}; };
    int fail = 0;
    std::string fail_what;
    auto fail_with = [&](int code, const std::string& what) {
        if (!fail) {
            fail = code;
            fail_what = what;
        }
    };
    // Re-send a tensor in place from its registered source.  The source is
    // the checkpoint, so what lands is the truth — unless the source carries
    // an expected (manifest) digest the bytes must match.  (A recorded digest
    // does not veto it: it may be a stale peer's claim.)
    auto repair = [&](const Key& k, Entry* e) {
        HostSource hs;
        if (!SourceRegistry::get().find(k, &hs) || hs.size != e->size) return false;
        fetch(hs, arena_ + e->off, e->size, s_main_);
        TG_CUDA(cudaStreamSynchronize(s_main_));
        rep->repaired_bytes += e->size;
        const Digest g = fingerprint_resident(k);
        if (hs.has_expected && !(hs.expected == g)) {
            ++rep->expected_mismatches;
            return false;
        }
        e->digest = g;
        e->has_digest = true;
        e->suspect = false;
        return true;
    };
    rep->digests.assign(m.tensors.size(), Digest{});
    for (std::size_t i = 0; i < np; ++i) {
        const TensorDesc& t = D.miss_desc[D.plan.placements[i].tensor];
        const u32 at = D.misses[D.plan.placements[i].tensor];  // position in m.tensors
        Entry* e = store_.entry(t.id);
        std::size_t slot = kNone;
        if (fp_of_placement[i] != kNone) slot = fp_of_placement[i];
        else if (ctask_of_placement[i] != kNone) slot = nf + ctask_of_placement[i];
        const bool pieces_fused = rep->placement_src[i] == 3 && fused && ctask_of_placement[i] == kNone &&
                                  fp_of_placement[i] == kNone;
        if (slot == kNone && !pieces_fused) {  // landed (the streams are joined), not fingerprinted by request
            e->suspect = false;
            continue;
        }
        Digest g;
        if (pieces_fused) {  // tgfp1 root of the summed raw leaf sums of the pieces and straddle leaves
            u64 sh = 0, sl = 0;
            for (std::size_t k : ctasks_of_reshard[i]) {
                sh += h_dig[2 * (nf + k)];
                sl += h_dig[2 * (nf + k) + 1];
            }
            u64 h1 = 0, h2 = 0;
            mm::body(h1, h2, sh, sl);
            mm::finish(h1, h2, t.size, 0, 8, 24);
            g = Digest{h1, h2};
        } else {
            g = digest_at(slot);
        }
        rep->digests[at] = g;
        rep->fingerprint_bytes += t.size;
        if (!has_truth[i]) {
            e->digest = g;
            e->has_digest = true;
            e->suspect = false;
        } else if (g == truth[i]) {
            e->suspect = false;
        } else if (rep->placement_src[i] == 1) {
            // The peer's index was stale (its bytes changed under us): fetch the
            // tensor from its host source instead.
            ++rep->verify_mismatches;
            if (repair(t.id, e)) rep->digests[at] = e->digest;
            else fail_with(kErrVerify, "peer bytes of " + t.id.hex() + " fail verification and no source repairs them");
        } else {
            // The registered source itself disagrees with its expected digest:
            // nothing here is the truth any more, so the tensor can only be
            // re-sent (from a corrected source) on its next reuse.
            ++rep->expected_mismatches;
            e->has_digest = false;
            fail_with(kErrVerify, "source bytes of " + t.id.hex() + " do not match the expected digest");
        }
    }
    std::vector<char> verified(rel.size(), 0);  // relocated hits settled here
    for (std::size_t hix = 0; fp_reuse && hix < hit_keys.size(); ++hix) {
        const Key& k = hit_keys[hix];
        const std::size_t slot = !fused                                 ? hit_base + hix
                                 : split && hix >= k_in && hix < n_still ? hit_base + (hix - k_in)
                                 : hix < n_still                         ? nf + ctask_of_still[hix]
                                                 : nf + ctask_of_reloc[hit_rel[hix]];
        const Digest g = digest_at(slot);
        Entry* e = store_.entry(k);
        if (hit_rel[hix] != kNone)
            for (std::size_t j = 0; j < rel.size(); ++j) verified[j] |= rel[j].tensor == k;
        rep->digests[hit_pos[hix]] = g;
        rep->fingerprint_bytes += e->size;
        // Whether the tensor was trustworthy before this load: a relocated one
        // is marked suspect by this load until its move is verified, so its
        // state from before the move is what counts.
        const bool was_suspect = hit_rel[hix] != kNone ? prior_suspect[hit_rel[hix]] != 0 : e->suspect;
        if (e->has_digest && e->digest == g) {
            e->suspect = false;
        } else if (!e->has_digest && !was_suspect) {
            // Placed without a fingerprint (kLoadFingerprintNew off) by a load
            // that completed: the first verification records the truth.
            e->digest = g;
            e->has_digest = true;
            e->suspect = false;
        } else {
            // Content drifted (the key says "reuse", the bytes disagree), or a
            // failed load left it unverifiable: re-send it in place from its
            // source (same plan, fresh bytes).
            ++rep->verify_mismatches;
            if (repair(k, e)) rep->digests[hit_pos[hix]] = e->digest;
            else fail_with(kErrVerify, "reused tensor " + k.hex() + " fails verification and cannot be repaired");
        }
    }
    // Relocated tensors not verified above: the load kernel hashed them from
    // the move's own read, so they are checked against their truth for free
    // (a mismatch leaves them suspect, to be repaired on their next reuse);
    // otherwise the completed move leaves them as they were.
    for (std::size_t j = 0; j < rel.size(); ++j) {
        const Key& k = rel[j].tensor;
        if (verified[j]) continue;
        Entry* e = store_.entry(k);
        if (fused && ctask_of_reloc[j] != kNone && e->has_digest) e->suspect = !(digest_at(nf + ctask_of_reloc[j]) == e->digest);
        else e->suspect = prior_suspect[j];
    }
    rep->suspect_after = 0;
    for (const auto& t : m.tensors)
        if (store_.entry(t.id)->suspect) ++rep->suspect_after;
    rep->t.host_total_us = std::chrono::duration<double, std::micro>(clk::now() - h0).count();
    totals_.loads += 1;
    totals_.data_plane_ms += rep->t.total_ms;
    totals_.pcie_bytes += rep->pcie_bytes;
    totals_.peer_bytes += rep->peer_bytes;
    totals_.device_src_bytes += rep->device_src_bytes;
    totals_.fingerprint_bytes += rep->fingerprint_bytes;
    totals_.relocated_bytes += D.plan.total_merge_cost;
    totals_.verify_mismatches += rep->verify_mismatches;
    totals_.repaired_bytes += rep->repaired_bytes;
    if (fail) throw DeviceError(fail, fail_what);
    resident_clean_ = lone;  // the kernel zeroed its sums and counters
    return 0;
    };
    if (flags & kLoadAsync) {
        pending_ = std::make_unique<PendingLoad>();
        pending_->report = *rep;  // the caller keeps the decision; digests / timings land here
        pending_->model = m;
        pending_->finish = std::move(finish);
        return ok();
    }
    finish(rep, m);
    return ok();
}

// Re-shard pull: cover tensor t's parent byte range with resident shards of
// the same parent in any TP layout — on peer pools, and (when `plan` is given)
// in this pool itself, where a shard this load neither evicts nor relocates
// keeps its bytes in place for the whole load (placements only fill free
// space).  Local pieces are preferred (HBM, not NVLink).  Pieces hold the
// source, the destination offset inside t, and the length; *local_bytes
// counts the bytes sourced from this pool.
bool Pool::assemble_shard(const TensorDesc& t, std::vector<MoveDesc>* pieces, const Plan* plan,
                          u64* local_bytes) const {
    ShardOf me;
    if (!ShardLineage::get().find(t.id, &me) || me.size != t.size || t.size == 0) return false;
    struct Cand {
        u64 b, e;
        const std::uint8_t* base;
        bool local;
    };
    std::unordered_map<Key, bool, KeyHash> touched;  // evicted or relocated by this load
    if (plan) {
        for (const Candidate& c : plan->evictions) touched[c.tensor] = true;
        for (const Move& m : plan->relocations) touched[m.tensor] = true;
    }
    std::vector<Cand> cands;
    for (const auto& [kid, of] : ShardLineage::get().children(me.parent)) {
        if (kid == t.id || of.begin >= me.begin + me.size || of.begin + of.size <= me.begin) continue;
        const std::uint8_t* base = nullptr;
        bool local = false;
        if (plan && !touched.count(kid)) {
            const auto it = store_.tensors().find(kid);
            if (it != store_.tensors().end() && it->second.size == of.size && it->second.has_digest &&
                !it->second.suspect) {
                base = arena_ + it->second.off;
                local = true;
            }
        }
        for (std::size_t k = 0; !base && k < peers_.size(); ++k) {
            const Entry* e = peers_[k]->store_.entry(kid);
            if (e && e->size == of.size && e->has_digest && !e->suspect) base = peers_[k]->arena_ + e->off;
        }
        for (std::size_t r = 0; !base && r < remotes_.size(); ++r) {
            auto it = remotes_[r].index.find(kid);
            if (it != remotes_[r].index.end() && it->second.size == of.size) base = remotes_[r].base + it->second.off;
        }
        if (base) cands.push_back(Cand{of.begin, of.begin + of.size, base, local});
    }
    std::vector<MoveDesc> out;
    u64 local = 0;
    const u64 end = me.begin + me.size;
    for (u64 pos = me.begin; pos < end;) {
        const Cand* best = nullptr;
        for (const Cand& c : cands)
            if (c.b <= pos && pos < c.e &&
                (!best || (c.local && !best->local) || (c.local == best->local && c.e > best->e)))
                best = &c;
        if (!best) return false;
        const u64 len = std::min(best->e, end) - pos;
        out.push_back(MoveDesc{reinterpret_cast<u64>(best->base + (pos - best->b)), pos - me.begin, len});
        if (best->local) local += len;
        pos += len;
    }
    *pieces = std::move(out);
    if (local_bytes) *local_bytes = local;
    return true;
}

// Bytes of a registered source into the arena (repair paths).
void Pool::fetch(const HostSource& hs, std::uint8_t* dst, u64 size, cudaStream_t s) {
    if (hs.is_file()) {
        if (!stager_) stager_ = make_stager(device_);
        stager_->stage(hs.path, hs.file_off, size, dst, s);
    } else {
        TG_CUDA(cudaMemcpyAsync(dst, hs.ptr, size, cudaMemcpyDefault, s));
    }
}

St Pool::move_tensor(const Key& k, u64 to) {
    complete_pending();
    const Entry* e = store_.entry(k);
    const u64 from = e ? e->off : 0, size = e ? e->size : 0;
    St st = store_.move_tensor(k, to);
    if (!st || !has_device()) return st;
    DeviceScope ds(device_);
    Entry* moved = store_.entry(k);
    const bool prior = moved->suspect;
    moved->suspect = true;  // until the bytes have moved (a failure leaves it suspect)
    wait_readers();
    MoveDesc md{reinterpret_cast<u64>(arena_ + from), reinterpret_cast<u64>(arena_ + to), size};
    relocate_launch(&md, 1, sm_count_, s_main_);
    TG_CUDA(cudaGetLastError());
    TG_CUDA(cudaStreamSynchronize(s_main_));
    moved->suspect = prior;
    return st;
}

Digest Pool::fingerprint_resident(const Key& k) {
    const Entry* e = store_.entry(k);
    if (!e) throw DeviceError(kErrNoSource, "tensor not resident");
    if (!has_device()) throw DeviceError(kErrNoDevice, "pool has no device");
    Digest d;
    fingerprint_device(arena_ + e->off, e->size, device_, &d);
    return d;
}

// Let this pool's kernels read (and write) HBM of device `other` over NVLink.
void Pool::enable_peer_access(int other) {
    if (other == device_ || std::find(peer_devices_.begin(), peer_devices_.end(), other) != peer_devices_.end())
        return;
    DeviceScope ds(device_);
    int can = 0;
    TG_CUDA(cudaDeviceCanAccessPeer(&can, device_, other));
    if (!can) throw DeviceError(kErrCuda, "no P2P path between devices");
    cudaError_t e = cudaDeviceEnablePeerAccess(other, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "cudaDeviceEnablePeerAccess");
    cudaGetLastError();
    peer_devices_.push_back(other);
}

void Pool::add_peer(Pool* p) {
    if (!has_device() || !p->has_device()) throw DeviceError(kErrNoDevice, "peer pools need devices");
    enable_peer_access(p->device_);
    peers_.push_back(p);
    p->peer_of_.push_back(this);
}

// This load read peer arenas: record the end of its data plane for them.
void Pool::note_readers() {
    if (!ev_reader_) TG_CUDA(cudaEventCreateWithFlags(&ev_reader_, cudaEventDisableTiming));
    TG_CUDA(cudaEventRecord(ev_reader_, s_main_));
    for (Pool* p : peers_) p->reader_events_[this] = ev_reader_;
}

// Before this pool's data plane writes its arena: wait (on the device) for
// every peer that read from it.
void Pool::wait_readers() {
    for (const auto& [q, e] : reader_events_) TG_CUDA(cudaStreamWaitEvent(s_main_, e));
}

int Pool::complete_pending() {
    if (!pending_) return 0;
    std::unique_ptr<PendingLoad> p = std::move(pending_);
    DeviceScope ds(device_);
    int rc = 0;
    last_async_err_.clear();
    try {
        p->finish(&p->report, p->model);
    } catch (const DeviceError& e) {
        rc = e.code;
        last_async_err_ = e.what();
    } catch (const std::exception& e) {
        rc = kErrCuda;
        last_async_err_ = e.what();
    }
    if (rc) {
        ++totals_.failed_loads;
        sync_all_streams();
        p->report.suspect_after = 0;
        for (const auto& t : p->model.tensors)
            if (const Entry* e = store_.entry(t.id); e && e->suspect) ++p->report.suspect_after;
    }
    last_async_ = std::move(p->report);
    last_async_rc_ = rc;
    return rc;
}

// Does this pool's in-flight asynchronous load place any of `keys`, or a
// shard sibling of one (same lineage parent)?
bool Pool::pending_shares(const std::vector<Key>& keys) const {
    if (!pending_) return false;
    std::unordered_map<Key, bool, KeyHash> mine, parents;
    for (const auto& t : pending_->model.tensors) {
        mine[t.id] = true;
        ShardOf s;
        if (ShardLineage::get().find(t.id, &s)) parents[s.parent] = true;
    }
    for (const Key& k : keys) {
        if (mine.count(k)) return true;
        ShardOf s;
        if (!parents.empty() && ShardLineage::get().find(k, &s) && parents.count(s.parent)) return true;
    }
    return false;
}

// S'_peer: bytes of m missing here but resident on a peer — verified there,
// or being placed by the peer's in-flight asynchronous load (which a load of
// ours lands before pulling, see load_model_impl).
u64 Pool::peer_reuse_size(const ModelDesc& m) const {
    u64 s = 0;
    for (const auto& t : m.tensors) {
        if (store_.tensors().count(t.id)) continue;
        bool found = false;
        for (Pool* p : peers_)
            if (const auto it = p->store_.tensors().find(t.id);
                it != p->store_.tensors().end() &&
                ((it->second.has_digest && !it->second.suspect) || p->pending_shares({t.id}))) {
                found = true;
                break;
            }
        for (const RemotePeer& r : remotes_)
            if (!found && r.index.count(t.id)) found = true;
        std::vector<MoveDesc> pieces;  // or assembled from peer shards of another layout
        if (found || (has_device() && assemble_shard(t, &pieces, nullptr, nullptr))) s += t.size;
    }
    return s;
}

// ---- cross-process peers (one process per GPU): CUDA IPC on the arena -----------
void Pool::export_handle(cudaIpcMemHandle_t* h) const {
    if (!has_device()) throw DeviceError(kErrNoDevice, "pool has no device");
    DeviceScope ds(device_);
    TG_CUDA(cudaIpcGetMemHandle(h, arena_));
}

std::vector<RemoteEntry> Pool::index() const {
    std::vector<RemoteEntry> out;
    out.reserve(store_.tensors().size());
    for (const auto& [k, e] : store_.tensors())
        if (e.has_digest && !e.suspect) out.push_back(RemoteEntry{k, e.off, e.size, e.digest});
    return out;
}

int Pool::attach_remote(const cudaIpcMemHandle_t& h, const std::vector<RemoteEntry>& idx) {
    if (!has_device()) throw DeviceError(kErrNoDevice, "pool has no device");
    DeviceScope ds(device_);
    RemotePeer r;
    void* p = nullptr;
    TG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    r.base = static_cast<std::uint8_t*>(p);
    for (const RemoteEntry& e : idx) r.index[e.id] = e;
    remotes_.push_back(std::move(r));
    return static_cast<int>(remotes_.size() - 1);
}

void Pool::update_remote(int id, const std::vector<RemoteEntry>& idx) {
    if (id < 0 || static_cast<std::size_t>(id) >= remotes_.size()) throw DeviceError(104, "bad remote peer id");
    auto& m = remotes_[static_cast<std::size_t>(id)].index;
    m.clear();
    for (const RemoteEntry& e : idx) m[e.id] = e;
}

struct Pool::Snapshot {
    Store store;
    std::uint8_t* bytes = nullptr;
    u64 n = 0;
};

Pool::Snapshot* Pool::snapshot() {
    auto* s = new Snapshot{store_, nullptr, 0};
    if (has_device()) {
        DeviceScope ds(device_);
        s->n = store_.pool_size();
        TG_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->bytes), s->n));
        TG_CUDA(cudaMemcpyAsync(s->bytes, arena_, s->n, cudaMemcpyDeviceToDevice, s_main_));
        TG_CUDA(cudaStreamSynchronize(s_main_));
    }
    return s;
}

void Pool::restore(const Snapshot* s) {
    store_ = s->store;
    if (has_device() && s->bytes) {
        DeviceScope ds(device_);
        TG_CUDA(cudaMemcpyAsync(arena_, s->bytes, s->n, cudaMemcpyDeviceToDevice, s_main_));
        TG_CUDA(cudaStreamSynchronize(s_main_));
    }
}

void Pool::drop(Snapshot* s) {
    if (!s) return;
    if (s->bytes) cudaFree(s->bytes);
    delete s;
}

void Pool::adopt_store(const Store& src) {
    Store next = src;
    if (has_device()) {
        for (const auto& [k, e] : src.tensors()) {
            Entry* n = next.entry(k);
            const Entry* cur = store_.entry(k);
            if (cur && cur->off == e.off && cur->size == e.size && !cur->suspect) {
                n->suspect = false;
                n->has_digest = cur->has_digest;
                n->digest = cur->digest;
            } else {
                n->suspect = true;
            }
        }
    }
    store_ = std::move(next);
}

std::unique_ptr<KvDevice> Pool::make_kv_device() {
    if (!has_device()) return nullptr;
    return tg::make_kv_device(device_, s_main_);
}

void fingerprint_device(const void* ptr, u64 n, int device, Digest* out) {
    DeviceScope ds(device);
    int sms = 148;
    TG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    std::vector<FpTask> t{FpTask{static_cast<const std::uint8_t*>(ptr), n, 0}};
    const u64 tiles = build_tasks(t);
    cudaStream_t s;
    TG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    void* d = nullptr;
    TG_CUDA(cudaMallocAsync(&d, sizeof(FpTask) + 6 * sizeof(u64), s));
    TG_CUDA(cudaMemcpyAsync(d, t.data(), sizeof(FpTask), cudaMemcpyHostToDevice, s));
    auto* sums = reinterpret_cast<u64*>(static_cast<std::uint8_t*>(d) + sizeof(FpTask));
    TG_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(u64), s));
    fp_launch(static_cast<const FpTask*>(d), 1, tiles, sums, sums + 2, sums + 4, sms, s);
    TG_CUDA(cudaGetLastError());
    u64 h[2];
    TG_CUDA(cudaMemcpyAsync(h, sums + 2, sizeof h, cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaFreeAsync(d, s));
    TG_CUDA(cudaStreamSynchronize(s));
    TG_CUDA(cudaStreamDestroy(s));
    *out = Digest{h[0], h[1]};
}

// Kernel-only timing of K1 / K3 for microbenchmarks: setup outside the timed
// region, `reps` back-to-back launches bracketed by CUDA events on the
// launching stream.  Returns the mean ms per launch.
double bench_fingerprint(const std::vector<std::pair<const void*, u64>>& bufs, int device, int reps,
                         std::vector<Digest>* out) {
    DeviceScope ds(device);
    int sms = 148;
    TG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    std::vector<FpTask> t;
    for (const auto& [p, n] : bufs) t.push_back(FpTask{static_cast<const std::uint8_t*>(p), n, 0});
    const u64 tiles = build_tasks(t);
    const u32 nt = static_cast<u32>(t.size());
    cudaStream_t s;
    TG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    void* d = nullptr;
    const std::size_t per = 4 * sizeof(u64) * nt;  // sums + digests per rep
    TG_CUDA(cudaMalloc(&d, sizeof(FpTask) * nt + per * (reps + 1) + 2 * sizeof(u64)));
    TG_CUDA(cudaMemcpyAsync(d, t.data(), sizeof(FpTask) * nt, cudaMemcpyHostToDevice, s));
    auto* sums = reinterpret_cast<u64*>(static_cast<std::uint8_t*>(d) + sizeof(FpTask) * nt);
    TG_CUDA(cudaMemsetAsync(sums, 0, per * (reps + 1), s));
    auto rep_sums = [&](int r) { return sums + static_cast<std::size_t>(r) * 4 * nt; };
    u64* sync = rep_sums(reps + 1);
    fp_launch(static_cast<const FpTask*>(d), nt, tiles, rep_sums(0), rep_sums(0) + 2 * nt, sync, sms, s);  // warm-up
    cudaEvent_t a, b;
    TG_CUDA(cudaEventCreate(&a));
    TG_CUDA(cudaEventCreate(&b));
    TG_CUDA(cudaEventRecord(a, s));
    for (int r = 1; r <= reps; ++r)
        fp_launch(static_cast<const FpTask*>(d), nt, tiles, rep_sums(r), rep_sums(r) + 2 * nt, sync, sms, s);
    TG_CUDA(cudaEventRecord(b, s));
    TG_CUDA(cudaGetLastError());
    std::vector<u64> h(2 * nt);
    TG_CUDA(cudaMemcpyAsync(h.data(), rep_sums(reps) + 2 * nt, 2 * nt * sizeof(u64), cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    TG_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    cudaStreamDestroy(s);
    if (out) {
        out->clear();
        for (u32 i = 0; i < nt; ++i) out->push_back(Digest{h[2 * i], h[2 * i + 1]});
    }
    return ms / reps;
}

// K3F over hazard-free moves: one warm-up launch (whose digests are returned)
// then `reps` timed launches; returns ms per launch (0 when reps == 0).
double bench_copy_fp(const std::vector<MoveDesc>& moves, int device, int reps, std::vector<Digest>* out) {
    DeviceScope ds(device);
    int sms = 148;
    TG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    std::vector<CopyFpTask> t;
    u64 tiles = 0;
    for (const MoveDesc& m : moves) {
        t.push_back(CopyFpTask{reinterpret_cast<const std::uint8_t*>(m.src), reinterpret_cast<std::uint8_t*>(m.dst),
                               m.len, tiles, -1, -1});
        tiles += ((m.len + kLeafBytes - 1) / kLeafBytes + kLeavesPerTile - 1) / kLeavesPerTile;
    }
    const u32 nt = static_cast<u32>(t.size());
    cudaStream_t s;
    TG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    void* d = nullptr;
    const std::size_t per = 4 * sizeof(u64) * nt;
    TG_CUDA(cudaMalloc(&d, sizeof(CopyFpTask) * nt + per * (reps + 1) + 2 * sizeof(u64)));
    TG_CUDA(cudaMemcpyAsync(d, t.data(), sizeof(CopyFpTask) * nt, cudaMemcpyHostToDevice, s));
    auto* sums = reinterpret_cast<u64*>(static_cast<std::uint8_t*>(d) + sizeof(CopyFpTask) * nt);
    TG_CUDA(cudaMemsetAsync(sums, 0, per * (reps + 1), s));
    auto rep_sums = [&](int r) { return sums + static_cast<std::size_t>(r) * 4 * nt; };
    u64* sync = rep_sums(reps + 1);
    const auto* dt = static_cast<const CopyFpTask*>(d);
    copy_fp_launch(dt, nt, tiles, rep_sums(0), rep_sums(0) + 2 * nt, sync, nullptr, 0, sms, s);
    cudaEvent_t a, b;
    TG_CUDA(cudaEventCreate(&a));
    TG_CUDA(cudaEventCreate(&b));
    TG_CUDA(cudaEventRecord(a, s));
    for (int r = 1; r <= reps; ++r)
        copy_fp_launch(dt, nt, tiles, rep_sums(r), rep_sums(r) + 2 * nt, sync, nullptr, 0, sms, s);
    TG_CUDA(cudaEventRecord(b, s));
    TG_CUDA(cudaGetLastError());
    std::vector<u64> h(2 * nt);
    TG_CUDA(cudaMemcpyAsync(h.data(), rep_sums(0) + 2 * nt, 2 * nt * sizeof(u64), cudaMemcpyDeviceToHost, s));
    TG_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    TG_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    cudaStreamDestroy(s);
    if (out) {
        out->clear();
        for (u32 i = 0; i < nt; ++i) out->push_back(Digest{h[2 * i], h[2 * i + 1]});
    }
    return reps ? ms / reps : 0.0;
}

double bench_relocate(const std::vector<MoveDesc>& moves, int device, int reps) {
    DeviceScope ds(device);
    int sms = 148;
    TG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cudaStream_t s;
    TG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int nm = static_cast<int>(moves.size());
    relocate_launch(moves.data(), nm, sms, s);  // warm-up
    cudaEvent_t a, b;
    TG_CUDA(cudaEventCreate(&a));
    TG_CUDA(cudaEventCreate(&b));
    TG_CUDA(cudaEventRecord(a, s));
    for (int r = 0; r < reps; ++r) relocate_launch(moves.data(), nm, sms, s);
    TG_CUDA(cudaEventRecord(b, s));
    TG_CUDA(cudaGetLastError());
    TG_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    TG_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(s);
    return ms / reps;
}

void synth_fill_device(const Key& k, u64 begin, u64 len, void* dst, int device) {
    DeviceScope ds(device);
    synth_launch(k.hi, k.lo, begin, len, static_cast<std::uint8_t*>(dst), nullptr);
    TG_CUDA(cudaGetLastError());
    TG_CUDA(cudaStreamSynchronize(nullptr));
}

}  // namespace tg
