// Launch interfaces of the sm_100a kernels (plain C++ so host code can call
// them without CUDA headers beyond cuda_runtime.h).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace tg {

// Number of kernels this library has launched (bench.py's gpu_launches).
extern std::atomic<std::uint64_t> g_kernel_launches;

// ---- K1: content fingerprint (tgfp1) -------------------------------------
// Leaf = 4096 B, leaf_i digest = murmur3_x64_128(leaf bytes, seed = i);
// tensor digest = murmur3(le64 ΣH ‖ le64 ΣL ‖ le64 n, seed 0).
constexpr std::uint64_t kLeafBytes = 4096;
constexpr std::uint32_t kLeavesPerTile = 32;

struct FpTask {
    const std::uint8_t* base;  // device pointer (any alignment)
    std::uint64_t n;           // bytes
    std::uint64_t tile0;       // first tile index of this task (prefix over tasks)
};

// sums: 2 u64 per task (must be zeroed), digests: 2 u64 per task, sync: two
// u64 of device scratch private to this launch (tile dispenser, finished
// CTAs; zeroed by it unless the caller did, sync_zeroed).  Runs the load
// kernel below with fingerprint-only tasks; its last CTA writes the digests.
void fp_launch(const FpTask* d_tasks, std::uint32_t n_tasks, std::uint64_t total_tiles, std::uint64_t* d_sums,
               std::uint64_t* d_digests, std::uint64_t* d_sync, int sm_count, cudaStream_t s,
               bool sync_zeroed = false, std::uint64_t* stamps = nullptr, bool clean = false);

// ---- K3F: copy + fingerprint in one pass — the load kernel ---------------
// Moves every task's n bytes src -> dst (any alignments) and produces the
// tgfp1 digest of the moved bytes, reading them once; dst == nullptr only
// fingerprints (a reused tensor verified in place).  One persistent launch
// runs a whole load: warps take 128 KiB tiles in task order from a counter,
// and a task with gate >= 0 writes nothing before every tile of WAR wave
// `gate` has finished (its sources read) — so relocation waves, the
// placements gated on them and the in-place verification share one launch.
struct CopyFpTask {
    const std::uint8_t* src;
    std::uint8_t* dst;    // nullptr: fingerprint only
    std::uint64_t n;
    std::uint64_t tile0;  // tile prefix (32 leaves per tile), relative to the launch
    std::int32_t gate;    // wave that must be complete before this task writes (-1: none)
    std::int32_t wave;    // wave this task belongs to (its tiles count towards need[wave]; -1: none)
    // Leaf index of byte 0 within its tensor (the murmur seed of leaf i is
    // leaf_base + i): a task may be a leaf-aligned piece of a tensor.  With
    // kRawSums set, the launch writes the task's raw (ΣH, ΣL) instead of a
    // digest; the host adds the pieces of one tensor and takes the root.
    std::uint64_t leaf_base = 0;
};
constexpr std::uint64_t kRawSums = std::uint64_t{1} << 63;
// sync: 2 + n_waves u64 of device scratch — tile dispenser, the finished
// tiles of each wave, finished CTAs — (zeroed by the launch unless
// sync_zeroed); need[w] = tiles of wave w's tasks.  sums: 2 u64 per task
// (zeroed by the caller).  The launch's last CTA to finish turns the sums
// into digests (no second kernel).
void copy_fp_launch(const CopyFpTask* d_tasks, std::uint32_t n_tasks, std::uint64_t total_tiles, std::uint64_t* d_sums,
                    std::uint64_t* d_digests, std::uint64_t* d_sync, const std::uint64_t* d_need,
                    std::uint32_t n_waves, int sm_count, cudaStream_t s, bool sync_zeroed = false,
                    std::uint64_t* stamps = nullptr,  // nullable: globaltimer ns at start / end
                    bool clean = false);  // zero sums and sync counters after the digests (no gated waiters)
// Warps one load-kernel launch keeps resident (tile-count sizing of the
// independent work placed between gated waves).
std::uint64_t copy_fp_resident_warps(int sm_count);

// ---- K3: relocation wave (batched misaligned memcpy) ---------------------
constexpr int kMaxMovesPerLaunch = 96;
struct MoveDesc {
    std::uint64_t src;  // device address
    std::uint64_t dst;  // device address
    std::uint64_t len;  // bytes
};
// All moves of one launch must be pairwise hazard-free (one WAR wave).
void relocate_launch(const MoveDesc* moves, int n_moves, int sm_count, cudaStream_t s);

// ---- K4: KV batch expansion ------------------------------------------------
struct KvGrantDev {
    std::uint64_t start;  // first global block index of this grant
    std::uint64_t lbn0;
    std::uint32_t slot;
    std::uint32_t pad;
};
struct KvRunDev {
    std::uint64_t start;  // first carved-block index (relative to pops) of this run
    std::uint64_t off;
    std::uint64_t first_pbn;
};
struct KvBatchArgs {
    const KvGrantDev* grants;
    std::uint32_t n_grants;
    const KvRunDev* runs;
    std::uint32_t n_runs;
    std::uint64_t total;
    std::uint64_t pops;
    std::uint64_t free_before;
    std::uint64_t block_bytes;
    std::uint64_t* tables;  // [slots][stride]
    std::uint64_t stride;
    std::uint64_t* free_list;
    std::uint64_t* addr;  // pbn -> offset
    std::uint64_t* out;   // optional: granted pbns in order
};
void kv_batch_launch(const KvBatchArgs& a, cudaStream_t s);

// ---- K4D: device-decided KV batches (the allocator decision on the GPU) -----
// Control block of an armed engine, resident in HBM.  The host writes the
// first part at arm time (pointers and limits, a mirror of the pool's free
// runs of at least one block in ascending (size, offset) order, the per-slot
// block and token counts); kv_device_batch_kernel advances the second part.
// Every pointer is read at run time, so a captured CUDA graph of batches stays
// valid across arms.
constexpr std::uint32_t kKvDevMaxRequests = 8192;  // per batch
constexpr std::uint32_t kKvDevMaxPieces = 64;      // carved pieces per batch
struct KvDevCtl {
    std::uint64_t* tables;
    std::uint64_t stride;
    std::uint64_t* free_list;
    std::uint64_t* addr;
    const std::uint64_t* run_off;
    const std::uint64_t* run_blocks;
    std::uint64_t n_runs;
    std::uint64_t* slot_blocks;
    std::uint64_t* slot_tokens;
    std::uint64_t* slot_mark;  // batch that last touched the slot (+1): duplicate detection
    std::uint64_t n_slots;
    std::uint8_t* log;
    std::uint64_t log_entry_bytes;
    std::uint64_t max_batches;
    std::uint64_t max_requests;
    std::uint64_t block_bytes;
    std::uint64_t block_tokens;
    // advanced by the kernel
    std::uint64_t free_top;
    std::uint64_t next_pbn;
    std::uint64_t run_cursor;
    std::uint64_t run_used;
    std::uint64_t blocks_left;
    std::uint64_t batches;
    std::uint64_t stalled;  // 0 ok, 1 a batch fell back to the host (later ones do nothing), 2 log overflow
};
// One log entry per batch: header, the batch's (slot, tokens) pairs
// (max_requests of them), then up to kKvDevMaxPieces carved pieces.
struct KvLogHeader {
    std::uint64_t n;
    std::uint64_t status;  // 0 applied on the device, 1 left to the host (replayed at sync)
    std::uint64_t total;
    std::uint64_t pops;
    std::uint64_t n_pieces;
    std::uint64_t pad[3];
};
struct KvPiece {
    std::uint64_t off;
    std::uint64_t count;
    std::uint64_t first_pbn;
};
inline std::uint64_t kv_log_entry_bytes(std::uint64_t max_requests) {
    return sizeof(KvLogHeader) + 16 * max_requests + sizeof(KvPiece) * kKvDevMaxPieces;
}
void kv_device_batch_launch(KvDevCtl* d_ctl, const std::uint64_t* d_slots, const std::uint64_t* d_tokens,
                            std::uint32_t n, cudaStream_t s);
// Block-table consumer (what a paged-attention cache write / gather does):
// token i of request-slot slots[i] at position pos[i] lives at
// arena + addr[tables[slot * stride + pos / block_tokens]] + (pos % block_tokens) * token_bytes.
// write: buf[i] -> that place; else that place -> buf[i] (token_bytes each).
// A reference outside the tables (slot or LBN past the table, PBN 0 = never
// granted, a PBN past the address table, a block outside the arena) moves
// nothing and counts one fault in *faults.
struct KvTokensArgs {
    const std::uint64_t* tables;
    std::uint64_t n_slots, stride;
    const std::uint64_t* addr;
    std::uint64_t n_pbns;
    std::uint8_t* arena;
    std::uint64_t arena_bytes;
    std::uint64_t block_tokens, token_bytes;
    const std::uint64_t* slots;
    const std::uint64_t* pos;
    std::uint8_t* buf;
    std::uint32_t n;
    bool write;
    unsigned long long* faults;
};
void kv_tokens_launch(const KvTokensArgs& a, cudaStream_t s);
void kv_release_launch(const std::uint64_t* table_row, std::uint64_t blocks, std::uint64_t* free_list_dst,
                       cudaStream_t s);

// ---- synthetic checkpoint bytes -------------------------------
void synth_launch(std::uint64_t hi, std::uint64_t lo, std::uint64_t begin, std::uint64_t len, std::uint8_t* dst,
                  cudaStream_t s);

// ---- K6: device tensor index lookup ------------------------------------------
// table: tg_index_slot[capacity] (include/tangram.h); keys: (hi, lo) pairs;
// out: 3 u64 per key = offset, size, found | flags << 32 (offset ~0 when absent).
void index_lookup_launch(const void* table, std::uint64_t capacity, const std::uint64_t* d_keys, std::uint32_t n,
                         std::uint64_t* d_out, cudaStream_t s);

// ---- K5: peer pull (SM copy over NVLink peer mappings) -----------------------
// Reuses the relocation kernel: the source address is a peer arena pointer.

}  // namespace tg
