// Two-stage allocation planner (MCMDKP heuristic) of the Tangram pool.
//
// Produces exactly the plan of the reference plan_allocation
// (packing.hpp:311-483): Stage 1 evicts cost-ordered candidates until the
// free total covers the new tensors; Stage 2 distributes the tensors over
// barrier-delimited root subspaces, refines them with partitioned-gain
// packing (Alg. 1, packing.hpp:180-214) and composes relocations (pack
// allocated regions to the subspace edges) and best-fit placements.  The
// plan is then executed by the B200 data plane (relocation waves on HBM,
// chunked H2D, fingerprints) in store.cpp / device/*.cu.
#pragma once

#include <string>
#include <unordered_set>
#include <vector>

#include "model.hpp"
#include "regions.hpp"

namespace tg {

struct Candidate {
    Key tensor;
    u64 size = 0;
    double cost = 0;
    double last_access = 0;
    std::string model_id;
};

// (cost ↑, size ↓, last_access ↑, id ↑) — packing.hpp:42-47.
bool candidate_before(const Candidate& a, const Candidate& b);

enum class Strictness : std::uint8_t { Functional = 0, LiteralGuard = 1 };
enum class MergeMode : std::uint8_t { PartitionedGain = 0, GlobalMerge = 1 };

struct Move {
    Key tensor;
    u64 from = 0, to = 0, size = 0;
};

struct Place {
    u32 tensor = 0;  // index into PlanInput::tensors
    u64 off = 0;
};

struct Plan {
    std::vector<Candidate> evictions;
    std::vector<Move> relocations;
    std::vector<Place> placements;
    double total_eviction_cost = 0;
    u64 total_merge_cost = 0;
    u64 pgp_merge_cost = 0;
    u64 initial_merge_cost = 0;
    u64 fallback_evictions = 0;
};

struct PlanInput {
    const PoolMap* pool = nullptr;               // current layout
    const std::vector<TensorDesc>* tensors = nullptr;  // new tensors, model order
    std::vector<Candidate> candidates;           // evictable residents
    std::unordered_set<Key, KeyHash> immovable;  // pinned tensors
    Strictness strictness = Strictness::Functional;
    MergeMode merge = MergeMode::PartitionedGain;
    bool keep_candidate_order = false;           // random-eviction mode
};

// Two-bin best-fit-decreasing used by Alg. 1 (packing.hpp:103-123); exposed
// for unit tests.  `sizes` are consumed in order; bins returned as index lists.
bool two_bin_pack(const std::vector<u64>& sizes, u64 cap1, u64 cap2, Strictness s, std::vector<u32>* first,
                  std::vector<u32>* second);

// On success *work holds the post-plan layout.
Res<Plan> make_plan(const PlanInput& in, PoolMap* work);

}  // namespace tg
