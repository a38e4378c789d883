#include "planner.hpp"

#include <algorithm>
#include <deque>
#include <numeric>
#include <unordered_map>

namespace tg {

bool candidate_before(const Candidate& a, const Candidate& b) {
    if (a.cost != b.cost) return a.cost < b.cost;
    if (a.size != b.size) return a.size > b.size;
    if (a.last_access != b.last_access) return a.last_access < b.last_access;
    return a.tensor < b.tensor;
}

bool two_bin_pack(const std::vector<u64>& sizes, u64 cap1, u64 cap2, Strictness s, std::vector<u32>* first,
                  std::vector<u32>* second) {
    first->clear();
    second->clear();
    for (u32 i = 0; i < sizes.size(); ++i) {
        const u64 need = sizes[i];
        if (s == Strictness::LiteralGuard && need >= std::min(cap1, cap2)) return false;
        const bool to_first = cap1 >= cap2;  // ties go to the first bin
        u64& cap = to_first ? cap1 : cap2;
        if (need > cap) return false;
        cap -= need;
        (to_first ? first : second)->push_back(i);
    }
    return true;
}

namespace {

// A run of consecutive extents that starts and ends with a free extent.
struct Span {
    std::vector<Extent> ext;
    u64 capacity = 0;   // free bytes inside
    u64 allocated = 0;  // bytes that a full merge would move
    std::vector<u32> tensors;  // indices into the size-sorted new tensors

    void tally() {
        capacity = allocated = 0;
        for (const auto& e : ext) (e.kind == Kind::Free ? capacity : allocated) += e.len;
    }
    u64 lo() const { return ext.front().off; }
    u64 hi() const { return ext.back().end(); }
};

// Maximal groups of adjacent allocated extents: candidate partition points,
// largest first, then lowest address (packing.hpp:151-169).
struct Cut {
    std::size_t a, b;  // inclusive extent index range
    u64 bytes, off;
};

std::vector<Cut> cuts_of(const Span& s) {
    std::vector<Cut> cuts;
    const auto& x = s.ext;
    std::size_t i = 0;
    while (i < x.size()) {
        if (x[i].kind == Kind::Free) {
            ++i;
            continue;
        }
        Cut c{i, i, 0, x[i].off};
        while (c.b + 1 < x.size() && x[c.b + 1].kind != Kind::Free) ++c.b;
        for (std::size_t k = c.a; k <= c.b; ++k) c.bytes += x[k].len;
        cuts.push_back(c);
        i = c.b + 1;
    }
    std::sort(cuts.begin(), cuts.end(), [](const Cut& p, const Cut& q) {
        return p.bytes != q.bytes ? p.bytes > q.bytes : p.off < q.off;
    });
    return cuts;
}

// Root subspaces: split the chain at barriers (KV blocks, pinned tensors)
// and trim each segment to free extents at both ends (packing.hpp:267-286).
std::vector<Span> roots_of(const PoolMap& pool, const std::unordered_set<Key, KeyHash>& immovable) {
    std::vector<Span> roots;
    Span cur;
    auto close = [&] {
        auto& x = cur.ext;
        std::size_t a = 0, b = x.size();
        while (a < b && x[a].kind != Kind::Free) ++a;
        while (b > a && x[b - 1].kind != Kind::Free) --b;
        if (a < b) {
            Span s;
            s.ext.assign(x.begin() + static_cast<long>(a), x.begin() + static_cast<long>(b));
            s.tally();
            roots.push_back(std::move(s));
        }
        x.clear();
    };
    for (const auto& [o, e] : pool.extents()) {
        const bool barrier = e.kind == Kind::Kv || (e.kind == Kind::Tensor && immovable.count(e.tensor));
        if (barrier) close();
        else cur.ext.push_back(e);
    }
    close();
    return roots;
}

}  // namespace

Res<Plan> make_plan(const PlanInput& in, PoolMap* work) {
    Plan plan;
    const auto& news = *in.tensors;
    if (news.empty()) return plan;
    *work = *in.pool;

    u64 needed = 0;
    for (const auto& t : news) needed += t.size;

    // ---- Stage 1: cheapest evictions until the free total suffices ----------
    std::vector<Candidate> order = in.candidates;
    if (!in.keep_candidate_order) std::sort(order.begin(), order.end(), candidate_before);
    std::unordered_map<Key, u64, KeyHash> where;  // resident tensor -> offset (pre-plan)
    for (const auto& [o, e] : in.pool->extents())
        if (e.kind == Kind::Tensor) where.emplace(e.tensor, e.off);
    std::unordered_map<Key, std::size_t, KeyHash> cand_index;
    for (std::size_t i = 0; i < order.size(); ++i) cand_index.emplace(order[i].tensor, i);

    std::unordered_set<Key, KeyHash> gone;
    std::size_t cursor = 0;
    auto evict_one = [&]() -> bool {
        for (; cursor < order.size(); ++cursor) {
            const Candidate& c = order[cursor];
            if (gone.count(c.tensor)) continue;
            auto w = where.find(c.tensor);
            if (w == where.end()) continue;
            work->release(w->second);
            gone.insert(c.tensor);
            plan.evictions.push_back(c);
            plan.total_eviction_cost += c.cost;
            ++cursor;
            return true;
        }
        return false;
    };
    while (work->free_total() < needed)
        if (!evict_one()) return Err::InsufficientMemory;

    // ---- Stage 2: distribute over roots (retry with one more eviction) -------
    std::vector<u32> by_size(news.size());
    std::iota(by_size.begin(), by_size.end(), 0u);
    std::stable_sort(by_size.begin(), by_size.end(),
                     [&](u32 a, u32 b) { return news[a].size > news[b].size; });

    std::vector<Span> roots;
    for (;;) {
        roots = roots_of(*work, in.immovable);
        bool fits = !roots.empty();
        if (fits) {
            std::vector<u64> room(roots.size());
            for (std::size_t i = 0; i < roots.size(); ++i) room[i] = roots[i].capacity;
            for (u32 t = 0; t < by_size.size() && fits; ++t) {
                std::size_t best = 0;
                for (std::size_t i = 1; i < roots.size(); ++i)
                    if (room[i] > room[best]) best = i;
                const u64 sz = news[by_size[t]].size;
                if (room[best] < sz) {
                    fits = false;
                    break;
                }
                roots[best].tensors.push_back(t);
                room[best] -= sz;
            }
        }
        if (fits) break;
        if (!evict_one()) return Err::InsufficientMemory;
    }

    // ---- Alg. 1: partitioned-gain packing -----------------------------------
    for (const auto& r : roots) plan.initial_merge_cost += r.allocated;
    u64 merge_cost = plan.initial_merge_cost;
    std::deque<Span> pending(std::make_move_iterator(roots.begin()), std::make_move_iterator(roots.end()));
    std::vector<Span> finals;
    std::vector<u64> sizes;
    std::vector<u32> b1, b2;
    while (!pending.empty()) {
        Span cur = std::move(pending.front());
        pending.pop_front();
        bool split = false;
        if (in.merge == MergeMode::PartitionedGain) {
            sizes.resize(cur.tensors.size());
            for (std::size_t i = 0; i < cur.tensors.size(); ++i) sizes[i] = news[by_size[cur.tensors[i]]].size;
            for (const Cut& c : cuts_of(cur)) {
                Span left, right;
                left.ext.assign(cur.ext.begin(), cur.ext.begin() + static_cast<long>(c.a));
                right.ext.assign(cur.ext.begin() + static_cast<long>(c.b) + 1, cur.ext.end());
                left.tally();
                right.tally();
                if (!two_bin_pack(sizes, left.capacity, right.capacity, in.strictness, &b1, &b2)) continue;
                merge_cost -= c.bytes;
                for (u32 i : b1) left.tensors.push_back(cur.tensors[i]);
                for (u32 i : b2) right.tensors.push_back(cur.tensors[i]);
                pending.push_back(std::move(left));
                pending.push_back(std::move(right));
                split = true;
                break;
            }
        }
        if (!split) finals.push_back(std::move(cur));
    }
    plan.pgp_merge_cost = merge_cost;

    // ---- compose relocations and placements per finalized subspace ----------
    for (const Span& sub : finals) {
        const u64 lo = sub.lo(), hi = sub.hi();
        std::vector<const Extent*> live;
        for (const auto& e : sub.ext)
            if (e.kind != Kind::Free) live.push_back(&e);

        // free bytes after each live extent on the original layout
        std::vector<u64> free_after(live.size(), 0);
        {
            u64 acc = 0;
            std::size_t j = live.size();
            for (auto it = sub.ext.rbegin(); it != sub.ext.rend(); ++it) {
                if (it->kind == Kind::Free) acc += it->len;
                else free_after[--j] = acc;
            }
        }

        auto relocate = [&](const Extent& r, u64 dst) {
            work->move(r.off, dst);
            plan.relocations.push_back(Move{r.tensor, r.off, dst, r.len});
            plan.total_merge_cost += r.len;
        };

        std::vector<std::size_t> rightward, leftward;
        for (std::size_t i = 0; i < live.size(); ++i) (live[i]->len <= free_after[i] ? rightward : leftward).push_back(i);

        u64 right_fill = 0;
        for (auto it = rightward.rbegin(); it != rightward.rend(); ++it) {
            const Extent& r = *live[*it];
            const u64 dst = hi - right_fill - r.len;
            if (work->is_free_range(dst, r.len)) {
                relocate(r, dst);
                right_fill += r.len;
            } else {
                leftward.push_back(*it);
            }
        }
        std::sort(leftward.begin(), leftward.end());

        u64 left_fill = 0;
        for (std::size_t i : leftward) {
            const Extent& r = *live[i];
            const u64 dst = lo + left_fill;
            if (work->is_free_range(dst, r.len)) {
                relocate(r, dst);
                left_fill += r.len;
                continue;
            }
            const u64 alt = hi - right_fill - r.len;
            if (alt >= lo && work->is_free_range(alt, r.len)) {
                relocate(r, alt);
                right_fill += r.len;
                continue;
            }
            // Neither edge has room: evict instead, if it is a candidate.
            auto ci = cand_index.find(r.tensor);
            if (ci == cand_index.end() || gone.count(r.tensor)) return Err::Infeasible;
            work->release(r.off);
            gone.insert(r.tensor);
            plan.evictions.push_back(order[ci->second]);
            plan.total_eviction_cost += order[ci->second].cost;
            plan.fallback_evictions++;
        }

        // best fit inside the subspace extent, lowest address on ties
        for (u32 t : sub.tensors) {
            const TensorDesc& td = news[by_size[t]];
            u64 best_off = 0, best_len = 0;
            bool found = false;
            work->for_each_free_in(lo, hi, [&](const Extent& f) {
                const u64 a = std::max(f.off, lo), b = std::min(f.end(), hi);
                if (b <= a || b - a < td.size) return;
                if (!found || b - a < best_len) {
                    found = true;
                    best_off = a;
                    best_len = b - a;
                }
            });
            if (!found) return Err::Infeasible;
            work->carve(best_off, td.size, Kind::Tensor, td.id, 0, 1);
            plan.placements.push_back(Place{by_size[t], best_off});
        }
    }
    return plan;
}

}  // namespace tg
