// Value-semantics check of the drop-in ReuseStore (reuse_store.hpp:336-344):
// the reference's stores are values — copied for rollback (kv_engine.hpp:
// 146-158) — so a copy must be independent of its original.  Built twice by
// integration/Makefile (pure reference / B200 bindings); tests/test_dropin.py
// requires byte-identical stdout.  The sequence:
//   s: load opt1.3B, end_instance, load qwen3B (relocations + evictions);
//   c = s (copy); c: end_instance, load llama3B        -> s unchanged
//   r = s (copy); r: evict a tensor, alloc a KV region  -> s unchanged
//   s = c (copy-assign back), then s = std::move(r)     -> s equals r
//   s: end_instance(llama3B) twice over, reload qwen3B and llama3B.
// Every dump goes to stdout.  With TANGRAM_SYNTH_SOURCES the binding build
// also reports on stderr, as JSON, the data plane of the last loads
// (tensors re-sent because the adopted layout was not in the arena).
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <optional>
#include <string>
#include <type_traits>

#include "json.hpp"
#include <warmsim/catalog.hpp>  // <>: never the directory of this file
#include <warmsim/reuse_store.hpp>

using namespace warmsim;

// containers move stores on reallocation (simulator.hpp:213, std::vector<Gpu>)
static_assert(std::is_nothrow_move_constructible_v<ReuseStore>);

static void show(const char* tag, const ReuseStore& s) { std::cout << tag << " " << s.dump().dump() << "\n"; }

int main(int argc, char** argv) {
    const double gib = argc > 1 ? std::atof(argv[1]) : 7.0;
    const auto cat = default_catalog();
    auto model = [&](const std::string& id) -> const ModelSpec& {
        for (const auto& m : cat)
            if (m.model_id == id) return m;
        std::abort();
    };
#ifdef TANGRAM_BINDING
    if (std::getenv("TANGRAM_SYNTH_SOURCES")) {
        for (const char* id : {"opt1.3B", "qwen3B", "llama3B"})
            for (const auto& t : model(id).tensors) {
                void* d = nullptr;
                const tg_tensor_id tid{t.id.hi, t.id.lo};
                if (tg_device_alloc(0, t.size, &d) || tg_synth_fill_device(tid, 0, t.size, d, 0) ||
                    tg_host_register(tid, d, t.size, nullptr)) {
                    std::fprintf(stderr, "source setup failed: %s\n", tg_last_error_detail());
                    return 3;
                }
            }
    }
#endif
    ModelStatsTable stats;
    ReuseStore s(GpuSpec{"gpu0", static_cast<Bytes>(gib * (1ull << 30)), 55e9, 3000e9, 12e9});
    double t = 0;
    auto load = [&](ReuseStore& st, const std::string& id) {
        stats.record_request(id, t);
        auto r = st.load_model(model(id), stats, t);
        t += 10;
        std::cout << "load " << id << " ok=" << static_cast<bool>(r);
        if (r) std::cout << " xfer=" << r.value().bytes_transferred << " merged=" << r.value().bytes_merged;
        std::cout << "\n";
        return r;
    };
    load(s, "opt1.3B");
    s.end_instance("opt1.3B");
    load(s, "qwen3B");
    show("s0", s);

    ReuseStore c = s;
    c.end_instance("qwen3B");
    load(c, "llama3B");
    show("s_after_c", s);
    show("c", c);

    ReuseStore r = s;
    TensorId victim{};
    for (const auto& x : model("opt1.3B").tensors)  // a resident, unpinned tensor
        if (s.tensor_map().count(x.id)) {
            victim = x.id;
            break;
        }
    std::cout << "evict ok=" << static_cast<bool>(r.evict_tensor(victim)) << "\n";
    auto kv = r.alloc_kv_region(1 << 20, 7);
    std::cout << "kv ok=" << static_cast<bool>(kv) << "\n";
    show("s_after_r", s);
    show("r", r);
    std::cout << "tensors s=" << s.tensor_map().size() << " c=" << c.tensor_map().size()
              << " r=" << r.tensor_map().size() << "\n";

    s = c;
    show("s_eq_c", s);
    s = std::move(r);
    show("s_eq_r", s);
    std::cout << "valid=" << static_cast<bool>(s.validate()) << "\n";

    s = c;
    s.end_instance("llama3B");
    auto q = load(s, "qwen3B");
    s.end_instance("qwen3B");
    auto l = load(s, "llama3B");
    show("s_final", s);
    std::cout << "valid=" << static_cast<bool>(s.validate()) << "\n";

    // the store keeps its state for a copy taken before it mutates
    ReuseStore backup = s;
    s.end_instance("llama3B");
    load(s, "opt1.3B");
    show("backup", backup);
    show("s_after_backup", s);

    // a copy that outlives its original carries on with the pool
    std::optional<ReuseStore> first(std::in_place, GpuSpec{"gpu0", static_cast<Bytes>(8.0 * (1ull << 30)), 55e9,
                                                            3000e9, 12e9});
    load(*first, "opt1.3B");
    ReuseStore second = *first;
    first.reset();
    second.end_instance("opt1.3B");
    auto w = load(second, "qwen3B");
    show("second", second);
#ifdef TANGRAM_BINDING
    if (q && l && w) {
        const auto& a = q.value().device;
        const auto& b = l.value().device;
        std::fprintf(stderr,
                     "{\"repaired\": [%llu, %llu], \"suspect\": [%u, %u], \"fingerprinted\": [%llu, %llu], "
                     "\"mismatches\": [%u, %u], \"second_placed\": %llu}\n",
                     (unsigned long long)a.repaired_bytes, (unsigned long long)b.repaired_bytes, a.suspect_tensors,
                     b.suspect_tensors, (unsigned long long)a.fingerprint_bytes,
                     (unsigned long long)b.fingerprint_bytes, a.verify_mismatches, b.verify_mismatches,
                     (unsigned long long)(w.value().device.pcie_bytes + w.value().device.device_src_bytes));
    }
#endif
    return 0;
}
