"""Host control plane: bit-exact against the reference (golden fixtures made by
the compiled reference, and live differential fuzzing against oracle/_ref).

Runs on CPU: pools are created control-plane-only (device=None), which take
exactly the same decisions as device pools (the data plane only executes
them); the GPU tests re-check the same sequences with bytes.
"""
import json
import os
import random

import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
GIB = 1 << 30


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def outcome_json(o):
    """Our LoadOutcome in the oracle's JSON shape."""
    p = o.plan
    return {
        "ok": True,
        "hits": [h.hex() for h in o.hit_tensors],
        "misses": [m.hex() for m in o.missed_tensors],
        "bytes_transferred": o.bytes_transferred,
        "bytes_merged": o.bytes_merged,
        "eviction_cost_total": o.eviction_cost_total,
        "plan": {
            "evictions": [{"tensor": e.tensor.hex(), "size": e.size, "cost": e.cost, "last_access": e.last_access,
                           "model": e.model_id} for e in p.evictions],
            "relocations": [{"tensor": r.tensor.hex(), "from": r.from_, "to": r.to, "size": r.size}
                            for r in p.relocations],
            "placements": [{"tensor": x.tensor.hex(), "offset": x.offset, "size": x.size} for x in p.placements],
            "total_eviction_cost": p.total_eviction_cost,
            "total_merge_cost": p.total_merge_cost,
            "pgp_merge_cost": p.pgp_merge_cost,
            "initial_merge_cost": p.initial_merge_cost,
            "fallback_evictions": p.fallback_evictions,
        },
    }


def result_json(r):
    if r.ok():
        return outcome_json(r.value())
    return {"ok": False, "error": int(r.error())}


def run_sequence(tg, pool_bytes, seq, merge=0, strictness=0, device=None):
    cat = {m.model_id: m for m in tg.default_catalog()}
    st = tg.ReuseStore(tg.GpuSpec(pool_size=pool_bytes), device=device)
    stats = tg.ModelStatsTable()
    out = []
    t = 0.0
    for mid in seq:
        stats.record_request(mid, t)
        stats.set_load_bandwidth(mid, 55e9)
        r = st.load_model(cat[mid], stats, t, tg.LoadPolicy(merge=merge, strictness=strictness))
        out.append(result_json(r))
        st.end_instance(mid)
        assert st.validate().ok()
        t += 10.0
    return {"loads": out, "final_dump": st.dump()}


CASES = {"pg_30": (30, 0, 0), "pg_32": (32, 0, 0), "pg_36": (36, 0, 0), "pg_40": (40, 0, 0),
         "gm_32": (32, 1, 0), "gm_36": (36, 1, 0), "lg_32": (32, 0, 1)}


@pytest.mark.parametrize("case", sorted(CASES))
def test_c2_switch_matches_golden(tg, case):
    g = _golden("c1_c2_loads.json")[case]
    gib, merge, strict = CASES[case]
    got = run_sequence(tg, gib * GIB, ["opt13B", "opt6.7B", "opt13B", "opt6.7B", "opt13B"], merge, strict)
    for i, (a, b) in enumerate(zip(got["loads"], g["loads"])):
        assert a == b, f"load {i}"
    assert got["final_dump"] == g["final_dump"]


def test_c2_appendix_a_numbers(tg):
    """SURVEY Appendix A, 32 GiB: load 3 = 28/13 hits, 5,351,666,658 B
    transferred, 7,620,833,334 B merged, 15 relocations, 3 WAR waves."""
    cat = {m.model_id: m for m in tg.default_catalog()}
    st = tg.ReuseStore(tg.GpuSpec(pool_size=32 * GIB), device=None)
    stats = tg.ModelStatsTable()
    outs = []
    for i, mid in enumerate(["opt13B", "opt6.7B", "opt13B"]):
        stats.record_request(mid, 10.0 * i)
        stats.set_load_bandwidth(mid, 55e9)
        outs.append(st.load_model(cat[mid], stats, 10.0 * i).value())
        st.end_instance(mid)
    o = outs[2]
    assert (len(o.hit_tensors), len(o.missed_tensors)) == (28, 13)
    assert o.bytes_transferred == 5_351_666_658 and o.bytes_merged == 7_620_833_334
    assert len(o.plan.relocations) == 15 and len(o.plan.evictions) == 18
    # wave structure is computed by the device path; the control-plane pool
    # reports it too (the planner output is identical)
    assert o.waves == 3


def test_c1_cold_then_warm(tg):
    g = _golden("c1_c2_loads.json")["c1_160"]
    got = run_sequence(tg, 160 * GIB, ["opt1.3B", "opt1.3B"])
    assert got == g
    cold, warm = got["loads"]
    assert len(cold["plan"]["placements"]) == 25 and cold["plan"]["placements"][0]["offset"] == 0
    assert warm["bytes_transferred"] == 0 and len(warm["hits"]) == 25


# ---- live differential fuzz against the compiled reference -------------------------

def _small_catalog(tg, rnd, n_models, scale=1):
    models = []
    for i in range(n_models):
        total = rnd.randint(2_000, 60_000) * scale + (rnd.randint(0, scale - 1) if scale > 1 else 0)
        layers = rnd.randint(1, 5)
        models.append(tg.make_model(f"m{i}", total, layers, rnd.choice([0, 16, 64]),
                                    latency_sensitivity=rnd.choice([1.0, 0.5, 0.25])))
    return models


def _fuzz_once(tg, ref, seed, n_ops=120, device=None, scale=1, sources=None, on_step=None, extra_flags=0):
    """Random op mix on our store and the compiled reference, compared after
    every op.  With a device: a pool in HBM whose bytes come from
    sources(models, pool) (anything with close()), load flags drawn from a
    second stream (| extra_flags), and on_step(pool, outcome) checking the
    bytes."""
    rnd = random.Random(seed)
    frnd = random.Random(seed ^ 0x5EED5EED)  # load-flag stream, independent of the op stream
    models = _small_catalog(tg, rnd, rnd.randint(2, 6), scale)
    pool = rnd.randint(40_000, 150_000) * scale
    mine = tg.ReuseStore(tg.GpuSpec(pool_size=pool, pcie_bandwidth=rnd.choice([55e9, 12e9])), device=device)
    src = sources(models, mine) if sources is not None else None
    try:
        _fuzz_ops(tg, ref, seed, n_ops, rnd, frnd, models, pool, mine, device, on_step, extra_flags)
    finally:
        if src is not None:
            src.close()
        mine.close()


def _fuzz_ops(tg, ref, seed, n_ops, rnd, frnd, models, pool, mine, device, on_step, extra_flags):
    theirs = ref.ReuseStore(pool, pcie=mine.spec.pcie_bandwidth)
    s_m, s_r = tg.ModelStatsTable(), ref.ModelStatsTable()
    rng_m, rng_r = tg.Rng(seed), ref.Rng(seed)
    t = 0.0
    active = set()
    for step in range(n_ops):
        op = rnd.random()
        m = rnd.choice(models)
        r = None
        if op < 0.45:
            t += rnd.choice([0.0, 0.5, 1.0, 10.0])
            s_m.record_request(m.model_id, t)
            s_r.record_request(m.model_id, t)
            if rnd.random() < 0.3:
                bw = rnd.choice([1e9, 55e9, 7e8])
                s_m.set_load_bandwidth(m.model_id, bw)
                s_r.set_load_bandwidth(m.model_id, bw)
            merge, strict, rand_ev = rnd.random() < 0.2, rnd.random() < 0.2, rnd.random() < 0.15
            flags = (frnd.choice([11, 3, 1, 9, 2 | 8]) | extra_flags) if device is not None else 11
            r = mine.load_model(m, s_m, t, tg.LoadPolicy(merge=int(merge), strictness=int(strict),
                                                         random_eviction=rand_ev, rng=rng_m, flags=flags))
            a = result_json(r)
            b = theirs.load_model(m.to_json(), s_r, t, merge=int(merge), strictness=int(strict),
                                  random_eviction=rand_ev, rng=rng_r)
            assert a == b, (seed, step, "load")
            if a["ok"]:
                active.add(m.model_id)
        elif op < 0.7:
            mine.end_instance(m.model_id)
            theirs.end_instance(m.model_id)
            active.discard(m.model_id)
        elif op < 0.78:
            dump = theirs.dump()
            if dump["tensor_map"]:
                e = rnd.choice(dump["tensor_map"])
                a = mine.evict_tensor(tg.TensorId.from_hex(e["tensor"]))
                b = theirs.evict_tensor(e["tensor"])
                assert (0 if a.ok() else int(a.error()) + 1) == b, (seed, step, "evict")
        elif op < 0.82:
            mine.evict_model(m.model_id)
            theirs.evict_model(m.model_id)
        elif op < 0.88:
            dump = theirs.dump()
            if dump["tensor_map"]:
                e = rnd.choice(dump["tensor_map"])
                to = rnd.randint(0, pool - 1)
                a = mine.move_tensor(tg.TensorId.from_hex(e["tensor"]), to)
                b = theirs.move_tensor(e["tensor"], to)
                assert (0 if a.ok() else int(a.error()) + 1) == b, (seed, step, "move")
        elif op < 0.95:
            size, bid = rnd.randint(1, 5000), rnd.randint(1, 99)
            a = mine.alloc_kv_region(size, bid)
            rc, off = theirs.alloc_kv_region(size, bid)
            assert (0 if a.ok() else int(a.error()) + 1) == rc, (seed, step, "kv alloc")
            if a.ok():
                assert a.value() == off
        else:
            regs = [r for r in theirs.dump()["regions"] if r["state"] == "kv_block"]
            if regs:
                off = rnd.choice(regs)["offset"]
                a = mine.free_kv_region(off)
                b = theirs.free_kv_region(off)
                assert (0 if a.ok() else int(a.error()) + 1) == b
        assert mine.validate().ok()
        assert mine.dump() == theirs.dump(), (seed, step)
        if on_step is not None:
            on_step(mine, r)
        mi, ri = mine.info(), theirs.info()
        for k in ("free_bytes", "kv_bytes", "pinned_bytes", "reusable_bytes", "bytes_merged_total",
                  "bytes_transferred_total", "evictions_total", "region_count", "largest_free"):
            assert mi[k] == ri[k], (seed, step, k)
        if rnd.random() < 0.1:
            ex = rnd.choice(models).model_id
            a = mine.eviction_candidates(s_m, ex)
            b = theirs.eviction_candidates(s_r, ex)
            assert [(c.tensor.hex(), c.size, c.cost, c.last_access, c.model_id) for c in a] == \
                   [(c["tensor"], c["size"], c["cost"], c["last_access"], c["model"]) for c in b]


@pytest.mark.parametrize("seed", range(60))
def test_store_differential_fuzz(tg, ref, seed):
    _fuzz_once(tg, ref, seed)


def test_evict_tensor_codes(tg, ref):
    m = tg.make_model("a", 10_000, 2, 16)
    mine = tg.ReuseStore(tg.GpuSpec(pool_size=50_000), device=None)
    theirs = ref.ReuseStore(50_000)
    s, r = tg.ModelStatsTable(), ref.ModelStatsTable()
    mine.load_model(m, s, 0.0)
    theirs.load_model(m.to_json(), r, 0.0)
    tid = m.tensors[0].id
    assert mine.evict_tensor(tid).error() == tg.Error.Pinned
    assert theirs.evict_tensor(tid.hex()) == 1 + int(tg.Error.Pinned)
    mine.end_instance("a")
    theirs.end_instance("a")
    assert mine.evict_tensor(tid).ok() and theirs.evict_tensor(tid.hex()) == 0
    assert mine.evict_tensor(tid).error() == tg.Error.NotFound
    assert mine.dump() == theirs.dump()


def test_capacity_check_counts_kv_and_pinned(tg, ref):
    """load_model checks the whole model against pool − pinned_other
    (reuse_store.hpp:124-130, Appendix B)."""
    a, b = tg.make_model("a", 30_000, 2, 16), tg.make_model("b", 30_000, 2, 16)
    mine = tg.ReuseStore(tg.GpuSpec(pool_size=70_000), device=None)
    s = tg.ModelStatsTable()
    assert mine.load_model(a, s, 0.0).ok()
    assert mine.alloc_kv_region(20_000, 1).ok()
    r = mine.load_model(b, s, 1.0)
    assert r.error() == tg.Error.InsufficientMemory
    theirs = ref.ReuseStore(70_000)
    rs = ref.ModelStatsTable()
    theirs.load_model(a.to_json(), rs, 0.0)
    theirs.alloc_kv_region(20_000, 1)
    assert theirs.load_model(b.to_json(), rs, 1.0) == {"ok": False, "error": 0}
    assert mine.dump() == theirs.dump()
