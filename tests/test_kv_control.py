"""KV block allocator, control half (CPU): counts, stats, carved runs, pool
dumps and address tables against the reference KvEngine (kv_engine.hpp:43-239).

The per-block tables (LBN→PBN) are materialised by the device kernel and are
compared in tests/test_gpu_load.py; here the engine runs on a control-plane
pool, where every host-visible effect must already be identical.
"""
import json
import os
import random

import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
GIB = 1 << 30


def _stats_tuple(s):
    return (s.pool_invocations, s.alloc_batches, s.blocks_from_free_list, s.blocks_from_pool, s.reclaim_events)


def _ref_stats_tuple(st):
    s = st["stats"]
    return (s["pool_invocations"], s["alloc_batches"], s["blocks_from_free_list"], s["blocks_from_pool"],
            s["reclaim_events"])


def test_c3_prefill_burst_matches_golden(tg):
    g = json.load(open(os.path.join(GOLDEN, "c3_kv.json")))
    model = tg.make_model("llama2-13B", 26_000_000_000, 40, 819_200)
    for n, case in g.items():
        pool = tg.ReuseStore(tg.GpuSpec(pool_size=160 * GIB), device=None)
        stats = tg.ModelStatsTable()
        stats.record_request("llama2-13B", 0.0)
        pool.load_model(model, stats, 0.0).value()
        kv = tg.KvEngine("llama2-13B", 16, 819_200)
        reqs = [tuple(r) for r in case["requests"]]
        burst = kv.batch_allocate(pool, stats, reqs).value()
        assert burst == [len(x) for x in case["burst"]]
        dec = kv.batch_allocate(pool, stats, [(r, (p + 15) // 16 * 16 + 1) for r, p in reqs]).value()
        assert dec == [len(x) for x in case["decode"]]
        assert _stats_tuple(kv.stats()) == _ref_stats_tuple(case["state"])
        at = kv.address_table()
        assert sorted(at.items()) == sorted((a[0], (a[1], a[2])) for a in case["state"]["address_table"])
        info = pool.info()
        for k in ("kv_bytes", "free_bytes", "pinned_bytes"):
            assert info[k] == case["info"][k]
        assert info["region_count"] == case["regions"]
        # compact representation: one extent per carve run, not per block
        assert info["extent_count"] < len(model.tensors) + 2 * len(reqs) + 2
        assert pool.validate().ok()
    # 1,504 / 7,032 blocks
    assert sum(len(x) for x in g["16"]["burst"]) == 1504 and sum(len(x) for x in g["64"]["burst"]) == 7032


def test_ensure_capacity_spec_examples(tg):
    """ceil(33/16)=3, 48→49 gives +1, 40→47 gives +0."""
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=1 << 20), device=None)
    st = tg.ModelStatsTable()
    kv = tg.KvEngine("m", 16, 8)
    assert kv.ensure_capacity(pool, st, 1, 33).value() == 3
    assert kv.ensure_capacity(pool, st, 2, 48).value() == 3
    assert kv.ensure_capacity(pool, st, 2, 49).value() == 1
    assert kv.ensure_capacity(pool, st, 3, 40).value() == 3
    assert kv.ensure_capacity(pool, st, 3, 47).value() == 0
    assert kv.ensure_capacity(pool, st, 3, 46).error() == tg.Error.InvalidArgument


def _kv_fuzz(tg, ref, seed, n_ops=150):
    rnd = random.Random(seed)
    pool_size = rnd.randint(30_000, 120_000)
    mine = tg.ReuseStore(tg.GpuSpec(pool_size=pool_size), device=None)
    theirs = ref.ReuseStore(pool_size)
    s_m, s_r = tg.ModelStatsTable(), ref.ModelStatsTable()
    # some resident, unpinned tensors of other models (reclaim candidates) and
    # the serving model itself
    others = [tg.make_model(f"o{i}", rnd.randint(3_000, 15_000), rnd.randint(1, 3), 0) for i in range(3)]
    t = 0.0
    for m in others:
        t += 1.0
        s_m.record_request(m.model_id, t)
        s_r.record_request(m.model_id, t)
        a = mine.load_model(m, s_m, t)
        b = theirs.load_model(m.to_json(), s_r, t)
        assert a.ok() == b["ok"]
        mine.end_instance(m.model_id)
        theirs.end_instance(m.model_id)
    serving = tg.make_model("serve", rnd.randint(2_000, 8_000), 2, 0)
    t += 1.0
    s_m.record_request("serve", t)
    s_r.record_request("serve", t)
    mine.load_model(serving, s_m, t)
    theirs.load_model(serving.to_json(), s_r, t)
    bs, bpt = rnd.choice([(4, 32), (16, 8), (8, 100)])
    kv_m, kv_r = tg.KvEngine("serve", bs, bpt), ref.KvEngine("serve", bs, bpt)
    live = {}
    next_rid = 1
    for step in range(n_ops):
        op = rnd.random()
        if op < 0.45:
            reqs = []
            for _ in range(rnd.randint(1, 5)):
                if live and rnd.random() < 0.5:
                    rid = rnd.choice(list(live))
                    tok = live[rid] + rnd.randint(0, 3 * bs)
                else:
                    rid = next_rid
                    next_rid += 1
                    tok = rnd.randint(0, 6 * bs)
                if rnd.random() < 0.03 and rid in live and live[rid] > 0:
                    tok = live[rid] - 1  # InvalidArgument path
                reqs.append((rid, tok))
            a = kv_m.batch_allocate(mine, s_m, reqs, want_pbns=False)
            b = kv_r.batch_allocate(theirs, s_r, reqs)
            if b["ok"]:
                assert a.ok(), (seed, step, a)
                assert a.value() == [len(g) for g in b["granted"]], (seed, step)
            else:
                assert not a.ok() and int(a.error()) == b["error"], (seed, step, a, b)
            for rid, tok in reqs:
                tb = kv_r.table(rid)
                if tb is not None:
                    live[rid] = tb["token_count"]
        elif op < 0.6:
            rid = rnd.choice(list(live)) if live and rnd.random() < 0.8 else next_rid + 5
            tok = live.get(rid, 0) + rnd.randint(0, 2 * bs)
            a = kv_m.ensure_capacity(mine, s_m, rid, tok, want_pbns=False)
            b = kv_r.ensure_capacity(theirs, s_r, rid, tok)
            assert a.ok() == b["ok"], (seed, step)
            if b["ok"]:
                assert a.value() == len(b["granted"])
            tb = kv_r.table(rid)
            if tb is not None:
                live[rid] = tb["token_count"]
        elif op < 0.8 and live:
            rid = rnd.choice(list(live))
            assert kv_m.release_request(rid).ok() == (kv_r.release_request(rid) == 0)
            live.pop(rid)
        elif op < 0.85:
            n = rnd.randint(1, 6)
            a = kv_m.urgent_reclaim(mine, s_m, n)
            b = kv_r.urgent_reclaim(theirs, s_r, n)
            assert (0 if a.ok() else int(a.error()) + 1) == b
        elif op < 0.88:
            kv_m.instance_teardown(mine)
            kv_r.instance_teardown(theirs)
            live.clear()
        assert mine.validate().ok()
        assert mine.dump() == theirs.dump(), (seed, step)
        st = kv_r.state()
        assert _stats_tuple(kv_m.stats()) == _ref_stats_tuple(st), (seed, step)
        assert kv_m.free_list_size() == st["free_list_size"]
        assert kv_m.active_requests() == st["active_requests"]
        assert sorted(kv_m.address_table().items()) == sorted((a[0], (a[1], a[2])) for a in st["address_table"])


@pytest.mark.parametrize("seed", range(40))
def test_kv_differential_fuzz(tg, ref, seed):
    _kv_fuzz(tg, ref, seed)
