"""Device tensor index: the host image of the open-addressing
table the pool publishes to HBM.  CPU half: the image mirrors the tensor map
(reuse_store.hpp:338, TensorEntry :26-32) after every kind of mutation, and is
a pure function of the store's state.  The GPU half (test_gpu_index.py)
checks the published device table and device lookups against it.
"""
import random

import pytest

MB = 1 << 20


def probe(cap, img, key):
    """Linear probe from key.lo & (cap - 1) — the consumer-side
    include/tangram_index.cuh, restated."""
    i = key[1] & (cap - 1)
    for _ in range(cap):
        s = img[i]
        if not s["flags"] & 1:
            return None
        if s["key"] == key:
            return s
        i = (i + 1) & (cap - 1)
    return None


def check_image(tg, cpu, pool, absent=()):
    cap, img = pool.index_image()
    dump = pool.dump()["tensor_map"]
    assert cap >= 1024 and cap & (cap - 1) == 0 and cap >= 2 * len(dump)
    assert sum(1 for s in img if s["flags"] & 1) == len(dump)
    for e in dump:
        t = tg.TensorId.from_hex(e["tensor"])
        s = probe(cap, img, (t.hi, t.lo))
        assert s is not None, e
        assert (s["offset"], s["size"], s["last_access"]) == (e["offset"], e["size"], e["last_access"])
        assert bool(s["flags"] & 2) == e["pinned"]
        assert s["model"] == cpu.murmur3(e["model"].encode(), 0)[1]
    for t in absent:
        assert probe(cap, img, (t.hi, t.lo)) is None
    return cap, img


@pytest.mark.parametrize("seed", range(6))
def test_index_image_tracks_every_mutation(tg, cpu, seed):
    rng = random.Random(seed)
    models = [tg.make_model(f"ix{seed}_{k}", rng.randrange(20 * MB, 60 * MB) | 1, rng.randrange(2, 7), 64)
              for k in range(4)]
    all_ids = {t.id for m in models for t in m.tensors}
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=rng.randrange(70 * MB, 120 * MB)), device=None)
    stats = tg.ModelStatsTable()
    for i in range(30):
        m = models[rng.randrange(4)]
        op = rng.random()
        if op < 0.55:
            stats.record_request(m.model_id, float(i))
            if pool.load_model(m, stats, float(i), tg.LoadPolicy(merge=i % 2)).ok():
                if rng.random() < 0.8:
                    pool.end_instance(m.model_id)
        elif op < 0.7:
            pool.end_instance(m.model_id)
        elif op < 0.8:
            pool.evict_model(m.model_id)
        elif op < 0.9:
            resident = [tg.TensorId.from_hex(e["tensor"]) for e in pool.dump()["tensor_map"] if not e["pinned"]]
            if resident:
                pool.evict_tensor(rng.choice(resident))
        else:
            runs = pool.dump()["regions"]
            free = [r for r in runs if r["state"] == "free"]
            movable = [tg.TensorId.from_hex(e["tensor"]) for e in pool.dump()["tensor_map"] if not e["pinned"]]
            if free and movable:
                pool.move_tensor(rng.choice(movable), rng.choice(free)["offset"])
        resident = {tg.TensorId.from_hex(e["tensor"]) for e in pool.dump()["tensor_map"]}
        check_image(tg, cpu, pool, absent=all_ids - resident)
    pool.close()


def test_index_image_is_a_function_of_state(tg):
    """Same operations → same image on a second pool; the table grows past
    1024 slots with the tensor count."""
    def build():
        pool = tg.ReuseStore(tg.GpuSpec(pool_size=4 << 30), device=None)
        stats = tg.ModelStatsTable()
        for k in range(3):
            m = tg.make_model(f"big{k}", 700 * MB + 13, 200, 64)  # ~600 tensors per model
            pool.load_model(m, stats, float(k))
            pool.end_instance(m.model_id)
        return pool
    a, b = build(), build()
    ca, ia = a.index_image()
    assert (ca, ia) == b.index_image()
    assert ca >= 2048 and sum(1 for s in ia if s["flags"] & 1) == len(a.dump()["tensor_map"])
    a.close()
    b.close()


def test_device_index_needs_a_device(tg):
    """Control-plane pools have no device table; nothing is emulated."""
    import ctypes as C
    from paper_2512_01357_b200 import _native as N
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=1 << 30), device=None)
    ptr, cap = C.c_void_p(), C.c_uint64()
    assert N.lib.tg_pool_device_index(pool._h, C.byref(ptr), C.byref(cap)) == 101  # TG_ERR_NO_DEVICE
    keys, out = (N.TensorIdC * 1)(), (N.IndexHitC * 1)()
    assert N.lib.tg_index_lookup(pool._h, keys, 1, out) == 101
    pool.close()
