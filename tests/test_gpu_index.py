"""Device tensor index on a B200: the table published in HBM
equals the host image byte for byte after every kind of mutation, and device
lookups (K6, through the consumer probe include/tangram_index.cuh) agree with
the pool's tensor map."""
import ctypes as C
import random

import pytest

from test_gpu_load import HbmCache
from test_index import check_image

pytestmark = pytest.mark.gpu
MB = 1 << 20


def check_device(tg, cpu, pool, ids):
    from paper_2512_01357_b200 import _native as N
    cap, img = check_image(tg, cpu, pool)
    ptr, dcap = pool.device_index()
    assert dcap == cap
    dev = (N.IndexSlotC * cap)()
    assert N.lib.tg_memcpy(C.cast(dev, C.c_void_p), C.c_void_p(ptr), cap * 64) == 0
    host = (N.IndexSlotC * cap)()
    n = C.c_uint64()
    assert N.lib.tg_pool_index_image(pool._h, host, cap, C.byref(n)) == 0
    assert bytes(dev) == bytes(host)
    hits = pool.index_lookup(ids)
    for t, h in zip(ids, hits):
        info = pool.tensor_info(t)
        if info is None:
            assert h is None, t
        else:
            assert h == {"offset": info["offset"], "size": info["size"], "pinned": info["pinned"]}, t


@pytest.mark.parametrize("seed", [0, 1])
def test_device_index_follows_the_pool(tg, cpu, seed):
    rng = random.Random(seed)
    models = [tg.make_model(f"dix{seed}_{k}", rng.randrange(20 * MB, 60 * MB) | 1, rng.randrange(2, 7), 64)
              for k in range(4)]
    ids = [t.id for m in models for t in m.tensors]
    cache = HbmCache(tg, models)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=rng.randrange(70 * MB, 120 * MB)), device=0)
    stats = tg.ModelStatsTable()
    snap = None
    try:
        for i in range(24):
            m = models[rng.randrange(4)]
            op = rng.random()
            if op < 0.55:
                stats.record_request(m.model_id, float(i))
                if pool.load_model(m, stats, float(i), tg.LoadPolicy(merge=i % 2)).ok() and rng.random() < 0.8:
                    pool.end_instance(m.model_id)
            elif op < 0.7:
                pool.evict_model(m.model_id)
            elif op < 0.8:
                movable = [tg.TensorId.from_hex(e["tensor"]) for e in pool.dump()["tensor_map"] if not e["pinned"]]
                free = [r for r in pool.dump()["regions"] if r["state"] == "free"]
                if movable and free:
                    pool.move_tensor(rng.choice(movable), rng.choice(free)["offset"])
            elif op < 0.9:
                snap = pool.snapshot()
            elif snap is not None:
                pool.restore(snap)
            check_device(tg, cpu, pool, ids)
    finally:
        pool.close()
        cache.close()
