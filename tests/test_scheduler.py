"""Affinity scheduler (scheduler.hpp:41-120) vs the reference on random
snapshots (SPEC acceptance criterion 5), plus the peer-term extension."""
import random

import pytest


def _rand_case(tg, rnd):
    models = {}
    for i in range(rnd.randint(1, 5)):
        m = tg.make_model(f"m{i}", rnd.randint(1_000, 100_000), rnd.randint(1, 3), rnd.choice([0, 8, 64]),
                          location=rnd.choice([tg.ModelLocation.ModelCache, tg.ModelLocation.ModelStore]))
        models[m.model_id] = m
    snaps = []
    for g in range(rnd.randint(1, 8)):
        pool = rnd.randint(2_000, 150_000)
        reuse = {mid: rnd.randint(0, m.total_size) if rnd.random() < 0.5 else 0 for mid, m in models.items()}
        snaps.append(tg.GpuSnapshot(f"gpu{rnd.randint(0, 9)}{g}", rnd.random() < 0.8, pool, rnd.randint(0, pool),
                                    reuse, rnd.choice([55e9, 12e9, 1e9]), rnd.choice([12e9, 3e9])))
    reqs = [rnd.choice(list(models) + ["unknown"]) for _ in range(rnd.randint(1, 8))]
    return models, snaps, reqs


def _ref_schedule(ref, models, snaps, reqs, batch, bs):
    out = ref.schedule({
        "requests": reqs,
        "snapshots": [{"gpu_id": s.gpu_id, "available": s.available, "pool_size": s.pool_size,
                       "free_bytes": s.free_bytes, "reuse": s.reuse_size_by_model, "pcie": s.pcie_bandwidth,
                       "store": s.store_bandwidth} for s in snaps],
        "models": [m.to_json() for m in models.values()], "batch_size": batch, "block_size_tokens": bs})
    return [tuple(a) for a in out["assignments"]], out["deferred"], out["entries"]


@pytest.mark.parametrize("chunk", range(10))
def test_schedule_matches_reference(tg, ref, chunk):
    rnd = random.Random(1000 + chunk)
    for _ in range(100):
        models, snaps, reqs = _rand_case(tg, rnd)
        batch, bs = rnd.randint(1, 4), rnd.choice([16, 32])
        a, d, est = tg.schedule(reqs, snaps, models, batch, bs)
        ra, rd, rent = _ref_schedule(ref, models, snaps, reqs, batch, bs)
        assert a == ra and d == rd
        for mine, theirs in zip(est, rent):
            assert mine == [tuple(c) for c in theirs["candidates"]]
        # ×10 bandwidth scale invariance of the argmin (criterion 5)
        for s in snaps:
            s.pcie_bandwidth *= 10
            s.store_bandwidth *= 10
        a10, d10, _ = tg.schedule(reqs, snaps, models, batch, bs)
        assert (a10, d10) == (a, d)


def test_estimate_load_time_spec_examples(tg):
    """0.5 s / 0 / 2.0 s."""
    m = tg.ModelSpec("m", [], total_size=10_000_000_000)
    g = tg.GpuSnapshot("g", pcie_bandwidth=10e9, store_bandwidth=2.5e9)
    assert tg.estimate_load_time(m, 5_000_000_000, g) == 0.5
    assert tg.estimate_load_time(m, 10_000_000_000, g) == 0.0
    ms = tg.ModelSpec("m", [], total_size=5_000_000_000, location=tg.ModelLocation.ModelStore)
    assert tg.estimate_load_time(ms, 0, g) == 2.0


def test_peer_term(tg):
    """Peer-resident bytes cost S'_peer / B_nvlink instead of / B_pcie; with
    B_nvlink = 0 the reference estimate is unchanged."""
    m = tg.ModelSpec("m", [], total_size=100_000_000_000)
    g = tg.GpuSnapshot("g", pcie_bandwidth=50e9, store_bandwidth=10e9)
    assert tg.estimate_load_time(m, 0, g, 60_000_000_000) == 2.0
    g.nvlink_bandwidth = 600e9
    assert abs(tg.estimate_load_time(m, 0, g, 60_000_000_000) - (0.8 + 0.1)) < 1e-12
    # the scheduler prefers the GPU whose peer can feed it
    models = {"m": tg.make_model("m", 100_000, 2, 0)}
    s0 = tg.GpuSnapshot("gpu0", True, 1 << 20, 0, {"m": 0}, 1e9, 1e9, 900e9, {"m": 80_000})
    s1 = tg.GpuSnapshot("gpu1", True, 1 << 20, 0, {"m": 10_000}, 1e9, 1e9, 900e9, {})
    a, _, _ = tg.schedule(["m"], [s0, s1], models)
    assert a == [("m", "gpu0")]
    s0.nvlink_bandwidth = s1.nvlink_bandwidth = 0.0
    a, _, _ = tg.schedule(["m"], [s0, s1], models)
    assert a == [("m", "gpu1")]
