"""Two-stage planner (plan_allocation, packing.hpp:311-483) directly:
SPEC known answers, bit-exact differential fuzz against the compiled
reference planner, and the reference's own brute-force optimality oracle
(packing_oracle.hpp:78-181, SPEC acceptance criteria 1-2)."""
import random

import pytest


def _ids(tg, n, base=7):
    return [tg.TensorId(base, i + 1) for i in range(n)]


def test_fig5_partitioned_gain(tg, ref):
    """Fig. 5: [F2][T1][F4][T3][F6] + {5,5} → final merge cost 1."""
    t1, t3 = tg.TensorId(1, 1), tg.TensorId(1, 3)
    regions = [(0, 2, "free", None, 0), (2, 1, "tensor", t1, 0), (3, 4, "free", None, 0),
               (7, 3, "tensor", t3, 0), (10, 6, "free", None, 0)]
    news = [tg.TensorSpec(tg.TensorId(2, 1), "m", "n1", 5), tg.TensorSpec(tg.TensorId(2, 2), "m", "n2", 5)]
    p = tg.pool.plan_allocation(regions, news).value()
    assert p.initial_merge_cost == 4 and p.pgp_merge_cost == 1 and p.total_merge_cost == 1
    assert len(p.relocations) == 1
    assert [(x.tensor, x.offset) for x in p.placements] == [(news[0].id, 0), (news[1].id, 10)]
    inst = {"regions": [{"offset": o, "size": s, "state": k, **({"tensor": t.hex()} if t else {})}
                        for o, s, k, t, _ in regions],
            "new_tensors": [{"id": t.id.hex(), "size": t.size} for t in news], "candidates": []}
    bf = ref.brute_force_oracle(inst)
    assert bf["feasible"] and bf["merge_bytes"] == 1


def test_try_packing_spec_examples(ref):
    """SPEC.md:278-279 through the reference itself (our copy is exercised by
    every split decision in the differential fuzz below)."""
    assert ref.try_packing([5, 3], 6, 4) == {"success": True, "first": [5], "second": [3]}
    assert ref.try_packing([7], 6, 4)["success"] is False


def _random_instance(tg, rnd, small=False):
    regions, residents = [], []
    off = 0
    n = rnd.randint(1, 10 if small else 24)
    prev_free = False
    tid = 1
    for i in range(n):
        size = rnd.randint(1, 40)
        kind = rnd.choices(["free", "tensor", "kv_block"], [0.4, 0.5, 0.1 if not small else 0.05])[0]
        if kind == "free" and prev_free:
            kind = "tensor"
        if kind == "tensor":
            t = tg.TensorId(3, tid)
            tid += 1
            regions.append((off, size, "tensor", t, 0))
            residents.append((t, size))
        elif kind == "kv_block":
            regions.append((off, size, "kv_block", None, rnd.randint(1, 9)))
        else:
            regions.append((off, size, "free", None, 0))
        prev_free = kind == "free"
        off += size
    if small:
        residents = residents[:10]
    cands = []
    immovable = []
    for t, size in residents:
        r = rnd.random()
        if r < 0.15:
            immovable.append(t)
        elif r < 0.85:
            cost = rnd.choice([0.0, 0.5, 1.0, 2.0, rnd.random()])
            cands.append(tg.pool.EvictionCandidate(t, size, cost, float(rnd.randint(0, 3)), "old"))
    news = [tg.TensorSpec(tg.TensorId(9, i + 1), "new", f"n{i}", rnd.randint(1, 30))
            for i in range(rnd.randint(1, 6 if small else 10))]
    return regions, news, cands, immovable


def _ref_request(regions, news, cands, immovable, strictness, merge, randomize):
    return {"regions": [{"offset": o, "size": s, "state": k, **({"tensor": t.hex()} if t else {}),
                         **({"block": b} if k == "kv_block" else {})} for o, s, k, t, b in regions],
            "new_tensors": [{"id": t.id.hex(), "size": t.size, "model_id": t.model_id, "name": t.name} for t in news],
            "candidates": [{"tensor": c.tensor.hex(), "size": c.size, "cost": c.cost, "last_access": c.last_access,
                            "model": c.model_id} for c in cands],
            "immovable": [t.hex() for t in immovable], "strictness": strictness, "merge_policy": merge,
            "randomize_eviction": randomize}


def _plan_json(p):
    return {"ok": True,
            "evictions": [{"tensor": e.tensor.hex(), "size": e.size, "cost": e.cost, "last_access": e.last_access,
                           "model": e.model_id} for e in p.evictions],
            "relocations": [{"tensor": r.tensor.hex(), "from": r.from_, "to": r.to, "size": r.size}
                            for r in p.relocations],
            "placements": [{"tensor": x.tensor.hex(), "offset": x.offset, "size": x.size} for x in p.placements],
            "total_eviction_cost": p.total_eviction_cost, "total_merge_cost": p.total_merge_cost,
            "pgp_merge_cost": p.pgp_merge_cost, "initial_merge_cost": p.initial_merge_cost,
            "fallback_evictions": p.fallback_evictions}


@pytest.mark.parametrize("chunk", range(10))
def test_planner_differential(tg, ref, chunk):
    rnd = random.Random(500 + chunk)
    for _ in range(200):
        regions, news, cands, imm = _random_instance(tg, rnd)
        strict, merge, randomize = rnd.random() < 0.2, rnd.random() < 0.2, rnd.random() < 0.1
        a = tg.pool.plan_allocation(regions, news, cands, imm, strict, merge, randomize)
        b = ref.plan_allocation(_ref_request(regions, news, cands, imm, int(strict), int(merge), randomize))
        if b["ok"]:
            assert a.ok() and _plan_json(a.value()) == b
        else:
            assert not a.ok() and int(a.error()) == b["error"]


def test_heuristic_never_beats_brute_force_oracle(tg, ref):
    """SPEC acceptance 2: on >= 500 small instances the exact oracle's optimum
    never exceeds the heuristic's objective (eviction cost + merged bytes /
    intra bandwidth, bandwidth 1)."""
    rnd = random.Random(77)
    checked = 0
    while checked < 500:
        regions, news, cands, imm = _random_instance(tg, rnd, small=True)
        a = tg.pool.plan_allocation(regions, news, cands, imm)
        if not a.ok():
            continue
        p = a.value()
        inst = _ref_request(regions, news, cands, imm, 0, 0, False)
        inst["intra_copy_bandwidth"] = 1.0
        bf = ref.brute_force_oracle(inst)
        if not bf.get("ok"):
            continue
        assert bf["feasible"]
        assert bf["best_cost"] <= p.total_eviction_cost + p.total_merge_cost + 1e-9
        checked += 1
