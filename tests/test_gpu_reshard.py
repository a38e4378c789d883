"""Re-shard pulls (SURVEY §8(d) C4 "shards resident on peers in a previous TP
layout", §8(e)): a pool loading the TP4 shards of a model whose TP2 shards
are resident on two peer pools assembles every tensor from the overlapping
TP2 pieces device-to-device (on one GPU the peers are pools on the same
device), with no host source registered.  Decisions equal the reference's
for the TP4 shard ModelSpecs; every assembled tensor fingerprints equal to the
CPU restatement of its byte range of the parent tensor.
"""
import os

import pytest

pytestmark = pytest.mark.gpu


def _expected(cpu, tg, t):
    parent, begin, size = tg.lineage(t.id)
    assert size == t.size
    return cpu.content_fingerprint(cpu.synth(parent.hi, parent.lo, size, begin), threads=8)[0]


@pytest.mark.parametrize("fused", [False, True], ids=["K3+K1", "K3F"])
def test_tp2_to_tp4_reshard_from_peers(tg, cpu, ref, fused):
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("reshard", 60_000_011, 3, 8192)
    tp2 = [tg.shard_model(m, r, 2) for r in range(2)]
    tp4 = [tg.shard_model(m, r, 4) for r in range(4)]
    peers = [tg.ReuseStore(tg.GpuSpec(f"gpu{r}", 40_000_000), device=0) for r in range(2)]
    with HostCheckpoint(tp2):
        for r, p in enumerate(peers):
            st = tg.ModelStatsTable()
            st.record_request(tp2[r].model_id, 0.0)
            o = p.load_model(tp2[r], st, 0.0).value()
            for i, t in enumerate(tp2[r].tensors):  # TP2 bytes = parent ranges
                assert o.digests[i] == _expected(cpu, tg, t)
    # sources unregistered: the TP4 bytes can only come from the peers
    c = tg.ReuseStore(tg.GpuSpec("gpu2", 64_000_000), device=0)
    for p in peers:
        c.add_peer(p)
    sc = tg.ModelStatsTable()
    r_pool, r_stats = ref.ReuseStore(64_000_000, gpu_id="gpu2"), ref.ModelStatsTable()
    for k, shard in enumerate(tp4):
        assert c.peer_reuse_size(shard) == shard.total_size  # the scheduler's S'_peer term
        sc.record_request(shard.model_id, float(k))
        o = c.load_model(shard, sc, float(k), tg.LoadPolicy(flags=1 | 2 | 4 | (8 if fused else 0))).value()
        assert o.peer_bytes == shard.total_size and o.pcie_bytes == 0
        assert all(p.source == 3 for p in o.plan.placements)
        for i, t in enumerate(shard.tensors):
            assert o.digests[i] == _expected(cpu, tg, t), (shard.model_id, t.name)
        c.end_instance(shard.model_id)
        r_stats.record_request(shard.model_id, float(k))
        r_pool.load_model(shard.to_json(), r_stats, float(k))
        r_pool.end_instance(shard.model_id)
        assert c.dump() == r_pool.dump()
    # a warm reload of a TP4 shard reuses in place (no peer bytes)
    sc.record_request(tp4[1].model_id, 9.0)
    o = c.load_model(tp4[1], sc, 9.0).value()
    assert o.bytes_transferred == 0 and o.verify_mismatches == 0
    c.close()
    for p in peers:
        p.close()


def test_reshard_needs_full_cover(tg):
    """A TP4 shard straddling a TP2 boundary with only one TP2 peer resident
    cannot be assembled: the load asks for a host source and, with none
    registered, fails leaving the pool unchanged."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("reshard-gap", 20_000_003, 2, 8192)
    tp2 = [tg.shard_model(m, r, 2) for r in range(2)]
    tp4 = [tg.shard_model(m, r, 4) for r in range(4)]
    a = tg.ReuseStore(tg.GpuSpec("gpu0", 20_000_000), device=0)
    with HostCheckpoint([tp2[0]]):
        st = tg.ModelStatsTable()
        st.record_request(tp2[0].model_id, 0.0)
        a.load_model(tp2[0], st, 0.0).value()
    c = tg.ReuseStore(tg.GpuSpec("gpu1", 20_000_000), device=0)
    c.add_peer(a)
    sc = tg.ModelStatsTable()
    sc.record_request(tp4[0].model_id, 0.0)
    assert c.load_model(tp4[0], sc, 0.0, tg.LoadPolicy(flags=1 | 2 | 4 | 8)).value().peer_bytes == tp4[0].total_size
    before = c.dump()
    sc.record_request(tp4[2].model_id, 1.0)  # bytes [n/2, 3n/4): on no peer
    with pytest.raises(N.TangramRuntimeError):
        c.load_model(tp4[2], sc, 1.0, tg.LoadPolicy(flags=1 | 2 | 4 | 8))
    assert c.dump() == before
    a.close()
    c.close()


def test_reshard_from_own_pool(tg, cpu, ref):
    """One GPU switching TP layout: the TP4 shards are assembled from the
    pool's own resident TP2 shards (device-to-device in HBM), which this load
    neither evicts nor relocates; decisions and dumps equal the reference's."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("reshard-self", 30_000_017, 2, 8192)
    tp2 = [tg.shard_model(m, r, 2) for r in range(2)]
    tp4 = [tg.shard_model(m, r, 4) for r in range(4)]
    size = 70_000_000
    c = tg.ReuseStore(tg.GpuSpec("gpu0", size), device=0)
    r_pool, r_stats, sc = ref.ReuseStore(size), ref.ModelStatsTable(), tg.ModelStatsTable()
    t = 0.0
    with HostCheckpoint(tp2):
        for sh in tp2:
            sc.record_request(sh.model_id, t)
            c.load_model(sh, sc, t).value()
            c.end_instance(sh.model_id)
            r_stats.record_request(sh.model_id, t)
            r_pool.load_model(sh.to_json(), r_stats, t)
            r_pool.end_instance(sh.model_id)
            t += 1.0
    for sh in tp4[:2]:
        sc.record_request(sh.model_id, t)
        o = c.load_model(sh, sc, t, tg.LoadPolicy(flags=1 | 2 | 4 | 8)).value()
        assert all(p.source == 3 for p in o.plan.placements)
        assert o.device_src_bytes == sh.total_size and o.peer_bytes == 0 and o.pcie_bytes == 0
        for i, tt in enumerate(sh.tensors):
            assert o.digests[i] == _expected(cpu, tg, tt)
        c.end_instance(sh.model_id)
        r_stats.record_request(sh.model_id, t)
        r_pool.load_model(sh.to_json(), r_stats, t)
        r_pool.end_instance(sh.model_id)
        assert c.dump() == r_pool.dump()
        t += 1.0
    c.close()


@pytest.mark.parametrize("src_tp,dst_tp", [(3, 2), (3, 5), (5, 3), (7, 2)])
@pytest.mark.parametrize("fused", [False, True], ids=["K3+K1", "fused"])
def test_reshard_piece_boundaries_inside_leaves(tg, cpu, ref, src_tp, dst_tp, fused):
    """Layouts whose shard boundaries fall inside 4 KiB leaves of the target
    shards (odd tensor sizes; tiny tensors whose pieces are shorter than a
    leaf).  Fused, every piece's leaf-aligned interior is copied and hashed by
    the load kernel with seeds from its leaf index, the straddling leaves are
    pre-copied and verified in place, and the host adds the raw sums: the
    digest equals the CPU restatement of the parent range, as on the K3 + K1
    path, and the decisions equal the reference's."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model(f"rs-{src_tp}-{dst_tp}", 30_000_037, 2, 8192)
    tiny = tg.make_model(f"rs-tiny-{src_tp}-{dst_tp}", 12_289, 1, 0)  # shards of a few KiB
    srcs = [tg.shard_model(x, r, src_tp) for x in (m, tiny) for r in range(src_tp)]
    dsts = [tg.shard_model(x, r, dst_tp) for x in (m, tiny) for r in range(dst_tp)]
    holder = tg.ReuseStore(tg.GpuSpec("gpu0", 64_000_000), device=0)
    with HostCheckpoint(srcs):
        st = tg.ModelStatsTable()
        for k, sm in enumerate(srcs):
            st.record_request(sm.model_id, float(k))
            holder.load_model(sm, st, float(k)).value()
            holder.end_instance(sm.model_id)
    c = tg.ReuseStore(tg.GpuSpec("gpu1", 64_000_000), device=0)
    c.add_peer(holder)
    sc = tg.ModelStatsTable()
    r_pool, r_stats = ref.ReuseStore(64_000_000, gpu_id="gpu1"), ref.ModelStatsTable()
    try:
        for k, shard in enumerate(dsts):
            sc.record_request(shard.model_id, float(k))
            o = c.load_model(shard, sc, float(k), tg.LoadPolicy(flags=1 | 2 | 4 | (8 if fused else 0))).value()
            assert o.peer_bytes == shard.total_size and o.pcie_bytes == 0 and o.verify_mismatches == 0
            for i, t in enumerate(shard.tensors):
                want = _expected(cpu, tg, t)
                assert o.digests[i] == want, (shard.model_id, t.name)
                assert c.fingerprint_tensor(t.id) == want, (shard.model_id, t.name)
            c.end_instance(shard.model_id)
            r_stats.record_request(shard.model_id, float(k))
            r_pool.load_model(shard.to_json(), r_stats, float(k))
            r_pool.end_instance(shard.model_id)
            assert c.dump() == r_pool.dump()
    finally:
        c.close()
        holder.close()


def _gated_pulls(o):
    """Placements of re-shard pulls (source 3) whose destination overlaps the
    source range of one of the load's relocations: bytes a WAR wave must read
    before the pull may write them."""
    rel = o.plan.relocations
    return [p for p in o.plan.placements if p.source == 3 and
            any(p.offset < r.from_ + r.size and r.from_ < p.offset + p.size for r in rel)]


@pytest.mark.parametrize("fused", [False, True], ids=["K3+K1", "fused"])
def test_reshard_pulls_gated_on_relocation_waves(tg, cpu, ref, fused):
    """Re-shard pulls into space a relocation wave of the same load vacates.
    A pool switching among TP4 shards of one model (assembled from TP2 peers,
    no host source) and three host-sourced models, under every merge policy,
    with random tensor evictions: fused, a gated pull's piece tasks and
    straddle fragments wait for the wave inside the load kernel and its
    straddle leaves are verified by a second launch behind it.  Decisions and
    dumps equal the reference's op by op; every resident tensor fingerprints
    equal to the CPU restatement; the sequence provably exercises gated
    pulls."""
    import random
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    base = tg.make_model("gr", 30_000_037, 3, 8192)
    tp2 = [tg.shard_model(base, r, 2) for r in range(2)]
    tp4 = [tg.shard_model(base, r, 4) for r in range(4)]
    others = [tg.make_model(f"o{i}", 9_000_000 + i * 1_000_003, 2, 4096) for i in range(3)]
    holder = tg.ReuseStore(tg.GpuSpec("peer", 64_000_000), device=0)
    with HostCheckpoint(tp2):
        st = tg.ModelStatsTable()
        for k, sm in enumerate(tp2):
            st.record_request(sm.model_id, float(k))
            holder.load_model(sm, st, float(k)).value()
            holder.end_instance(sm.model_id)
    expected = {}

    def want(tid, size):
        if tid not in expected:
            lin = tg.lineage(tid)
            data = cpu.synth(lin[0].hi, lin[0].lo, size, lin[1]) if lin else cpu.synth(tid.hi, tid.lo, size)
            expected[tid] = cpu.content_fingerprint(data, threads=8)[0]
        return expected[tid]

    gated = 0
    flags = 1 | 2 | 4 | (8 if fused else 0)
    try:
        with HostCheckpoint(others):
            for seed in range(int(os.environ.get("TANGRAM_RESHARD_SEEDS", "6"))):
                rnd = random.Random(seed)
                size = rnd.choice([24_000_000, 28_000_000, 32_000_000])
                c = tg.ReuseStore(tg.GpuSpec("gpu1", size), device=0)
                c.add_peer(holder)
                r_pool, r_stats, sc = ref.ReuseStore(size, gpu_id="gpu1"), ref.ModelStatsTable(), tg.ModelStatsTable()
                try:
                    for k in range(14):
                        t = float(k + 1)
                        m = rnd.choice(tp4[:2] + others)
                        merge = rnd.choice([0, 1])
                        sc.record_request(m.model_id, t)
                        r_stats.record_request(m.model_id, t)
                        r = c.load_model(m, sc, t, tg.LoadPolicy(merge=tg.MergePolicy(merge), flags=flags))
                        rr = r_pool.load_model(m.to_json(), r_stats, t, merge=merge)
                        assert r.ok() == rr["ok"], (seed, k)
                        if r.ok():
                            o = r.value()
                            assert o.verify_mismatches == 0 and o.pcie_bytes + o.peer_bytes + o.device_src_bytes \
                                == o.bytes_transferred
                            gated += len(_gated_pulls(o))
                            for i, tt in enumerate(m.tensors):
                                assert o.digests[i] == want(tt.id, tt.size), (seed, k, tt.name)
                            c.end_instance(m.model_id)
                            r_pool.end_instance(m.model_id)
                        if rnd.random() < 0.4 and c.dump()["tensor_map"]:
                            e = rnd.choice(c.dump()["tensor_map"])
                            c.evict_tensor(tg.TensorId.from_hex(e["tensor"]))
                            r_pool.evict_tensor(e["tensor"])
                        assert c.dump() == r_pool.dump(), (seed, k)
                        for e in c.dump()["tensor_map"]:
                            tid = tg.TensorId.from_hex(e["tensor"])
                            assert c.fingerprint_tensor(tid) == want(tid, e["size"]), (seed, k, e)
                finally:
                    c.close()
    finally:
        holder.close()
    assert gated > 0
