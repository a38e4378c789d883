"""Device load path on a B200: decisions bit-exact with the reference
(golden fixtures from oracle/_ref), pooled bytes bit-exact with the CPU
restatement (every resident tensor's device fingerprint equals tgfp1 of its
synthetic checkpoint bytes computed on the CPU), block tables equal to the
reference's.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from test_control_plane import _fuzz_once, result_json

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
GIB = 1 << 30


def _expected_digest(cpu, tid, size):
    data = cpu.synth(tid.hi, tid.lo, size)
    return cpu.content_fingerprint(data, threads=16)[0]


class HbmCache:
    """Device-resident synthetic sources for a set of models."""

    def __init__(self, tg, models, device=0):
        from paper_2512_01357_b200 import _native as N
        from paper_2512_01357_b200.checkpoint import DeviceBuffer
        self.bufs = {}
        for m in models:
            for t in m.tensors:
                if t.id in self.bufs:
                    continue
                b = DeviceBuffer(t.size, device)
                assert N.lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), device) == 0
                assert N.lib.tg_host_register(t.id.c(), C.c_void_p(b.ptr), t.size, None) == 0
                self.bufs[t.id] = b

    def close(self):
        from paper_2512_01357_b200 import _native as N
        for tid, b in self.bufs.items():
            N.lib.tg_host_unregister(tid.c())
            b.free()


def _check_pooled_bytes(tg, cpu, pool, expected_cache):
    """Every resident tensor: device fingerprint == CPU tgfp1 of its bytes."""
    dump = pool.dump()
    for e in dump["tensor_map"]:
        tid = tg.TensorId.from_hex(e["tensor"])
        if tid not in expected_cache:
            expected_cache[tid] = _expected_digest(cpu, tid, e["size"])
        assert pool.fingerprint_tensor(tid) == expected_cache[tid], e
        assert pool.tensor_info(tid)["digest"] == expected_cache[tid]


@pytest.mark.parametrize("fused", [False, True], ids=["K3+K1", "K3F"])
@pytest.mark.parametrize("case,merge", [("pg_32", 0), ("gm_36", 1)])
def test_c2_switch_bytes_and_decisions(tg, cpu, case, merge, fused):
    g = json.load(open(os.path.join(GOLDEN, "c1_c2_loads.json")))[case]
    gib = int(case.split("_")[1])
    cat = {m.model_id: m for m in tg.default_catalog()}
    seq = ["opt13B", "opt6.7B", "opt13B", "opt6.7B", "opt13B"]
    cache = HbmCache(tg, [cat["opt13B"], cat["opt6.7B"]])
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=gib * GIB), device=0)
    stats = tg.ModelStatsTable()
    expected = {}
    try:
        for i, mid in enumerate(seq):
            stats.record_request(mid, 10.0 * i)
            stats.set_load_bandwidth(mid, 55e9)
            r = pool.load_model(cat[mid], stats, 10.0 * i,
                                tg.LoadPolicy(merge=merge, flags=1 | 2 | (8 if fused else 0)))
            assert result_json(r) == g["loads"][i], f"load {i}"
            o = r.value()
            assert o.verify_mismatches == 0 and o.repaired_bytes == 0
            assert o.device_src_bytes == o.bytes_transferred
            _check_pooled_bytes(tg, cpu, pool, expected)
            pool.end_instance(mid)
        assert pool.dump() == g["final_dump"]
    finally:
        pool.close()
        cache.close()


def test_c1_cold_then_warm_from_host(tg, cpu):
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    g = json.load(open(os.path.join(GOLDEN, "c1_c2_loads.json")))["c1_160"]
    m = {x.model_id: x for x in tg.default_catalog()}["opt1.3B"]
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=160 * GIB), device=0)
    stats = tg.ModelStatsTable()
    with HostCheckpoint([m]) as ck:
        outs = []
        for i in range(2):
            stats.record_request(m.model_id, 10.0 * i)
            stats.set_load_bandwidth(m.model_id, 55e9)
            r = pool.load_model(m, stats, 10.0 * i)
            assert result_json(r) == g["loads"][i]
            outs.append(r.value())
            pool.end_instance(m.model_id)
        cold, warm = outs
        assert cold.pcie_bytes == m.total_size and warm.pcie_bytes == 0
        for i, t in enumerate(m.tensors):
            want = cpu.content_fingerprint(ck.view(t.id), threads=16)[0]
            assert cold.digests[i] == want and warm.digests[i] == want
        assert warm.fingerprint_bytes == m.total_size and warm.verify_mismatches == 0
    pool.close()


def test_verification_repairs_drifted_bytes(tg, cpu):
    """A reused tensor whose bytes no longer match its recorded fingerprint is
    re-sent from its host source (content decides reuse vs transfer)."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("drift", 40_000_017, 3, 64)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=64 << 20), device=0)
    stats = tg.ModelStatsTable()
    with HostCheckpoint([m]) as ck:
        cold = pool.load_model(m, stats, 0.0).value()
        pool.end_instance("drift")
        victim = m.tensors[1]
        info = pool.tensor_info(victim.id)
        junk = np.full(4096, 0xAB, dtype=np.uint8)
        N.lib.tg_memcpy(C.c_void_p(info["device_ptr"] + 1000), junk.ctypes.data_as(C.c_void_p), junk.size)
        warm = pool.load_model(m, stats, 1.0).value()
        assert warm.bytes_transferred == 0  # the key still says "hit"
        assert warm.verify_mismatches == 1 and warm.repaired_bytes == victim.size
        assert pool.fingerprint_tensor(victim.id) == cold.digests[1]
        assert pool.fingerprint_tensor(victim.id) == cpu.content_fingerprint(ck.view(victim.id), threads=8)[0]
    pool.close()


def test_snapshot_restore_roundtrip(tg):
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    a, b = tg.make_model("a", 30_000_001, 2, 0), tg.make_model("b", 30_000_003, 3, 0)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=70_000_000), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([a, b]):
        pool.load_model(a, st, 0.0).value()
        pool.end_instance("a")
        snap = pool.snapshot()
        d0 = pool.dump()
        fps = {t.id: pool.fingerprint_tensor(t.id) for t in a.tensors}
        st.record_request("b", 1.0)
        pool.load_model(b, st, 1.0).value()  # evicts / moves a's tensors
        assert pool.dump() != d0
        pool.restore(snap)
        assert pool.dump() == d0
        assert {t.id: pool.fingerprint_tensor(t.id) for t in a.tensors} == fps
    pool.close()


@pytest.mark.parametrize("fused", [False, True], ids=["K3+K1", "K3F"])
def test_peer_pull_same_device(tg, cpu, fused):
    """Misses resident in a peer pool are pulled device-to-device (K5 path;
    on one GPU the peer is a second pool on the same device)."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("peer", 50_000_021, 3, 0)
    a = tg.ReuseStore(tg.GpuSpec("gpu0", 80_000_000), device=0)
    b = tg.ReuseStore(tg.GpuSpec("gpu1", 80_000_000), device=0)
    b.add_peer(a)
    sa, sb = tg.ModelStatsTable(), tg.ModelStatsTable()
    with HostCheckpoint([m]) as ck:
        oa = a.load_model(m, sa, 0.0).value()
        assert b.peer_reuse_size(m) == m.total_size
        ob = b.load_model(m, sb, 0.0, tg.LoadPolicy(flags=1 | 2 | 4 | (8 if fused else 0))).value()
        assert ob.peer_bytes == m.total_size and ob.pcie_bytes == 0
        assert all(p.source == 1 for p in ob.plan.placements)
        assert ob.digests == oa.digests
        for i, t in enumerate(m.tensors):
            assert ob.digests[i] == cpu.content_fingerprint(ck.view(t.id), threads=8)[0]
    a.close()
    b.close()


def test_c3_kv_tables_match_reference(tg):
    """Llama-2-13B + prefill burst (16 / 64 ShareGPT prompts, seed 7) and one
    decode-step batch: device block tables equal the reference's."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    g = json.load(open(os.path.join(GOLDEN, "c3_kv.json")))
    model = tg.make_model("llama2-13B", 26_000_000_000, 40, 819_200)
    with HostCheckpoint([model]):
        for n, case in g.items():
            pool = tg.ReuseStore(tg.GpuSpec(pool_size=160 * GIB), device=0)
            stats = tg.ModelStatsTable()
            stats.record_request("llama2-13B", 0.0)
            pool.load_model(model, stats, 0.0).value()
            kv = tg.KvEngine("llama2-13B", 16, 819_200)
            reqs = [tuple(r) for r in case["requests"]]
            assert kv.batch_allocate(pool, stats, reqs).value() == case["burst"]
            dec = [(r, (p + 15) // 16 * 16 + 1) for r, p in reqs]
            assert kv.batch_allocate(pool, stats, dec).value() == case["decode"]
            for rid, want in case["tables"].items():
                t = kv.table(int(rid))
                assert t.token_count == want["token_count"]
                assert [[k, v] for k, v in sorted(t.lbn_to_pbn.items())] == want["lbn_to_pbn"]
            # address table in HBM agrees with the host's carve runs
            tables, stride, addr = kv.device_tables()
            at = kv.address_table()
            from paper_2512_01357_b200 import _native as N
            hi = max(at) + 1
            buf = (C.c_uint64 * hi)()
            N.lib.tg_memcpy(buf, C.c_void_p(addr), 8 * hi)
            assert all(buf[p] == off for p, (off, _) in at.items())
            kv.instance_teardown(pool)
            assert pool.kv_bytes() == 0 and pool.validate().ok()
            pool.close()


def test_kv_device_fuzz_vs_reference(tg, ref):
    """Random batches / releases / teardowns on a device pool: every table
    read back from HBM equals the reference's."""
    import random
    rnd = random.Random(11)
    for trial in range(6):
        pool_size = rnd.randint(40_000, 100_000)
        mine = tg.ReuseStore(tg.GpuSpec(pool_size=pool_size), device=0)
        theirs = ref.ReuseStore(pool_size)
        sm, sr = tg.ModelStatsTable(), ref.ModelStatsTable()
        kvm, kvr = tg.KvEngine("s", 8, 100), ref.KvEngine("s", 8, 100)
        live, nxt = {}, 1
        for step in range(60):
            op = rnd.random()
            if op < 0.6:
                reqs = []
                for _ in range(rnd.randint(1, 4)):
                    if live and rnd.random() < 0.5:
                        rid = rnd.choice(list(live))
                        reqs.append((rid, live[rid] + rnd.randint(0, 20)))
                    else:
                        reqs.append((nxt, rnd.randint(0, 40)))
                        nxt += 1
                a = kvm.batch_allocate(mine, sm, reqs)
                b = kvr.batch_allocate(theirs, sr, reqs)
                assert a.ok() == b["ok"]
                if b["ok"]:
                    assert a.value() == b["granted"]
                for rid, tok in reqs:
                    tb = kvr.table(rid)
                    if tb:
                        live[rid] = tb["token_count"]
            elif op < 0.9 and live:
                rid = rnd.choice(list(live))
                kvm.release_request(rid)
                kvr.release_request(rid)
                live.pop(rid)
            else:
                kvm.instance_teardown(mine)
                kvr.instance_teardown(theirs)
                live.clear()
            for rid in live:
                t, rt = kvm.table(rid), kvr.table(rid)
                assert [[k, v] for k, v in sorted(t.lbn_to_pbn.items())] == rt["lbn_to_pbn"]
            assert mine.dump() == theirs.dump()
        mine.close()


def test_missing_source_leaves_pool_unchanged(tg):
    """A miss without a byte source fails with TG_ERR_NO_SOURCE before any
    state changes (like a failed plan, reuse_store.hpp:117-119)."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    a, b = tg.make_model("src-a", 20_000_003, 2, 0), tg.make_model("src-b", 20_000_011, 2, 0)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=30_000_000), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([a]):
        pool.load_model(a, st, 0.0).value()
        pool.end_instance("src-a")
        before = pool.dump()
        st.record_request("src-b", 1.0)
        with pytest.raises(N.TangramRuntimeError) as ei:
            pool.load_model(b, st, 1.0)
        assert ei.value.code == 102
        assert pool.dump() == before and pool.validate().ok()
    pool.close()


def test_insufficient_memory_is_a_domain_error(tg, ref):
    """Planning failures come back as the reference's Error values, the pool
    untouched, on a device pool too."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    a = tg.make_model("big", 50_000_000, 2, 0)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=40_000_000), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([a]):
        before = pool.dump()
        r = pool.load_model(a, st, 0.0)
        assert r.error() == tg.Error.InsufficientMemory and pool.dump() == before
    rr = ref.ReuseStore(40_000_000)
    assert rr.load_model(a.to_json(), ref.ModelStatsTable(), 0.0) == {"ok": False, "error": 0}
    pool.close()


def test_kv_tables_survive_engine_copy_and_pool_teardown(tg):
    """KvEngine value semantics (copied in kv_engine.hpp:146 rollback and by
    the simulator): a clone owns independent device tables."""
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=1 << 24), device=0)
    st = tg.ModelStatsTable()
    kv = tg.KvEngine("m", 4, 64)
    a = kv.batch_allocate(pool, st, [(1, 10), (2, 30)]).value()
    c = kv.clone()
    assert c.table(1).lbn_to_pbn == kv.table(1).lbn_to_pbn
    kv.release_request(1)
    kv.batch_allocate(pool, st, [(3, 8)])
    assert c.table(1) is not None and [c.table(1).lbn_to_pbn[i] for i in range(3)] == a[0]
    pool.close()
    del c, kv


def test_model_store_file_sources(tg, cpu, tmp_path):
    """Model Store placement (§8(f) row 2): tensors registered as ranges of a
    checkpoint file stream file → pinned ring → HBM; bytes and fingerprints
    equal the CPU restatement, decisions unchanged."""
    from paper_2512_01357_b200 import _native as N
    m = tg.make_model("store-model", 90_000_029, 4, 0, location=tg.ModelLocation.ModelStore)
    path = tmp_path / "ckpt.bin"
    with open(path, "wb") as f:
        f.write(b"HDR!" * 3)  # odd header so tensor offsets in the file are unaligned
        offs = {}
        for t in m.tensors:
            offs[t.id] = f.tell()
            f.write(cpu.synth(t.id.hi, t.id.lo, t.size).tobytes())
    for t in m.tensors:
        assert N.lib.tg_file_register(t.id.c(), str(path).encode(), offs[t.id], t.size, None) == 0
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=128 << 20), device=0)
    st = tg.ModelStatsTable()
    o = pool.load_model(m, st, 0.0).value()
    assert o.pcie_bytes == m.total_size
    for i, t in enumerate(m.tensors):
        assert o.digests[i] == cpu.content_fingerprint(cpu.synth(t.id.hi, t.id.lo, t.size), threads=8)[0]
    for t in m.tensors:
        N.lib.tg_host_unregister(t.id.c())
    pool.close()


def test_model_store_pipelined_ranges_across_files(tg, cpu, tmp_path):
    """The stager's readers run ahead of the issue loop over every file range
    of a load: tensors from 0 B to several 8 MiB chunks, split over two files
    at unaligned offsets, a second model's ranges interleaved in the same
    files.  Every placed byte equals the CPU restatement."""
    from paper_2512_01357_b200 import _native as N
    sizes = [0, 1, 4095, 8 << 20, (8 << 20) + 17, 3 * (8 << 20) - 5, 50_000_011, 123_457, 33_554_433, 7]
    m = tg.make_model("store-pipe", sum(sizes), len(sizes), 0, location=tg.ModelLocation.ModelStore)
    # make_model splits the total evenly; re-cut it to the sizes above
    ts = [tg.TensorSpec(id=t.id, model_id=m.model_id, name=t.name, size=sz) for t, sz in zip(m.tensors, sizes)]
    m = tg.ModelSpec(model_id=m.model_id, tensors=ts, total_size=sum(sizes), location=tg.ModelLocation.ModelStore)
    files = [tmp_path / "a.bin", tmp_path / "b.bin"]
    handles = [open(f, "wb") for f in files]
    for i, h in enumerate(handles):
        h.write(b"x" * (3 + 5 * i))
    offs = {}
    for i, t in enumerate(m.tensors):
        h = handles[i % 2]
        offs[t.id] = (str(files[i % 2]), h.tell())
        h.write(cpu.synth(t.id.hi, t.id.lo, t.size).tobytes() if t.size else b"")
        h.write(b"pad")
    for h in handles:
        h.close()
    for t in m.tensors:
        path, off = offs[t.id]
        assert N.lib.tg_file_register(t.id.c(), path.encode(), off, t.size, None) == 0
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=256 << 20), device=0)
    st = tg.ModelStatsTable()
    st.record_request(m.model_id, 0.0)
    try:
        o = pool.load_model(m, st, 0.0).value()
        assert o.pcie_bytes == m.total_size and o.verify_mismatches == 0
        for i, t in enumerate(m.tensors):
            want = cpu.content_fingerprint(cpu.synth(t.id.hi, t.id.lo, t.size), threads=8)[0]
            assert o.digests[i] == want, t.name
            assert pool.fingerprint_tensor(t.id) == want, t.name
    finally:
        for t in m.tensors:
            N.lib.tg_host_unregister(t.id.c())
        pool.close()


@pytest.mark.parametrize("source", ["hbm", "host"])
@pytest.mark.parametrize("seed", [52, 51, 13, 7, 99, 1234])
def test_fused_load_kernel_fuzz(tg, cpu, seed, source):
    """Odd-sized models rotating through a small pool: loads with up to 8 WAR
    waves, device-source placements gated on them and in-place verification,
    all in one load-kernel launch (TG_LOAD_FUSED).  Decisions and digests
    equal the unfused path (K3 waves + K1) load by load, and every resident
    tensor's bytes equal the CPU restatement's.  (Seeds 52, 51 and 13 were
    chosen on the control plane for their wave counts; the others are random.)"""
    import random
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    mb = 1 << 20
    rng = random.Random(seed)
    models = [tg.make_model(f"m{seed}_{k}", rng.randrange(40 * mb, 90 * mb) | 1, rng.randrange(2, 6), 64)
              for k in range(4)]
    size = rng.randrange(120 * mb, 170 * mb)
    seq = [rng.randrange(4) for _ in range(12)]
    src = HbmCache(tg, models) if source == "hbm" else HostCheckpoint(models).__enter__()
    pools = {f: tg.ReuseStore(tg.GpuSpec(pool_size=size), device=0) for f in (False, True)}
    stats = {f: tg.ModelStatsTable() for f in pools}
    expected, waves = {}, 0
    try:
        for i, k in enumerate(seq):
            m = models[k]
            res = {}
            for f, pool in pools.items():
                stats[f].record_request(m.model_id, 10.0 * i)
                stats[f].set_load_bandwidth(m.model_id, 55e9)
                res[f] = pool.load_model(m, stats[f], 10.0 * i, tg.LoadPolicy(merge=i % 2, flags=1 | 2 | (8 if f else 0)))
            assert result_json(res[True]) == result_json(res[False]), f"load {i}"
            if not res[True].ok():
                continue
            o, u = res[True].value(), res[False].value()
            waves = max(waves, o.waves)
            assert o.digests == u.digests, f"load {i}"
            assert o.verify_mismatches == 0 and o.repaired_bytes == 0
            _check_pooled_bytes(tg, cpu, pools[True], expected)
            for pool in pools.values():
                pool.end_instance(m.model_id)
        assert pools[True].dump() == pools[False].dump()
        assert waves >= {52: 4, 51: 4, 13: 4}.get(seed, 1)  # the first seeds were picked for deep wave chains
    finally:
        for pool in pools.values():
            pool.close()
        if source == "hbm":
            src.close()
        else:
            src.__exit__(None, None, None)


def test_edge_models_match_reference(tg, ref, cpu):
    """Ragged edges: a model with no tensors, one with a single 1-byte tensor,
    and one whose tensors are 15, 16, 17, 4095, 4096 and 4097 bytes — loaded,
    reloaded and switched against the reference on a small device pool."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    def spec(mid, sizes):
        ts = [tg.TensorSpec(tg.tensor_key(mid, f"t{i}", [max(1, n // 2)]), mid, f"t{i}", n) for i, n in enumerate(sizes)]
        ts.sort(key=lambda t: t.name)
        return tg.ModelSpec(mid, ts, sum(sizes))
    models = [spec("empty", []), spec("one", [1]), spec("ragged", [15, 16, 17, 4095, 4096, 4097])]
    size = 64 * 1024
    mine, theirs = tg.ReuseStore(tg.GpuSpec(pool_size=size), device=0), ref.ReuseStore(size)
    sm, sr = tg.ModelStatsTable(), ref.ModelStatsTable()
    with HostCheckpoint(models[1:]) as ck:
        t = 0.0
        for m in models + models[::-1]:
            sm.record_request(m.model_id, t)
            sr.record_request(m.model_id, t)
            a = mine.load_model(m, sm, t)
            b = theirs.load_model(m.to_json(), sr, t)
            assert a.ok() == b["ok"]
            if a.ok():
                o = a.value()
                assert o.bytes_transferred == b["bytes_transferred"] and o.verify_mismatches == 0
                for i, tt in enumerate(m.tensors):
                    assert o.digests[i] == cpu.content_fingerprint(ck.view(tt.id), threads=1)[0]
            mine.end_instance(m.model_id)
            theirs.end_instance(m.model_id)
            assert mine.dump() == theirs.dump()
            t += 1.0
    assert mine.validate().ok()
    mine.close()


def test_concurrent_load_kernels_on_one_gpu(tg, ref):
    """Two pools on one GPU load concurrently from two host threads (ctypes
    drops the GIL), each with multi-wave GlobalMerge plans: the gated load
    kernels share the SMs without deadlock (a gated tile only waits for tiles
    taken earlier by running warps), and both pools end equal to the
    reference with every reused tensor verified."""
    import random
    import threading
    mb = 1 << 20
    rng = random.Random(52)
    models = [tg.make_model(f"cc_{k}", rng.randrange(40 * mb, 90 * mb) | 1, rng.randrange(2, 6), 64) for k in range(4)]
    size = rng.randrange(120 * mb, 170 * mb)
    seq = [rng.randrange(4) for _ in range(12)]
    cache = HbmCache(tg, models)
    pools = [tg.ReuseStore(tg.GpuSpec(f"gpu{i}", size), device=0) for i in range(2)]
    errors, waves = [], [0, 0]

    def run(i):
        try:
            st = tg.ModelStatsTable()
            for j, k in enumerate(seq):
                m = models[k]
                st.record_request(m.model_id, 10.0 * j)
                st.set_load_bandwidth(m.model_id, 55e9)
                r = pools[i].load_model(m, st, 10.0 * j, tg.LoadPolicy(merge=1))
                if r.ok():
                    assert r.value().verify_mismatches == 0
                    waves[i] = max(waves[i], r.value().waves)
                pools[i].end_instance(m.model_id)
        except Exception as e:  # pragma: no cover
            errors.append(e)
    try:
        threads = [threading.Thread(target=run, args=(i,)) for i in range(2)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert not errors and not any(t.is_alive() for t in threads)
        theirs = ref.ReuseStore(size)
        rs = ref.ModelStatsTable()
        for j, k in enumerate(seq):
            m = models[k]
            rs.record_request(m.model_id, 10.0 * j)
            rs.set_load_bandwidth(m.model_id, 55e9)
            theirs.load_model(m.to_json(), rs, 10.0 * j, merge=1)
            theirs.end_instance(m.model_id)
        for p in pools:
            d, r = p.dump(), theirs.dump()
            d.pop("gpu_id", None), r.pop("gpu_id", None)
            assert d == r
            assert p.validate().ok()
        assert max(waves) >= 2
    finally:
        for p in pools:
            p.close()
        cache.close()


def test_kv_pressure_reclaims_tensors_then_reload(tg, ref, cpu):
    """On-demand KV under pressure (urgent reclaim, kv_engine.hpp:183-194)
    evicts resident tensors of an idle model on a device pool; after the KV
    teardown the model reloads — evicted tensors re-sent, survivors verified in
    place — every step equal to the reference, and every resident tensor's
    bytes equal to the CPU restatement."""
    mb = 1 << 20
    idle = tg.make_model("idle", 90 * mb + 7, 3, 64)
    busy = tg.make_model("busy", 30 * mb + 3, 2, 4096)
    size = 150 * mb
    cache = HbmCache(tg, [idle, busy])
    mine, theirs = tg.ReuseStore(tg.GpuSpec(pool_size=size), device=0), ref.ReuseStore(size)
    sm, sr = tg.ModelStatsTable(), ref.ModelStatsTable()
    expected = {}
    try:
        for t, m in ((0.0, idle), (1.0, busy)):
            sm.record_request(m.model_id, t)
            sr.record_request(m.model_id, t)
            assert mine.load_model(m, sm, t).ok() and theirs.load_model(m.to_json(), sr, t)["ok"]
        mine.end_instance(idle.model_id)
        theirs.end_instance(idle.model_id)
        kvm, kvr = tg.KvEngine("busy", 16, 4096), ref.KvEngine("busy", 16, 4096)
        reqs = [(i + 1, 2000) for i in range(8)]  # 8 x 125 blocks x 64 KiB: forces reclaim
        a, b = kvm.batch_allocate(mine, sm, reqs), kvr.batch_allocate(theirs, sr, reqs)
        assert a.ok() == b["ok"]
        assert kvm.stats().reclaim_events == kvr.state()["stats"]["reclaim_events"] >= 1
        assert mine.dump() == theirs.dump()
        _check_pooled_bytes(tg, cpu, mine, expected)
        kvm.instance_teardown(mine)
        kvr.instance_teardown(theirs)
        sm.record_request(idle.model_id, 2.0)
        sr.record_request(idle.model_id, 2.0)
        o = mine.load_model(idle, sm, 2.0).value()
        r = theirs.load_model(idle.to_json(), sr, 2.0)
        assert o.bytes_transferred == r["bytes_transferred"] > 0 and o.verify_mismatches == 0
        assert mine.dump() == theirs.dump()
        _check_pooled_bytes(tg, cpu, mine, expected)
    finally:
        mine.close()
        cache.close()


SOAK_SEEDS = int(os.environ.get("TANGRAM_SOAK_SEEDS", "6"))


@pytest.mark.parametrize("seed", range(SOAK_SEEDS))
def test_device_store_differential_fuzz(tg, ref, cpu, seed):
    """The control-plane differential fuzz (loads under every merge /
    strictness / random-eviction policy, end_instance, evict_tensor,
    evict_model, move_tensor, KV regions) on a device pool with real bytes:
    every op equals the reference (outcome, dump, accessors), load flags are
    drawn from {verify+fingerprint+fused, unfused, verify-only, fused}, and
    after every op each resident tensor's device bytes fingerprint to the CPU
    restatement's digest of its checkpoint bytes (and to the digest the pool
    recorded, when it has one).  TANGRAM_SOAK_SEEDS widens the seed range."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    expected = {}

    def sources(models, pool):
        return HbmCache(tg, models) if seed % 2 else HostCheckpoint(models)

    _fuzz_once(tg, ref, 1000 + seed, n_ops=150, device=0, scale=257, sources=sources,
               on_step=_soak_checker(tg, cpu, seed, {}))


@pytest.mark.parametrize("seed", [36])
def test_device_store_fuzz_regressions(tg, ref, cpu, seed):
    """Soak seeds that once failed, kept in the default run.  Seed 36: a
    tensor placed without a fingerprint (a load without
    TG_LOAD_FINGERPRINT_NEW) is relocated by a later load of its model; the
    relocation marks it suspect until the move is verified, which must not
    count as a content mismatch (nothing is re-sent)."""
    test_device_store_differential_fuzz(tg, ref, cpu, seed)


@pytest.mark.parametrize("seed", range(max(1, SOAK_SEEDS // 2)))
def test_device_store_fuzz_async(tg, ref, cpu, seed):
    """The device fuzz with every load asynchronous (TG_LOAD_ASYNC): decisions
    and dumps still equal the reference op by op (they are final when the
    call returns).  After half of the ops the pending load is finished
    explicitly (tg_pool_sync: no mismatch, nothing left suspect) and every
    resident tensor is checked against the CPU restatement; after the other
    half nothing is checked, so the next op — a load, an eviction, a move, a
    KV region — has to land the previous load itself."""
    import random
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    pick = random.Random(7000 + seed)
    check = _soak_checker(tg, cpu, seed, {})

    def sources(models, pool):
        return HbmCache(tg, models) if seed % 2 else HostCheckpoint(models)

    def on_step(pool, r):
        if pick.random() < 0.5:
            return
        done = pool.sync()
        if done is not None:
            assert done.verify_mismatches == 0 and done.suspect_tensors == 0
        check(pool, r)

    _fuzz_once(tg, ref, 3000 + seed, n_ops=120, device=0, scale=257, sources=sources, on_step=on_step,
               extra_flags=16)


def _soak_checker(tg, cpu, seed, expected, peer_bytes=None):
    def on_step(pool, r):
        if r is not None and r.ok():
            o = r.value()
            assert o.verify_mismatches == 0 and o.repaired_bytes == 0
        for e in pool.dump()["tensor_map"]:
            tid = tg.TensorId.from_hex(e["tensor"])
            if tid not in expected:
                expected[tid] = _expected_digest(cpu, tid, e["size"])
            assert pool.fingerprint_tensor(tid) == expected[tid], (seed, e)
            info = pool.tensor_info(tid)
            if info["has_digest"]:
                assert info["digest"] == expected[tid], (seed, e)
        if r is not None and r.ok() and peer_bytes is not None:
            peer_bytes.append(r.value().peer_bytes)
    return on_step


class _PeerHolder:
    """A second device pool holding every model (loaded from an HBM cache that
    is then dropped), attached as the fuzz pool's peer: the fuzz pool's misses
    can only be served over the peer mapping."""

    def __init__(self, tg, models, pool, size):
        self.peer = tg.ReuseStore(tg.GpuSpec("peer", size), device=0)
        cache = HbmCache(tg, models)
        try:
            st = tg.ModelStatsTable()
            for i, m in enumerate(models):
                st.record_request(m.model_id, float(i))
                assert self.peer.load_model(m, st, float(i)).ok()
                self.peer.end_instance(m.model_id)
        finally:
            cache.close()
        pool.add_peer(self.peer)

    def close(self):
        self.peer.close()


@pytest.mark.parametrize("seed", range(max(1, SOAK_SEEDS // 2)))
def test_device_store_fuzz_peer_sourced(tg, ref, cpu, seed):
    """The same fuzz with no registered byte source: every miss is pulled from
    a peer pool that holds all models (TG_LOAD_PEER).  Decisions still equal
    the reference's, the pulled bytes fingerprint to the CPU restatement, and
    the misses are counted as peer bytes."""
    pulled = []

    def sources(models, pool):
        return _PeerHolder(tg, models, pool, sum(m.total_size for m in models) + (1 << 20))

    _fuzz_once(tg, ref, 2000 + seed, n_ops=120, device=0, scale=257, sources=sources,
               on_step=_soak_checker(tg, cpu, seed, {}, pulled), extra_flags=4)
    assert sum(pulled) > 0
