"""Asynchronous loads (TG_LOAD_ASYNC, §8(f) row 1: loads overlapped across
GPUs during a trace replay).

tg_load_model with TG_LOAD_ASYNC returns once the reference's decision is
committed and the data plane is enqueued; the wait and the digest
bookkeeping run at the pool's next operation or tg_pool_sync.  Checked here:

* decisions and dumps are those of the synchronous path (and of the compiled
  reference) load by load, and the completed outcome carries the same digests;
* two pools on one device with loads in flight at once both land byte-exact;
* a pool that pulls from a peer asynchronously is never overwritten under its
  reads: the peer's next load waits (on the device) for the reader's event;
* a load that fails while asynchronous reports the error at tg_pool_sync, its
  tensors stay suspect, and the next reload repairs them.
"""
import pytest

pytestmark = pytest.mark.gpu

ASYNC = 16


def _seq(tg):
    """The shrunken C2 switch (qwen3B <-> opt1.3B in 7 GiB: relocation waves,
    evictions, placements) run back and forth."""
    cat = {m.model_id: m for m in tg.default_catalog()}
    a, b = cat["qwen3B"], cat["opt1.3B"]
    return [a, b, a, b, a]


def _cpu_digest(cpu, tid, size):
    return cpu.content_fingerprint(cpu.synth(tid.hi, tid.lo, size), threads=16)[0]


def test_async_loads_match_sync_loads(tg, cpu):
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    seq = _seq(tg)
    models = {m.model_id: m for m in seq}.values()
    pools = [tg.ReuseStore(tg.GpuSpec("gpu0", 7 << 30), device=0) for _ in range(2)]
    stats = [tg.ModelStatsTable(), tg.ModelStatsTable()]
    with HostCheckpoint(list(models)):
        for i, m in enumerate(seq):
            outs = []
            for k, (pool, st) in enumerate(zip(pools, stats)):
                st.record_request(m.model_id, 10.0 * i)
                flags = 1 | 2 | 8 | (ASYNC if k else 0)
                outs.append(pool.load_model(m, st, 10.0 * i, tg.LoadPolicy(flags=flags)).value())
            o_sync, o_async = outs
            if i == 2:
                assert o_sync.plan.relocations  # the switch really compacts            # the decision is final when the call returns; the bytes may still move
            assert o_async.hit_tensors == o_sync.hit_tensors
            assert o_async.bytes_transferred == o_sync.bytes_transferred
            assert o_async.bytes_merged == o_sync.bytes_merged
            assert o_async.plan.relocations == o_sync.plan.relocations
            assert pools[1].dump() == pools[0].dump()  # reads of the committed state do not wait
            done = pools[1].sync(details=True)
            assert done is not None and done.verify_mismatches == 0 and done.suspect_tensors == 0
            assert done.digests == o_sync.digests
            assert pools[1].sync() is None  # nothing left in flight
            for pool in pools:
                pool.end_instance(m.model_id)
        for t in seq[-1].tensors:
            assert pools[1].fingerprint_tensor(t.id) == _cpu_digest(cpu, t.id, t.size)
    for p in pools:
        p.close()


def test_async_loads_on_two_pools_overlap_and_land(tg, cpu):
    """Both pools' loads are in flight at once (one device here; on a box
    with more GPUs each pool has its own)."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m1 = tg.make_model("ovl-1", 400_000_019, 6, 0)
    m2 = tg.make_model("ovl-2", 300_000_007, 5, 0)
    p1 = tg.ReuseStore(tg.GpuSpec("gpu0", 500_000_000), device=0)
    p2 = tg.ReuseStore(tg.GpuSpec("gpu1", 500_000_000), device=0)
    s1, s2 = tg.ModelStatsTable(), tg.ModelStatsTable()
    s1.record_request(m1.model_id, 0.0)
    s2.record_request(m2.model_id, 0.0)
    pol = tg.LoadPolicy(flags=1 | 2 | 8 | ASYNC)
    with HostCheckpoint([m1, m2]):
        o1 = p1.load_model(m1, s1, 0.0, pol).value()
        o2 = p2.load_model(m2, s2, 0.0, pol).value()
        assert o1.bytes_transferred == m1.total_size and o2.bytes_transferred == m2.total_size
        d1, d2 = p1.sync(details=True), p2.sync(details=True)
        assert d1.pcie_bytes == m1.total_size and d2.pcie_bytes == m2.total_size
        for m, d in ((m1, d1), (m2, d2)):
            for i, t in enumerate(m.tensors):
                assert d.digests[i] == _cpu_digest(cpu, t.id, t.size), t.name
    p1.close()
    p2.close()


def test_async_peer_reads_are_not_overwritten(tg, cpu):
    """b pulls m from a (TG_LOAD_PEER, async); a at once evicts m and loads
    another model over the same bytes.  a's load waits for b's reads on the
    device, so b's pulled bytes verify against a's digests (no repair)."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("peer-src", 300_000_013, 4, 0)
    x = tg.make_model("peer-over", 300_000_001, 4, 0)
    a = tg.ReuseStore(tg.GpuSpec("gpu0", 320_000_000), device=0)
    b = tg.ReuseStore(tg.GpuSpec("gpu1", 320_000_000), device=0)
    b.add_peer(a)
    sa, sb = tg.ModelStatsTable(), tg.ModelStatsTable()
    with HostCheckpoint([m, x]):
        sa.record_request(m.model_id, 0.0)
        a.load_model(m, sa, 0.0).value()
        a.end_instance(m.model_id)
        offs = {t.id: a.tensor_info(t.id)["offset"] for t in m.tensors}
        sb.record_request(m.model_id, 1.0)
        ob = b.load_model(m, sb, 1.0, tg.LoadPolicy(flags=1 | 2 | 4 | 8 | ASYNC)).value()
        assert ob.bytes_transferred == m.total_size
        a.evict_model(m.model_id)
        sa.record_request(x.model_id, 2.0)
        ox = a.load_model(x, sa, 2.0).value()  # overwrites m's old bytes in a's arena
        assert {p.offset for p in ox.plan.placements} & set(offs.values())  # x lands where m was
        done = b.sync(details=True)
        assert done.peer_bytes == m.total_size and done.pcie_bytes == 0
        assert done.verify_mismatches == 0 and done.repaired_bytes == 0
        for i, t in enumerate(m.tensors):
            assert done.digests[i] == _cpu_digest(cpu, t.id, t.size), t.name
            assert b.fingerprint_tensor(t.id) == _cpu_digest(cpu, t.id, t.size), t.name
        for t in x.tensors:
            assert a.fingerprint_tensor(t.id) == _cpu_digest(cpu, t.id, t.size), t.name
    a.close()
    b.close()


def test_async_failure_reported_at_sync_then_repaired(tg, cpu):
    """A source whose bytes miss their manifest digest, loaded asynchronously:
    tg_load_model already returned 0; tg_pool_sync reports the failure, the
    tensor is suspect, and once the source is corrected the next reload
    re-sends it."""
    import ctypes as C
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint, synth_host
    m = tg.make_model("async-fail", 80_000_009, 4, 0)
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", 100_000_000), device=0)
    st = tg.ModelStatsTable()
    t0 = m.tensors[0]
    with HostCheckpoint([m]):
        buf = synth_host(t0.id, t0.size)
        bad = N.DigestC(1, 2)
        N.check_runtime(N.lib.tg_host_register(t0.id.c(), C.c_void_p(buf.ctypes.data), t0.size, C.byref(bad)))
        st.record_request(m.model_id, 0.0)
        o = pool.load_model(m, st, 0.0, tg.LoadPolicy(flags=1 | 2 | 8 | ASYNC)).value()
        assert o.bytes_transferred == m.total_size
        with pytest.raises(N.TangramRuntimeError):
            pool.sync()
        assert pool.tensor_info(t0.id)["suspect"]
        N.check_runtime(N.lib.tg_host_register(t0.id.c(), C.c_void_p(buf.ctypes.data), t0.size, None))
        pool.end_instance(m.model_id)
        st.record_request(m.model_id, 1.0)
        o2 = pool.load_model(m, st, 1.0, tg.LoadPolicy(flags=1 | 2 | 8 | ASYNC)).value()
        assert o2.bytes_transferred == 0
        d2 = pool.sync(details=True)
        assert d2.repaired_bytes >= t0.size and d2.suspect_tensors == 0
        for t in m.tensors:
            assert pool.fingerprint_tensor(t.id) == _cpu_digest(cpu, t.id, t.size), t.name
    pool.close()
