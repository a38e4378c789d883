"""Cross-process peer pull: one process per GPU in
production; here two processes share cuda:0, which exercises the same CUDA
IPC mapping, index exchange and K3 pull over the peer arena.  Process A loads
a model from host; process B attaches A's arena + index and loads the same
model with TG_LOAD_PEER: every byte comes from A's pool, fingerprints equal
A's and the CPU restatement's.  A stale index (A evicts + overwrites) is
caught by the post-pull fingerprint and repaired from the host source."""
import multiprocessing as mp
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _model(tg):
    return tg.make_model("ipc-model", 48_000_037, 3, 0)


def _owner(q, done):
    sys.path.insert(0, ROOT)
    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = _model(tg)
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", 64 << 20), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([m]):
        o = pool.load_model(m, st, 0.0).value()
        q.put((pool.export_ipc(), pool.index(), o.digests))
        done.wait(120)
    pool.close()


def test_ipc_peer_pull(tg, cpu):
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    ctx = mp.get_context("spawn")
    q, done = ctx.Queue(), ctx.Event()
    a = ctx.Process(target=_owner, args=(q, done))
    a.start()
    try:
        handle, index, a_digests = q.get(timeout=120)
        m = _model(tg)
        pool = tg.ReuseStore(tg.GpuSpec("gpu1", 64 << 20), device=0)
        pid = pool.attach_remote(handle, index)
        assert pid == 0 and pool.peer_reuse_size(m) == m.total_size
        st = tg.ModelStatsTable()
        o = pool.load_model(m, st, 0.0, tg.LoadPolicy(flags=1 | 2 | 4)).value()
        assert o.peer_bytes == m.total_size and o.pcie_bytes == 0
        assert all(p.source == 1 for p in o.plan.placements)
        assert o.digests == a_digests and o.verify_mismatches == 0
        with HostCheckpoint([m]) as ck:
            for i, t in enumerate(m.tensors):
                assert o.digests[i] == cpu.content_fingerprint(ck.view(t.id), threads=8)[0]
            # stale index: pretend A's tensor 0 holds other bytes
            pool.end_instance(m.model_id)
            pool.evict_model(m.model_id)
            bad = [(tid, off, size, (dig[0] ^ 1, dig[1])) if k == 0 else (tid, off, size, dig)
                   for k, (tid, off, size, dig) in enumerate(index)]
            pool.update_remote(pid, bad)
            o2 = pool.load_model(m, st, 1.0, tg.LoadPolicy(flags=1 | 2 | 4)).value()
            assert o2.verify_mismatches == 1 and o2.repaired_bytes > 0
            assert o2.digests == a_digests
        pool.close()
    finally:
        done.set()
        a.join(timeout=60)
    assert a.exitcode == 0


def _reshard_model(tg):
    return tg.make_model("ipc-reshard", 40_000_003, 2, 8192)


def _shard_owner(q, done):
    sys.path.insert(0, ROOT)
    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = _reshard_model(tg)
    tp2 = [tg.shard_model(m, r, 2) for r in range(2)]
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", 48 << 20), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint(tp2):
        for sh in tp2:
            st.record_request(sh.model_id, 0.0)
            pool.load_model(sh, st, 0.0).value()
            pool.end_instance(sh.model_id)
    q.put((pool.export_ipc(), pool.index()))
    done.wait(120)
    pool.close()


@pytest.mark.parametrize("fused", [False, True], ids=["K3+K1", "K3F"])
def test_ipc_reshard_pull(tg, cpu, fused):
    """Re-shard across processes: process A holds the TP2 shards; process B
    attaches A's arena and index and loads the TP4 shards — every tensor
    assembled from A's overlapping TP2 pieces (no host source registered in
    B), fingerprints equal to the CPU restatement of the parent ranges."""
    ctx = mp.get_context("spawn")
    q, done = ctx.Queue(), ctx.Event()
    a = ctx.Process(target=_shard_owner, args=(q, done))
    a.start()
    try:
        handle, index = q.get(timeout=120)
        m = _reshard_model(tg)
        [tg.shard_model(m, r, 2) for r in range(2)]  # lineage of A's shards, known in this process too
        tp4 = [tg.shard_model(m, r, 4) for r in range(4)]
        pool = tg.ReuseStore(tg.GpuSpec("gpu1", 48 << 20), device=0)
        pool.attach_remote(handle, index)
        st = tg.ModelStatsTable()
        for k, sh in enumerate(tp4):
            assert pool.peer_reuse_size(sh) == sh.total_size
            st.record_request(sh.model_id, float(k))
            o = pool.load_model(sh, st, float(k), tg.LoadPolicy(flags=1 | 2 | 4 | (8 if fused else 0))).value()
            assert o.peer_bytes == sh.total_size and o.pcie_bytes == 0
            assert all(p.source == 3 for p in o.plan.placements)
            for i, t in enumerate(sh.tensors):
                parent, begin, size = tg.lineage(t.id)
                want = cpu.content_fingerprint(cpu.synth(parent.hi, parent.lo, size, begin), threads=8)[0]
                assert o.digests[i] == want
            pool.end_instance(sh.model_id)
        pool.close()
    finally:
        done.set()
        a.join(timeout=60)
    assert a.exitcode == 0
