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
