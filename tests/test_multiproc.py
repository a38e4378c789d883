"""N>1 host logic over torch.distributed (gloo, world size 2, CPU).

C4: GPT-20B tensor-sharded over N ranks; each rank owns an
independent pool and loads its shard ModelSpec — no data-path collective.
Per-rank LoadOutcome / dump must equal the reference ReuseStore run on that
rank's shard.  The affinity scheduler runs on snapshots gathered from all
ranks and must pick the same GPU on every rank (and match the reference)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

GIB = 1 << 30


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2512_01357_b200 as tg
        from oracle import ref
        from test_control_plane import outcome_json
        gpt = {m.model_id: m for m in tg.default_catalog()}["gpt20B"]
        shard = tg.shard_model(gpt, rank, world)
        pool = tg.ReuseStore(tg.GpuSpec(f"gpu{rank}", 160 * GIB), device=None)
        st = tg.ModelStatsTable()
        st.record_request(shard.model_id, 0.0)
        cold = pool.load_model(shard, st, 0.0).value()
        pool.end_instance(shard.model_id)
        st.record_request(shard.model_id, 1.0)
        warm = pool.load_model(shard, st, 1.0).value()
        # reference on the same shard
        r = ref.ReuseStore(160 * GIB, gpu_id=f"gpu{rank}")
        rs = ref.ModelStatsTable()
        rs.record_request(shard.model_id, 0.0)
        rc = r.load_model(shard.to_json(), rs, 0.0)
        r.end_instance(shard.model_id)
        rs.record_request(shard.model_id, 1.0)
        rw = r.load_model(shard.to_json(), rs, 1.0)
        ok = outcome_json(cold) == rc and outcome_json(warm) == rw and pool.dump() == r.dump()
        # gather (shard bytes, outcome ok, reuse of the full model on this pool)
        mine = {"rank": rank, "bytes": shard.total_size, "ok": ok, "cold_xfer": cold.bytes_transferred,
                "warm_xfer": warm.bytes_transferred, "free": pool.free_bytes(),
                "reuse": {m.model_id: pool.reuse_size(m) for m in tg.default_catalog()}}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        # global affinity decision from gathered snapshots, identical on every rank
        snaps = [tg.GpuSnapshot(f"gpu{v['rank']}", True, 160 * GIB, v["free"], v["reuse"]) for v in allv]
        reg = {m.model_id: m for m in tg.default_catalog()}
        a, d, _ = tg.schedule(["opt1.3B", "gpt20B"], snaps, reg, 1, 16)
        decisions = [None] * world
        dist.all_gather_object(decisions, a)
        q.put((rank, allv, decisions))
    finally:
        dist.destroy_process_group()


def test_sharded_gpt20b_two_ranks(ref):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, allv, decisions in res:
        assert all(v["ok"] for v in allv)
        assert sum(v["bytes"] for v in allv) == 40_000_000_000
        assert all(v["cold_xfer"] == v["bytes"] and v["warm_xfer"] == 0 for v in allv)
        assert decisions[0] == decisions[1]
    # pools hold disjoint shards (no cross-rank reuse of the full model)
    assert all(v["reuse"]["gpt20B"] == 0 for v in res[0][1])
