"""K4D — device-decided KV batches (tg_kv_batch_allocate_device) on a B200.

Batches enqueued between arm and sync are decided by the kernel alone; after
sync the engine must be indistinguishable from the reference KvEngine
(kv_engine.hpp:107-161) driven with the same batches: block tables (read back
from HBM), address table, counters, free list, and the pool dump.  Batches
the device cannot decide alone (contended pool -> urgent reclaim, a request
twice, a shrinking token count) are replayed on the host path at sync, with
the reference's error semantics.
"""
import random

import pytest

pytestmark = pytest.mark.gpu

BS, BPT = 8, 100  # 8 tokens x 100 B = 800 B blocks


def _dev(values):
    import torch
    return torch.tensor(values, dtype=torch.int64, device="cuda:0")


def _fragment(rnd, mine, theirs, n_ops):
    """Identical random alloc/free sequences on both pools -> holes of mixed sizes."""
    held = []
    for i in range(n_ops):
        if held and rnd.random() < 0.45:
            off = held.pop(rnd.randrange(len(held)))
            assert mine.free_kv_region(off).ok() == (theirs.free_kv_region(off) == 0)
        else:
            size = rnd.randint(300, 5000)
            a = mine.alloc_kv_region(size, 10_000 + i)
            rc, off = theirs.alloc_kv_region(size, 10_000 + i)
            assert a.ok() == (rc == 0)
            if a.ok():
                assert a.value() == off
                held.append(off)
    assert mine.dump() == theirs.dump()


def _same_engine(kvm, kvr, mine, theirs, live):
    for rid in live:
        t, rt = kvm.table(rid), kvr.table(rid)
        assert rt, rid
        assert t.token_count == rt["token_count"], rid
        assert [[k, v] for k, v in sorted(t.lbn_to_pbn.items())] == rt["lbn_to_pbn"], rid
    st = kvr.state()
    assert sorted([p, o, s] for p, (o, s) in kvm.address_table().items()) == st["address_table"]
    s = kvm.stats()
    assert [s.pool_invocations, s.alloc_batches, s.blocks_from_free_list, s.blocks_from_pool,
            s.reclaim_events] == [st["stats"][k] for k in ("pool_invocations", "alloc_batches",
                                                          "blocks_from_free_list", "blocks_from_pool",
                                                          "reclaim_events")]
    assert kvm.free_list_size() == st["free_list_size"]
    assert mine.dump() == theirs.dump()


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6, 7, 8])
def test_device_batches_equal_reference(tg, ref, seed):
    rnd = random.Random(seed)
    pool_size = rnd.randint(150_000, 500_000)
    mine = tg.ReuseStore(tg.GpuSpec(pool_size=pool_size), device=0)
    theirs = ref.ReuseStore(pool_size)
    sm, sr = tg.ModelStatsTable(), ref.ModelStatsTable()
    _fragment(rnd, mine, theirs, 40)
    kvm, kvr = tg.KvEngine("s", BS, BPT), ref.KvEngine("s", BS, BPT)
    live, nxt = {}, 1
    applied_total = replayed_total = 0
    for session in range(6):
        # host-path batch: new requests (prefill), releases
        reqs = [(nxt + i, rnd.randint(0, 40)) for i in range(rnd.randint(1, 5))]
        nxt += len(reqs)
        a, b = kvm.batch_allocate(mine, sm, reqs), kvr.batch_allocate(theirs, sr, reqs)
        assert a.ok() == b["ok"]
        for rid, _ in reqs:
            tb = kvr.table(rid)
            if tb:
                live[rid] = tb["token_count"]
        for rid in [r for r in live if rnd.random() < 0.2]:
            assert kvm.release_request(rid).ok() and kvr.release_request(rid) == 0
            live.pop(rid)
        if not live:
            continue
        # device session
        assert kvm.device_arm(mine, 64, 32, 16).ok()
        keep, first_err = [], None
        for step in range(rnd.randint(1, 10)):
            rids = [r for r in live if rnd.random() < 0.7] or [next(iter(live))]
            batch = [(r, live[r] + rnd.choice([0, 1, 1, 2, 7, 15, 30])) for r in rids]
            x = rnd.random()
            if x < 0.08:  # a request twice: the device leaves the batch to the host
                batch.append((batch[0][0], batch[0][1] + 3))
            elif x < 0.12:  # shrinking token count: InvalidArgument (partial effects kept)
                batch.append((batch[0][0], 0))
            slots = _dev([kvm.request_slot(r) for r, _ in batch])
            toks = _dev([t for _, t in batch])
            keep += [slots, toks]
            kvm.batch_allocate_device(slots.data_ptr(), toks.data_ptr(), len(batch))
            rr = kvr.batch_allocate(theirs, sr, batch)
            if not rr["ok"] and first_err is None:
                first_err = rr["error"]
            for r in rids:
                tb = kvr.table(r)
                live[r] = tb["token_count"]
        res = kvm.device_sync(mine, sm)
        if first_err is None:
            assert res.ok(), res
            applied, replayed = res.value()
            applied_total += applied
            replayed_total += replayed
        else:
            assert not res.ok() and res.error().value == first_err
        _same_engine(kvm, kvr, mine, theirs, live)
        assert mine.validate().ok()
    assert applied_total > 0
    mine.close()


def test_device_batches_in_a_cuda_graph(tg, ref):
    """A decode loop captured once (tokens += 1 per step on the device, then
    the batch) and replayed: the sync'ed engine equals the reference fed the
    same 4 x replays batches."""
    import torch
    rnd = random.Random(7)
    pool_size = 800_000
    mine = tg.ReuseStore(tg.GpuSpec(pool_size=pool_size), device=0)
    theirs = ref.ReuseStore(pool_size)
    sm, sr = tg.ModelStatsTable(), ref.ModelStatsTable()
    _fragment(rnd, mine, theirs, 60)
    kvm, kvr = tg.KvEngine("s", BS, BPT), ref.KvEngine("s", BS, BPT)
    reqs = [(i + 1, rnd.randint(1, 60)) for i in range(24)]
    assert kvm.batch_allocate(mine, sm, reqs).ok() and kvr.batch_allocate(theirs, sr, reqs)["ok"]
    live = dict(reqs)
    rids = [r for r, _ in reqs]
    assert kvm.device_arm(mine, 256, 32, 64).ok()
    slots = _dev([kvm.request_slot(r) for r in rids])
    toks = _dev([live[r] for r in rids])
    inc = _dev([rnd.randint(1, 3) for _ in rids])
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            for _ in range(4):
                toks.add_(inc)
                kvm.batch_allocate_device(slots.data_ptr(), toks.data_ptr(), len(rids),
                                          stream=torch.cuda.current_stream().cuda_stream)
    incs = inc.tolist()
    replays = 5
    for _ in range(replays):
        g.replay()
    for _ in range(replays * 4):
        for i, r in enumerate(rids):
            live[r] += incs[i]
        assert kvr.batch_allocate(theirs, sr, [(r, live[r]) for r in rids])["ok"]
    torch.cuda.synchronize()
    applied, replayed = kvm.device_sync(mine, sm).value()
    assert applied == replays * 4 and replayed == 0
    _same_engine(kvm, kvr, mine, theirs, live)
    mine.close()


def test_armed_engine_freezes_the_pool(tg):
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=100_000), device=0)
    st = tg.ModelStatsTable()
    kv = tg.KvEngine("s", BS, BPT)
    assert kv.batch_allocate(pool, st, [(1, 20)]).ok()
    assert kv.device_arm(pool, 16, 8, 4).ok()
    from paper_2512_01357_b200 import _native as N
    with pytest.raises(N.TangramRuntimeError):
        pool.alloc_kv_region(800, 5)
    with pytest.raises(N.TangramRuntimeError):
        kv.batch_allocate(pool, st, [(2, 8)])
    other = tg.KvEngine("t", BS, BPT)
    with pytest.raises(N.TangramRuntimeError):
        other.batch_allocate(pool, st, [(9, 8)])
    # unknown slot: the batch is left to the host, which cannot map it
    bad = _dev([99])
    t = _dev([8])
    kv.batch_allocate_device(bad.data_ptr(), t.data_ptr(), 1)
    r = kv.device_sync(pool, st)
    assert not r.ok() and r.error().name == "InvalidArgument"
    assert pool.alloc_kv_region(800, 5).ok()  # disarmed
    # log overflow is reported
    assert kv.device_arm(pool, 16, 8, 2).ok()
    s1 = _dev([kv.request_slot(1)])
    for k in range(3):
        tk = _dev([24 + 8 * k])
        kv.batch_allocate_device(s1.data_ptr(), tk.data_ptr(), 1)
        torch_sync()
    with pytest.raises(N.TangramRuntimeError):
        kv.device_sync(pool, st)
    pool.close()


def torch_sync():
    import torch
    torch.cuda.synchronize()


def test_destroying_an_armed_engine_releases_the_pool(tg):
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=50_000), device=0)
    st = tg.ModelStatsTable()
    kv = tg.KvEngine("s", BS, BPT)
    assert kv.batch_allocate(pool, st, [(1, 20)]).ok()
    assert kv.device_arm(pool, 16, 8, 4).ok()
    from paper_2512_01357_b200 import _native as N
    with pytest.raises(N.TangramRuntimeError):
        pool.alloc_kv_region(800, 5)
    del kv
    import gc
    gc.collect()
    assert pool.alloc_kv_region(800, 5).ok()
    pool.close()


@pytest.mark.parametrize("token_bytes", [48, 64])
def test_block_tables_drive_a_paged_cache(tg, cpu, token_bytes):
    """The allocator's block tables, consumed the way a paged-attention cache
    write / gather does (tg_kv_write_tokens / tg_kv_read_tokens): every token
    of every live request gets its own bytes, nothing overlaps — not other
    requests' tokens, not the resident model's tensors — across host-decided
    batches, device-decided decode steps, releases and free-list reuse."""
    import numpy as np
    import torch
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    rnd = random.Random(token_bytes)
    model = tg.make_model("paged", 3_000_011, 2, token_bytes)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=3_000_011 + 600_000), device=0)
    st = tg.ModelStatsTable()
    st.record_request(model.model_id, 0.0)
    with HostCheckpoint([model]):
        digests = pool.load_model(model, st, 0.0).value().digests
    kv = tg.KvEngine(model.model_id, 8, token_bytes)
    live = {}

    def write(rids_tokens):
        slots, pos, pat = [], [], []
        for rid, (lo, hi) in rids_tokens.items():
            for p in range(lo, hi):
                slots.append(kv.request_slot(rid))
                pos.append(p)
                pat.append(np.full(token_bytes, (rid * 131 + p * 7) % 251, dtype=np.uint8))
                pat[-1][:8] = np.frombuffer(np.int64(rid * 100000 + p).tobytes(), dtype=np.uint8)
        if not slots:
            return
        s_d, p_d = _dev(slots), _dev(pos)
        buf = torch.from_numpy(np.concatenate(pat)).cuda()
        kv.write_tokens(pool, s_d.data_ptr(), p_d.data_ptr(), buf.data_ptr(), len(slots))
        torch.cuda.synchronize()

    def check():
        slots, pos, want = [], [], []
        for rid, n in live.items():
            for p in range(n):
                slots.append(kv.request_slot(rid))
                pos.append(p)
                w = np.full(token_bytes, (rid * 131 + p * 7) % 251, dtype=np.uint8)
                w[:8] = np.frombuffer(np.int64(rid * 100000 + p).tobytes(), dtype=np.uint8)
                want.append(w)
        out = torch.empty(len(slots) * token_bytes, dtype=torch.uint8, device="cuda:0")
        s_d, p_d = _dev(slots), _dev(pos)
        kv.read_tokens(pool, s_d.data_ptr(), p_d.data_ptr(), out.data_ptr(), len(slots))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), np.concatenate(want))
        for i, t in enumerate(model.tensors):  # KV blocks never overlap the resident tensors
            assert pool.fingerprint_tensor(t.id) == digests[i]

    nxt = 1
    for rnd_i in range(4):
        reqs = [(nxt + i, rnd.randint(1, 60)) for i in range(12)]
        nxt += len(reqs)
        assert kv.batch_allocate(pool, st, reqs, want_pbns=False).ok()
        write({r: (0, n) for r, n in reqs})
        live.update(dict(reqs))
        # device-decided decode steps
        assert kv.device_arm(pool, 64, 64, 8).ok()
        grown = {}
        for step in range(3):
            batch = [(r, live[r] + rnd.randint(1, 9)) for r in live]
            s_d, t_d = _dev([kv.request_slot(r) for r, _ in batch]), _dev([t for _, t in batch])
            kv.batch_allocate_device(s_d.data_ptr(), t_d.data_ptr(), len(batch))
            torch.cuda.synchronize()  # the inputs must live until the batch ran
            for r, t in batch:
                grown[r] = (grown.get(r, (live[r], live[r]))[0], t)
                live[r] = t
        assert kv.device_sync(pool, st).ok()
        write(grown)
        check()
        for r in [r for r in list(live) if rnd.random() < 0.4]:
            assert kv.release_request(r).ok()
            live.pop(r)
        check()
    pool.close()


def test_token_consumer_rejects_references_outside_the_tables(tg):
    """an unset LBN (PBN 0), an unknown slot or a position past the
    table moves nothing (it would otherwise land at arena offset 0, inside a
    resident tensor) and is counted as a fault."""
    import numpy as np
    import torch
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    model = tg.make_model("faults", 2_000_003, 2, 64)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=4_000_000), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([model]):
        digests = pool.load_model(model, st, 0.0).value().digests
    kv = tg.KvEngine(model.model_id, 8, 64)
    assert kv.batch_allocate(pool, st, [(1, 20), (2, 5)]).ok()  # slot 0: 3 blocks, slot 1: 1 block
    s0, s1 = kv.request_slot(1), kv.request_slot(2)
    slots = [s0, s1, s1, 77, s0]
    pos = [3, 2, 9, 0, 10_000]  # ok, ok, LBN 1 of slot 1 never granted, unknown slot, past the table
    buf = torch.full((len(slots) * 64,), 0xEE, dtype=torch.uint8, device="cuda:0")
    s_d, p_d = _dev(slots), _dev(pos)  # kept alive until the kernels ran
    kv.write_tokens(pool, s_d.data_ptr(), p_d.data_ptr(), buf.data_ptr(), len(slots))
    assert kv.token_faults() == 3
    for i, t in enumerate(model.tensors):
        assert pool.fingerprint_tensor(t.id) == digests[i]
    out = torch.zeros(2 * 64, dtype=torch.uint8, device="cuda:0")
    s2, p2 = _dev(slots[:2]), _dev(pos[:2])
    kv.read_tokens(pool, s2.data_ptr(), p2.data_ptr(), out.data_ptr(), 2)
    assert kv.token_faults() == 3 and np.all(out.cpu().numpy() == 0xEE)
    pool.close()


def test_reserved_tables_never_move_and_consumers_on_other_streams(tg):
    """tg_kv_reserve pins the device tables' addresses; a consumer on another
    stream is ordered after the table updates of the batches before it."""
    import numpy as np
    import torch
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=64 << 20), device=0)
    st = tg.ModelStatsTable()
    kv = tg.KvEngine("r", 16, 128)
    kv.reserve(pool, 64, 64, 4096)
    ptrs = kv.device_tables()
    side = torch.cuda.Stream()
    rid = 1
    for step in range(10):
        reqs = [(rid + i, 16 * (step + 1)) for i in range(6)]
        rid += 6
        assert kv.batch_allocate(pool, st, reqs, want_pbns=False).ok()
        # no host sync between the table update and the consumer on `side`
        slots = [kv.request_slot(r) for r, n in reqs for p in range(n)]
        pos = [p for r, n in reqs for p in range(n)]
        src = torch.arange(len(slots) * 128, device="cuda:0").to(torch.uint8)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            s_d, p_d = _dev(slots), _dev(pos)
            kv.write_tokens(pool, s_d.data_ptr(), p_d.data_ptr(), src.data_ptr(), len(slots),
                            stream=side.cuda_stream)
            back = torch.empty_like(src)
            kv.read_tokens(pool, s_d.data_ptr(), p_d.data_ptr(), back.data_ptr(), len(slots),
                           stream=side.cuda_stream)
        side.synchronize()
        assert torch.equal(back, src)
        assert kv.device_tables() == ptrs
    assert kv.token_faults() == 0
    pool.close()


def test_device_sync_rejects_another_pool(tg):
    """the device-decided carves are folded only into the pool the
    engine was armed on."""
    import torch
    from paper_2512_01357_b200 import _native as N
    a = tg.ReuseStore(tg.GpuSpec("a", 32 << 20), device=0)
    b = tg.ReuseStore(tg.GpuSpec("b", 32 << 20), device=0)
    st = tg.ModelStatsTable()
    kv = tg.KvEngine("x", 16, 256)
    assert kv.batch_allocate(a, st, [(1, 16)]).ok()
    assert kv.device_arm(a, 64, 8, 4).ok()
    s_d, t_d = _dev([kv.request_slot(1)]), _dev([200])
    kv.batch_allocate_device(s_d.data_ptr(), t_d.data_ptr(), 1)
    torch.cuda.synchronize()
    dump_b = b.dump()
    with pytest.raises(N.TangramRuntimeError) as ei:
        kv.device_sync(b, st)
    assert ei.value.code == 104 and b.dump() == dump_b
    assert kv.device_sync(a, st).ok()
    assert a.validate().ok() and b.validate().ok()
    a.close()
    b.close()
