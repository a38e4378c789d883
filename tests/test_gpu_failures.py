"""Failure atomicity of the device load path (reuse_store.hpp:117-119 for the
reference's own failure rule).

Faults are injected where the data plane can really fail once bytes move: a
checkpoint file that reads short mid-load, a CUDA copy error, a stale peer
index with nothing to repair it, and a source whose bytes miss their manifest
digest.  After each:

* ``tg_load_model`` returns a runtime code (>= 100);
* the pool holds the reference's decision for that load (dump equal to the
  compiled reference run on the same sequence), and every tensor whose bytes
  the load could not verify is *suspect*: not exported to peers, not a byte
  source;
* the next reload of the model re-sends exactly those tensors
  (``repaired_bytes``), after which every resident tensor's device bytes
  fingerprint equal to the CPU restatement and nothing is suspect.

Failures found before the commit (no source, a missing or short file) leave
the pool unchanged.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cpu_digest(cpu, tid, size):
    return cpu.content_fingerprint(cpu.synth(tid.hi, tid.lo, size), threads=16)[0]


def _check_bytes(tg, cpu, pool, models, others=()):
    """Resident tensors of `models` are verified and byte-exact.  Tensors of
    `others` (relocated by a failed load, not reused since) are either
    byte-exact or still suspect — and then not exported."""
    exported = {e[0] for e in pool.index()}
    for m in list(models) + list(others):
        for t in m.tensors:
            info = pool.tensor_info(t.id)
            if info is None:
                continue
            if m in others and info["suspect"]:
                assert t.id not in exported, t.name
                continue
            assert not info["suspect"], t.name
            assert pool.fingerprint_tensor(t.id) == _cpu_digest(cpu, t.id, t.size), t.name


def _ref_dump(ref, ops, pool_size, gpu_id="gpu0"):
    """Dump of the compiled reference after (kind, model, clock) ops."""
    r = ref.ReuseStore(pool_size, gpu_id=gpu_id)
    st = ref.ModelStatsTable()
    for kind, m, t in ops:
        if kind == "load":
            st.record_request(m.model_id, t)
            r.load_model(m.to_json(), st, t)
        else:
            r.end_instance(m.model_id)
    return r.dump()


def _write_ckpt(cpu, path, models):
    offs = {}
    with open(path, "wb") as f:
        f.write(b"TG" * 7)  # unaligned tensor offsets in the file
        for m in models:
            for t in m.tensors:
                offs[t.id] = f.tell()
                f.write(cpu.synth(t.id.hi, t.id.lo, t.size).tobytes())
    return offs


def _register_file(tg, path, offs, models):
    from paper_2512_01357_b200 import _native as N
    for m in models:
        for t in m.tensors:
            assert N.lib.tg_file_register(t.id.c(), str(path).encode(), offs[t.id], t.size, None) == 0


def _unregister(models):
    from paper_2512_01357_b200 import _native as N
    for m in models:
        for t in m.tensors:
            N.lib.tg_host_unregister(t.id.c())


def test_missing_or_short_file_leaves_pool_unchanged(tg, cpu, tmp_path):
    """A checkpoint file that is missing or too short when the load is
    planned is a no-source failure: code 102 and the pool untouched."""
    from paper_2512_01357_b200 import _native as N
    a = tg.make_model("fa", 30_000_019, 2, 0)
    b = tg.make_model("fb", 20_000_011, 2, 0)
    path = tmp_path / "ck.bin"
    offs = _write_ckpt(cpu, path, [a, b])
    _register_file(tg, path, offs, [a, b])
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=64 << 20), device=0)
    st = tg.ModelStatsTable()
    try:
        pool.load_model(a, st, 0.0).value()
        pool.end_instance("fa")
        before = pool.dump()
        os.truncate(path, offs[b.tensors[-1].id] + 5)  # the file lost its tail
        with pytest.raises(N.TangramRuntimeError) as ei:
            pool.load_model(b, st, 1.0)
        assert ei.value.code == 102 and ei.value.outcome is None
        assert pool.dump() == before
        os.remove(path)
        with pytest.raises(N.TangramRuntimeError) as ei:
            pool.load_model(b, st, 1.0)
        assert ei.value.code == 102 and pool.dump() == before
        _check_bytes(tg, cpu, pool, [a])
    finally:
        _unregister([a, b])
        pool.close()


@pytest.mark.parametrize("nth", [1, 3])
def test_short_read_mid_load_is_repaired_on_reload(tg, cpu, ref, tmp_path, nth):
    """A chunk of the checkpoint file reads short while the load runs (the
    file shrank under it): the load fails after its commit, its tensors are
    suspect, and the reload re-sends them."""
    from paper_2512_01357_b200 import _native as N
    a = tg.make_model("sa", 70_000_023, 3, 0)
    b = tg.make_model("sb", 50_000_017, 3, 0)
    path = tmp_path / "ck.bin"
    offs = _write_ckpt(cpu, path, [a, b])
    _register_file(tg, path, offs, [a, b])
    size = 100_000_000  # b evicts part of a
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=size), device=0)
    st = tg.ModelStatsTable()
    try:
        st.record_request("sa", 0.0)
        pool.load_model(a, st, 0.0).value()
        pool.end_instance("sa")
        st.record_request("sb", 1.0)
        tg.failpoint("file_read", nth)
        with pytest.raises(N.TangramRuntimeError) as ei:
            pool.load_model(b, st, 1.0)
        tg.failpoint("file_read", 0)
        err = ei.value
        assert err.code >= 100 and err.outcome is not None
        assert err.outcome.suspect_tensors > 0
        ops = [("load", a, 0.0), ("end", a, 0), ("load", b, 1.0)]
        assert pool.dump() == _ref_dump(ref, ops, size)  # the reference's decision stands
        suspect = [t for t in b.tensors if pool.tensor_info(t.id)["suspect"]]
        assert len(suspect) == err.outcome.suspect_tensors
        exported = {e[0] for e in pool.index()}
        assert not exported & {t.id for t in suspect}
        # reload: the suspect tensors (no digest was ever recorded) are re-sent
        pool.end_instance("sb")
        st.record_request("sb", 2.0)
        o = pool.load_model(b, st, 2.0).value()
        assert o.bytes_transferred == 0 and o.suspect_tensors == 0
        assert o.repaired_bytes == sum(t.size for t in suspect)
        ops += [("end", b, 0), ("load", b, 2.0)]
        assert pool.dump() == _ref_dump(ref, ops, size)
        _check_bytes(tg, cpu, pool, [b], others=[a])
        assert {e[0] for e in pool.index()} >= {t.id for t in b.tensors}
    finally:
        tg.failpoint("file_read", 0)
        _unregister([a, b])
        pool.close()


def test_copy_error_mid_load(tg, cpu, ref):
    """A host->device copy fails in the middle of a switch that also relocates
    resident tensors: every tensor the load wrote is suspect afterwards; the
    next loads verify and repair them."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    cat = {m.model_id: m for m in tg.default_catalog()}
    x, y = cat["qwen3B"], cat["opt1.3B"]
    size = 7 << 30
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=size), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([x, y]):
        try:
            st.record_request(x.model_id, 0.0)
            pool.load_model(x, st, 0.0).value()
            pool.end_instance(x.model_id)
            st.record_request(y.model_id, 10.0)
            pool.load_model(y, st, 10.0).value()
            pool.end_instance(y.model_id)
            st.record_request(x.model_id, 20.0)
            tg.failpoint("h2d", 2)
            with pytest.raises(N.TangramRuntimeError) as ei:
                pool.load_model(x, st, 20.0)
            err = ei.value
            assert err.code == 100 and err.outcome.suspect_tensors > 0
            assert err.outcome.plan.relocations and err.outcome.plan.placements
            ops = [("load", x, 0.0), ("end", x, 0), ("load", y, 10.0), ("end", y, 0), ("load", x, 20.0)]
            assert pool.dump() == _ref_dump(ref, ops, size)
            moved = {r.tensor for r in err.outcome.plan.relocations}
            placed = {p.tensor for p in err.outcome.plan.placements}
            for tid in moved | placed:
                assert pool.tensor_info(tid)["suspect"]
            pool.end_instance(x.model_id)
            st.record_request(x.model_id, 30.0)
            o = pool.load_model(x, st, 30.0).value()
            assert o.suspect_tensors == 0 and o.bytes_transferred == 0
            # placements never got a digest: always re-sent; relocated ones only if their bytes differ
            assert o.repaired_bytes >= sum(p.size for p in err.outcome.plan.placements)
            _check_bytes(tg, cpu, pool, [x], others=[y])
        finally:
            tg.failpoint("h2d", 0)
            pool.close()


def test_stale_peer_without_source(tg, cpu, ref):
    """Peer bytes that fail their digest with no host source: the load fails
    with TG_ERR_VERIFY, the victim is suspect and keeps the peer's digest as
    its truth (never its own bad bytes'), and is not exported; once a source
    exists the reload repairs it."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("stale", 60_000_013, 3, 0)
    a = tg.ReuseStore(tg.GpuSpec("gpu0", 80_000_000), device=0)
    b = tg.ReuseStore(tg.GpuSpec("gpu1", 80_000_000), device=0)
    b.add_peer(a)
    sa, sb = tg.ModelStatsTable(), tg.ModelStatsTable()
    ck = HostCheckpoint([m])
    try:
        oa = a.load_model(m, sa, 0.0).value()
        victim = m.tensors[2]
        info = a.tensor_info(victim.id)
        junk = np.full(8192, 0x5A, dtype=np.uint8)
        N.lib.tg_memcpy(C.c_void_p(info["device_ptr"] + 12345), junk.ctypes.data_as(C.c_void_p), junk.size)
        _unregister([m])  # no host source anywhere
        sb.record_request(m.model_id, 0.0)
        with pytest.raises(N.TangramRuntimeError) as ei:
            b.load_model(m, sb, 0.0, tg.LoadPolicy(flags=1 | 2 | 4 | 8))
        err = ei.value
        assert err.code == 105 and err.outcome.peer_bytes == m.total_size
        assert err.outcome.verify_mismatches == 1 and err.outcome.suspect_tensors == 1
        assert b.dump() == _ref_dump(ref, [("load", m, 0.0)], 80_000_000, "gpu1")
        vi = b.tensor_info(victim.id)
        assert vi["suspect"] and vi["has_digest"] and vi["digest"] == oa.digests[2]
        assert victim.id not in {e[0] for e in b.index()}
        for i, t in enumerate(m.tensors):
            if t.id != victim.id:
                assert not b.tensor_info(t.id)["suspect"] and b.tensor_info(t.id)["digest"] == oa.digests[i]
        # without a source the reload cannot repair it either (and says so)
        b.end_instance(m.model_id)
        sb.record_request(m.model_id, 1.0)
        with pytest.raises(N.TangramRuntimeError) as ei:
            b.load_model(m, sb, 1.0)
        assert ei.value.code == 105 and b.tensor_info(victim.id)["suspect"]
        ck.register()
        b.end_instance(m.model_id)
        sb.record_request(m.model_id, 2.0)
        o = b.load_model(m, sb, 2.0).value()
        assert o.repaired_bytes == victim.size and o.suspect_tensors == 0
        assert b.fingerprint_tensor(victim.id) == _cpu_digest(cpu, victim.id, victim.size) == oa.digests[2]
        ops = [("load", m, 0.0), ("end", m, 0), ("load", m, 1.0), ("end", m, 0), ("load", m, 2.0)]
        assert b.dump() == _ref_dump(ref, ops, 80_000_000, "gpu1")
    finally:
        ck.close()
        a.close()
        b.close()


def test_expected_digest_mismatch_is_a_hard_error(tg, cpu, ref):
    """A source whose bytes miss their manifest digest fails the load
    (TG_ERR_VERIFY); the corrupt tensor is suspect with no recorded truth and
    is re-sent, from the corrected source, on the reload."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("manifest", 45_000_007, 3, 0)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=64 << 20), device=0)
    st = tg.ModelStatsTable()
    ck = HostCheckpoint([m], register=False)
    try:
        want = {t.id: _cpu_digest(cpu, t.id, t.size) for t in m.tensors}
        for t in m.tensors:
            d = N.DigestC(*want[t.id])
            assert N.lib.tg_host_register(t.id.c(), C.c_void_p(ck.entries[t.id][0]), t.size, C.byref(d)) == 0
        victim = m.tensors[1]
        view = ck.view(victim.id)
        good = view.copy()
        view[777:777 + 64] ^= 0xFF  # the checkpoint is corrupt
        st.record_request(m.model_id, 0.0)
        with pytest.raises(N.TangramRuntimeError) as ei:
            pool.load_model(m, st, 0.0)
        err = ei.value
        assert err.code == 105 and err.outcome.expected_mismatches == 1 and err.outcome.suspect_tensors == 1
        vi = pool.tensor_info(victim.id)
        assert vi["suspect"] and not vi["has_digest"]
        assert pool.dump() == _ref_dump(ref, [("load", m, 0.0)], 64 << 20)
        view[:] = good  # the checkpoint is fixed
        pool.end_instance(m.model_id)
        st.record_request(m.model_id, 1.0)
        o = pool.load_model(m, st, 1.0).value()
        assert o.repaired_bytes == victim.size and o.suspect_tensors == 0 and o.expected_mismatches == 0
        _check_bytes(tg, cpu, pool, [m])
        assert pool.tensor_info(victim.id)["digest"] == want[victim.id]
    finally:
        _unregister([m])
        ck.close()
        pool.close()


def test_suspect_is_verified_even_without_verify_flag(tg, cpu):
    """Suspect tensors are verified on reuse whatever the flags say, and a
    load with TG_LOAD_EXPLICIT and no other flag does no optional work."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    m = tg.make_model("noflag", 30_000_001, 2, 0)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=40 << 20), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([m]):
        try:
            tg.failpoint("h2d", 1)
            with pytest.raises(N.TangramRuntimeError):
                pool.load_model(m, st, 0.0)
            tg.failpoint("h2d", 0)
            pool.end_instance(m.model_id)
            none = tg.LoadPolicy(flags=tg.pool.LOAD_EXPLICIT)
            o = pool.load_model(m, st, 1.0, none).value()
            assert o.repaired_bytes == m.total_size and o.suspect_tensors == 0
            pool.end_instance(m.model_id)
            o = pool.load_model(m, st, 2.0, none).value()
            assert o.fingerprint_bytes == 0 and o.repaired_bytes == 0 and o.timings["total_ms"] >= 0
            _check_bytes(tg, cpu, pool, [m])
        finally:
            tg.failpoint("h2d", 0)
            pool.close()
