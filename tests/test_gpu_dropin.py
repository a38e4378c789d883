"""C5 trace replay with real bytes: the unmodified
reference Simulator over the B200 bindings, pool gpu0 on CUDA device 0 with
every catalog tensor's bytes synthesised in HBM, the other seven pools
control-plane-only (one GPU in this run).  RunMetrics must stay byte-identical
to the pure-reference build while gpu0 really moves and fingerprints bytes."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")


@pytest.mark.parametrize("mode,async_loads", [("reuse_odkv", "0"), ("reuse_odkv", "1"), ("reuse", "1"),
                                              ("baseline", "0")])
def test_c5_replay_moves_bytes_and_matches_reference(mode, async_loads):
    """reuse_odkv is C5 (on-demand KV through KvEngine); reuse and baseline
    take the simulator's reserve_kv pre-reservation path (simulator.hpp:606-637:
    eviction_candidates, evict_tensor, alloc_kv_region, free runs) against the
    device pool."""
    ref_bin, tg_bin = os.path.join(BUILD, "sim_reference"), os.path.join(BUILD, "sim_tangram")
    if not (os.path.exists(ref_bin) and os.path.exists(tg_bin)):
        pytest.skip("drop-in binaries not built (make -C integration)")
    args = [mode, "8", "48", "4", "2", "2000", "42", "0", "0", "L3"]
    a = subprocess.run([ref_bin] + args, capture_output=True, check=True, timeout=600)
    env = dict(os.environ, TANGRAM_DEVICE="auto", TANGRAM_SYNTH_SOURCES="1", TANGRAM_ASYNC_LOADS=async_loads)
    b = subprocess.run([tg_bin] + args, capture_output=True, check=True, timeout=600, env=env)
    assert a.stdout == b.stdout
    pools = json.loads(b.stderr.decode().strip().splitlines()[-1])["pools"]
    g0 = [p for p in pools if p["gpu_id"] == "gpu0"][0]
    assert g0["device"] == 0 and g0["loads"] > 0
    assert g0["device_src_bytes"] > 0 and g0["fingerprint_bytes"] > 0
    assert g0["verify_mismatches"] == 0 and g0["failed_loads"] == 0
    print(json.dumps(g0))


SMALL = ["opt1.3B", "qwen3B", "llama3B", "opt6.7B", "llama8B", "yi9B"]


def _small_replay(extra_env, args):
    tg_bin = os.path.join(BUILD, "sim_tangram")
    env = dict(os.environ, TANGRAM_DEVICE="0", TANGRAM_SYNTH_SOURCES="host", **extra_env)
    b = subprocess.run([tg_bin] + args, capture_output=True, check=True, timeout=900, env=env)
    rep = json.loads(b.stderr.decode().strip().splitlines()[-1])
    return b.stdout, rep


def test_c5_small_all_pools_real_async_and_peer_schedule():
    """A C5-shaped replay whose every pool holds real bytes on this one GPU
    (4 pools x 24 GiB, the six smallest catalog models — 62 GB, so models
    migrate between pools — sources in pinned host memory): synchronous and asynchronous loads give the reference's
    RunMetrics byte for byte; with the peer-aware schedule
    (TANGRAM_PEER_SCHEDULE) misses resident on another pool come from it
    instead of over PCIe — PCIe bytes saved, nothing fails verification."""
    ref_bin, tg_bin = os.path.join(BUILD, "sim_reference"), os.path.join(BUILD, "sim_tangram")
    if not (os.path.exists(ref_bin) and os.path.exists(tg_bin)):
        pytest.skip("drop-in binaries not built (make -C integration)")
    args = ["reuse_odkv", "4", "24", "4", "2", "400", "42", "0", "0", "L3", ",".join(SMALL)]
    a = subprocess.run([ref_bin] + args, capture_output=True, check=True, timeout=600)
    out_sync, r_sync = _small_replay({"TANGRAM_ASYNC_LOADS": "0"}, args)
    out_async, r_async = _small_replay({"TANGRAM_ASYNC_LOADS": "1"}, args)
    assert out_sync == a.stdout and out_async == a.stdout
    out_peer, r_peer = _small_replay({"TANGRAM_ASYNC_LOADS": "1", "TANGRAM_PEER_SCHEDULE": "700"}, args)
    for r in (r_sync, r_async, r_peer):
        assert all(p["device"] == 0 for p in r["pools"]) and len(r["pools"]) == 4
        assert sum(p["verify_mismatches"] + p["failed_loads"] for p in r["pools"]) == 0
    pcie = {k: sum(p["pcie_bytes"] for p in r["pools"]) for k, r in (("sync", r_sync), ("peer", r_peer))}
    peer = sum(p["peer_bytes"] for p in r_peer["pools"])
    assert sum(p["peer_bytes"] for p in r_sync["pools"]) == 0
    assert peer > 0  # misses pulled from another pool
    assert pcie["peer"] < pcie["sync"]  # ... instead of over PCIe
    print(json.dumps({"replay_s": {"sync": r_sync["replay_s"], "async": r_async["replay_s"],
                                   "peer": r_peer["replay_s"]}, "pcie_bytes": pcie, "peer_bytes": peer}))


def test_store_copy_semantics_on_a_device_pool():
    """The drop-in store's value semantics with real bytes: stdout (every
    dump) equals the reference's; the copies were control-plane clones, so the
    layout adopted back into the device pool is re-sent where the arena does
    not hold it, and the final loads leave nothing suspect."""
    ref_bin, tg_bin = os.path.join(BUILD, "copy_reference"), os.path.join(BUILD, "copy_tangram")
    if not (os.path.exists(ref_bin) and os.path.exists(tg_bin)):
        pytest.skip("copy_check binaries not built (make -C integration)")
    a = subprocess.run([ref_bin], capture_output=True, check=True, timeout=300)
    env = dict(os.environ, TANGRAM_DEVICE="0", TANGRAM_SYNTH_SOURCES="1")
    b = subprocess.run([tg_bin], capture_output=True, check=True, timeout=300, env=env)
    assert a.stdout == b.stdout
    rep = json.loads(b.stderr.decode().strip().splitlines()[-1])
    assert rep["suspect"] == [0, 0] and sum(rep["repaired"]) > 0 and min(rep["fingerprinted"]) > 0
    assert rep["second_placed"] > 0  # the surviving copy kept the device pool (bytes really placed)
    print(rep)


def test_clone_and_assign_keep_bytes_honest(tg, cpu):
    """tg_pool_clone / tg_pool_assign through the Python mirror: a clone's
    loads move no bytes and leave the device pool alone; assigning it back
    marks exactly the tensors the arena does not hold at their adopted
    offsets suspect; the next reloads re-send them and every resident tensor
    then fingerprints equal to the CPU restatement."""
    from paper_2512_01357_b200.checkpoint import HostCheckpoint
    a = tg.make_model("ca", 40_000_003, 3, 0)
    b = tg.make_model("cb", 30_000_001, 3, 0)
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=60_000_000), device=0)
    st = tg.ModelStatsTable()
    with HostCheckpoint([a, b]):
        st.record_request("ca", 0.0)
        pool.load_model(a, st, 0.0).value()
        pool.end_instance("ca")
        before = pool.dump()
        c = pool.clone()
        assert c.dump() == before and c.device is None
        st.record_request("cb", 1.0)
        oc = c.load_model(b, st, 1.0).value()
        assert oc.bytes_transferred == b.total_size and oc.pcie_bytes == 0  # control plane only
        assert pool.dump() == before
        layout = pool.tensor_map()
        pool.assign(c)
        assert pool.dump() == c.dump()
        tm = pool.tensor_map()
        for tid, e in tm.items():
            held = tid in layout and layout[tid]["offset"] == e["offset"] and not layout[tid]["suspect"]
            assert e["suspect"] == (not held), tid
        pool.end_instance("cb")
        st.record_request("cb", 2.0)
        o = pool.load_model(b, st, 2.0).value()
        assert o.bytes_transferred == 0 and o.repaired_bytes == b.total_size and o.suspect_tensors == 0
        for m in (a, b):
            for t in m.tensors:
                if t.id in tm and not pool.tensor_info(t.id)["suspect"]:
                    want = cpu.content_fingerprint(cpu.synth(t.id.hi, t.id.lo, t.size), threads=8)[0]
                    assert pool.fingerprint_tensor(t.id) == want
        c.close()
    pool.close()
