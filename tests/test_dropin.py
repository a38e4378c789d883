"""Drop-in boundary: the reference's own Simulator (simulator.hpp, unmodified)
compiled against the B200 bindings in integration/warmsim/ produces
byte-identical RunMetrics (per-request records, aggregates, KV counters,
schedule log, allocation log, utilisation series) to the pure-reference build.
Pools are control-plane-only here (TANGRAM_DEVICE=none): the simulator models
8 GPUs in one process; the byte-moving path is covered by the GPU tests."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")

CONFIGS = [
    # mode, n_gpus, pool_gib, batch, keep_alive, n_requests, seed, eviction, merge, locality
    ("reuse_odkv", 8, 48, 4, 2, 2000, 42, 0, 0, "L3"),   # C5
    ("reuse", 8, 48, 4, 2, 2000, 42, 0, 0, "L3"),
    ("baseline", 8, 48, 4, 2, 2000, 42, 0, 0, "L3"),
    ("reuse_odkv", 4, 48, 2, 1, 800, 7, 1, 0, "L1"),     # random eviction (simulator Rng stream)
    ("reuse", 4, 48, 2, 2, 600, 3, 0, 1, "L2"),          # global merge
    ("reuse", 8, 48, 1, 2, 600, 3, 0, 1, "L2"),
    ("baseline", 4, 64, 2, 1, 500, 9, 1, 0, "L1"),
    ("reuse_odkv", 1, 64, 8, 0.5, 600, 11, 0, 0, "L4"),
    ("reuse_odkv", 3, 48, 4, 1, 500, 5, 1, 1, "L3"),
    ("reuse_odkv", 4, 40, 2, 1, 800, 7, 1, 0, "L1"),     # RuntimeInfeasible in both builds
]


@pytest.fixture(scope="module")
def binaries():
    if not os.path.isdir("/root/reference/proj/include/warmsim"):
        if not (os.path.exists(os.path.join(BUILD, "sim_reference")) and
                os.path.exists(os.path.join(BUILD, "sim_tangram"))):
            pytest.skip("reference headers absent and drop-in binaries not prebuilt")
    else:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration")], check=True)
    return os.path.join(BUILD, "sim_reference"), os.path.join(BUILD, "sim_tangram")


@pytest.mark.parametrize("cfg", CONFIGS, ids=[f"{c[0]}-{c[1]}x{c[2]}G-ev{c[7]}-gm{c[8]}-{c[9]}" for c in CONFIGS])
def test_simulator_runmetrics_identical(binaries, cfg):
    ref_bin, tg_bin = binaries
    args = [str(x) for x in cfg]
    env = dict(os.environ, TANGRAM_DEVICE="none")
    a = subprocess.run([ref_bin] + args, capture_output=True, check=True, timeout=300).stdout
    b = subprocess.run([tg_bin] + args, capture_output=True, check=True, timeout=300, env=env).stdout
    assert a.strip()
    assert a == b


@pytest.mark.parametrize("async_loads", ["0", "1"])
def test_peer_term_without_peer_bytes_is_the_reference(binaries, async_loads):
    """integration/warmsim/scheduler.hpp routes schedule / estimate_load_time
    through tg_schedule.  With the peer term switched on
    (TANGRAM_PEER_SCHEDULE) but no device pool holding bytes, S'_peer = 0 for
    every (GPU, model) and the estimate (S - S' - S'_peer)/B + S'_peer/B_nvlink
    reduces to the reference's (S - S')/B (scheduler.hpp:41-48): RunMetrics
    stay byte-identical.  TG_LOAD_ASYNC on control-plane pools is a no-op."""
    ref_bin, tg_bin = binaries
    args = [str(x) for x in ("reuse_odkv", 4, 24, 4, 2, 400, 42, 0, 0, "L3")] + [
        "opt1.3B,qwen3B,llama3B,opt6.7B,llama8B,yi9B"]
    env = dict(os.environ, TANGRAM_DEVICE="none", TANGRAM_PEER_SCHEDULE="700", TANGRAM_ASYNC_LOADS=async_loads)
    a = subprocess.run([ref_bin] + args, capture_output=True, check=True, timeout=300).stdout
    b = subprocess.run([tg_bin] + args, capture_output=True, check=True, timeout=300, env=env).stdout
    assert a.strip() and b"exception" not in a
    assert a == b


def test_store_copies_are_independent_values():
    """reuse_store.hpp:336-344: a copied store is independent of its original
    (the reference copies stores for rollback, kv_engine.hpp:146-158).  The
    same driver (integration/copy_check.cpp: copy, mutate the copy, assign
    back by copy and by move, reload) prints byte-identical dumps against the
    reference and against the bindings."""
    ref_bin = os.path.join(BUILD, "copy_reference")
    tg_bin = os.path.join(BUILD, "copy_tangram")
    if os.path.isdir("/root/reference/proj/include/warmsim"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration")], check=True)
    if not (os.path.exists(ref_bin) and os.path.exists(tg_bin)):
        pytest.skip("copy_check binaries not built")
    a = subprocess.run([ref_bin], capture_output=True, check=True, timeout=120).stdout
    b = subprocess.run([tg_bin], capture_output=True, check=True, timeout=120,
                       env=dict(os.environ, TANGRAM_DEVICE="none")).stdout
    assert a == b
    dumps = {}
    for line in a.decode().splitlines():
        tag, _, rest = line.partition(" ")
        if rest.startswith("{"):
            dumps[tag] = rest
    assert dumps["s0"] == dumps["s_after_c"] == dumps["s_after_r"]  # mutating a copy leaves the original
    assert dumps["c"] != dumps["s0"] and dumps["r"] != dumps["s0"]
    assert dumps["s_eq_c"] == dumps["c"] and dumps["s_eq_r"] == dumps["r"]
    assert b"evict ok=1" in a and b"kv ok=1" in a
    assert dumps["backup"] == dumps["s_final"] != dumps["s_after_backup"]  # a copy taken before a mutation
