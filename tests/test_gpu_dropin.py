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


@pytest.mark.parametrize("mode", ["reuse_odkv", "reuse", "baseline"])
def test_c5_replay_moves_bytes_and_matches_reference(mode):
    """reuse_odkv is C5 (on-demand KV through KvEngine); reuse and baseline
    take the simulator's reserve_kv pre-reservation path (simulator.hpp:606-637:
    eviction_candidates, evict_tensor, alloc_kv_region, free runs) against the
    device pool."""
    ref_bin, tg_bin = os.path.join(BUILD, "sim_reference"), os.path.join(BUILD, "sim_tangram")
    if not (os.path.exists(ref_bin) and os.path.exists(tg_bin)):
        pytest.skip("drop-in binaries not built (make -C integration)")
    args = [mode, "8", "48", "4", "2", "2000", "42", "0", "0", "L3"]
    a = subprocess.run([ref_bin] + args, capture_output=True, check=True, timeout=600)
    env = dict(os.environ, TANGRAM_DEVICE="auto", TANGRAM_SYNTH_SOURCES="1")
    b = subprocess.run([tg_bin] + args, capture_output=True, check=True, timeout=600, env=env)
    assert a.stdout == b.stdout
    pools = json.loads(b.stderr.decode().strip().splitlines()[-1])["pools"]
    g0 = [p for p in pools if p["gpu_id"] == "gpu0"][0]
    assert g0["device"] == 0 and g0["loads"] > 0
    assert g0["device_src_bytes"] > 0 and g0["fingerprint_bytes"] > 0
    print(json.dumps(g0))
