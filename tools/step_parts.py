"""Diagnostics: the bench step's load kernel with its parts switched on and
off (policy flags), kernel time per variant (median of 5), same pool state.
    python tools/step_parts.py
"""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    lib = N.lib
    cat = bench.catalog(tg)
    for m in (cat["opt13B"], cat["opt6.7B"]):
        for t in m.tensors:
            b = DeviceBuffer(t.size, 0)
            lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), 0)
            lib.tg_host_register(t.id.c(), C.c_void_p(b.ptr), t.size, None)
            globals().setdefault("_keep", []).append(b)
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", bench.POOL), device=0)
    for i, mid in enumerate(bench.SEQ[:2]):
        pool.load_model(cat[mid], bench.fresh_stats(tg, i + 1), 10.0 * i).value()
        pool.end_instance(mid)
    snap = pool.snapshot()
    target = cat[bench.SEQ[2]]
    out = {}
    for name, flags in (("full", 1 | 2 | 8), ("no_reuse_verify", 2 | 8), ("no_fingerprints", 8)):
        ks = []
        for _ in range(6):
            pool.restore(snap)
            torch.cuda.synchronize()
            o = pool.load_model(target, bench.fresh_stats(tg, 3), 20.0, tg.LoadPolicy(flags=flags), details=False).value()
            ks.append(o.timings["relocate_ms"])
        out[name] = {"kernel_ms": statistics.median(ks[1:]), "fingerprint_bytes": o.fingerprint_bytes}
    # the same moves through the load kernel alone: each WAR wave, then the
    # HBM-cache placements (copy + fingerprint, tg_copy_fingerprint)
    pool.restore(snap)
    o = pool.load_model(target, bench.fresh_stats(tg, 3), 20.0, tg.LoadPolicy(flags=1 | 2 | 8)).value()
    plan = o.plan
    pool.restore(snap)
    arena = pool.info()["arena"]
    waves = {}
    for r in plan.relocations:
        waves.setdefault(r.wave, []).append((arena + r.from_, arena + r.to, r.size))
    src_of = {t.id: b for t, b in zip([t for m in (cat["opt13B"], cat["opt6.7B"]) for t in m.tensors], _keep)}
    groups = {f"wave{w}": mv for w, mv in sorted(waves.items())}
    groups["placements"] = [(src_of[p.tensor].ptr, arena + p.offset, p.size) for p in plan.placements]
    for name, mv in groups.items():
        arr = (C.c_uint64 * (3 * len(mv)))(*[x for m in mv for x in m])
        dg = (N.DigestC * len(mv))()
        ms = C.c_double()
        N.check_runtime(lib.tg_copy_fingerprint(arr, len(mv), 0, 5, C.byref(ms), dg), name)
        nbytes = sum(m[2] for m in mv)
        out[name] = {"moves": len(mv), "ms": ms.value, "GBps_rw": 2 * nbytes / ms.value / 1e6}
        pool.restore(snap)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
