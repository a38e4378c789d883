"""Microbenchmarks of the hot kernels in isolation (CUDA events, after warm-up,
inputs >> L2): K1 fingerprint at several source alignments, K3 relocation at
several (src, dst) alignment classes, and the KV batch kernel.  Prints one
JSON object; also the target of the ncu captures in tools/profile.sh.

    python tools/kernel_bench.py [--gib 16] [--only fp|reloc|kv]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=16)
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    lib = N.lib
    dev = 0
    torch.cuda.set_device(dev)
    out = {}
    n = int(args.gib * (1 << 30))

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return min(ts), sum(ts) / len(ts)

    if args.only in ("", "fp"):
        buf = DeviceBuffer(n + 64, dev)
        lib.tg_synth_fill_device(tg.TensorId(1, 2).c(), 0, n + 64, C.c_void_p(buf.ptr), dev)
        res = {}
        for shift in (0, 3, 8):
            d = N.DigestC()
            f = lambda: lib.tg_fingerprint_device(C.c_void_p(buf.ptr + shift), n, dev, C.byref(d))
            f()
            best, mean = timed(f, args.reps)
            res[f"shift{shift}"] = {"ms": best, "GBps": n / best / 1e6, "mean_GBps": n / mean / 1e6}
        out["fp"] = {"bytes": n, **res}
        buf.free()

    if args.only in ("", "reloc"):
        # one tensor of n/2 bytes moved back and forth inside a pool of n+ bytes
        size = n // 2 - 4096
        res = {}
        for src_mis, dst_mis in ((0, 0), (0, 5), (3, 11), (7, 7)):
            pool = tg.ReuseStore(tg.GpuSpec(pool_size=n + 8192), device=dev)
            m = tg.ModelSpec("r", [tg.TensorSpec(tg.TensorId(5, src_mis * 16 + dst_mis), "r", "t", size)], size)
            src = DeviceBuffer(size, dev)
            lib.tg_host_register(m.tensors[0].id.c(), C.c_void_p(src.ptr), size, None)
            if src_mis:
                pool.alloc_kv_region(src_mis, 1)
            o = pool.load_model(m, tg.ModelStatsTable(), 0.0).value()
            pool.end_instance("r")
            a_off = o.plan.placements[0].offset
            b_off = n // 2 + 1024 + dst_mis
            tid = m.tensors[0].id
            state = {"at": a_off}

            def move():
                to = b_off if state["at"] == a_off else a_off
                assert pool.move_tensor(tid, to).ok()
                state["at"] = to

            move()
            best, mean = timed(move, args.reps)
            res[f"src{a_off % 16}_dst{b_off % 16}"] = {"ms": best, "GBps_rw": 2 * size / best / 1e6,
                                                      "mean_GBps_rw": 2 * size / mean / 1e6}
            lib.tg_host_unregister(tid.c())
            src.free()
            pool.close()
        out["reloc"] = {"bytes_moved": size, **res}

    if args.only in ("", "kv"):
        model = tg.make_model("kvm", 1 << 30, 8, 819_200)
        src = DeviceBuffer(1 << 30, dev)
        for t in model.tensors:
            pass
        pool = tg.ReuseStore(tg.GpuSpec(pool_size=64 << 30), device=dev)
        st = tg.ModelStatsTable()
        from paper_2512_01357_b200.checkpoint import HostCheckpoint
        with HostCheckpoint([model], device=dev):
            pool.load_model(model, st, 0.0).value()
        res = {}
        for nreq in (16, 64, 256):
            kv = tg.KvEngine("kvm", 16, 819_200 // 16)
            reqs = [(i + 1, 1500 + 37 * i) for i in range(nreq)]
            torch.cuda.synchronize()
            import time
            t0 = time.perf_counter()
            r = kv.batch_allocate(pool, st, reqs, want_pbns=False).value()
            t1 = time.perf_counter()
            res[str(nreq)] = {"blocks": sum(r), "host_us_incl_launch": (t1 - t0) * 1e6}
            kv.instance_teardown(pool)
        out["kv"] = res
        pool.close()
        src.free()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
