"""Microbenchmarks of the hot kernels in isolation: K1 fingerprint at several
source alignments and K3 relocation at several (src, dst) alignment classes.
Kernel-only timing (tg_bench_*: reps back-to-back launches bracketed by CUDA
events on the launching stream, after a warm-up launch); inputs >> L2.
Prints one JSON object.

    python tools/kernel_bench.py [--gib 16] [--only fp|reloc]  (reloc also times the fused K3F) [--reps 5]
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
    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    lib = N.lib
    dev = 0
    out = {"peak_hbm_GBps": None}
    try:
        out["peak_hbm_GBps"] = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    n = int(args.gib * (1 << 30))
    if args.only in ("", "fp"):
        buf = DeviceBuffer(n + 64, dev)
        lib.tg_synth_fill_device(tg.TensorId(1, 2).c(), 0, n + 64, C.c_void_p(buf.ptr), dev)
        res = {}
        for shift in (3, 0, 8, 13, 0):
            ms = C.c_double()
            d = N.DigestC()
            ptrs = (C.c_void_p * 1)(buf.ptr + shift)
            ns = (C.c_uint64 * 1)(n)
            N.check_runtime(lib.tg_bench_fingerprint(ptrs, ns, 1, dev, args.reps, C.byref(ms), C.byref(d)),
                            "bench fp")
            res[f"shift{shift}"] = {"ms": ms.value, "GBps": n / ms.value / 1e6}
        out["fp"] = {"bytes_per_launch": n, **res}
        buf.free()
    if args.only in ("", "reloc"):
        size = n // 2
        a = DeviceBuffer(size + 64, dev)
        b = DeviceBuffer(size + 64, dev)
        res = {}
        for so, do in ((0, 0), (0, 5), (3, 11), (7, 7), (13, 2)):
            ms = C.c_double()
            mv = (C.c_uint64 * 3)(a.ptr + so, b.ptr + do, size)
            N.check_runtime(lib.tg_bench_relocate(mv, 1, dev, args.reps, C.byref(ms)), "bench reloc")
            res[f"src{so}_dst{do}"] = {"ms": ms.value, "GBps_rw": 2 * size / ms.value / 1e6}
        out["reloc"] = {"bytes_per_launch": size, **res}
        res = {}
        for so, do in ((0, 0), (3, 3), (0, 8), (3, 11), (13, 2)):
            ms = C.c_double()
            mv = (C.c_uint64 * 3)(a.ptr + so, b.ptr + do, size)
            dg = (N.DigestC * 1)()
            N.check_runtime(lib.tg_copy_fingerprint(mv, 1, dev, args.reps, C.byref(ms), dg), "bench K3F")
            res[f"src{so}_dst{do}"] = {"ms": ms.value, "GBps_rw": 2 * size / ms.value / 1e6}
        for so in (0, 3):  # in-place verification through the load kernel (dst = nullptr)
            ms = C.c_double()
            mv = (C.c_uint64 * 3)(a.ptr + so, 0, size)
            dg = (N.DigestC * 1)()
            N.check_runtime(lib.tg_copy_fingerprint(mv, 1, dev, args.reps, C.byref(ms), dg), "bench K3F verify")
            res[f"verify_src{so}"] = {"ms": ms.value, "GBps_read": size / ms.value / 1e6}
        out["copy_fp"] = {"bytes_per_launch": size, **res}
        a.free()
        b.free()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
