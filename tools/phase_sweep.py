"""Diagnostics: load-kernel rates by 128-byte line phase of the source (p)
and destination (q): copies (r+w GB/s, 4 GiB) and in-place verification
(read GB/s).  python tools/phase_sweep.py"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2512_01357_b200 as tg
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    lib = N.lib
    size = 4 << 30
    a, b = DeviceBuffer(size + 4096, 0), DeviceBuffer(size + 4096, 0)
    lib.tg_synth_fill_device(tg.TensorId(5, 6).c(), 0, size + 4096, C.c_void_p(a.ptr), 0)
    out = {}
    for p in (0, 3, 64, 67):
        for q in (0, 11, 64, 75):
            arr = (C.c_uint64 * 3)(a.ptr + p, b.ptr + q, size)
            dg = (N.DigestC * 1)()
            ms = C.c_double()
            N.check_runtime(lib.tg_copy_fingerprint(arr, 1, 0, 5, C.byref(ms), dg), "copy")
            out[f"copy_p{p}_q{q}"] = round(2 * size / ms.value / 1e6)
        arr = (C.c_uint64 * 3)(a.ptr + p, 0, size)
        dg = (N.DigestC * 1)()
        ms = C.c_double()
        N.check_runtime(lib.tg_copy_fingerprint(arr, 1, 0, 5, C.byref(ms), dg), "verify")
        out[f"verify_p{p}"] = round(size / ms.value / 1e6)
        ptrs = (C.c_void_p * 1)(a.ptr + p)
        ns = (C.c_uint64 * 1)(size)
        N.check_runtime(lib.tg_bench_fingerprint(ptrs, ns, 1, 0, 5, C.byref(ms), dg), "k1")
        out[f"k1_p{p}"] = round(size / ms.value / 1e6)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
