"""Diagnostics: load-kernel (copy + fingerprint) and K3 rates for move lists
of different geometry inside one 32 GiB arena-like buffer, modelled on the C2
step's relocation waves (5 moves of 530 MB shifted by the same 2.80 GB).
    python tools/move_geometry.py
"""
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
    n = 32 << 30
    buf = DeviceBuffer(n + 4096, 0)
    lib.tg_synth_fill_device(tg.TensorId(3, 4).c(), 0, n, C.c_void_p(buf.ptr), 0)
    a = buf.ptr
    D, S, base = 2_797_238_364, 530_416_667, 26_258_333_334 - 2_797_238_364 * 4
    cases = {
        "wave_like_5x530MB_same_shift": [(a + 26_258_333_334 + i * S, a + 26_258_333_334 + i * S + D, S) for i in range(5)],
        "one_2.65GB_move_same_shift": [(a + 20_000_000_003, a + 20_000_000_003 + D, 5 * S)],
        "5x530MB_far_apart": [(a + 1_000_000_003 + i * 3 * S, a + 17_000_000_007 + i * 2 * S, S) for i in range(5)],
        "5x530MB_shift_8GiB": [(a + 1_000_000_003 + i * S, a + 1_000_000_003 + i * S + (8 << 30) + 12, S) for i in range(5)],
    }
    out = {}
    for name, mv in cases.items():
        arr = (C.c_uint64 * (3 * len(mv)))(*[x for m in mv for x in m])
        nbytes = sum(m[2] for m in mv)
        dg = (N.DigestC * len(mv))()
        ms = C.c_double()
        N.check_runtime(lib.tg_copy_fingerprint(arr, len(mv), 0, 5, C.byref(ms), dg), name)
        k3 = C.c_double()
        N.check_runtime(lib.tg_bench_relocate(arr, len(mv), 0, 5, C.byref(k3)), name)
        out[name] = {"load_kernel_GBps_rw": 2 * nbytes / ms.value / 1e6, "k3_GBps_rw": 2 * nbytes / k3.value / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
