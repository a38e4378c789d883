"""K1 fixed cost vs size: the fingerprint-only load kernel over one buffer of
0.25 .. 8 GiB (source phase 3, the catalog's common case) and over C1's own
25-tensor layout, kernel-only (tg_bench_fingerprint: back-to-back launches
bracketed by CUDA events).  A linear fit t = t0 + n / R separates the launch's
fixed cost (ramp + tail) from its streaming rate.

    python tools/fp_size_sweep.py  -> stdout JSON
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import paper_2512_01357_b200 as tg  # noqa: E402
from paper_2512_01357_b200 import _native as N  # noqa: E402
from paper_2512_01357_b200.checkpoint import DeviceBuffer  # noqa: E402

lib = N.lib
GIB = 1 << 30


def bench(ptrs, ns, reps=10):
    ms = C.c_double()
    digs = (N.DigestC * len(ptrs))()
    N.check_runtime(lib.tg_bench_fingerprint((C.c_void_p * len(ptrs))(*ptrs), (C.c_uint64 * len(ns))(*ns),
                                             len(ptrs), 0, reps, C.byref(ms), digs), "bench")
    return ms.value


def main():
    buf = DeviceBuffer(8 * GIB + 4096, 0)
    lib.tg_synth_fill_device(tg.TensorId(1, 2).c(), 0, 8 * GIB + 4096, C.c_void_p(buf.ptr), 0)
    rows = []
    for gib in (0.25, 0.5, 1, 2, 2.6e9 / GIB, 4, 8):
        n = int(gib * GIB)
        ms = bench([buf.ptr + 3], [n])
        rows.append({"bytes": n, "ms": ms, "GBps": n / ms / 1e6})
    # C1 layout: opt1.3B's 25 tensors packed size-descending from offset 0
    m = {x.model_id: x for x in tg.default_catalog()}["opt1.3B"]
    sizes = sorted((t.size for t in m.tensors), reverse=True)
    ptrs, off = [], 0
    for s in sizes:
        ptrs.append(buf.ptr + off)
        off += s
    c1 = bench(ptrs, sizes)
    # the same tensors dispensed grouped by source phase class (hash variant)
    order = sorted(range(len(ptrs)), key=lambda i: (0 if ptrs[i] % 16 == 0 else 1 + (ptrs[i] % 16) // 4, i))
    c1_sorted = bench([ptrs[i] for i in order], [sizes[i] for i in order])
    # the same sizes, every tensor at source phase 3 (one hash variant)
    ptrs3, off = [], 0
    for s in sizes:
        ptrs3.append(buf.ptr + off + 3)
        off += (s + 4095) // 4096 * 4096
    c1_phase3 = bench(ptrs3, sizes)
    xs = [r["bytes"] for r in rows]
    ys = [r["ms"] for r in rows]
    k = len(xs)
    mx, my = sum(xs) / k, sum(ys) / k
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    t0 = my - slope * mx
    print(json.dumps({"single_buffer_phase3": rows, "fit": {"fixed_us": t0 * 1e3, "stream_GBps": 1 / slope / 1e6},
                      "c1_layout": {"tensors": len(sizes), "bytes": sum(sizes), "ms": c1,
                                    "GBps": sum(sizes) / c1 / 1e6},
                      "c1_layout_grouped_by_phase": {"ms": c1_sorted, "GBps": sum(sizes) / c1_sorted / 1e6},
                      "c1_sizes_all_phase3": {"ms": c1_phase3, "GBps": sum(sizes) / c1_phase3 / 1e6}}))
    buf.free()


if __name__ == "__main__":
    main()
