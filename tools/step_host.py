"""Diagnostics: host-side phases of the bench step (C2 load #3).  python tools/step_host.py"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2512_01357_b200 as tg
from paper_2512_01357_b200 import _native as N
from paper_2512_01357_b200.checkpoint import DeviceBuffer
lib = N.lib
cat = bench.catalog(tg); keep = []
for m in (cat["opt13B"], cat["opt6.7B"]):
    for t in m.tensors:
        b = DeviceBuffer(t.size, 0); lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), 0)
        lib.tg_host_register(t.id.c(), C.c_void_p(b.ptr), t.size, None); keep.append(b)
pool = tg.ReuseStore(tg.GpuSpec("gpu0", bench.POOL), device=0)
for i, mid in enumerate(bench.SEQ[:2]):
    pool.load_model(cat[mid], bench.fresh_stats(tg, i + 1), 10.0 * i).value(); pool.end_instance(mid)
snap = pool.snapshot(); out = []
for k in range(5):
    pool.restore(snap); torch.cuda.synchronize()
    o = pool.load_model(cat["opt13B"], bench.fresh_stats(tg, 3), 20.0, details=False).value()
    out.append({a: round(b, 3) for a, b in o.timings.items() if a in ("plan_us", "total_ms", "relocate_ms", "host_issue_us", "host_wait_us", "host_total_us")})
print(json.dumps(out[-3:]))
