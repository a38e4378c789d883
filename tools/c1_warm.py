"""C1 warm-reload breakdown: for each small catalog
model, the 100 %-reuse reload timed as bench.py does (CUDA events on the pool
stream around the Python call) next to the library's own device timeline
(entry -> load kernel end -> all done) and host timings.

    python tools/c1_warm.py [model ...]   -> gpurun_out/c1_warm.json
"""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2512_01357_b200 as tg  # noqa: E402
from paper_2512_01357_b200.checkpoint import HostCheckpoint  # noqa: E402

HBM = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6536.4
names = sys.argv[1:] or ["opt1.3B", "qwen3B", "llama3B", "opt13B"]
cat = {m.model_id: m for m in tg.default_catalog()}
out = {}
for name in names:
    m = cat[name]
    pool = tg.ReuseStore(tg.GpuSpec("gpu0", m.total_size + (64 << 20)), device=0)
    st = tg.ModelStatsTable()
    rows = []
    with HostCheckpoint([m]):
        st.record_request(m.model_id, 0.0)
        pool.load_model(m, st, 0.0, details=False).value()
        pool.end_instance(m.model_id)
        s = torch.cuda.ExternalStream(pool.stream(), device=0)
        for k in range(12):
            st.record_request(m.model_id, 1.0 + k)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            o = pool.load_model(m, st, 1.0 + k, details=False).value()
            b.record(s)
            b.synchronize()
            pool.end_instance(m.model_id)
            rows.append(dict(event_ms=a.elapsed_time(b), **{k2: v for k2, v in o.timings.items()}))
    pool.close()
    first, rest = rows[0], rows[2:]
    med = {k: statistics.median(r[k] for r in rest) for k in rest[0]}
    out[name] = {"bytes": m.total_size, "first": first, "median": med,
                 "frac_event": m.total_size / med["event_ms"] / 1e6 / HBM,
                 "frac_total": m.total_size / med["total_ms"] / 1e6 / HBM,
                 "frac_kernel": m.total_size / med["relocate_ms"] / 1e6 / HBM}
    print(name, json.dumps({k: round(v, 4) for k, v in med.items()}), round(out[name]["frac_event"], 3),
          round(out[name]["frac_kernel"], 3))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c1_warm.json", "w"), indent=1)
