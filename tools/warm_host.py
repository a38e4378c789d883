"""Diagnostics: host-side phases of an OPT-1.3B 100 %-reuse reload (LoadOutcome timings).
    python tools/warm_host.py"""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_01357_b200 as tg
from paper_2512_01357_b200.checkpoint import HostCheckpoint
m = {x.model_id: x for x in tg.default_catalog()}["opt1.3B"]
pool = tg.ReuseStore(tg.GpuSpec("gpu0", 8 << 30), device=0)
st = tg.ModelStatsTable()
with HostCheckpoint([m]):
    st.record_request(m.model_id, 0.0); pool.load_model(m, st, 0.0).value(); pool.end_instance(m.model_id)
    out = []
    for k in range(6):
        st.record_request(m.model_id, 1.0 + k)
        torch.cuda.synchronize()
        o = pool.load_model(m, st, 1.0 + k, details=False).value()
        pool.end_instance(m.model_id)
        out.append({a: round(b, 3) for a, b in o.timings.items()})
print(json.dumps(out[-3:]))
