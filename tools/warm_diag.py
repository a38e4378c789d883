import ctypes as C, json, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_01357_b200 as tg
from paper_2512_01357_b200 import _native as N
from paper_2512_01357_b200.checkpoint import DeviceBuffer
lib = N.lib
m = {x.model_id: x for x in tg.default_catalog()}["opt13B"]
bufs = []
for t in m.tensors:
    b = DeviceBuffer(t.size, 0); lib.tg_synth_fill_device(t.id.c(), 0, t.size, C.c_void_p(b.ptr), 0)
    lib.tg_host_register(t.id.c(), C.c_void_p(b.ptr), t.size, None); bufs.append(b)
pool = tg.ReuseStore(tg.GpuSpec("gpu0", m.total_size + (64 << 20)), device=0)
st = tg.ModelStatsTable(); st.record_request(m.model_id, 0.0)
pool.load_model(m, st, 0.0).value(); pool.end_instance(m.model_id)
for b in bufs: b.free()
out = []
for k in range(6):
    st.record_request(m.model_id, 1.0 + k)
    torch.cuda.synchronize()
    o = pool.load_model(m, st, 1.0 + k, details=False).value()
    pool.end_instance(m.model_id)
    out.append({kk: round(v, 4) for kk, v in o.timings.items()})
infos = [pool.tensor_info(t.id) for t in m.tensors]
ptrs = (C.c_void_p * len(infos))(*[i["device_ptr"] for i in infos])
ns = (C.c_uint64 * len(infos))(*[i["size"] for i in infos])
digs = (N.DigestC * len(infos))()
ms = C.c_double()
lib.tg_bench_fingerprint(ptrs, ns, len(infos), 0, 5, C.byref(ms), digs)
print(json.dumps({"loads": out, "k1_alone_ms": ms.value, "k1_GBps": m.total_size / ms.value / 1e6,
                  "aligned16": sum(1 for i in infos if i["device_ptr"] % 16 == 0)}))
