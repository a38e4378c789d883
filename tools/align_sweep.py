import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import paper_2512_01357_b200 as tg
from paper_2512_01357_b200 import _native as N
from paper_2512_01357_b200.checkpoint import DeviceBuffer
lib = N.lib
n = 32 << 30
buf = DeviceBuffer(n + 4096, 0)
lib.tg_synth_fill_device(tg.TensorId(3, 4).c(), 0, n, C.c_void_p(buf.ptr), 0)
a = buf.ptr
D, S = 2_797_238_364, 5 * 530_416_667
out = {}
for x in list(range(0, 16)) + [64, 96]:
    mv = [(a + 20_000_000_000 + x, a + 20_000_000_000 + x + D, S)]
    arr = (C.c_uint64 * 3)(*mv[0])
    dg = (N.DigestC * 1)()
    ms = C.c_double()
    N.check_runtime(lib.tg_copy_fingerprint(arr, 1, 0, 5, C.byref(ms), dg), "x")
    out[x] = round(2 * S / ms.value / 1e6)
# same split into 5 tasks at S/5 boundaries (leaf grid per task)
for x in (0, 3):
    s5 = S // 5
    mv = [(a + 20_000_000_000 + x + i * s5, a + 20_000_000_000 + x + i * s5 + D, s5) for i in range(5)]
    arr = (C.c_uint64 * 15)(*[v for m in mv for v in m])
    dg = (N.DigestC * 5)()
    ms = C.c_double()
    N.check_runtime(lib.tg_copy_fingerprint(arr, 5, 0, 5, C.byref(ms), dg), "x5")
    out[f"split5_x{x}"] = round(2 * S / ms.value / 1e6)
    s5 = (S // 5) // 4096 * 4096
    mv = [(a + 20_000_000_000 + x + i * s5, a + 20_000_000_000 + x + i * s5 + D, s5) for i in range(5)]
    arr = (C.c_uint64 * 15)(*[v for m in mv for v in m])
    N.check_runtime(lib.tg_copy_fingerprint(arr, 5, 0, 5, C.byref(ms), dg), "x5a")
    out[f"split5_leafaligned_x{x}"] = round(2 * 5 * s5 / ms.value / 1e6)
print(json.dumps(out))
