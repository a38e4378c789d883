"""The C-ABI library loads without a GPU and exports every symbol that
include/tangram.h declares; control-plane-only calls work on CPU and
data-plane calls fail loudly (no silent fallback)."""
import ctypes as C
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "tangram.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(tg):
    from paper_2512_01357_b200 import _native as N
    names = _declared()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(N.lib, n)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert set(names) == set(N.EXPORTED), set(names) ^ set(N.EXPORTED)


def test_version_and_errors(tg):
    from paper_2512_01357_b200 import _native as N
    assert N.lib.tg_version() == 1
    assert N.lib.tg_error_string(1) == b"insufficient memory"
    assert N.lib.tg_error_string(10) == b"invalid argument"
    assert N.lib.tg_error_string(101) == b"no device"
    assert N.lib.tg_error_string(107) == b"a KV engine is armed for device batches"


def test_kv_device_path_needs_a_device(tg):
    """K4D (device-decided KV batches) refuses control-plane-only pools."""
    from paper_2512_01357_b200 import _native as N
    import pytest
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=1 << 20), device=None)
    st = tg.ModelStatsTable()
    kv = tg.KvEngine("s", 8, 100)
    assert kv.batch_allocate(pool, st, [(1, 20)]).ok()
    assert kv.request_slot(1) == 0
    with pytest.raises(N.TangramRuntimeError):
        kv.device_arm(pool, 16, 8, 4)
    assert pool.alloc_kv_region(800, 5).ok()  # not armed
    # the paged-cache consumers need device tables too
    assert N.lib.tg_kv_write_tokens(kv._h, pool._h, None, None, None, 0, None) == 101
    assert N.lib.tg_kv_read_tokens(kv._h, pool._h, None, None, None, 0, None) == 101


def test_data_plane_fails_loudly_without_device(tg):
    """A control-plane-only pool refuses byte-level requests instead of
    faking them."""
    from paper_2512_01357_b200 import _native as N
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=1 << 20), device=None)
    m = tg.make_model("x", 1000, 2, 16)
    st = tg.ModelStatsTable()
    assert pool.load_model(m, st, 0.0).ok()
    d = N.DigestC()
    rc = N.lib.tg_fingerprint_tensor(pool._h, m.tensors[0].id.c(), C.byref(d))
    assert rc == 101
    s = C.c_void_p()
    assert N.lib.tg_pool_stream(pool._h, C.byref(s)) == 101


def test_device_pool_without_gpu_errors(tg):
    from paper_2512_01357_b200 import _native as N
    if N.device_count() > 0:
        return
    import pytest
    with pytest.raises(N.TangramRuntimeError):
        tg.ReuseStore(tg.GpuSpec(pool_size=1 << 20), device=0)


def test_plain_c_client(tmp_path):
    """include/tangram.h is plain C11: a C client compiles with -Wall -Werror,
    links libtangram.so and loads a catalog model on a control-plane pool."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        import pytest
        pytest.skip("no gcc")
    exe = tmp_path / "load_c11"
    lib = os.path.join(ROOT, "paper_2512_01357_b200")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "load_c11.c"), "-L", lib, "-ltangram",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "rc=0 xfer=2600000000 hits=0", out
