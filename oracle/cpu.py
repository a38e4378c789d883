"""ORACLE / TEST INFRASTRUCTURE ONLY: ctypes driver for oracle/cpu_oracle.c.

The plain-C restatement of murmur3 (types.hpp:64-124), the tgfp1 content
fingerprint (SURVEY §8 a2′), the synthetic checkpoint stream and
the CPU data plane of apply_plan (reuse_store.hpp:316-334).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "_build", "libtangram_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            raise RuntimeError(f"CPU oracle not built: {_PATH} (run `make -C oracle`)")
        L = ctypes.CDLL(_PATH)
        c = ctypes
        u64p = c.POINTER(c.c_uint64)
        L.orc_murmur3_x64_128.argtypes = [c.c_void_p, c.c_uint64, c.c_uint64, u64p]
        L.orc_content_fingerprint.argtypes = [c.c_void_p, c.c_uint64, c.c_int, u64p, u64p]
        L.orc_fingerprint_finalize.argtypes = [c.c_uint64, c.c_uint64, c.c_uint64, u64p]
        L.orc_synth_fill.argtypes = [c.c_uint64, c.c_uint64, c.c_uint64, c.c_uint64, c.c_void_p]
        L.orc_copy.argtypes = [c.c_void_p, c.c_void_p, c.c_uint64, c.c_int]
        L.orc_replay_plan.argtypes = [c.c_void_p, c.c_uint64, u64p, c.c_uint64, u64p,
                                      c.POINTER(c.c_void_p), c.c_int]
        for f in (L.orc_murmur3_x64_128, L.orc_content_fingerprint, L.orc_fingerprint_finalize,
                  L.orc_synth_fill, L.orc_copy, L.orc_replay_plan):
            f.restype = None
        _lib = L
    return _lib


def _ptr(a):
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if isinstance(a, (bytes, bytearray)):
        return ctypes.cast(ctypes.create_string_buffer(bytes(a), len(a)), ctypes.c_void_p).value
    return int(a)


def murmur3(data, seed=0):
    buf = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    out = (ctypes.c_uint64 * 2)()
    lib().orc_murmur3_x64_128(buf.ctypes.data if buf.size else None, buf.size, seed, out)
    return out[0], out[1]


def content_fingerprint(data, threads=1, n=None):
    """tgfp1 fingerprint of a numpy uint8 array (or raw pointer + n)."""
    out = (ctypes.c_uint64 * 2)()
    sums = (ctypes.c_uint64 * 2)()
    if isinstance(data, np.ndarray):
        n = data.nbytes
        p = data.ctypes.data if n else None
    else:
        p = int(data)
    lib().orc_content_fingerprint(p, n, threads, out, sums)
    return (out[0], out[1]), (sums[0], sums[1])


def synth(hi, lo, size, begin=0):
    """Synthetic checkpoint bytes [begin, begin+size) of tensor (hi, lo)."""
    out = np.empty(size, dtype=np.uint8)
    lib().orc_synth_fill(hi, lo, begin, size, out.ctypes.data if size else None)
    return out


def synth_into(hi, lo, dst_ptr, size, begin=0):
    lib().orc_synth_fill(hi, lo, begin, size, dst_ptr)


def copy(dst_ptr, src_ptr, n, threads=1):
    lib().orc_copy(dst_ptr, src_ptr, n, threads)
