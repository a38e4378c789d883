"""Synthetic host checkpoints for the load path.

Bytes of tensor t are the little-endian u64 stream
splitmix64(t.hi ^ rotl(t.lo, 17) ^ (w * 0x9E3779B97F4A7C15)), truncated to
t.size — content is a pure function of the TensorId, so "same content" and
"same key" coincide and content-keyed reuse decisions equal the reference's
key-based ones.  A tensor-parallel shard (shard_model) holds its byte range
of the parent tensor's stream, so shards of one tensor in different layouts
agree byte for byte where they overlap.  Buffers are pinned (cudaMallocHost) and registered with the
library as the byte source of each tensor (tg_host_register).  Large
checkpoints are generated on the GPU (synth kernel) and copied down once.
"""
import ctypes as C

import numpy as np

from . import _native as N
from .pool import ModelSpec, TensorId, lineage

lib = N.lib


def host_array(ptr, n):
    """numpy uint8 view of n bytes at a host address."""
    if n == 0:
        return np.empty(0, dtype=np.uint8)
    return np.ctypeslib.as_array((C.c_uint8 * n).from_address(ptr))


class PinnedBuffer:
    def __init__(self, n):
        self.n = n
        self.ptr = C.c_void_p()
        N.check_runtime(lib.tg_host_alloc(max(1, n), C.byref(self.ptr)), "tg_host_alloc")
        self.ptr = self.ptr.value

    def array(self):
        return host_array(self.ptr, self.n)

    def free(self):
        if self.ptr:
            lib.tg_host_free(C.c_void_p(self.ptr))
            self.ptr = None

    __del__ = free


class DeviceBuffer:
    def __init__(self, n, device=0):
        self.n, self.device = n, device
        p = C.c_void_p()
        N.check_runtime(lib.tg_device_alloc(device, max(1, n), C.byref(p)), "tg_device_alloc")
        self.ptr = p.value

    def free(self):
        if self.ptr:
            lib.tg_device_free(self.device, C.c_void_p(self.ptr))
            self.ptr = None

    __del__ = free


def content_of(tid: TensorId):
    """(stream id, offset) of a tensor's synthetic bytes: its own stream, or
    its parent's at the shard's offset."""
    lin = lineage(tid)
    return (tid, 0) if lin is None else (lin[0], lin[1])


def synth_host(tid: TensorId, n, begin=0, threads=8):
    out = np.empty(n, dtype=np.uint8)
    if n:
        lib.tg_synth_fill_host(tid.c(), begin, n, out.ctypes.data, threads)
    return out


class HostCheckpoint:
    """Pinned synthetic bytes for every tensor of `models`, registered as sources."""

    def __init__(self, models, device=0, fill="device", register=True):
        self.models = list(models)
        self.entries = {}
        seen = set()
        tensors = []
        for m in self.models:
            for t in m.tensors:
                if t.id not in seen:
                    seen.add(t.id)
                    tensors.append(t)
        total = sum(t.size for t in tensors)
        self.slab = PinnedBuffer(total)
        scratch = None
        if fill == "device" and tensors:
            scratch = DeviceBuffer(max(t.size for t in tensors), device)
        off = 0
        for t in tensors:
            ptr = self.slab.ptr + off
            sid, begin = content_of(t.id)
            if fill == "device":
                N.check_runtime(lib.tg_synth_fill_device(sid.c(), begin, t.size, C.c_void_p(scratch.ptr), device))
                N.check_runtime(lib.tg_memcpy(C.c_void_p(ptr), C.c_void_p(scratch.ptr), t.size), "tg_memcpy")
            else:
                lib.tg_synth_fill_host(sid.c(), begin, t.size, C.c_void_p(ptr), 8)
            if register:
                N.check_runtime(lib.tg_host_register(t.id.c(), C.c_void_p(ptr), t.size, None), "tg_host_register")
            self.entries[t.id] = (ptr, t.size)
            off += t.size
        if scratch is not None:
            scratch.free()
        self.registered = register

    def register(self):
        """(Re-)register every tensor's pinned bytes as its source."""
        for tid, (ptr, n) in self.entries.items():
            N.check_runtime(lib.tg_host_register(tid.c(), C.c_void_p(ptr), n, None), "tg_host_register")
        self.registered = True

    def view(self, tid: TensorId):
        ptr, n = self.entries[tid]
        return host_array(ptr, n)

    def close(self):
        if self.registered:
            for tid in self.entries:
                lib.tg_host_unregister(tid.c())
            self.registered = False
        self.slab.free()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
