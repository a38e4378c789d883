"""K1 fingerprint and K3 relocation kernels against the CPU oracle.

Parity bar: bit-exact (integer/byte work).  Oracle: oracle/cpu_oracle.c
(murmur3 restated from types.hpp:77-124, tgfp1 content fingerprint,
synthetic bytes) — itself pinned to the compiled reference in test_oracle.py.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev_fp(tg, dptr, n):
    from paper_2512_01357_b200 import _native as N
    d = N.DigestC()
    rc = N.lib.tg_fingerprint_device(C.c_void_p(dptr), n, 0, C.byref(d))
    assert rc == 0, N.lib.tg_last_error_detail()
    return (d.hi, d.lo)


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 4095, 4096, 4097, 4096 * 32, 4096 * 32 + 5, 131072 * 3 + 77,
                               (1 << 22) + 12345])
@pytest.mark.parametrize("shift", [0, 1, 3, 4, 7, 8, 13, 15])
def test_fingerprint_matches_cpu(tg, cpu, n, shift):
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    from paper_2512_01357_b200 import _native as N
    rng = np.random.default_rng(n * 31 + shift)
    data = rng.integers(0, 256, size=n, dtype=np.uint8)
    buf = DeviceBuffer(n + 64)
    N.lib.tg_memcpy(C.c_void_p(buf.ptr + shift), data.ctypes.data_as(C.c_void_p), n)
    got = _dev_fp(tg, buf.ptr + shift, n)
    want, _ = cpu.content_fingerprint(data, threads=4)
    assert got == want


def test_fingerprint_large_synthetic(tg, cpu):
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    from paper_2512_01357_b200 import _native as N
    tid = tg.TensorId(0x1234, 0x5678)
    n = 68_611_111  # odd catalog size (opt1.3B layer attn)
    buf = DeviceBuffer(n + 64)
    assert N.lib.tg_synth_fill_device(tid.c(), 0, n, C.c_void_p(buf.ptr + 3), 0) == 0
    host = np.empty(n, dtype=np.uint8)
    N.lib.tg_memcpy(host.ctypes.data_as(C.c_void_p), C.c_void_p(buf.ptr + 3), n)
    assert np.array_equal(host[:1 << 20], cpu.synth(tid.hi, tid.lo, 1 << 20))
    assert np.array_equal(host[-4099:], cpu.synth(tid.hi, tid.lo, 4099, begin=n - 4099))
    assert _dev_fp(tg, buf.ptr + 3, n) == cpu.content_fingerprint(host, threads=8)[0]


def _relocate_case(tg, moves, arena_n, seed):
    """Apply moves (src_off, dst_off, len) through tg_move_tensor on a pool and
    compare the arena with a numpy memmove replay."""
    from paper_2512_01357_b200 import _native as N
    pool = tg.ReuseStore(tg.GpuSpec(pool_size=arena_n), device=0)
    arena = pool.info()["arena"]
    rng = np.random.default_rng(seed)
    data = rng.integers(0, 256, size=arena_n, dtype=np.uint8)
    N.lib.tg_memcpy(C.c_void_p(arena), data.ctypes.data_as(C.c_void_p), arena_n)
    return pool, arena, data


def test_relocation_kernel_random_alignments(tg):
    """Single moves of every alignment class through tg_move_tensor (K3)."""
    from paper_2512_01357_b200 import _native as N
    rng = np.random.default_rng(7)
    arena_n = 8 << 20
    for case in range(40):
        size = int(rng.integers(1, 300_000)) if case % 4 else int(rng.integers(1, 40))
        pool = tg.ReuseStore(tg.GpuSpec(pool_size=arena_n), device=0)
        arena = pool.info()["arena"]
        m = tg.ModelSpec("m", [tg.TensorSpec(tg.TensorId(1, case), "m", "t", size)], size)
        from paper_2512_01357_b200.checkpoint import PinnedBuffer
        src = PinnedBuffer(size)
        src.array()[:] = rng.integers(0, 256, size=size, dtype=np.uint8)
        N.lib.tg_host_register(tg.TensorId(1, case).c(), C.c_void_p(src.ptr), size, None)
        st = tg.ModelStatsTable()
        pre = int(rng.integers(0, 64))
        # occupy [0, pre) with a kv region so the tensor lands at an odd offset
        if pre:
            assert pool.alloc_kv_region(pre, 1).ok()
        o = pool.load_model(m, st, 0.0).value()
        pool.end_instance("m")
        off = o.plan.placements[0].offset
        to = int(rng.integers(off + size, arena_n - size))
        assert pool.move_tensor(tg.TensorId(1, case), to).ok()
        out = np.empty(size, dtype=np.uint8)
        N.lib.tg_memcpy(out.ctypes.data_as(C.c_void_p), C.c_void_p(arena + to), size)
        assert np.array_equal(out, src.array()), (case, size, off, to)
        assert pool.fingerprint_tensor(tg.TensorId(1, case)) == o.digests[0]
        N.lib.tg_host_unregister(tg.TensorId(1, case).c())
        pool.close()


@pytest.mark.parametrize("n", [0, 1, 15, 17, 4095, 4096, 4097, 8192, 4096 * 31 + 7, 4096 * 32, 4096 * 33 + 1,
                               (1 << 21) + 4093, 131072 * 5 + 999])
@pytest.mark.parametrize("so,do", [(0, 0), (0, 5), (5, 0), (3, 11), (11, 3), (7, 7), (15, 1), (1, 15), (0, 8),
                                   (4, 0), (12, 4), (8, 12), (6, 2)])
@pytest.mark.parametrize("pad", [16, 32, 64, 112])
def test_copy_fingerprint_fused(tg, cpu, n, so, do, pad):
    """K3F moves the bytes exactly (including head/tail bytes, neighbours
    untouched) and returns the same digest as tgfp1 on the CPU.  `pad` moves
    the destination across the 128-byte line phases the line stores use."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    rng = np.random.default_rng(n * 131 + so * 17 + do)
    data = rng.integers(0, 256, size=n + 64, dtype=np.uint8)
    src, dst = DeviceBuffer(n + 128), DeviceBuffer(n + 256)
    N.lib.tg_memcpy(C.c_void_p(src.ptr), data.ctypes.data_as(C.c_void_p), n + 64)
    guard = np.full(n + 256, 0x5A, dtype=np.uint8)
    N.lib.tg_memcpy(C.c_void_p(dst.ptr), guard.ctypes.data_as(C.c_void_p), n + 256)
    mv = (C.c_uint64 * 3)(src.ptr + so, dst.ptr + pad + do, n)
    dig = (N.DigestC * 1)()
    assert N.lib.tg_copy_fingerprint(mv, 1, 0, 0, None, dig) == 0, N.lib.tg_last_error_detail()
    out = np.empty(n + 256, dtype=np.uint8)
    N.lib.tg_memcpy(out.ctypes.data_as(C.c_void_p), C.c_void_p(dst.ptr), n + 256)
    assert np.array_equal(out[pad + do:pad + do + n], data[so:so + n])
    assert np.all(out[:pad + do] == 0x5A) and np.all(out[pad + do + n:] == 0x5A)
    assert (dig[0].hi, dig[0].lo) == cpu.content_fingerprint(data[so:so + n].copy(), threads=4)[0]


def test_copy_fingerprint_batched_moves(tg, cpu):
    """Several hazard-free moves in one launch (a relocation wave)."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    rng = np.random.default_rng(3)
    sizes = [68_611_111 % (1 << 22), 4097, 1, 300_001, 4096 * 64 + 3]
    bufs, moves, datas = [], [], []
    for k, n in enumerate(sizes):
        s, d = DeviceBuffer(n + 64), DeviceBuffer(n + 64)
        # the whole source buffer is initialised: realigning reads touch the
        # bytes before the tensor inside its first 16-byte word (discarded)
        pad = rng.integers(0, 256, size=n + 64, dtype=np.uint8)
        N.lib.tg_memcpy(C.c_void_p(s.ptr), pad.ctypes.data_as(C.c_void_p), n + 64)
        dat = rng.integers(0, 256, size=n, dtype=np.uint8)
        N.lib.tg_memcpy(C.c_void_p(s.ptr + k), dat.ctypes.data_as(C.c_void_p), n)
        moves += [s.ptr + k, d.ptr + 2 * k + 1, n]
        bufs += [s, d]
        datas.append(dat)
    arr = (C.c_uint64 * len(moves))(*moves)
    dig = (N.DigestC * len(sizes))()
    assert N.lib.tg_copy_fingerprint(arr, len(sizes), 0, 0, None, dig) == 0
    for k, n in enumerate(sizes):
        out = np.empty(n, dtype=np.uint8)
        N.lib.tg_memcpy(out.ctypes.data_as(C.c_void_p), C.c_void_p(moves[3 * k + 1]), n)
        assert np.array_equal(out, datas[k])
        assert (dig[k].hi, dig[k].lo) == cpu.content_fingerprint(datas[k], threads=4)[0]


def test_copy_fingerprint_mixed_verify(tg, cpu):
    """One writing launch mixing moves and in-place verification tasks (dst =
    0) at every phase class and ragged sizes, as a load's single launch does:
    verify tiles realign from the next stage while move tiles keep the paired
    ring, tiles of both kinds interleave in a warp's stream, and every digest
    equals the CPU restatement."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    rng = np.random.default_rng(17)
    specs = [(4096 * 33 + 5, 3, 9), (131077, 0, None), (4097, 13, None), (4096 * 40, 8, 0), (393293, 7, None),
             (1, 1, None), (4096 * 64 + 15, 0, 5), (200_003, 12, None), (16, 5, None), (4096 * 32, 11, 11)]
    bufs, moves, datas = [], [], []
    for n, so, do in specs:
        s_ = DeviceBuffer(n + 64)
        raw = rng.integers(0, 256, size=n + 64, dtype=np.uint8)
        N.lib.tg_memcpy(C.c_void_p(s_.ptr), raw.ctypes.data_as(C.c_void_p), n + 64)
        bufs.append(s_)
        dst = 0
        if do is not None:
            d_ = DeviceBuffer(n + 64)
            bufs.append(d_)
            dst = d_.ptr + do
        moves += [s_.ptr + so, dst, n]
        datas.append(raw[so:so + n].copy())
    arr = (C.c_uint64 * len(moves))(*moves)
    dig = (N.DigestC * len(specs))()
    assert N.lib.tg_copy_fingerprint(arr, len(specs), 0, 0, None, dig) == 0, N.lib.tg_last_error_detail()
    for k, (n, so, do) in enumerate(specs):
        assert (dig[k].hi, dig[k].lo) == cpu.content_fingerprint(datas[k], threads=4)[0], k
        if do is not None:
            out = np.empty(n, dtype=np.uint8)
            N.lib.tg_memcpy(out.ctypes.data_as(C.c_void_p), C.c_void_p(moves[3 * k + 1]), n)
            assert np.array_equal(out, datas[k]), k


def test_tensor_beyond_4gib(tg, cpu):
    """A 4.5 GB tensor (byte offsets, leaf and tile counts past 2^32): K1 and
    the load kernel's move + fingerprint agree with the CPU restatement, and
    the moved bytes match around the 4 GiB boundary and at both ends."""
    from paper_2512_01357_b200 import _native as N
    from paper_2512_01357_b200.checkpoint import DeviceBuffer
    n = 4_500_000_007
    tid = tg.TensorId(0xABCD, 0x4242)
    src, dst = DeviceBuffer(n + 64), DeviceBuffer(n + 64)
    assert N.lib.tg_synth_fill_device(tid.c(), 0, n, C.c_void_p(src.ptr + 5), 0) == 0
    host = np.empty(n, dtype=np.uint8)
    N.lib.tg_memcpy(host.ctypes.data_as(C.c_void_p), C.c_void_p(src.ptr + 5), n)
    want = cpu.content_fingerprint(host, threads=16)[0]
    assert _dev_fp(tg, src.ptr + 5, n) == want
    mv = (C.c_uint64 * 3)(src.ptr + 5, dst.ptr + 14, n)
    dig = (N.DigestC * 1)()
    assert N.lib.tg_copy_fingerprint(mv, 1, 0, 0, None, dig) == 0, N.lib.tg_last_error_detail()
    assert (dig[0].hi, dig[0].lo) == want
    for lo in (0, (1 << 32) - 4099, n - 5000):
        w = np.empty(4099, dtype=np.uint8)
        N.lib.tg_memcpy(w.ctypes.data_as(C.c_void_p), C.c_void_p(dst.ptr + 14 + lo), 4099)
        assert np.array_equal(w, host[lo:lo + 4099]), lo
    assert _dev_fp(tg, dst.ptr + 14, n) == want
