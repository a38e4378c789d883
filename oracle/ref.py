"""ORACLE / TEST INFRASTRUCTURE ONLY: ctypes driver for the reference.

Loads oracle/_ref/libwarmsim_ref.so (the unmodified reference headers behind a
JSON C-ABI, see ref_capi.cpp) and exposes the reference's own objects:
ReuseStore (reuse_store.hpp:50), KvEngine (kv_engine.hpp:43), ModelStatsTable
(model.hpp:70), plan_allocation (packing.hpp:311), schedule (scheduler.hpp:79),
brute_force_oracle (packing_oracle.hpp:78), Simulator (simulator.hpp:202).
"""
import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "_ref", "libwarmsim_ref.so")
_lib = None

ERRORS = ["InsufficientMemory", "PoolExhausted", "Infeasible", "Pinned", "NotFound", "OverlapMove",
          "DestinationOccupied", "OrderingError", "InstanceTooLarge", "InvalidArgument"]


def available():
    return os.path.exists(_PATH)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            raise RuntimeError(f"reference oracle not built: {_PATH} (run `make -C oracle`)")
        L = ctypes.CDLL(_PATH)
        c = ctypes
        sig = {
            "ref_murmur3": (None, [c.c_void_p, c.c_uint64, c.c_uint64, c.POINTER(c.c_uint64)]),
            "ref_fingerprint": (c.c_char_p, [c.c_char_p, c.c_char_p, c.POINTER(c.c_int64), c.c_int, c.c_int]),
            "ref_default_catalog": (c.c_char_p, []),
            "ref_make_model": (c.c_char_p, [c.c_char_p, c.c_uint64, c.c_int, c.c_uint64]),
            "ref_stats_create": (c.c_int, [c.c_double]),
            "ref_stats_record_request": (c.c_int, [c.c_int, c.c_char_p, c.c_double]),
            "ref_stats_record_eviction": (c.c_int, [c.c_int, c.c_char_p, c.c_double]),
            "ref_stats_set_load_bandwidth": (None, [c.c_int, c.c_char_p, c.c_double]),
            "ref_stats_miss_probability": (c.c_double, [c.c_int, c.c_char_p]),
            "ref_rng_create": (c.c_int, [c.c_uint64]),
            "ref_store_create": (c.c_int, [c.c_char_p, c.c_uint64, c.c_double, c.c_double, c.c_double]),
            "ref_store_clone": (c.c_int, [c.c_int]),
            "ref_destroy": (None, [c.c_int]),
            "ref_load_model": (c.c_char_p, [c.c_int, c.c_char_p, c.c_int, c.c_double, c.c_char_p]),
            "ref_load_model_timed": (c.c_char_p, [c.c_int, c.c_char_p, c.c_int, c.c_double, c.c_char_p]),
            "ref_end_instance": (None, [c.c_int, c.c_char_p]),
            "ref_evict_tensor": (c.c_int, [c.c_int, c.c_char_p]),
            "ref_evict_model": (None, [c.c_int, c.c_char_p]),
            "ref_move_tensor": (c.c_int, [c.c_int, c.c_char_p, c.c_uint64]),
            "ref_alloc_kv_region": (c.c_int, [c.c_int, c.c_uint64, c.c_uint64, c.POINTER(c.c_uint64)]),
            "ref_free_kv_region": (c.c_int, [c.c_int, c.c_uint64]),
            "ref_validate": (c.c_int, [c.c_int]),
            "ref_dump": (c.c_char_p, [c.c_int]),
            "ref_store_info": (c.c_char_p, [c.c_int]),
            "ref_lookup": (c.c_char_p, [c.c_int, c.c_char_p]),
            "ref_eviction_candidates": (c.c_char_p, [c.c_int, c.c_int, c.c_char_p]),
            "ref_kv_create": (c.c_int, [c.c_char_p, c.c_uint64, c.c_uint64]),
            "ref_kv_batch_allocate": (c.c_char_p, [c.c_int, c.c_int, c.c_int, c.POINTER(c.c_uint64),
                                                   c.POINTER(c.c_uint64), c.c_uint64]),
            "ref_kv_ensure_capacity": (c.c_char_p, [c.c_int, c.c_int, c.c_int, c.c_uint64, c.c_uint64]),
            "ref_kv_release_request": (c.c_int, [c.c_int, c.c_uint64]),
            "ref_kv_teardown": (None, [c.c_int, c.c_int]),
            "ref_kv_urgent_reclaim": (c.c_int, [c.c_int, c.c_int, c.c_int, c.c_uint64]),
            "ref_kv_table": (c.c_char_p, [c.c_int, c.c_uint64]),
            "ref_kv_state": (c.c_char_p, [c.c_int]),
            "ref_plan_allocation": (c.c_char_p, [c.c_char_p]),
            "ref_try_packing": (c.c_char_p, [c.POINTER(c.c_uint64), c.c_uint64, c.c_uint64, c.c_uint64, c.c_int]),
            "ref_brute_force_oracle": (c.c_char_p, [c.c_char_p]),
            "ref_schedule": (c.c_char_p, [c.c_char_p]),
            "ref_sample_lengths": (c.c_char_p, [c.c_uint64, c.c_char_p, c.c_uint64]),
            "ref_simulate": (c.c_char_p, [c.c_char_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _j(b):
    return json.loads(b.decode())


def _e(b):
    return b if isinstance(b, bytes) else str(b).encode()


def murmur3(data: bytes, seed=0):
    out = (ctypes.c_uint64 * 2)()
    buf = ctypes.create_string_buffer(data, len(data))
    lib().ref_murmur3(ctypes.cast(buf, ctypes.c_void_p), len(data), seed, out)
    return out[0], out[1]


def fingerprint(model_id, name, shape, etype=1):
    arr = (ctypes.c_int64 * len(shape))(*shape)
    return json.loads(lib().ref_fingerprint(_e(model_id), _e(name), arr, len(shape), etype).decode())


def default_catalog():
    return _j(lib().ref_default_catalog())


def make_model(model_id, total, layers, bpt):
    return _j(lib().ref_make_model(_e(model_id), total, layers, bpt))


def sample_lengths(seed, dataset, n):
    return _j(lib().ref_sample_lengths(seed, _e(dataset), n))


def plan_allocation(request: dict):
    return _j(lib().ref_plan_allocation(_e(json.dumps(request))))


def try_packing(sizes, c1, c2, strictness=0):
    arr = (ctypes.c_uint64 * max(1, len(sizes)))(*sizes)
    return _j(lib().ref_try_packing(arr, len(sizes), c1, c2, strictness))


def brute_force_oracle(instance: dict):
    return _j(lib().ref_brute_force_oracle(_e(json.dumps(instance))))


def schedule(request: dict):
    return _j(lib().ref_schedule(_e(json.dumps(request))))


def simulate(request: dict):
    return _j(lib().ref_simulate(_e(json.dumps(request))))


class _Handle:
    h = 0

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.ref_destroy(self.h)
        except Exception:
            pass


class Rng(_Handle):
    def __init__(self, seed):
        self.h = lib().ref_rng_create(seed)


class ModelStatsTable(_Handle):
    def __init__(self, decay=0.95):
        self.h = lib().ref_stats_create(decay)

    def record_request(self, model_id, t):
        return lib().ref_stats_record_request(self.h, _e(model_id), t)

    def record_eviction(self, model_id, t):
        return lib().ref_stats_record_eviction(self.h, _e(model_id), t)

    def set_load_bandwidth(self, model_id, b):
        lib().ref_stats_set_load_bandwidth(self.h, _e(model_id), b)

    def miss_probability(self, model_id):
        return lib().ref_stats_miss_probability(self.h, _e(model_id))


def _policy(merge=0, strictness=0, random_eviction=False, rng=None):
    return json.dumps({"merge": merge, "strictness": strictness, "random_eviction": random_eviction,
                       "rng": rng.h if rng is not None else 0}).encode()


class ReuseStore(_Handle):
    def __init__(self, pool_size, gpu_id="gpu0", pcie=55e9, intra=3000e9, store=12e9, _h=None):
        self.h = _h if _h is not None else lib().ref_store_create(_e(gpu_id), pool_size, pcie, intra, store)

    def clone(self):
        return ReuseStore(0, _h=lib().ref_store_clone(self.h))

    def load_model(self, model, stats, clock, merge=0, strictness=0, random_eviction=False, rng=None, timed=False):
        f = lib().ref_load_model_timed if timed else lib().ref_load_model
        return _j(f(self.h, _e(json.dumps(model)), stats.h, clock,
                    _policy(merge, strictness, random_eviction, rng)))

    def end_instance(self, model_id):
        lib().ref_end_instance(self.h, _e(model_id))

    def evict_tensor(self, hexid):
        return lib().ref_evict_tensor(self.h, _e(hexid))

    def evict_model(self, model_id):
        lib().ref_evict_model(self.h, _e(model_id))

    def move_tensor(self, hexid, to):
        return lib().ref_move_tensor(self.h, _e(hexid), to)

    def alloc_kv_region(self, size, block_id):
        off = ctypes.c_uint64(0)
        rc = lib().ref_alloc_kv_region(self.h, size, block_id, ctypes.byref(off))
        return rc, off.value

    def free_kv_region(self, off):
        return lib().ref_free_kv_region(self.h, off)

    def validate(self):
        return lib().ref_validate(self.h)

    def dump(self):
        return _j(lib().ref_dump(self.h))

    def info(self):
        return _j(lib().ref_store_info(self.h))

    def lookup(self, model):
        return _j(lib().ref_lookup(self.h, _e(json.dumps(model))))

    def eviction_candidates(self, stats, exclude):
        return _j(lib().ref_eviction_candidates(self.h, stats.h, _e(exclude)))


class KvEngine(_Handle):
    def __init__(self, model_id, block_size_tokens, bytes_per_token):
        self.h = lib().ref_kv_create(_e(model_id), block_size_tokens, bytes_per_token)

    def batch_allocate(self, store, stats, requests):
        n = len(requests)
        rids = (ctypes.c_uint64 * max(1, n))(*[r for r, _ in requests])
        toks = (ctypes.c_uint64 * max(1, n))(*[t for _, t in requests])
        return _j(lib().ref_kv_batch_allocate(self.h, store.h, stats.h, rids, toks, n))

    def ensure_capacity(self, store, stats, rid, tokens):
        return _j(lib().ref_kv_ensure_capacity(self.h, store.h, stats.h, rid, tokens))

    def release_request(self, rid):
        return lib().ref_kv_release_request(self.h, rid)

    def instance_teardown(self, store):
        lib().ref_kv_teardown(self.h, store.h)

    def urgent_reclaim(self, store, stats, blocks):
        return lib().ref_kv_urgent_reclaim(self.h, store.h, stats.h, blocks)

    def table(self, rid):
        return _j(lib().ref_kv_table(self.h, rid))

    def state(self):
        return _j(lib().ref_kv_state(self.h))
