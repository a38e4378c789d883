"""Python mirror of the reference's pool / loader API over libtangram.so.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/warmsim):

* ``Result`` / ``Error``      — types.hpp:155-217
* ``TensorId``, ``TensorSpec``, ``ModelSpec``, ``GpuSpec`` — types.hpp:46-60, model.hpp:17-45
* ``ModelStatsTable``        — model.hpp:70-133
* ``ReuseStore``             — reuse_store.hpp:50-345 (bytes move on the B200 arena)
* ``KvEngine``               — kv_engine.hpp:43-239 (tables live in HBM)
* ``LoadPolicy``             — reuse_store.hpp:43-48
* ``make_model`` / ``default_catalog`` — catalog.hpp:37-90
* ``schedule`` / ``estimate_load_time`` — scheduler.hpp:41-120

``ReuseStore(spec, device=0)`` owns a device-resident arena on that GPU; every
load moves real bytes (H2D / relocation / peer pull kernels) and fingerprints
them.  ``device=None`` gives a control-plane-only store that takes the same
decisions but has no arena (used to test the host logic without a GPU and to
model several GPUs in one process); it never pretends to move bytes.
"""
import ctypes as C
import enum
import json
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from . import _native as N

lib = N.lib


class Error(enum.IntEnum):
    InsufficientMemory = 0
    PoolExhausted = 1
    Infeasible = 2
    Pinned = 3
    NotFound = 4
    OverlapMove = 5
    DestinationOccupied = 6
    OrderingError = 7
    InstanceTooLarge = 8
    InvalidArgument = 9


class Result:
    """Result<T> (types.hpp:197-213)."""

    __slots__ = ("_v", "_e")

    def __init__(self, value=None, error: Optional[Error] = None):
        self._v, self._e = value, error

    def ok(self):
        return self._e is None

    __bool__ = ok

    def value(self):
        if self._e is not None:
            raise ValueError(f"Result holds error {self._e.name}")
        return self._v

    def error(self):
        return self._e

    def __repr__(self):
        return f"Result(ok={self.ok()}, {'value' if self.ok() else 'error'}={self._v if self.ok() else self._e})"


def _result(rc, value=None, where=""):
    N.check_runtime(rc, where)
    return Result(value) if rc == 0 else Result(error=Error(rc - 1))


@dataclass(frozen=True, order=True)
class TensorId:
    hi: int = 0
    lo: int = 0

    def hex(self):
        return f"{self.hi:016x}{self.lo:016x}"

    @staticmethod
    def from_hex(h):
        return TensorId(int(h[:16], 16), int(h[16:32], 16))

    def c(self):
        return N.TensorIdC(self.hi, self.lo)


@dataclass
class TensorSpec:
    id: TensorId
    model_id: str
    name: str
    size: int


class ModelLocation(enum.IntEnum):
    ModelCache = 0
    ModelStore = 1


@dataclass
class ModelSpec:
    model_id: str
    tensors: List[TensorSpec] = field(default_factory=list)
    total_size: int = 0
    latency_sensitivity: float = 1.0
    location: ModelLocation = ModelLocation.ModelCache
    bytes_per_token: int = 0

    def c(self):
        """tg_model_spec view (cached; rebuild if the tensor list changes)."""
        key = (len(self.tensors), self.total_size, self.latency_sensitivity, int(self.location))
        if getattr(self, "_ckey", None) != key:
            self._names = [t.name.encode() for t in self.tensors]
            self._mids = [t.model_id.encode() for t in self.tensors]
            arr = (N.TensorSpecC * max(1, len(self.tensors)))()
            for i, t in enumerate(self.tensors):
                arr[i] = N.TensorSpecC(t.id.c(), self._names[i], t.size, self._mids[i])
            self._arr = arr
            self._mid = self.model_id.encode()
            self._spec = N.ModelSpecC(self._mid, arr, len(self.tensors), self.total_size,
                                      self.latency_sensitivity, int(self.location), self.bytes_per_token)
            self._ckey = key
        return self._spec

    def to_json(self):
        return {"model_id": self.model_id, "total_size": self.total_size,
                "latency_sensitivity": self.latency_sensitivity,
                "location": "model_store" if self.location else "model_cache",
                "bytes_per_token": self.bytes_per_token,
                "tensors": [{"id": t.id.hex(), "name": t.name, "size": t.size, "model_id": t.model_id}
                            for t in self.tensors]}


@dataclass
class GpuSpec:
    gpu_id: str = "gpu0"
    pool_size: int = 0
    pcie_bandwidth: float = 55e9
    intra_copy_bandwidth: float = 3000e9
    store_bandwidth: float = 12e9


def _model_from_handle(h):
    spec = N.ModelSpecC()
    N.check_runtime(lib.tg_model_view(h, C.byref(spec)), "tg_model_view")
    ts = []
    for i in range(spec.n_tensors):
        t = spec.tensors[i]
        ts.append(TensorSpec(TensorId(t.id.hi, t.id.lo), t.model_id.decode(), t.name.decode(), t.size))
    m = ModelSpec(spec.model_id.decode(), ts, spec.total_size, spec.latency_sensitivity,
                  ModelLocation(spec.location), spec.bytes_per_token)
    lib.tg_model_destroy(h)
    return m


def make_model(model_id, total_size, layers, bytes_per_token, location=ModelLocation.ModelCache,
               latency_sensitivity=1.0) -> ModelSpec:
    """catalog.hpp:37-67."""
    h = C.c_void_p()
    N.check_runtime(lib.tg_model_make(model_id.encode(), total_size, layers, bytes_per_token, int(location),
                                      latency_sensitivity, C.byref(h)), "tg_model_make")
    return _model_from_handle(h)


def default_catalog() -> List[ModelSpec]:
    """catalog.hpp:72-90."""
    out = []
    for i in range(lib.tg_model_catalog_size()):
        h = C.c_void_p()
        N.check_runtime(lib.tg_model_default_catalog(i, C.byref(h)), "tg_model_default_catalog")
        out.append(_model_from_handle(h))
    return out


def shard_model(model: ModelSpec, rank: int, world: int) -> ModelSpec:
    """Tensor-parallel shard ``rank`` of ``world``; same rule as tg_model_shard."""
    suffix = f"#tp{world}.{rank}"
    ts = []
    for t in model.tensors:
        chunk = (t.size + world - 1) // world
        b, e = min(t.size, rank * chunk), min(t.size, (rank + 1) * chunk)
        if e <= b:
            continue
        name = t.name + suffix
        tid = tensor_key(model.model_id + suffix, name, [(e - b) // 2])
        lib.tg_lineage_register(tid.c(), t.id.c(), b, e - b)  # shard = bytes [b, e) of t
        ts.append(TensorSpec(tid, model.model_id + suffix, name, e - b))
    ts.sort(key=lambda t: t.name)
    return ModelSpec(model.model_id + suffix, ts, sum(t.size for t in ts), model.latency_sensitivity,
                     model.location, model.bytes_per_token // world)


def lineage(tid: TensorId):
    """(parent TensorId, begin, size) if `tid` is a shard of another tensor, else None."""
    p, b, n = N.TensorIdC(), C.c_uint64(), C.c_uint64()
    if lib.tg_lineage_get(tid.c(), C.byref(p), C.byref(b), C.byref(n)) != 0:
        return None
    return TensorId(p.hi, p.lo), b.value, n.value


def failpoint(name: str, nth: int = 1):
    """Arm a test failpoint (tg_failpoint): its nth hit from now fails; nth <= 0 disarms."""
    N.check_runtime(lib.tg_failpoint(name.encode(), nth), "tg_failpoint")


def tensor_key(model_id, name, shape, dtype=1) -> TensorId:
    """fingerprint(model, name, shape, etype) (types.hpp:131-146); dtype 1 = f16."""
    arr = (C.c_int64 * max(1, len(shape)))(*shape)
    out = N.TensorIdC()
    N.check_runtime(lib.tg_tensor_key(model_id.encode(), name.encode(), arr, len(shape), dtype, C.byref(out)))
    return TensorId(out.hi, out.lo)


def murmur3_x64_128(data: bytes, seed=0) -> Tuple[int, int]:
    buf = C.create_string_buffer(bytes(data), len(data))
    out = N.DigestC()
    lib.tg_murmur3_x64_128(C.cast(buf, C.c_void_p), len(data), seed, C.byref(out))
    return out.hi, out.lo


class ModelStatsTable:
    """model.hpp:70-133."""

    def __init__(self, decay=0.95):
        self._h = C.c_void_p()
        lib.tg_stats_create(decay, C.byref(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.tg_stats_destroy(self._h)
            self._h = None

    def record_request(self, model_id, t) -> Result:
        return _result(lib.tg_stats_record_request(self._h, model_id.encode(), t))

    def record_eviction(self, model_id, t) -> Result:
        return _result(lib.tg_stats_record_eviction(self._h, model_id.encode(), t))

    def set_load_bandwidth(self, model_id, b):
        lib.tg_stats_set_load_bandwidth(self._h, model_id.encode(), b)

    def miss_probability(self, model_id):
        return lib.tg_stats_miss_probability(self._h, model_id.encode())


class Rng:
    """rng.hpp:18-73 (mt19937_64 stream)."""

    def __init__(self, seed):
        self._h = C.c_void_p()
        lib.tg_rng_create(seed, C.byref(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.tg_rng_destroy(self._h)
            self._h = None

    def uniform_below(self, n):
        return lib.tg_rng_uniform_below(self._h, n)


class MergePolicy(enum.IntEnum):
    PartitionedGain = 0
    GlobalMerge = 1


class PackingStrictness(enum.IntEnum):
    Functional = 0
    LiteralGuard = 1


LOAD_VERIFY_REUSE, LOAD_FINGERPRINT_NEW, LOAD_PEER, LOAD_FUSED, LOAD_ASYNC = 1, 2, 4, 8, 16
LOAD_EXPLICIT = 0x80000000  # flags taken literally (LOAD_EXPLICIT alone: no optional work)


@dataclass
class LoadPolicy:
    merge: MergePolicy = MergePolicy.PartitionedGain
    strictness: PackingStrictness = PackingStrictness.Functional
    random_eviction: bool = False
    rng: Optional[Rng] = None
    flags: int = LOAD_VERIFY_REUSE | LOAD_FINGERPRINT_NEW | LOAD_FUSED

    def c(self):
        return N.LoadPolicyC(int(self.merge), int(self.strictness), int(self.random_eviction),
                             self.rng._h if self.rng is not None else None, self.flags)


@dataclass
class EvictionCandidate:
    tensor: TensorId
    size: int
    cost: float
    last_access: float
    model_id: str


@dataclass
class Relocation:
    tensor: TensorId
    from_: int
    to: int
    size: int
    wave: int = 0


@dataclass
class Placement:
    tensor: TensorId
    offset: int
    size: int
    source: int = 0  # 0 host/PCIe, 1 peer/NVLink, 2 HBM source, 3 re-shard pieces from peer shards


@dataclass
class AllocationPlan:
    evictions: List[EvictionCandidate]
    relocations: List[Relocation]
    placements: List[Placement]
    total_eviction_cost: float
    total_merge_cost: int
    pgp_merge_cost: int
    initial_merge_cost: int
    fallback_evictions: int


@dataclass
class LoadOutcome:
    """reuse_store.hpp:34-41 plus the measured data plane."""
    hit_tensors: List[TensorId]
    missed_tensors: List[TensorId]
    bytes_transferred: int
    bytes_merged: int
    eviction_cost_total: float
    plan: AllocationPlan
    waves: int = 0
    pcie_bytes: int = 0
    peer_bytes: int = 0
    device_src_bytes: int = 0
    fingerprint_bytes: int = 0
    repaired_bytes: int = 0
    verify_mismatches: int = 0
    expected_mismatches: int = 0
    timings: dict = field(default_factory=dict)
    digests: List[Tuple[int, int]] = field(default_factory=list)
    suspect_tensors: int = 0


REGION_KIND = {0: "free", 1: "tensor", 2: "kv_block"}


class ReuseStore:
    """reuse_store.hpp:50-345 on a B200 arena.  ``device=None``: control plane only."""

    def __init__(self, spec: GpuSpec, device: Optional[int] = 0):
        self.spec = spec
        self._h = C.c_void_p()
        g = N.GpuSpecC(spec.gpu_id.encode(), spec.pool_size, spec.pcie_bandwidth, spec.intra_copy_bandwidth,
                       spec.store_bandwidth)
        N.check_runtime(lib.tg_pool_create(C.byref(g), -1 if device is None else device, C.byref(self._h)),
                        "tg_pool_create")
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib.tg_pool_destroy(self._h)
            self._h = None

    __del__ = close

    # -- value semantics (reuse_store.hpp:336-344)
    def clone(self) -> "ReuseStore":
        """Independent control-plane copy of this store's metadata (tg_pool_clone)."""
        c = ReuseStore.__new__(ReuseStore)
        c.spec, c.device, c._h = self.spec, None, C.c_void_p()
        N.check_runtime(lib.tg_pool_clone(self._h, C.byref(c._h)), "tg_pool_clone")
        return c

    def assign(self, other: "ReuseStore"):
        """Take other's metadata; tensors not already held here at the same
        offset become suspect (tg_pool_assign)."""
        N.check_runtime(lib.tg_pool_assign(self._h, other._h), "tg_pool_assign")

    def tensor_map(self) -> dict:
        """TensorId -> {offset, size, model, last_access, pinned, suspect} (tensor_map(), reuse_store.hpp:66)."""
        n = C.c_uint64()
        lib.tg_pool_tensors(self._h, None, 0, C.byref(n))
        buf = (N.TensorEntryC * max(1, n.value))()
        N.check_runtime(lib.tg_pool_tensors(self._h, buf, n.value, C.byref(n)), "tg_pool_tensors")
        return {TensorId(e.id.hi, e.id.lo): {"offset": e.offset, "size": e.size, "model": e.model_id.decode(),
                                             "last_access": e.last_access, "pinned": bool(e.pinned),
                                             "suspect": bool(e.suspect)} for e in buf[:n.value]}

    # -- accessors (reuse_store.hpp:56-74)
    def info(self):
        i = N.PoolInfoC()
        lib.tg_pool_info_get(self._h, C.byref(i))
        return {f: getattr(i, f) for f, _ in N.PoolInfoC._fields_}

    def pool_size(self): return self.info()["pool_size"]
    def free_bytes(self): return self.info()["free_bytes"]
    def kv_bytes(self): return self.info()["kv_bytes"]
    def pinned_tensor_bytes(self): return self.info()["pinned_tensor_bytes"]
    def pinned_bytes(self): return self.info()["pinned_bytes"]
    def reusable_bytes(self): return self.info()["reusable_bytes"]
    def bytes_merged_total(self): return self.info()["bytes_merged_total"]
    def bytes_transferred_total(self): return self.info()["bytes_transferred_total"]
    def evictions_total(self): return self.info()["evictions_total"]

    def stream(self):
        s = C.c_void_p()
        N.check_runtime(lib.tg_pool_stream(self._h, C.byref(s)), "tg_pool_stream")
        return s.value

    def set_model_alpha(self, model_id, alpha):
        lib.tg_set_model_alpha(self._h, model_id.encode(), alpha)

    def load_model(self, model: ModelSpec, stats: ModelStatsTable, clock: float,
                   policy: Optional[LoadPolicy] = None, details=True) -> Result:
        """load_model (reuse_store.hpp:120-174)."""
        pol = (policy or LoadPolicy()).c()
        out = N.LoadOutcomeC()
        rc = lib.tg_load_model(self._h, C.byref(model.c()), stats._h, clock, C.byref(pol), C.byref(out))
        if rc >= 100:
            # after the commit the outcome still describes the decision (see tangram.h)
            committed = out.n_hits + out.n_misses > 0
            raise N.TangramRuntimeError(rc, "tg_load_model", self._outcome(out, details) if committed else None)
        if rc:
            return Result(error=Error(rc - 1))
        return Result(self._outcome(out, details))

    def sync(self, details=False):
        """Finish an asynchronous load (LoadPolicy(flags=... | LOAD_ASYNC)) still
        in flight: its completed outcome (digests verified, timings), or None
        when none was pending.  Raises TangramRuntimeError if it failed."""
        out = N.LoadOutcomeC()
        rc = lib.tg_pool_sync(self._h, C.byref(out))
        if rc >= 100:
            raise N.TangramRuntimeError(rc, "tg_pool_sync", None)
        if out.n_hits + out.n_misses == 0:
            return None
        return self._outcome(out, details)

    def _outcome(self, o, details):
        h = self._h
        ids = lambda f, n: [TensorId(x.hi, x.lo) for x in _fetch(f, h, N.TensorIdC, n)]
        hits = ids(lib.tg_last_hits, o.n_hits) if details else []
        misses = ids(lib.tg_last_misses, o.n_misses) if details else []
        evs = [EvictionCandidate(TensorId(e.tensor.hi, e.tensor.lo), e.size, e.cost, e.last_access,
                                 e.model_id.decode()) for e in _fetch(lib.tg_last_evictions, h, N.EvictionC,
                                                                      o.n_evictions)] if details else []
        rels = [Relocation(TensorId(r.tensor.hi, r.tensor.lo), r.from_, r.to, r.size, r.wave)
                for r in _fetch(lib.tg_last_relocations, h, N.RelocationC, o.n_relocations)] if details else []
        pls = [Placement(TensorId(p.tensor.hi, p.tensor.lo), p.offset, p.size, p.source)
               for p in _fetch(lib.tg_last_placements, h, N.PlacementC, o.n_placements)] if details else []
        nd = lib.tg_last_digests(h, None, 0)
        digs = [(d.hi, d.lo) for d in _fetch(lib.tg_last_digests, h, N.DigestC, nd)] if details else []
        plan = AllocationPlan(evs, rels, pls, o.total_eviction_cost, o.total_merge_cost, o.pgp_merge_cost,
                              o.initial_merge_cost, o.fallback_evictions)
        t = {k: getattr(o, k) for k in ("plan_us", "total_ms", "relocate_ms", "h2d_ms", "peer_ms", "fp_kernel_ms",
                                        "fp_reuse_ms", "fp_reuse_max_ms", "host_issue_us", "host_wait_us",
                                        "host_total_us", "kernel_end_ms", "gated_h2d_start_ms")}
        return LoadOutcome(hits, misses, o.bytes_transferred, o.bytes_merged, o.eviction_cost_total, plan,
                           o.n_waves, o.pcie_bytes, o.peer_bytes, o.device_src_bytes, o.fingerprint_bytes, o.repaired_bytes,
                           o.verify_mismatches, o.expected_mismatches, t, digs, o.suspect_tensors)

    def end_instance(self, model_id):
        lib.tg_end_instance(self._h, model_id.encode())

    def evict_tensor(self, tid: TensorId) -> Result:
        return _result(lib.tg_evict_tensor(self._h, tid.c()))

    def evict_model(self, model_id):
        lib.tg_evict_model(self._h, model_id.encode())

    def move_tensor(self, tid: TensorId, new_offset) -> Result:
        return _result(lib.tg_move_tensor(self._h, tid.c(), new_offset), None, "tg_move_tensor")

    def alloc_kv_region(self, size, block_id) -> Result:
        off = C.c_uint64()
        rc = lib.tg_alloc_kv_region(self._h, size, block_id, C.byref(off))
        return _result(rc, off.value)

    def free_kv_region(self, offset) -> Result:
        return _result(lib.tg_free_kv_region(self._h, offset))

    def lookup(self, model: ModelSpec):
        mask = (C.c_uint8 * max(1, len(model.tensors)))()
        lib.tg_lookup(self._h, C.byref(model.c()), mask, None)
        hits = [t.id for i, t in enumerate(model.tensors) if mask[i]]
        misses = [t for i, t in enumerate(model.tensors) if not mask[i]]
        return hits, misses

    def reuse_size(self, model: ModelSpec) -> int:
        v = C.c_uint64()
        lib.tg_reuse_size(self._h, C.byref(model.c()), C.byref(v))
        return v.value

    def peer_reuse_size(self, model: ModelSpec) -> int:
        v = C.c_uint64()
        lib.tg_peer_reuse_size(self._h, C.byref(model.c()), C.byref(v))
        return v.value

    def eviction_candidates(self, stats: ModelStatsTable, exclude_model: str):
        n = C.c_uint32()
        lib.tg_eviction_candidates(self._h, stats._h, exclude_model.encode(), None, 0, C.byref(n))
        buf = (N.EvictionC * max(1, n.value))()
        lib.tg_eviction_candidates(self._h, stats._h, exclude_model.encode(), buf, n.value, C.byref(n))
        return [EvictionCandidate(TensorId(e.tensor.hi, e.tensor.lo), e.size, e.cost, e.last_access,
                                  e.model_id.decode()) for e in buf[:n.value]]

    def validate(self) -> Result:
        return _result(lib.tg_validate(self._h))

    def dump(self) -> dict:
        need = C.c_uint64()
        lib.tg_dump(self._h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        N.check_runtime(lib.tg_dump(self._h, buf, need.value, C.byref(need)), "tg_dump")
        return json.loads(buf.value.decode())

    def regions(self):
        n = C.c_uint64()
        lib.tg_regions(self._h, None, 0, C.byref(n))
        buf = (N.RegionC * max(1, n.value))()
        lib.tg_regions(self._h, buf, n.value, C.byref(n))
        return [(r.offset, r.size, REGION_KIND[r.kind], TensorId(r.tensor.hi, r.tensor.lo), r.block_id)
                for r in buf[:n.value]]

    def tensor_info(self, tid: TensorId):
        i = N.TensorInfoC()
        rc = lib.tg_tensor_info_get(self._h, tid.c(), C.byref(i))
        if rc:
            return None
        return {"offset": i.offset, "size": i.size, "last_access": i.last_access, "pinned": bool(i.pinned),
                "has_digest": bool(i.has_digest), "digest": (i.digest.hi, i.digest.lo),
                "device_ptr": i.device_ptr, "suspect": bool(i.suspect)}

    # -- device tensor index ------------------------------------------
    def index_image(self):
        """(capacity, [slot dicts]) of the open-addressing table the device holds
        (built on the host; available on control-plane pools too)."""
        cap = C.c_uint64()
        N.check_runtime(lib.tg_pool_index_image(self._h, None, 0, C.byref(cap)), "tg_pool_index_image")
        buf = (N.IndexSlotC * cap.value)()
        N.check_runtime(lib.tg_pool_index_image(self._h, buf, cap.value, C.byref(cap)), "tg_pool_index_image")
        return cap.value, [{"key": (b.key_hi, b.key_lo), "offset": b.offset, "size": b.size,
                            "last_access": b.last_access, "model": b.model, "flags": b.flags} for b in buf]

    def device_index(self):
        """(device pointer, capacity) of the published table (tg_index_slot[capacity])."""
        ptr, cap = C.c_void_p(), C.c_uint64()
        N.check_runtime(lib.tg_pool_device_index(self._h, C.byref(ptr), C.byref(cap)), "tg_pool_device_index")
        return ptr.value, cap.value

    def index_lookup(self, ids):
        """Device lookups (K6): [None | {"offset", "size", "pinned"}] per TensorId."""
        n = len(ids)
        keys = (N.TensorIdC * max(1, n))(*[t.c() for t in ids])
        out = (N.IndexHitC * max(1, n))()
        N.check_runtime(lib.tg_index_lookup(self._h, keys, n, out), "tg_index_lookup")
        return [{"offset": h.offset, "size": h.size, "pinned": bool(h.flags & 2)} if h.found else None
                for h in out[:n]]

    def fingerprint_tensor(self, tid: TensorId):
        d = N.DigestC()
        rc = lib.tg_fingerprint_tensor(self._h, tid.c(), C.byref(d))
        N.check_runtime(rc, "tg_fingerprint_tensor")
        return (d.hi, d.lo) if rc == 0 else None

    def add_peer(self, other: "ReuseStore"):
        N.check_runtime(lib.tg_pool_add_peer(self._h, other._h), "tg_pool_add_peer")

    # -- peers in other processes (CUDA IPC + index exchange) ----------------------
    def export_ipc(self) -> bytes:
        h = (C.c_uint8 * 64)()
        N.check_runtime(lib.tg_pool_export_ipc(self._h, h), "tg_pool_export_ipc")
        return bytes(h)

    def index(self):
        """[(TensorId, offset, size, digest)] of fingerprinted residents."""
        n = C.c_uint64()
        lib.tg_pool_index(self._h, None, 0, C.byref(n))
        buf = (N.IndexEntryC * max(1, n.value))()
        lib.tg_pool_index(self._h, buf, n.value, C.byref(n))
        return [(TensorId(e.id.hi, e.id.lo), e.offset, e.size, (e.digest.hi, e.digest.lo)) for e in buf[:n.value]]

    @staticmethod
    def _index_c(entries):
        arr = (N.IndexEntryC * max(1, len(entries)))()
        for i, (tid, off, size, dig) in enumerate(entries):
            arr[i] = N.IndexEntryC(tid.c(), off, size, N.DigestC(*dig))
        return arr

    def attach_remote(self, handle: bytes, entries) -> int:
        hb = (C.c_uint8 * 64)(*handle)
        pid = C.c_int32()
        N.check_runtime(lib.tg_pool_attach_remote(self._h, hb, self._index_c(entries), len(entries),
                                                  C.byref(pid)), "tg_pool_attach_remote")
        return pid.value

    def update_remote(self, peer_id, entries):
        N.check_runtime(lib.tg_pool_update_remote(self._h, peer_id, self._index_c(entries), len(entries)),
                        "tg_pool_update_remote")

    def snapshot(self):
        s = C.c_void_p()
        N.check_runtime(lib.tg_pool_snapshot(self._h, C.byref(s)), "tg_pool_snapshot")
        return _Snapshot(s)

    def restore(self, snap):
        N.check_runtime(lib.tg_pool_restore(self._h, snap._h), "tg_pool_restore")


class _Snapshot:
    def __init__(self, h):
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.tg_snapshot_destroy(self._h)
            self._h = None


def _fetch(fn, h, ctype, n):
    if n == 0:
        return []
    buf = (ctype * n)()
    fn(h, buf, n)
    return list(buf)


@dataclass
class KvAllocStats:
    pool_invocations: int
    alloc_batches: int
    blocks_from_free_list: int
    blocks_from_pool: int
    reclaim_events: int


@dataclass
class KvBlockTable:
    request_id: int
    block_size_tokens: int
    lbn_to_pbn: dict
    token_count: int


class KvEngine:
    """kv_engine.hpp:43-239; block tables and the free list live in HBM."""

    def __init__(self, model_id, block_size_tokens, bytes_per_token, _h=None):
        self.model_id = model_id
        self._bs = block_size_tokens
        self._h = C.c_void_p(_h) if _h is not None else C.c_void_p()
        if _h is None:
            N.check_runtime(lib.tg_kv_create(model_id.encode(), block_size_tokens, bytes_per_token,
                                             C.byref(self._h)), "tg_kv_create")

    def __del__(self):
        if getattr(self, "_h", None):
            lib.tg_kv_destroy(self._h)
            self._h = None

    def clone(self):
        h = C.c_void_p()
        N.check_runtime(lib.tg_kv_clone(self._h, C.byref(h)), "tg_kv_clone")
        return KvEngine(self.model_id, self._bs, 0, _h=h.value)

    @staticmethod
    def blocks_for(tokens, block_size):
        return (tokens + block_size - 1) // block_size

    def ensure_capacity(self, store: ReuseStore, stats: ModelStatsTable, request_id, tokens,
                        want_pbns=True) -> Result:
        have = self._blocks(request_id)
        cap = max(0, self.blocks_for(tokens, self._bs) - have)
        buf = (C.c_uint64 * max(1, cap))()
        n = C.c_uint64()
        rc = lib.tg_kv_ensure_capacity(self._h, store._h, stats._h, request_id, tokens,
                                       buf if (want_pbns and store.device is not None) else None, cap, C.byref(n))
        N.check_runtime(rc, "tg_kv_ensure_capacity")
        if rc:
            return Result(error=Error(rc - 1))
        return Result(list(buf[:n.value]) if (want_pbns and store.device is not None) else n.value)

    def batch_allocate(self, store: ReuseStore, stats: ModelStatsTable, requests: Sequence[Tuple[int, int]],
                       want_pbns=True) -> Result:
        n = len(requests)
        rids = (C.c_uint64 * max(1, n))(*[r for r, _ in requests])
        toks = (C.c_uint64 * max(1, n))(*[t for _, t in requests])
        counts = (C.c_uint64 * max(1, n))()
        cap = sum(self.blocks_for(t, self._bs) for _, t in requests)
        pb = (C.c_uint64 * max(1, cap))() if (want_pbns and store.device is not None) else None
        total = C.c_uint64()
        rc = lib.tg_kv_batch_allocate(self._h, store._h, stats._h, rids, toks, n, counts, pb, cap, C.byref(total))
        N.check_runtime(rc, "tg_kv_batch_allocate")
        if rc:
            return Result(error=Error(rc - 1))
        if pb is None:
            return Result([counts[i] for i in range(n)])
        out, k = [], 0
        for i in range(n):
            out.append(list(pb[k:k + counts[i]]))
            k += counts[i]
        return Result(out)

    def release_request(self, request_id) -> Result:
        return _result(lib.tg_kv_release_request(self._h, request_id), None, "tg_kv_release_request")

    def instance_teardown(self, store: ReuseStore):
        N.check_runtime(lib.tg_kv_teardown(self._h, store._h), "tg_kv_teardown")

    def urgent_reclaim(self, store: ReuseStore, stats: ModelStatsTable, needed_blocks) -> Result:
        return _result(lib.tg_kv_urgent_reclaim(self._h, store._h, stats._h, needed_blocks), None,
                       "tg_kv_urgent_reclaim")

    def _blocks(self, rid):
        n = C.c_uint64()
        rc = lib.tg_kv_table(self._h, rid, None, 0, C.byref(n), None)
        return n.value if rc == 0 else 0

    def table(self, request_id) -> Optional[KvBlockTable]:
        n, tok = C.c_uint64(), C.c_uint64()
        rc = lib.tg_kv_table(self._h, request_id, None, 0, C.byref(n), C.byref(tok))
        if rc:
            return None
        buf = (C.c_uint64 * max(1, n.value))()
        N.check_runtime(lib.tg_kv_table(self._h, request_id, buf, n.value, C.byref(n), C.byref(tok)), "tg_kv_table")
        return KvBlockTable(request_id, self._bs, {i: buf[i] for i in range(n.value)}, tok.value)

    # ---- device-decided batches (K4D; include/tangram.h) ---------------------------
    def request_slot(self, request_id) -> int:
        """Table row of a known request (its LBN->PBN row in the device tables)."""
        s = C.c_uint32()
        N.check_runtime(lib.tg_kv_request_slot(self._h, request_id, C.byref(s)), "tg_kv_request_slot")
        return s.value

    def device_arm(self, store: ReuseStore, max_blocks_per_request, max_requests, max_batches):
        rc = lib.tg_kv_device_arm(self._h, store._h, max_blocks_per_request, max_requests, max_batches)
        N.check_runtime(rc, "tg_kv_device_arm")
        return Result(None) if rc == 0 else Result(error=Error(rc - 1))

    def batch_allocate_device(self, slots_ptr, tokens_ptr, n, stream=None):
        """Enqueue one batch: `slots_ptr`/`tokens_ptr` are device pointers to n
        u64 each (e.g. torch int64 tensors' data_ptr()); no host round trip."""
        N.check_runtime(lib.tg_kv_batch_allocate_device(self._h, C.c_void_p(slots_ptr), C.c_void_p(tokens_ptr), n,
                                                        C.c_void_p(stream) if stream else None),
                        "tg_kv_batch_allocate_device")

    def write_tokens(self, store: ReuseStore, slots_ptr, positions_ptr, buf_ptr, n, stream=None):
        """Paged-cache write through the block tables (device pointers; see tangram.h)."""
        N.check_runtime(lib.tg_kv_write_tokens(self._h, store._h, C.c_void_p(slots_ptr), C.c_void_p(positions_ptr),
                                               C.c_void_p(buf_ptr), n, C.c_void_p(stream) if stream else None),
                        "tg_kv_write_tokens")

    def read_tokens(self, store: ReuseStore, slots_ptr, positions_ptr, buf_ptr, n, stream=None):
        """Paged-cache gather through the block tables (device pointers)."""
        N.check_runtime(lib.tg_kv_read_tokens(self._h, store._h, C.c_void_p(slots_ptr), C.c_void_p(positions_ptr),
                                              C.c_void_p(buf_ptr), n, C.c_void_p(stream) if stream else None),
                        "tg_kv_read_tokens")

    def device_sync(self, store: ReuseStore, stats: ModelStatsTable) -> Result:
        """Fold the device's decisions into the host state; replay the batches
        the device left to the host.  Value: (applied, replayed) batch counts."""
        a, r = C.c_uint64(), C.c_uint64()
        rc = lib.tg_kv_device_sync(self._h, store._h, stats._h, C.byref(a), C.byref(r))
        N.check_runtime(rc, "tg_kv_device_sync")
        if rc:
            return Result(error=Error(rc - 1))
        return Result((a.value, r.value))

    def address_table(self) -> dict:
        n = C.c_uint64()
        lib.tg_kv_address_table(self._h, None, 0, C.byref(n))
        buf = (C.c_uint64 * max(1, 3 * n.value))()
        lib.tg_kv_address_table(self._h, buf, n.value, C.byref(n))
        return {buf[3 * i]: (buf[3 * i + 1], buf[3 * i + 2]) for i in range(n.value)}

    def _stats(self):
        s = N.KvStatsC()
        lib.tg_kv_stats_get(self._h, C.byref(s))
        return s

    def stats(self) -> KvAllocStats:
        s = self._stats()
        return KvAllocStats(s.pool_invocations, s.alloc_batches, s.blocks_from_free_list, s.blocks_from_pool,
                            s.reclaim_events)

    def free_list_size(self):
        return self._stats().free_list_size

    def active_requests(self):
        return self._stats().active_requests

    def block_bytes(self):
        return self._stats().block_bytes

    def token_faults(self) -> int:
        """Block-table consumer references outside the granted blocks so far."""
        n = C.c_uint64()
        N.check_runtime(lib.tg_kv_token_faults(self._h, C.byref(n)), "tg_kv_token_faults")
        return n.value

    def wait_tables(self, stream):
        """Make a CUDA stream wait for the table updates enqueued so far."""
        N.check_runtime(lib.tg_kv_wait_tables(self._h, C.c_void_p(stream)), "tg_kv_wait_tables")

    def reserve(self, store: ReuseStore, max_requests, max_blocks_per_request, max_blocks):
        """Pre-size the device tables so their pointers never move."""
        N.check_runtime(lib.tg_kv_reserve(self._h, store._h, max_requests, max_blocks_per_request, max_blocks),
                        "tg_kv_reserve")

    def device_tables(self):
        t, a = C.c_void_p(), C.c_void_p()
        s = C.c_uint64()
        N.check_runtime(lib.tg_kv_device_tables(self._h, C.byref(t), C.byref(s), C.byref(a)), "tg_kv_device_tables")
        return t.value, s.value, a.value


KIND_CODE = {"free": 0, "tensor": 1, "kv_block": 2}


def plan_allocation(regions, new_tensors: Sequence[TensorSpec], candidates: Sequence[EvictionCandidate] = (),
                    immovable: Sequence[TensorId] = (), strictness=0, merge=0, randomize_eviction=False) -> Result:
    """plan_allocation (packing.hpp:311-483) over an explicit region tiling.
    regions: [(offset, size, kind, TensorId|None, block_id)] with kind in
    {"free", "tensor", "kv_block"}."""
    R = (N.RegionC * max(1, len(regions)))()
    for i, (off, size, kind, tid, blk) in enumerate(regions):
        R[i] = N.RegionC(off, size, KIND_CODE[kind], (tid or TensorId()).c(), blk or 0)
    keep = [t.name.encode() for t in new_tensors], [t.model_id.encode() for t in new_tensors]
    T = (N.TensorSpecC * max(1, len(new_tensors)))()
    for i, t in enumerate(new_tensors):
        T[i] = N.TensorSpecC(t.id.c(), keep[0][i], t.size, keep[1][i])
    mids = [c.model_id.encode() for c in candidates]
    E = (N.EvictionC * max(1, len(candidates)))()
    for i, c in enumerate(candidates):
        E[i] = N.EvictionC(c.tensor.c(), c.size, c.cost, c.last_access, mids[i])
    I = (N.TensorIdC * max(1, len(immovable)))(*[t.c() for t in immovable])
    h = C.c_void_p()
    rc = lib.tg_plan_allocation(R, len(regions), T, len(new_tensors), E, len(candidates), I, len(immovable),
                                int(strictness), int(merge), int(randomize_eviction), C.byref(h))
    N.check_runtime(rc, "tg_plan_allocation")
    if rc:
        return Result(error=Error(rc - 1))
    try:
        ev = [EvictionCandidate(TensorId(e.tensor.hi, e.tensor.lo), e.size, e.cost, e.last_access,
                                e.model_id.decode()) for e in _fetch(lib.tg_plan_evictions, h,
                                                                     N.EvictionC, lib.tg_plan_evictions(h, None, 0))]
        rl = [Relocation(TensorId(r.tensor.hi, r.tensor.lo), r.from_, r.to, r.size)
              for r in _fetch(lib.tg_plan_relocations, h, N.RelocationC, lib.tg_plan_relocations(h, None, 0))]
        pl = [Placement(TensorId(p.tensor.hi, p.tensor.lo), p.offset, p.size)
              for p in _fetch(lib.tg_plan_placements, h, N.PlacementC, lib.tg_plan_placements(h, None, 0))]
        ec, tm, pgp, init, fb = C.c_double(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib.tg_plan_costs(h, C.byref(ec), C.byref(tm), C.byref(pgp), C.byref(init), C.byref(fb))
        return Result(AllocationPlan(ev, rl, pl, ec.value, tm.value, pgp.value, init.value, fb.value))
    finally:
        lib.tg_plan_destroy(h)


@dataclass
class GpuSnapshot:
    """scheduler.hpp:22-36 (+ nvlink_bandwidth for the peer term)."""
    gpu_id: str
    available: bool = True
    pool_size: int = 0
    free_bytes: int = 0
    reuse_size_by_model: dict = field(default_factory=dict)
    pcie_bandwidth: float = 55e9
    store_bandwidth: float = 12e9
    nvlink_bandwidth: float = 0.0
    peer_reuse_by_model: dict = field(default_factory=dict)

    def c(self):
        self._gid = self.gpu_id.encode()
        return N.GpuSnapshotC(self._gid, int(self.available), self.pool_size, self.free_bytes,
                              self.pcie_bandwidth, self.store_bandwidth, self.nvlink_bandwidth)


def estimate_load_time(model: ModelSpec, reuse_size: int, gpu: GpuSnapshot, peer_reuse=0) -> float:
    g = gpu.c()
    return lib.tg_estimate_load_time(C.byref(model.c()), reuse_size, C.byref(g), peer_reuse)


def schedule(requests: Sequence[str], snapshots: Sequence[GpuSnapshot], registry: dict, batch_size=1,
             block_size_tokens=16):
    """scheduler.hpp:79-120; returns (assignments [(model, gpu_id)], deferred [model], estimates)."""
    names = sorted(registry)
    index = {m: i for i, m in enumerate(names)}
    models = (N.ModelSpecC * max(1, len(names)))(*[registry[m].c() for m in names])
    req = (C.c_uint32 * max(1, len(requests)))(*[index.get(m, 0xFFFFFFFF) for m in requests])
    gs = (N.GpuSnapshotC * max(1, len(snapshots)))(*[g.c() for g in snapshots])
    G, M = len(snapshots), len(names)
    reuse = (C.c_uint64 * max(1, G * M))(*[g.reuse_size_by_model.get(m, 0) for g in snapshots for m in names])
    peer = None
    if any(g.peer_reuse_by_model for g in snapshots):
        peer = (C.c_uint64 * max(1, G * M))(*[g.peer_reuse_by_model.get(m, 0) for g in snapshots for m in names])
    assign = (C.c_int32 * max(1, len(requests)))()
    est = (C.c_double * max(1, len(requests) * G))()
    N.check_runtime(lib.tg_schedule(req, len(requests), gs, G, models, M, reuse, peer, batch_size,
                                    block_size_tokens, assign, est), "tg_schedule")
    assignments, deferred, estimates = [], [], []
    for i, m in enumerate(requests):
        a = assign[i]
        estimates.append([(snapshots[g].gpu_id, est[i * G + g]) for g in range(G) if est[i * G + g] >= 0])
        if a < 0:
            deferred.append(m)
        else:
            assignments.append((m, snapshots[a].gpu_id))
    return assignments, deferred, estimates
