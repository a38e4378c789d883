"""ctypes binding of libtangram.so (include/tangram.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2512_01357_b200/csrc``).  There is no Python fallback for
any of it: if the shared object is missing, importing this module fails.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtangram.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtangram.so not built at {LIB_PATH}; run __graft_entry__.build() "
                      f"or `make -C paper_2512_01357_b200/csrc`")

lib = C.CDLL(LIB_PATH)

u64, u32, i32, i64, dbl = C.c_uint64, C.c_uint32, C.c_int32, C.c_int64, C.c_double
vp, cp = C.c_void_p, C.c_char_p
P = C.POINTER


class TensorIdC(C.Structure):
    _fields_ = [("hi", u64), ("lo", u64)]


DigestC = TensorIdC


class GpuSpecC(C.Structure):
    _fields_ = [("gpu_id", cp), ("pool_size", u64), ("pcie_bandwidth", dbl), ("intra_copy_bandwidth", dbl),
                ("store_bandwidth", dbl)]


class TensorSpecC(C.Structure):
    _fields_ = [("id", TensorIdC), ("name", cp), ("size", u64), ("model_id", cp)]


class ModelSpecC(C.Structure):
    _fields_ = [("model_id", cp), ("tensors", P(TensorSpecC)), ("n_tensors", u32), ("total_size", u64),
                ("latency_sensitivity", dbl), ("location", i32), ("bytes_per_token", u64)]


class LoadPolicyC(C.Structure):
    _fields_ = [("merge", i32), ("strictness", i32), ("random_eviction", i32), ("rng", vp), ("flags", u32),
                ("uniform_below", vp), ("rng_ctx", vp)]


class LoadOutcomeC(C.Structure):
    _fields_ = [("n_hits", u32), ("n_misses", u32), ("n_evictions", u32), ("n_relocations", u32),
                ("n_placements", u32), ("n_waves", u32), ("fallback_evictions", u64),
                ("bytes_transferred", u64), ("bytes_merged", u64), ("eviction_cost_total", dbl),
                ("total_merge_cost", u64), ("pgp_merge_cost", u64), ("initial_merge_cost", u64),
                ("total_eviction_cost", dbl),
                ("pcie_bytes", u64), ("peer_bytes", u64), ("device_src_bytes", u64), ("fingerprint_bytes", u64), ("repaired_bytes", u64),
                ("verify_mismatches", u32), ("expected_mismatches", u32),
                ("plan_us", dbl), ("total_ms", dbl), ("relocate_ms", dbl), ("h2d_ms", dbl), ("peer_ms", dbl),
                ("fp_kernel_ms", dbl), ("fp_reuse_ms", dbl), ("fp_reuse_max_ms", dbl),
                ("host_issue_us", dbl), ("host_wait_us", dbl), ("host_total_us", dbl),
                ("suspect_tensors", u32), ("reserved0", u32), ("kernel_end_ms", dbl), ("gated_h2d_start_ms", dbl)]


class EvictionC(C.Structure):
    _fields_ = [("tensor", TensorIdC), ("size", u64), ("cost", dbl), ("last_access", dbl), ("model_id", cp)]


class RelocationC(C.Structure):
    _fields_ = [("tensor", TensorIdC), ("from_", u64), ("to", u64), ("size", u64), ("wave", u32)]


class PlacementC(C.Structure):
    _fields_ = [("tensor", TensorIdC), ("offset", u64), ("size", u64), ("source", u32)]


class RegionC(C.Structure):
    _fields_ = [("offset", u64), ("size", u64), ("kind", i32), ("tensor", TensorIdC), ("block_id", u64)]


class PoolInfoC(C.Structure):
    _fields_ = [("pool_size", u64), ("free_bytes", u64), ("kv_bytes", u64), ("pinned_tensor_bytes", u64),
                ("pinned_bytes", u64), ("reusable_bytes", u64), ("bytes_merged_total", u64),
                ("bytes_transferred_total", u64), ("evictions_total", u64), ("region_count", u64),
                ("extent_count", u64), ("tensor_count", u64), ("largest_free", u64), ("device", i32),
                ("arena", vp), ("loads", u64), ("data_plane_ms", dbl), ("pcie_bytes", u64), ("peer_bytes", u64),
                ("device_src_bytes", u64), ("fingerprint_bytes", u64), ("relocated_bytes", u64), ("epoch", u64),
                ("verify_mismatches", u64), ("repaired_bytes", u64), ("failed_loads", u64)]


class TensorEntryC(C.Structure):
    _fields_ = [("id", TensorIdC), ("offset", u64), ("size", u64), ("last_access", dbl), ("pinned", i32),
                ("suspect", i32), ("model_id", cp)]


class TensorInfoC(C.Structure):
    _fields_ = [("offset", u64), ("size", u64), ("last_access", dbl), ("pinned", i32), ("has_digest", i32),
                ("digest", DigestC), ("device_ptr", vp), ("suspect", i32), ("reserved0", i32)]


class KvStatsC(C.Structure):
    _fields_ = [("pool_invocations", u64), ("alloc_batches", u64), ("blocks_from_free_list", u64),
                ("blocks_from_pool", u64), ("reclaim_events", u64), ("free_list_size", u64),
                ("active_requests", u64), ("next_pbn", u64), ("block_bytes", u64)]


class IndexEntryC(C.Structure):
    _fields_ = [("id", TensorIdC), ("offset", u64), ("size", u64), ("digest", DigestC)]


class IndexSlotC(C.Structure):
    _fields_ = [("key_hi", u64), ("key_lo", u64), ("offset", u64), ("size", u64), ("last_access", dbl),
                ("model", u64), ("flags", u32), ("reserved0", u32), ("reserved1", u64)]


class IndexHitC(C.Structure):
    _fields_ = [("offset", u64), ("size", u64), ("found", u32), ("flags", u32)]


class GpuSnapshotC(C.Structure):
    _fields_ = [("gpu_id", cp), ("available", i32), ("pool_size", u64), ("free_bytes", u64),
                ("pcie_bandwidth", dbl), ("store_bandwidth", dbl), ("nvlink_bandwidth", dbl)]


_SIGS = {
    "tg_version": (C.c_int, []),
    "tg_error_string": (cp, [C.c_int]),
    "tg_last_error_detail": (cp, []),
    "tg_device_count": (C.c_int, [P(C.c_int)]),
    "tg_kernel_launches": (u64, []),
    "tg_murmur3_x64_128": (C.c_int, [vp, u64, u64, P(DigestC)]),
    "tg_tensor_key": (C.c_int, [cp, cp, P(i64), i32, i32, P(TensorIdC)]),
    "tg_model_make": (C.c_int, [cp, u64, i32, u64, i32, dbl, P(vp)]),
    "tg_model_default_catalog": (C.c_int, [u32, P(vp)]),
    "tg_model_catalog_size": (u32, []),
    "tg_model_destroy": (None, [vp]),
    "tg_model_view": (C.c_int, [vp, P(ModelSpecC)]),
    "tg_model_shard": (C.c_int, [vp, u32, u32, P(vp)]),
    "tg_stats_create": (C.c_int, [dbl, P(vp)]),
    "tg_stats_destroy": (None, [vp]),
    "tg_stats_create_external": (C.c_int, [vp, vp, vp, P(vp)]),
    "tg_stats_record_request": (C.c_int, [vp, cp, dbl]),
    "tg_stats_record_eviction": (C.c_int, [vp, cp, dbl]),
    "tg_stats_set_load_bandwidth": (C.c_int, [vp, cp, dbl]),
    "tg_stats_miss_probability": (dbl, [vp, cp]),
    "tg_rng_create": (C.c_int, [u64, P(vp)]),
    "tg_rng_destroy": (None, [vp]),
    "tg_rng_uniform_below": (u64, [vp, u64]),
    "tg_pool_create": (C.c_int, [P(GpuSpecC), i32, P(vp)]),
    "tg_pool_destroy": (None, [vp]),
    "tg_pool_info_get": (C.c_int, [vp, P(PoolInfoC)]),
    "tg_pool_clone": (C.c_int, [vp, P(vp)]),
    "tg_pool_assign": (C.c_int, [vp, vp]),
    "tg_pool_tensors": (C.c_int, [vp, P(TensorEntryC), u64, P(u64)]),
    "tg_pool_stream": (C.c_int, [vp, P(vp)]),
    "tg_set_model_alpha": (C.c_int, [vp, cp, dbl]),
    "tg_load_model": (C.c_int, [vp, P(ModelSpecC), vp, dbl, P(LoadPolicyC), P(LoadOutcomeC)]),
    "tg_pool_sync": (C.c_int, [vp, P(LoadOutcomeC)]),
    "tg_last_hits": (u32, [vp, P(TensorIdC), u32]),
    "tg_last_misses": (u32, [vp, P(TensorIdC), u32]),
    "tg_last_evictions": (u32, [vp, P(EvictionC), u32]),
    "tg_last_relocations": (u32, [vp, P(RelocationC), u32]),
    "tg_last_placements": (u32, [vp, P(PlacementC), u32]),
    "tg_last_digests": (u32, [vp, P(DigestC), u32]),
    "tg_end_instance": (C.c_int, [vp, cp]),
    "tg_evict_tensor": (C.c_int, [vp, TensorIdC]),
    "tg_evict_model": (C.c_int, [vp, cp]),
    "tg_move_tensor": (C.c_int, [vp, TensorIdC, u64]),
    "tg_alloc_kv_region": (C.c_int, [vp, u64, u64, P(u64)]),
    "tg_free_kv_region": (C.c_int, [vp, u64]),
    "tg_lookup": (C.c_int, [vp, P(ModelSpecC), P(C.c_uint8), P(u64)]),
    "tg_reuse_size": (C.c_int, [vp, P(ModelSpecC), P(u64)]),
    "tg_peer_reuse_size": (C.c_int, [vp, P(ModelSpecC), P(u64)]),
    "tg_eviction_candidates": (C.c_int, [vp, vp, cp, P(EvictionC), u32, P(u32)]),
    "tg_validate": (C.c_int, [vp]),
    "tg_dump": (C.c_int, [vp, C.c_char_p, u64, P(u64)]),
    "tg_regions": (C.c_int, [vp, P(RegionC), u64, P(u64)]),
    "tg_tensor_info_get": (C.c_int, [vp, TensorIdC, P(TensorInfoC)]),
    "tg_pool_index_image": (C.c_int, [vp, P(IndexSlotC), u64, P(u64)]),
    "tg_pool_device_index": (C.c_int, [vp, P(vp), P(u64)]),
    "tg_index_lookup": (C.c_int, [vp, P(TensorIdC), u32, P(IndexHitC)]),
    "tg_fingerprint_tensor": (C.c_int, [vp, TensorIdC, P(DigestC)]),
    "tg_pool_add_peer": (C.c_int, [vp, vp]),
    "tg_pool_export_ipc": (C.c_int, [vp, vp]),
    "tg_pool_index": (C.c_int, [vp, P(IndexEntryC), u64, P(u64)]),
    "tg_pool_attach_remote": (C.c_int, [vp, vp, P(IndexEntryC), u64, P(i32)]),
    "tg_pool_update_remote": (C.c_int, [vp, i32, P(IndexEntryC), u64]),
    "tg_pool_snapshot": (C.c_int, [vp, P(vp)]),
    "tg_pool_restore": (C.c_int, [vp, vp]),
    "tg_snapshot_destroy": (None, [vp]),
    "tg_host_register": (C.c_int, [TensorIdC, vp, u64, P(DigestC)]),
    "tg_file_register": (C.c_int, [TensorIdC, cp, u64, u64, P(DigestC)]),
    "tg_host_unregister": (C.c_int, [TensorIdC]),
    "tg_host_clear": (C.c_int, []),
    "tg_host_alloc": (C.c_int, [u64, P(vp)]),
    "tg_host_free": (C.c_int, [vp]),
    "tg_fingerprint_device": (C.c_int, [vp, u64, i32, P(DigestC)]),
    "tg_synth_fill_device": (C.c_int, [TensorIdC, u64, u64, vp, i32]),
    "tg_bench_fingerprint": (C.c_int, [P(vp), P(u64), u32, i32, i32, P(dbl), P(DigestC)]),
    "tg_bench_relocate": (C.c_int, [P(u64), u32, i32, i32, P(dbl)]),
    "tg_copy_fingerprint": (C.c_int, [P(u64), u32, i32, i32, P(dbl), P(DigestC)]),
    "tg_synth_fill_host": (C.c_int, [TensorIdC, u64, u64, vp, i32]),
    "tg_device_alloc": (C.c_int, [i32, u64, P(vp)]),
    "tg_device_free": (C.c_int, [i32, vp]),
    "tg_memcpy": (C.c_int, [vp, vp, u64]),
    "tg_failpoint": (C.c_int, [cp, i64]),
    "tg_kv_create": (C.c_int, [cp, u64, u64, P(vp)]),
    "tg_kv_destroy": (None, [vp]),
    "tg_kv_clone": (C.c_int, [vp, P(vp)]),
    "tg_kv_ensure_capacity": (C.c_int, [vp, vp, vp, u64, u64, P(u64), u64, P(u64)]),
    "tg_kv_batch_allocate": (C.c_int, [vp, vp, vp, P(u64), P(u64), u64, P(u64), P(u64), u64, P(u64)]),
    "tg_kv_release_request": (C.c_int, [vp, u64]),
    "tg_kv_teardown": (C.c_int, [vp, vp]),
    "tg_kv_urgent_reclaim": (C.c_int, [vp, vp, vp, u64]),
    "tg_kv_table": (C.c_int, [vp, u64, P(u64), u64, P(u64), P(u64)]),
    "tg_kv_address_table": (C.c_int, [vp, P(u64), u64, P(u64)]),
    "tg_kv_stats_get": (C.c_int, [vp, P(KvStatsC)]),
    "tg_kv_device_tables": (C.c_int, [vp, P(vp), P(u64), P(vp)]),
    "tg_lineage_register": (C.c_int, [TensorIdC, TensorIdC, u64, u64]),
    "tg_lineage_get": (C.c_int, [TensorIdC, P(TensorIdC), P(u64), P(u64)]),
    "tg_kv_write_tokens": (C.c_int, [vp, vp, vp, vp, vp, C.c_uint32, vp]),
    "tg_kv_read_tokens": (C.c_int, [vp, vp, vp, vp, vp, C.c_uint32, vp]),
    "tg_kv_token_faults": (C.c_int, [vp, P(u64)]),
    "tg_kv_wait_tables": (C.c_int, [vp, vp]),
    "tg_kv_reserve": (C.c_int, [vp, vp, u32, u64, u64]),
    "tg_kv_request_slot": (C.c_int, [vp, u64, P(C.c_uint32)]),
    "tg_kv_device_arm": (C.c_int, [vp, vp, u64, C.c_uint32, C.c_uint32]),
    "tg_kv_batch_allocate_device": (C.c_int, [vp, vp, vp, C.c_uint32, vp]),
    "tg_kv_device_sync": (C.c_int, [vp, vp, vp, P(u64), P(u64)]),
    "tg_plan_allocation": (C.c_int, [P(RegionC), u64, P(TensorSpecC), u32, P(EvictionC), u32, P(TensorIdC), u32,
                                     i32, i32, i32, P(vp)]),
    "tg_plan_evictions": (u32, [vp, P(EvictionC), u32]),
    "tg_plan_relocations": (u32, [vp, P(RelocationC), u32]),
    "tg_plan_placements": (u32, [vp, P(PlacementC), u32]),
    "tg_plan_costs": (C.c_int, [vp, P(dbl), P(u64), P(u64), P(u64), P(u64)]),
    "tg_plan_destroy": (None, [vp]),
    "tg_schedule": (C.c_int, [P(u32), u32, P(GpuSnapshotC), u32, P(ModelSpecC), u32, P(u64), P(u64), u32, u64,
                              P(i32), P(dbl)]),
    "tg_estimate_load_time": (dbl, [P(ModelSpecC), u64, P(GpuSnapshotC), u64]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)

ERROR_NAMES = ["InsufficientMemory", "PoolExhausted", "Infeasible", "Pinned", "NotFound", "OverlapMove",
               "DestinationOccupied", "OrderingError", "InstanceTooLarge", "InvalidArgument"]


class TangramRuntimeError(RuntimeError):
    """A TG_ERR_* runtime failure (CUDA error, missing source, no device...)."""

    def __init__(self, code, where="", outcome=None):
        self.code = code
        self.outcome = outcome  # tg_load_model after its commit: the decision taken (suspect_tensors > 0)
        detail = lib.tg_last_error_detail().decode(errors="replace")
        super().__init__(f"{where}: {lib.tg_error_string(code).decode()} ({code}) {detail}".strip())


def check_runtime(rc, where=""):
    """Raise for runtime codes (>= 100); return domain codes (0..10) unchanged."""
    if rc >= 100:
        raise TangramRuntimeError(rc, where)
    return rc


def device_count():
    n = C.c_int(0)
    lib.tg_device_count(C.byref(n))
    return n.value
