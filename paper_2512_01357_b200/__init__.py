"""B200-native Tangram model-loading hot path (arXiv 2512.01357).

The product is libtangram.so (C-ABI in include/tangram.h): a bit-exact host
control plane (pool regions, two-stage planner, reuse index, KV allocator,
affinity scheduler) driving sm_100a kernels for content fingerprints,
relocation/compaction, KV block tables and NVLink peer pulls.  This package is
the thin Python mirror of the reference's C++ API used by tests and bench.py.
"""
from . import pool
from .pool import (AllocationPlan, Error, GpuSnapshot, GpuSpec, KvEngine, LoadOutcome, LoadPolicy, MergePolicy,
                   ModelLocation, ModelSpec, ModelStatsTable, PackingStrictness, Result, ReuseStore, Rng,
                   TensorId, TensorSpec, default_catalog, estimate_load_time, make_model, murmur3_x64_128,
                   schedule, shard_model, tensor_key, lineage, failpoint)
from ._native import LIB_PATH, device_count

__all__ = ["AllocationPlan", "Error", "GpuSnapshot", "GpuSpec", "KvEngine", "LoadOutcome", "LoadPolicy",
           "MergePolicy", "ModelLocation", "ModelSpec", "ModelStatsTable", "PackingStrictness", "Result",
           "ReuseStore", "Rng", "TensorId", "TensorSpec", "default_catalog", "estimate_load_time", "make_model",
           "murmur3_x64_128", "schedule", "shard_model", "tensor_key", "lineage", "failpoint", "LIB_PATH", "device_count"]
