#!/bin/bash
# compute-sanitizer over the final kernels (run on the GPU box):
#  memcheck : load kernel (paired stores, tail staging) at partial-leaf sizes and
#             several alignments / line phases; K4D device KV batches
#  racecheck: load kernel shared-memory ring (paired stores, tail staging)
#  synccheck: same
S=/usr/local/cuda/bin/compute-sanitizer
OUT=gpurun_out/sanitizer.txt
{
echo "# compute-sanitizer on the B200 (round 2: K3 TMA bulk copies, load-kernel stamps / self-cleaning lone launches, warm reloads as K1, async loads, pipelined file stager)"
echo "## memcheck: copy_fingerprint_fused at partial-leaf sizes"
timeout 900 $S --tool memcheck --error-exitcode 1 python -m pytest tests/test_gpu_kernels.py -q -k "copy_fingerprint_fused and (4097 or 135169 or 656359) and (16 or 112)" 2>&1 | tail -4
echo "## memcheck / racecheck: K1 fingerprint-only ring (next-stage realignment words) at partial-leaf sizes and phases"
timeout 900 $S --tool memcheck --error-exitcode 1 python -m pytest tests/test_gpu_kernels.py -q -k "fingerprint_matches_cpu and (4097 or 131077 or 393293)" 2>&1 | tail -2
timeout 900 $S --tool racecheck python -m pytest tests/test_gpu_kernels.py -q -k "fingerprint_matches_cpu and (131077 or 393293) and (3- or 0-)" 2>&1 | tail -2
echo "## memcheck / racecheck: verify and move tiles in one writing launch"
timeout 900 $S --tool memcheck --error-exitcode 1 python -m pytest -q tests/test_gpu_kernels.py::test_copy_fingerprint_mixed_verify 2>&1 | tail -2
timeout 900 $S --tool racecheck python -m pytest -q tests/test_gpu_kernels.py::test_copy_fingerprint_mixed_verify 2>&1 | tail -2
echo "## memcheck: verify tiles in writing launches (device store fuzz, one seed)"
timeout 900 $S --tool memcheck --error-exitcode 1 python -m pytest -q "tests/test_gpu_load.py::test_device_store_differential_fuzz[1]" 2>&1 | tail -2
echo "## memcheck: K4D device KV batches"
timeout 900 $S --tool memcheck --error-exitcode 1 python -m pytest -q "tests/test_gpu_kv_device.py::test_device_batches_equal_reference[1]" tests/test_gpu_kv_device.py::test_device_batches_in_a_cuda_graph 2>&1 | tail -4
echo "## memcheck: fused vs unfused load fuzz (K3 device-source placements), re-shard, paged cache, peer pulls"
timeout 1500 $S --tool memcheck --error-exitcode 1 python -m pytest -q "tests/test_gpu_load.py::test_fused_load_kernel_fuzz[52-hbm]" tests/test_gpu_reshard.py::test_reshard_from_own_pool "tests/test_gpu_kv_device.py::test_block_tables_drive_a_paged_cache[48]" tests/test_gpu_load.py::test_peer_pull_same_device 2>&1 | tail -4
echo "## racecheck: load kernel ring"
timeout 900 $S --tool racecheck python -m pytest -q "tests/test_gpu_kernels.py::test_copy_fingerprint_fused[16-3-11-135169]" "tests/test_gpu_kernels.py::test_copy_fingerprint_fused[112-0-8-656359]" 2>&1 | tail -4
echo "## synccheck: load kernel ring"
timeout 900 $S --tool synccheck python -m pytest -q "tests/test_gpu_kernels.py::test_copy_fingerprint_fused[16-3-11-135169]" "tests/test_gpu_kernels.py::test_copy_fingerprint_fused[112-0-8-656359]" 2>&1 | tail -4
echo "## racecheck / synccheck / initcheck: K4D, batched moves, device index (+ load fuzz, C1, peer pulls for initcheck)"
timeout 900 $S --tool racecheck python -m pytest -q tests/test_gpu_kv_device.py "tests/test_gpu_kernels.py::test_copy_fingerprint_batched_moves" tests/test_gpu_index.py 2>&1 | tail -2
timeout 900 $S --tool synccheck python -m pytest -q tests/test_gpu_kv_device.py "tests/test_gpu_kernels.py::test_copy_fingerprint_batched_moves" tests/test_gpu_index.py 2>&1 | tail -2
timeout 1500 $S --tool initcheck python -m pytest -q tests/test_gpu_kv_device.py "tests/test_gpu_kernels.py::test_copy_fingerprint_batched_moves" tests/test_gpu_index.py "tests/test_gpu_load.py::test_fused_load_kernel_fuzz[52-hbm]" tests/test_gpu_load.py::test_c1_cold_then_warm_from_host tests/test_gpu_load.py::test_peer_pull_same_device 2>&1 | tail -2
echo "## round 2 — memcheck / racecheck / synccheck: K3 relocate_bulk_kernel (cp.async.bulk + mbarrier ring) at random alignments"
timeout 900 $S --tool memcheck --error-exitcode 1 python -m pytest -q tests/test_gpu_kernels.py::test_relocation_kernel_random_alignments 2>&1 | tail -2
timeout 900 $S --tool racecheck python -m pytest -q tests/test_gpu_kernels.py::test_relocation_kernel_random_alignments 2>&1 | tail -2
timeout 900 $S --tool synccheck python -m pytest -q tests/test_gpu_kernels.py::test_relocation_kernel_random_alignments 2>&1 | tail -2
echo "## round 2 — memcheck / initcheck: warm reloads as K1 with stamps and self-cleaning resident descriptors (C1), async loads, file stager"
timeout 1500 $S --tool memcheck --error-exitcode 1 python -m pytest -q tests/test_gpu_load.py::test_c1_cold_then_warm_from_host tests/test_gpu_async.py tests/test_gpu_load.py::test_model_store_pipelined_ranges_across_files "tests/test_gpu_load.py::test_device_store_fuzz_async[0]" 2>&1 | tail -2
timeout 1500 $S --tool initcheck python -m pytest -q tests/test_gpu_load.py::test_c1_cold_then_warm_from_host tests/test_gpu_async.py::test_async_loads_match_sync_loads 2>&1 | tail -2
} > $OUT
cat $OUT
