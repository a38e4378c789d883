#!/bin/bash
# compute-sanitizer over the last round-2 changes (run on the GPU box):
# K1 on the three-slot / eight-warp ring, and re-shard pulls gated on
# relocation waves (in-kernel fragments + the post-kernel straddle launch).
S=/usr/local/cuda/bin/compute-sanitizer
OUT=gpurun_out/sanitizer_r02b.txt
{
echo "## memcheck / racecheck / synccheck: K1 three-slot ring at partial-leaf sizes and phases"
timeout 900 $S --tool memcheck --error-exitcode 1 python -m pytest tests/test_gpu_kernels.py -q -k "fingerprint_matches_cpu and (4097 or 131077 or 393293)" 2>&1 | tail -2
timeout 900 $S --tool racecheck python -m pytest tests/test_gpu_kernels.py -q -k "fingerprint_matches_cpu and (131077 or 393293) and (3- or 0-)" 2>&1 | tail -2
timeout 900 $S --tool synccheck python -m pytest tests/test_gpu_kernels.py -q -k "fingerprint_matches_cpu and (131077 or 393293) and (3- or 0-)" 2>&1 | tail -2
echo "## memcheck / racecheck: re-shard pulls gated on relocation waves (fused)"
timeout 1500 $S --tool memcheck --error-exitcode 1 python -m pytest -q "tests/test_gpu_reshard.py::test_reshard_pulls_gated_on_relocation_waves[fused]" 2>&1 | tail -2
timeout 1500 $S --tool racecheck python -m pytest -q "tests/test_gpu_reshard.py::test_reshard_pulls_gated_on_relocation_waves[fused]" 2>&1 | tail -2
} > $OUT
cat $OUT
