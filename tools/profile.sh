#!/bin/bash
# Run on the GPU box (gpurun).  Produces in gpurun_out/:
#   launches.csv        — every kernel of a short bench run with its device time
#                         (cold-cache, serialised: compare SHARES)
#   prof_load.ncu-rep   — ncu --set full of the bench step's load-kernel launch
#   prof_k1.ncu-rep     — ncu --set full of a fingerprint-only (K1) launch, unfused A/B run
#   prof_k3.ncu-rep     — ncu --set full of K3 (relocate_bulk_kernel), misaligned src0 -> dst5, 4 GiB
#   kernel_bench.json   — isolated kernel bandwidths
set -x
mkdir -p gpurun_out
python tools/kernel_bench.py > gpurun_out/kernel_bench.json 2> gpurun_out/kernel_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
# copy_fp_kernel launch order in bench --profile --steps 1 --warmup 0: load #1
# (0), load #2 (1) (no reused tensors: one load-kernel launch each), the
# measured step: its load kernel (2) and the concurrent K1 launch verifying
# the untouched reused tensors (3)
ncu --set full --clock-control none --import-source on -k regex:copy_fp_kernel -s 2 -c 2 -o gpurun_out/prof_load -f \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_load.log 2>&1
# unfused A/B (the step only; loads #1, #2 keep the default): copy_fp_kernel
# launches are load #1 (0), load #2 (1), the step's 13 K1 placements (2..14),
# then its reuse verification of the untouched tensors (15)
TANGRAM_UNFUSED=1 ncu --set full --clock-control none --import-source on -k regex:copy_fp_kernel -s 15 -c 1 \
    -o gpurun_out/prof_k1 -f python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline \
    > gpurun_out/prof_k1.log 2>&1
# K3 alone: kernel_bench --only reloc launches warm-up + 1 rep per (src, dst)
# class; launch 2 is the (0, 5) class's first
ncu --set full --clock-control none --import-source on -k regex:relocate -s 2 -c 1 -o gpurun_out/prof_k3 -f \
    python tools/kernel_bench.py --only reloc --gib 8 --reps 1 > gpurun_out/prof_k3.log 2>&1
ls -la gpurun_out
