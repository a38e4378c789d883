#!/bin/bash
# Run on the GPU box (gpurun).  Produces in gpurun_out/:
#   launches.csv        — every kernel of a short bench run with its device time
#                         (cold-cache, serialised: compare SHARES)
#   prof_fp.ncu-rep     — ncu --set full of the bench step's two K1 reuse-verification launches
#   prof_reloc.ncu-rep  — ncu --set full of the bench step's first K3 relocation wave
#   kernel_bench.json   — isolated kernel bandwidths
set -x
mkdir -p gpurun_out
python tools/kernel_bench.py > gpurun_out/kernel_bench.json 2> gpurun_out/kernel_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
# K1 (fp_v4_kernel) launch order in bench --profile --steps 1 --warmup 0:
#   load #1: 41 placements, load #2: 33 placements, step: 13 placements (74..86),
#   then the reuse verification: 87 = untouched tensors, 88 = relocated tensors
ncu --set full --clock-control none --import-source on -k regex:fp_v4 -s 87 -c 2 -o gpurun_out/prof_fp -f \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_fp.log 2>&1
# K3: load #2 has 2 waves (launches 0, 1); the step's first wave is launch 2
ncu --set full --clock-control none --import-source on -k regex:relocate -s 2 -c 1 -o gpurun_out/prof_reloc -f \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_reloc.log 2>&1
ls -la gpurun_out
