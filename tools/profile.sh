#!/bin/bash
# Run on the GPU box (gpurun).  Produces in gpurun_out/:
#   launches.csv        — every kernel of a short bench run with its device time
#                         (cold-cache, serialised: compare SHARES)
#   prof_fp.ncu-rep     — ncu --set full of the bench's K1 reuse-verification launch
#   prof_reloc.ncu-rep  — ncu --set full of one K3 relocation wave launch
#   kernel_bench.json   — isolated kernel bandwidths
set -x
mkdir -p gpurun_out
python tools/kernel_bench.py > gpurun_out/kernel_bench.json 2> gpurun_out/kernel_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
# K1 launches in bench --profile --steps 1 --warmup 0: load1 41 + load2 33 placements,
# then value-step: 13 placements, then the reuse verification (index 87)
ncu --set full --clock-control none --import-source on -k regex:fp_leaves -s 87 -c 1 -o gpurun_out/prof_fp -f \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_fp.log 2>&1
# K3: loads 1..2 relocation launches = 2 (load2 has 2 relocations: waves?), capture the first wave of load #3
ncu --set full --clock-control none --import-source on -k regex:relocate -s 2 -c 1 -o gpurun_out/prof_reloc -f \
    python bench.py --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_reloc.log 2>&1
ls -la gpurun_out
