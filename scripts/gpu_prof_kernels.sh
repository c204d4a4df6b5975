#!/bin/bash
# One ncu --set full capture (with source) per named kernel at the bench
# workload (4096 bits, 2^20 instances).  Usage: gpu_prof_kernels.sh tag k1 k2 ...
tag=$1; shift
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu"
for k in "$@"; do
  timeout 900 ncu --set full --metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.sum \
    --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
    -o gpurun_out/prof_${k}_$tag $B --steps 1 --warmup 3 > gpurun_out/ncu_${k}_$tag.log 2>&1; echo ncu_${k}_rc=$?
done
