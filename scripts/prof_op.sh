#!/bin/bash
# ncu --set full of one op at one size (quick_time invocation, 1 timed rep).
# Usage: prof_op.sh tag op bits kernel_regex
tag=$1; op=$2; bits=$3; k=$4
mkdir -p gpurun_out
timeout 900 ncu --set full --metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -o gpurun_out/prof_${tag} \
  python scripts/quick_time.py --ops $op --bits $bits --reps 1 > gpurun_out/ncu_${tag}.log 2>&1
echo ncu_${tag}_rc=$?
