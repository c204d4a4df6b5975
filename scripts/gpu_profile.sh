#!/bin/bash
# Profiling pass: sweep + ncu launch list of the bench command + one --set full
# capture per kernel at the bench workload (4096 bits, 2^20 instances).
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu"
timeout 900 $B --steps 20 --warmup 3 --sweep > gpurun_out/sweep.log 2>&1; echo sweep_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file gpurun_out/launches.csv $B --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches_rc=$?
for k in mul_ntt_kernel mul_classical_kernel add_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/prof_${k}_4k $B --steps 1 --warmup 3 > gpurun_out/ncu_full_$k.log 2>&1; echo full_${k}_rc=$?
done
ls -la gpurun_out
