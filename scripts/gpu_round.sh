#!/bin/bash
# Round evidence: smoke, gpu tests, the default bench line (e2e + cpu
# baseline), a sweep, the ncu launch list of the bench command and one
# ncu --set full capture per main kernel at the bench workload.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
B="python bench.py --no-e2e --no-cpu --no-fused"
timeout 900 python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 --sweep > gpurun_out/sweep.log 2>&1; echo sweep_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file gpurun_out/launches.csv $B --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches_rc=$?
for k in mul_ntt_kernel mul_classical_kernel add_kernel; do
  timeout 900 ncu --set full --metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --import-source on -k regex:"^$k" -s 3 -c 1 \
    -o gpurun_out/prof_${k}_4k $B --steps 1 --warmup 3 > gpurun_out/ncu_full_$k.log 2>&1; echo full_${k}_rc=$?
done
