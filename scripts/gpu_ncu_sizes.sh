#!/bin/bash
# Pipe / issue / DRAM counters of one launch per (op, size), 1K..256K bits
# (ncu --metrics only: fast), for profiles/ncu_kernels.json (bench.py per_size).
mkdir -p gpurun_out
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for op in ${NCU_OPS:-add mul_classical mul_ntt add6 poly_ntt mul_wide_ntt}; do
  case $op in
    add) k="add_kernel|add_cluster" ;;
    mul_classical) k="mul_classical" ;;
    mul_ntt) k="mul_ntt" ;;
    add6) k="add6" ;;
    poly_ntt) k="poly_ntt" ;;
    mul_wide_ntt) k="mul_wide_ntt" ;;
  esac
  for bits in ${NCU_BITS:-1024 2048 4096 8192 16384 32768 65536 131072 262144}; do
    timeout 300 ncu --metrics $MET --clock-control none -k regex:"$k" -s 2 -c 1 --csv \
      --log-file gpurun_out/m_${op}_${bits}.csv python scripts/quick_time.py --ops $op --bits $bits --reps 1 \
      > /dev/null 2>&1
    echo ${op}_${bits}_rc=$?
  done
done
