#!/bin/bash
# Round-2 evidence pass (everything summarised on the box; gpurun_out <= 64 MiB):
#  smoke, pytest -m gpu, the default bench line, the ncu launch list of the
#  bench command, ncu --set full of every kernel the line and DESIGN cite
#  (summaries, raw CSV, gzipped SASS source page), sanitizers (--big).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/pytest_gpu.log
s0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$? wall=$(( $(date +%s) - s0 ))s
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"add_kernel|mul_classical|mul_ntt" -c 24 --csv \
  --log-file gpurun_out/launches.csv python bench.py --no-e2e --no-cpu --no-per-size --steps 5 --warmup 3 \
  > gpurun_out/ncu_launch.log 2>&1; echo launches_rc=$?
M="--metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"
prof() {  # tag op bits kernel_regex
  timeout 600 ncu --set full $M --clock-control none --import-source on -k regex:"$4" -s 2 -c 1 \
    -o gpurun_out/prof_$1 python scripts/quick_time.py --ops $2 --bits $3 --reps 1 > gpurun_out/ncu_$1.log 2>&1
  echo ncu_$1_rc=$?
  python tools/ncu_summary.py gpurun_out/prof_$1.ncu-rep > gpurun_out/sum_$1.txt 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/raw_$1.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1.csv 2>/dev/null
  gzip -f gpurun_out/src_$1.csv
  rm -f gpurun_out/prof_$1.ncu-rep
}
SPECS=${PROF_SPECS:-"ntt_4k mul_ntt 4096 ^mul_ntt_kernel;classical_4k mul_classical 4096 ^mul_classical_kernel;add_4k add 4096 ^add_kernel;ntt_128k mul_ntt 131072 ^mul_ntt_r32;ntt_256k mul_ntt 262144 ^mul_ntt_r32;add6_128k add6 131072 ^add6;add6_256k add6 262144 ^add6;polyntt_4k poly_ntt 4096 ^poly_ntt;polyntt_256k poly_ntt 262144 ^poly_ntt;widentt_256k mul_wide_ntt 262144 ^mul_wide_ntt;addbig_64m add_big 67108864 ^add_lookback;classical_64k mul_classical 65536 ^mul_classical_kernel"}
IFS=';' read -ra SPEC_LIST <<< "$SPECS"
for spec in "${SPEC_LIST[@]}"; do prof $spec; done
if [ "${SANITIZE:-1}" = 1 ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    echo "### compute-sanitizer --tool $tool python scripts/sanitize_cases.py --big" >> gpurun_out/sanitizer.log
    timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python scripts/sanitize_cases.py --big > gpurun_out/sanitize_$tool.log 2>&1
    echo ${tool}_rc=$?
    tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitizer.log
  done
fi
du -sh gpurun_out
