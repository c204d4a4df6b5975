#!/bin/bash
# ncu --set full (with SASS source) of one launch per spec, summarised on the
# box: PROF_SPECS="tag op bits kernel_regex;..." bash scripts/prof_specs.sh
# -> gpurun_out/{sum,raw,src}_<tag>.*  (LIB=path optionally selects a variant)
mkdir -p gpurun_out
M="--metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"
prof() {  # tag op bits kernel_regex
  BN_LIB_PATH=${LIB:-} timeout 600 ncu --set full $M --clock-control none --import-source on -k regex:"$4" -s 2 -c 1 \
    -o gpurun_out/prof_$1 python scripts/quick_time.py --ops $2 --bits $3 --reps 1 > gpurun_out/ncu_$1.log 2>&1
  echo ncu_$1_rc=$?
  python tools/ncu_summary.py gpurun_out/prof_$1.ncu-rep > gpurun_out/sum_$1.txt 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/raw_$1.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1.csv 2>/dev/null
  gzip -f gpurun_out/src_$1.csv
  rm -f gpurun_out/prof_$1.ncu-rep
}
IFS=';' read -ra SPEC_LIST <<< "$PROF_SPECS"
for spec in "${SPEC_LIST[@]}"; do prof $spec; done
