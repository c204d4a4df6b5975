#!/bin/bash
# Round-2 baseline evidence: ncu --set full of the kernels VERDICT r01 names
# (NTT at 4K / 128K / 256K, 6-Add at 256K, Poly-NTT at 4K) + a quick timing.
# Summaries are written on the box (tools/ncu_summary.py, raw + source CSV);
# the .ncu-rep files are dropped unless KEEP_REP=1 (gpurun_out is capped at 64 MiB).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python scripts/quick_time.py --ops ${QT_OPS:-add,mul_classical,mul_ntt,add6,poly_ntt} --bits ${QT_BITS:-4096,131072,262144} --reps 10 > gpurun_out/qt.log 2>&1; echo qt_rc=$?
M="--metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"
prof() {  # tag op bits kernel_regex
  timeout 600 ncu --set full $M --clock-control none --import-source on -k regex:"$4" -s 2 -c 1 \
    -o gpurun_out/prof_$1 python scripts/quick_time.py --ops $2 --bits $3 --reps 1 > gpurun_out/ncu_$1.log 2>&1
  echo ncu_$1_rc=$?
  python tools/ncu_summary.py gpurun_out/prof_$1.ncu-rep > gpurun_out/sum_$1.txt 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/raw_$1.csv 2>/dev/null
  ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1.csv 2>/dev/null
  gzip -f gpurun_out/src_$1.csv
  [ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/prof_$1.ncu-rep
}
# PROF_SPECS: ';'-separated "tag op bits kernel_regex" entries
SPECS=${PROF_SPECS:-"ntt_4k mul_ntt 4096 ^mul_ntt_kernel;ntt_128k mul_ntt 131072 ^mul_ntt_r32;ntt_256k mul_ntt 262144 ^mul_ntt_r32;add6_256k add6 262144 ^add6;polyntt_4k poly_ntt 4096 ^poly_ntt"}
IFS=';' read -ra SPEC_LIST <<< "$SPECS"
for spec in "${SPEC_LIST[@]}"; do
  prof $spec
done
du -sh gpurun_out; ls gpurun_out
