#!/bin/bash
# compute-sanitizer passes over scripts/sanitize_cases.py (T5 in SURVEY §4).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python scripts/sanitize_cases.py --big > gpurun_out/sanitize_$tool.log 2>&1
  echo ${tool}_rc=$?
  tail -3 gpurun_out/sanitize_$tool.log
done
