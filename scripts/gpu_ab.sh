#!/bin/bash
# A/B of library builds + optional parity tests / bench.
# env: AB_ARGS (quick_time args), AB_LIBS (space-separated .so paths),
#      TESTS (pytest -k expression, empty = skip), BENCH=1 to run bench.py
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$TESTS" > gpurun_out/pytest_ab.log 2>&1; echo pytest_rc=$?
  tail -3 gpurun_out/pytest_ab.log
fi
if [ -n "$AB_LIBS" ]; then
  bash scripts/ab.sh "$AB_ARGS" $AB_LIBS > gpurun_out/ab.log 2>&1; echo ab_rc=$?
fi
if [ "$BENCH" = 1 ]; then
  s0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$? wall=$(( $(date +%s) - s0 ))s
fi
