#!/bin/bash
# A/B timing of library builds on one box: ab.sh "<quick_time args>" lib1.so lib2.so ...
# Runs each library twice, interleaved (A B A B), to separate drift from effect.
args=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    echo "## $lib round $round"
    BN_LIB_PATH=$lib python scripts/quick_time.py $args
  done
done
