#!/bin/bash
# Debug build with device-side bounds asserts (-DBN_BOUNDS_CHECK), then the
# parity tests of the kernels that carry them (compute-sanitizer is closed on
# the GPU pool; a failed device assert aborts the test process).
python tools/variant_build.py bounds zzz -DBN_BOUNDS_CHECK > /dev/null || exit 1
BN_LIB_PATH=ab/libbn_bounds.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
  -k "add6 or fused or in_place" 2>&1 | tail -2
