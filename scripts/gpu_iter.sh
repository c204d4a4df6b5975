#!/bin/bash
# Iteration pass: GPU tests, a short bench, one ncu --set full capture per
# multiplication kernel at the bench workload.  Usage: gpu_iter.sh [tag]
tag=${1:-iter}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$tag.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$tag.log 2>&1; echo bench_rc=$?
grep '^{' gpurun_out/bench_$tag.log | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print('value %.4g mults/s  ms/step %.3f' % (d['value'], d['ms_per_step']))
for k, v in d['ops'].items(): print(' ', k, {a: round(b, 4) for a, b in v.items()})
print('  roofline', d['roofline']['kernel'], round(d['roofline']['frac'], 3), 'clocks', d['clocks'])
"
for k in ${KERNELS:-mul_ntt_kernel mul_classical_kernel}; do
  timeout 900 ncu --set full --metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.sum --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/prof_${k}_$tag python bench.py --no-e2e --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_${k}_$tag.log 2>&1; echo ncu_${k}_rc=$?
done
