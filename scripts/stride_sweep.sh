#!/bin/bash
# bench value vs the per-kernel timing sample stride (events end PDL overlap)
mkdir -p gpurun_out
for s in ${STRIDES:-13 31 100000}; do
  APPO_BENCH_TIMING_STRIDE=$s timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/stride_$s.log 2>&1
  tail -1 gpurun_out/stride_$s.log | python -c "
import json, sys
d = json.loads(sys.stdin.read())
r = d['roofline']
print('$s', round(d['value']), round(d['ms_per_step'], 2), r.get('kernel'), r.get('launches'), round(r.get('frac', 0), 3))"
done
