#!/bin/bash
# bench throughput vs the sampler's SM budget (persistent grids of the sampler context)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for n in ${SMS:-24 32 40 48 64}; do
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-e2e --sampler-sms $n > gpurun_out/bench_sms_$n.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bench_sms_$n.log').read().strip().splitlines()[-1]); print('sms $n value', round(d['value']), 'ms', round(d['ms_per_step'],2))"
done
