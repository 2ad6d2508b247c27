#!/bin/bash
# bench value vs the sampler context's SM budget (--sampler-sms)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for s in ${SMS:-40 48 56 64 80}; do
  timeout -s KILL 300 python bench.py --sampler-sms $s --no-cpu-baseline --no-e2e > gpurun_out/sms_$s.log 2>&1
  echo "sms=$s $(tail -1 gpurun_out/sms_$s.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3))')"
done
