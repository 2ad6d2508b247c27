#!/bin/bash
# A/B of learner-backward GEMM tile widths with the two-stream backward
# (bench value, 5 timed iterations each; APPO_BN_* overrides in model.cu)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for cfg in "X=0" "APPO_BN_FCD=256" "APPO_BN_FCD=192" "APPO_BN_DX=128" "APPO_BN_DW=128" "APPO_BN_FCW=128" "X=0" "APPO_BN_FCD=256" "APPO_BN_DX=128"; do
  env $cfg timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bn.log 2>&1
  echo "$cfg rc=$? $(tail -1 gpurun_out/bn.log | cut -c90-115)"
done
for s in 48 80; do
  timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 --sampler-sms $s > gpurun_out/bn.log 2>&1
  echo "sampler-sms=$s rc=$? $(tail -1 gpurun_out/bn.log | cut -c90-115)"
done
