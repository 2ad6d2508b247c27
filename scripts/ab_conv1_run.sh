#!/bin/bash
# Run the conv1 A/B variants built by ab_conv1_build.sh (VARIANTS="a b a b").
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in $VARIANTS; do
  APPO_LIB=abtest/libappo_$v.so timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/ab_$v.txt 2>&1
  echo "== $v: $(grep -E 'conv1_s2d_wgrad' gpurun_out/ab_$v.txt | head -1 | awk '{print $5}' | tr '\n' ' ')"
done
