#!/bin/bash
# A/B of two library builds on the same box: warm per-kernel durations + GRU phases
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in ${VARIANTS:-A B A B}; do
  export APPO_LIB=abtest/libappo_$v.so
  APPO_GRU_PROF=1 timeout -s KILL 300 python scripts/_prof_gru.py > gpurun_out/gru_prof_$v.log 2>&1; echo "== $v"; grep "gru prof" gpurun_out/gru_prof_$v.log | tail -2 | cut -c1-220
  timeout -s KILL 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/warm_$v.csv python scripts/traffic_step.py > /dev/null 2>&1
  python scripts/warm_summary.py gpurun_out/warm_$v.csv 2>/dev/null | head -12 | tail -10
  python scripts/warm_summary.py gpurun_out/warm_$v.csv 2>/dev/null | tail -1
done
