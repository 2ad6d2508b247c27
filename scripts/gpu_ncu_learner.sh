#!/bin/bash
# ncu --set full capture of every kernel of one learner step
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 120 python scripts/ncu_learner.py || exit 1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/${NAME:-learner_full} python scripts/ncu_learner.py > gpurun_out/${NAME:-learner_full}.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${NAME:-learner_full}.log
