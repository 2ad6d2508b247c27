#!/bin/bash
# warm per-kernel durations of the learner step (ncu, serialised launches) and
# one --set full capture of the fused loss kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ENVS=2048 timeout -s KILL 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics gpu__time_duration.sum,launch__grid_size --csv --log-file gpurun_out/tail_warm.csv python scripts/traffic_step.py > gpurun_out/tail_warm.log 2>&1; echo "warm rc=$?"
KREGEX=traj_loss NAME=traj_loss_full SKIP=2 bash scripts/gpu_ncu_kernel.sh
