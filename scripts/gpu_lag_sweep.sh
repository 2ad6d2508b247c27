#!/bin/bash
# bench value and policy lag vs envs per GPU (C4 is 16,384 envs: 256 learner
# steps per rollout, so the last trajectories train ~500 versions after they
# were acted on; fewer envs -> fewer learner steps per rollout -> lower lag)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for e in ${ENVS_LIST:-2048 4096 8192 16384}; do
  timeout -s KILL 300 python bench.py --envs $e --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/lag_$e.log 2>&1
  tail -1 gpurun_out/lag_$e.log | ENVS=$e python -c '
import json, os, sys
d = json.loads(sys.stdin.read()); l = d["last_step"]
print("envs", os.environ["ENVS"], "value_Mfps", round(d["value"] / 1e6, 3), "lag_mean", l["lag_mean"],
      "lag_max", l["lag_max"], "learner_steps_per_iter", d["config"]["learner_steps_per_step"])'
done
