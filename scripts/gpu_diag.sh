#!/bin/bash
# diagnostics: GRU per-phase cycles, warm-cache per-kernel durations of the
# learner step, --set full captures of the small learner kernels
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
APPO_GRU_PROF=1 timeout -s KILL 300 python scripts/_prof_gru.py > gpurun_out/gru_prof.log 2>&1; echo "gru prof rc=$?"; grep "gru prof" gpurun_out/gru_prof.log
timeout -s KILL 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/warm_step.csv python scripts/traffic_step.py > gpurun_out/warm_step.log 2>&1; echo "warm rc=$?"
timeout -s KILL 600 ncu --profile-from-start off --set full --cache-control none --clock-control none -k regex:"heads_|ppo_loss|gather_slots|publish_derived|returns|splitk|sumsq" -c 12 -o gpurun_out/prof_small python scripts/traffic_step.py > gpurun_out/prof_small.log 2>&1; echo "small rc=$?"
timeout -s KILL 300 python scripts/hbm_sweep.py > gpurun_out/hbm_sweep.jsonl 2> gpurun_out/hbm_sweep.err; echo "sweep rc=$?"; cut -c1-200 gpurun_out/hbm_sweep.jsonl
