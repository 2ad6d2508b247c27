#!/bin/bash
# ncu evidence set (VERDICT r1 "next" item 2): HBM sweep of the memory-bound
# kernels (event timing + ncu DRAM bytes), --set full captures of both GRU
# recurrence kernels, and tensor-pipe / DRAM counters for every kernel of one
# inference step + 8 learner steps at the bench shapes.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/hbm_sweep.py > gpurun_out/hbm_sweep.jsonl 2> gpurun_out/hbm_sweep.err; echo "sweep rc=$?"
cat gpurun_out/hbm_sweep.jsonl | cut -c1-200
timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"returns_kernel|ppo_loss|adam_kernel|sumsq" --csv --log-file gpurun_out/hbm_sweep_ncu.csv python scripts/hbm_sweep.py --quick > gpurun_out/hbm_sweep_ncu.log 2>&1; echo "sweep ncu rc=$?"
ENVS=2048 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gru_seq -s 4 -c 2 -o gpurun_out/prof_gru python scripts/profile_step.py > gpurun_out/ncu_gru.log 2>&1; echo "ncu gru rc=$?"
timeout -s KILL 900 ncu --profile-from-start off --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tensor_pipe.csv python scripts/traffic_step.py > gpurun_out/tensor_pipe.log 2>&1; echo "ncu tensor rc=$?"
ls -la gpurun_out
