#!/bin/bash
# Round-2 evidence set: GPU tests (observed parity errors logged), bench (both
# arms), per-kernel step profile, ncu launch list of the bench command, DRAM
# traffic + tensor-pipe per kernel class, --set full captures of conv1 forward
# (inference launch) and the GRU recurrence kernels.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/parity_errors.jsonl
APPO_PARITY_LOG=gpurun_out/parity_errors.jsonl timeout -s KILL 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final_bench.log | cut -c1-200
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_bench_ref.log | cut -c1-200
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/final_profile_step.txt 2>&1; echo "profile rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --envs 2048 > gpurun_out/final_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_traffic.csv python scripts/traffic_step.py > gpurun_out/final_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout -s KILL 900 ncu --profile-from-start off --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_tensor_pipe.csv python scripts/traffic_step.py > gpurun_out/final_tensor_pipe.log 2>&1; echo "ncu tensor rc=$?"
KREGEX="conv1_s2d_kernel" NAME=final_conv1 SKIP=2 COUNT=1 bash scripts/gpu_ncu_kernel.sh
ENVS=2048 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gru_g_ -s 4 -c 2 -o gpurun_out/final_gru python scripts/profile_step.py > gpurun_out/final_ncu_gru.log 2>&1; echo "ncu gru rc=$?"
APPO_GRU_PROF=1 timeout -s KILL 120 python scripts/_prof_gru.py 2>&1 | grep "gru prof" > gpurun_out/final_gru_phases.txt
KREGEX="traj_loss_kernel" NAME=final_traj_loss SKIP=2 COUNT=1 bash scripts/gpu_ncu_kernel.sh
timeout -s KILL 300 python scripts/hbm_sweep.py > gpurun_out/final_hbm_sweep.jsonl 2>&1; echo "hbm sweep rc=$?"
# (learner --set full capture: scripts/gpu_ncu_learner.sh, separate call: 64 MB report)
ls -la gpurun_out | head -40
