#!/bin/bash
# Round-end measurement set: GPU tests, bench (both arms), per-kernel step
# profile, ncu launch list of the bench command and the DRAM-traffic capture.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_tests.log
timeout -s KILL 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final_bench.log | cut -c1-300
timeout -s KILL 900 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_bench_ref.log | cut -c1-200
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/final_profile_step.txt 2>&1; echo "profile rc=$?"; tail -2 gpurun_out/final_profile_step.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --envs 2048 > gpurun_out/final_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_traffic.csv python scripts/traffic_step.py > gpurun_out/final_traffic.log 2>&1; echo "ncu traffic rc=$?"
