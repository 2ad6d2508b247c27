cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -4 gpurun_out/t_all.log
timeout -s KILL 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench_full.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --envs 2048 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launch rc=$?"
ENVS=2048 timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_bf16 --csv --log-file gpurun_out/gemm_traffic.csv python scripts/profile_step.py > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 30 -c 2 -o gpurun_out/prof_gemm_bench python bench.py --envs 2048 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
