cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -8 gpurun_out/t_all.log
timeout -s KILL 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench_full.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --envs 2048 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu rc=$?"
