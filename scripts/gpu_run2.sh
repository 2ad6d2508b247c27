cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/t_all.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --envs 2048 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo "bench small rc=$?"
tail -c 3000 gpurun_out/bench_small.log
