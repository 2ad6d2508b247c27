cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -4 gpurun_out/t_all.log
timeout -s KILL 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -c 2800 gpurun_out/bench_full.log
timeout -s KILL 1200 python bench.py --no-overlap --no-e2e --no-cpu-baseline > gpurun_out/bench_nooverlap.log 2>&1; echo "bench2 rc=$?"
tail -c 600 gpurun_out/bench_nooverlap.log | head -c 300
