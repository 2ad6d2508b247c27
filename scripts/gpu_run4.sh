cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/t_all.log
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/profile_step.txt 2>&1; echo "profile rc=$?"
grep -A12 "learner step (2048 samples) \[None\]" gpurun_out/profile_step.txt; tail -3 gpurun_out/profile_step.txt
timeout -s KILL 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_full.log
