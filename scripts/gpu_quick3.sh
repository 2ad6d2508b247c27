cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -4 gpurun_out/t_all.log
ENVS=2048 timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/profile_step.txt 2>&1; echo "profile rc=$?"
grep -A6 "learner step (2048 samples) \[None\]" gpurun_out/profile_step.txt; tail -3 gpurun_out/profile_step.txt
