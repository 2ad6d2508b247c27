cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -8 gpurun_out/t_all.log
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/profile_step.txt 2>&1; echo "profile rc=$?"
grep -A10 "inference step (16384 envs) \[gemm_shapes\]" gpurun_out/profile_step.txt; tail -3 gpurun_out/profile_step.txt
timeout -s KILL 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])"
