#!/bin/bash
# One build->measure iteration on the GPU box: GPU tests, per-kernel step profile, short bench.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "gpu tests rc=$?"
tail -8 gpurun_out/t_all.log
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/profile_step.txt 2>&1; echo "profile rc=$?"
grep -B2 -A40 "learner step (2048 samples) \[gemm_shapes\]" gpurun_out/profile_step.txt | head -50; tail -3 gpurun_out/profile_step.txt
if [ "${BENCH:-1}" = "1" ]; then
timeout -s KILL 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'])"
fi
