#!/bin/bash
# build -> measure iteration: focused GPU tests, HBM sweep, per-kernel step profile, bench
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest ${TESTS:-tests/test_offpolicy_gpu.py tests/test_model_gpu.py tests/test_rollout_gpu.py} -q -p no:cacheprovider -x > gpurun_out/t_iter.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t_iter.log
timeout -s KILL 300 python scripts/hbm_sweep.py > gpurun_out/hbm_sweep.jsonl 2> gpurun_out/hbm_sweep.err; echo "sweep rc=$?"; cut -c1-160 gpurun_out/hbm_sweep.jsonl
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/profile_step.txt 2>&1; echo "profile rc=$?"
grep -A32 "learner step (2048 samples) \[gemm_shapes\]" gpurun_out/profile_step.txt | head -34; tail -3 gpurun_out/profile_step.txt
if [ "${BENCH:-1}" = "1" ]; then
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['h2d_gbps'], d['roofline']['kernel'], d['roofline']['frac'])"
fi
