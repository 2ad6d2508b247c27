#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest ${TESTS:-tests/test_offpolicy_gpu.py tests/test_model_gpu.py tests/test_rollout_gpu.py tests/test_gemm_gpu.py tests/test_parity_prod_gpu.py} -q -p no:cacheprovider -x > gpurun_out/t_iter.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t_iter.log
APPO_GRU_PROF=1 timeout -s KILL 300 python scripts/_prof_gru.py > gpurun_out/gru_prof.log 2>&1; grep "gru prof" gpurun_out/gru_prof.log | tail -2
timeout -s KILL 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/warm_step.csv python scripts/traffic_step.py > gpurun_out/warm_step.log 2>&1; echo "warm rc=$?"
python scripts/warm_summary.py gpurun_out/warm_step.csv | head -24
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['h2d_gbps'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['avg_us'])"
