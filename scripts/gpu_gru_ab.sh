#!/bin/bash
# grouped vs legacy GRU recurrence kernels on one box: parity tests, phases, warm durations
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_model_gpu.py tests/test_parity_prod_gpu.py tests/test_dp_gpu.py tests/test_checkpoint_gpu.py -q -p no:cacheprovider -x > gpurun_out/t_gru.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_gru.log
for L in 0 1 0 1; do
  export APPO_GRU_LEGACY=$L
  APPO_GRU_PROF=1 timeout -s KILL 300 python scripts/_prof_gru.py > gpurun_out/gru_prof_$L.log 2>&1; echo "== legacy=$L"; grep "gru prof" gpurun_out/gru_prof_$L.log | tail -2 | cut -c1-220
  timeout -s KILL 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/warm_g$L.csv python scripts/traffic_step.py > /dev/null 2>&1
  python scripts/warm_summary.py gpurun_out/warm_g$L.csv 2>/dev/null | grep "gru_seq\|total"
done
unset APPO_GRU_LEGACY
timeout -s KILL 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('value', d['value'], 'ms', d['ms_per_step'])"
