cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for S in 0 116 96 64; do
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --sampler-sms $S > gpurun_out/bench_s$S.log 2>&1; echo "sms=$S rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_s$S.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['last_step']['lag_mean'])"
done
