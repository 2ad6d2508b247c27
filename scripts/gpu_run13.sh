cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_sampler_gpu.py tests/test_model_gpu.py -q -p no:cacheprovider -x > gpurun_out/t_s.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_s.log
for S in 0 116 80; do
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --sampler-sms $S > gpurun_out/bench_s$S.log 2>&1; echo "sms=$S rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_s$S.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['last_step']['lag_mean'], d['last_step']['lag_max'])"
done
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --no-overlap > gpurun_out/bench_no.log 2>&1; echo "noov rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_no.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['last_step']['lag_mean'])"
