#!/bin/bash
# full GPU suite + bench + step profile
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest -x -q -m gpu tests > gpurun_out/full_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/full_tests.log
timeout -s KILL 300 python bench.py --no-cpu-baseline > gpurun_out/full_bench.log 2>&1
tail -1 gpurun_out/full_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks'])
for k in [d['roofline']]+d['roofline_kernels']: print(k['kernel'], k['bound'], round(k['frac'],3), round(k['avg_us'],1), k['launches'], round(k['share_of_step'],3))"
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/full_prof.txt 2>&1; grep wall gpurun_out/full_prof.txt
