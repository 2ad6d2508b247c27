#!/bin/bash
# fused loss block: learner parity tests, vtrace tests, HBM sweep, bench
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest -x -q tests/test_model_gpu.py tests/test_parity_prod_gpu.py tests/test_shapes_gpu.py tests/test_offpolicy_gpu.py > gpurun_out/tl_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tl_tests.log
timeout -s KILL 300 python scripts/hbm_sweep.py > gpurun_out/tl_hbm.jsonl 2>&1; grep returns gpurun_out/tl_hbm.jsonl | cut -c1-200
timeout -s KILL 300 python bench.py --no-cpu-baseline > gpurun_out/tl_bench.log 2>&1
tail -1 gpurun_out/tl_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks'])
for k in [d['roofline']]+d['roofline_kernels']: print(k['kernel'], k['bound'], round(k['frac'],3), round(k['avg_us'],1), k['launches'], round(k['share_of_step'],3))"
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/tl_prof.txt 2>&1; head -40 gpurun_out/tl_prof.txt | grep -v "^$" | head -34 | tail -24
