#!/bin/bash
# conv1 kernels: model parity tests + per-kernel timing (+ optional ncu capture: NCU=name KREGEX=...)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 150 python -m pytest tests/test_model_gpu.py tests/test_parity_prod_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/c1_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c1_tests.log
timeout -s KILL 120 python scripts/profile_step.py > gpurun_out/c1_prof.txt 2>&1; echo "prof rc=$?"; grep -E "conv1|conv2|dgrad|gru_infer|taps|wall" gpurun_out/c1_prof.txt | head -8
if [ -n "$NCU" ]; then KREGEX="${KREGEX:-conv1_s2d}" NAME=$NCU SKIP=${SKIP:-2} COUNT=1 bash scripts/gpu_ncu_kernel.sh; fi
