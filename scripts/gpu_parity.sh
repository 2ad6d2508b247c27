#!/bin/bash
# GPU parity run: the whole -m gpu suite, observed errors logged to gpurun_out/
mkdir -p gpurun_out
export APPO_PARITY_LOG=$PWD/gpurun_out/parity_errors.jsonl
rm -f $APPO_PARITY_LOG
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout ${1:-1500} python -m pytest tests -m gpu -q -rA ${@:2} > gpurun_out/gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/gpu_tests.log
tail -30 gpurun_out/gpu_tests.log
