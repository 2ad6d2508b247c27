#!/bin/bash
# Quick health check on a fresh box: GPU tests + one bench line.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/check_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/check_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/check_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/check_bench.log | cut -c1-400
