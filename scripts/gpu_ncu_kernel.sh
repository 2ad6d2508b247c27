#!/bin/bash
# ncu --set full capture of one kernel (regex $KREGEX) from profile_step.py; report to gpurun_out/$NAME.ncu-rep
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${KREGEX}" -s ${SKIP:-2} -c ${COUNT:-1} -o gpurun_out/${NAME} python scripts/profile_step.py > gpurun_out/${NAME}.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${NAME}.log
