cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
ENVS=2048 timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/profile_step.txt 2>&1; echo "profile rc=$?"
grep -A40 "learner step (2048 samples) \[gemm_shapes\]" gpurun_out/profile_step.txt | head -42
ENVS=2048 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gru_seq -s 4 -c 2 -o gpurun_out/prof_gru python scripts/profile_step.py > gpurun_out/ncu_gru.log 2>&1; echo "ncu rc=$?"
