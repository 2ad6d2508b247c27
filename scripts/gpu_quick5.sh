cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_model_gpu.py tests/test_sampler_gpu.py -q -p no:cacheprovider -x > gpurun_out/t_m.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/t_m.log
timeout -s KILL 300 python scripts/profile_step.py > gpurun_out/profile_step.txt 2>&1; echo "profile rc=$?"
grep -A10 "inference step (16384 envs) \[gemm_shapes\]" gpurun_out/profile_step.txt; tail -3 gpurun_out/profile_step.txt
