cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:gemm_bf16_kernel<32, false, false, 3, 2>|gen_obs" -s 2 -c 2 -o gpurun_out/prof_conv1 python scripts/profile_step.py > gpurun_out/ncu_conv1.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/ncu_conv1.log
