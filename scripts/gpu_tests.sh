cd $GRAFT_REPO_ROOT
nvidia-smi -L
export PYTHONUNBUFFERED=1
timeout -s KILL 300 python -m pytest tests/test_offpolicy_gpu.py -x -q -p no:cacheprovider > gpurun_out/t_off.log 2>&1; echo "offpolicy rc=$?"
tail -5 gpurun_out/t_off.log
timeout -s KILL 300 python -m pytest tests/test_gemm_gpu.py -q -p no:cacheprovider > gpurun_out/t_gemm.log 2>&1; echo "gemm rc=$?"
tail -25 gpurun_out/t_gemm.log
timeout -s KILL 400 python -m pytest tests/test_model_gpu.py -q -x -p no:cacheprovider > gpurun_out/t_model.log 2>&1; echo "model rc=$?"
tail -30 gpurun_out/t_model.log
