cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_cpp_host_gpu.py -q -p no:cacheprovider > gpurun_out/t_cpp.log 2>&1; echo "cpp rc=$?"; tail -3 gpurun_out/t_cpp.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_r2a.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r2a.log | cut -c1-3000
bash scripts/gpu_evidence.sh
