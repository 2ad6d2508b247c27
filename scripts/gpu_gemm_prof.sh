cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench.txt 2>&1; cat gpurun_out/gemm_bench.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/prof_gi python scripts/gemm_bench.py gi_infer > gpurun_out/ncu_gi.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/prof_c2 python scripts/gemm_bench.py conv2_dcol > gpurun_out/ncu_c2.log 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out/
