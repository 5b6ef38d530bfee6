cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm or forward_tn or dgrad or wgrad or gelu_epilogue or simt" > gpurun_out/t_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/t_gemm.log
python scratch/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
python scratch/gemm_ts.py > gpurun_out/gemm_ts.log 2>&1
