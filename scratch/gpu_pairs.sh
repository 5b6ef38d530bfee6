cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm" > gpurun_out/pairs.log 2>&1; echo "rc=$?" >> gpurun_out/pairs.log
for pp in 1 2; do echo "PAIRS=$pp" >> gpurun_out/pairs.log; SB_GEMM_DBG=1 SB_GEMM_PAIRS=$pp timeout 200 python scratch/gemm_bench.py >> gpurun_out/pairs.log 2>&1; done
