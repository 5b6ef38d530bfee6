cd $GRAFT_REPO_ROOT
for pp in 1 0; do echo "PERSIST=$pp"; SB_ATTN_BWD_PERSIST=$pp timeout 300 python scratch/attn_bench.py 2>&1 | head -1; done > gpurun_out/bwdp.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "flash or attention" >> gpurun_out/bwdp.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q >> gpurun_out/bwdp.log 2>&1
