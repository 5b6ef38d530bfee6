cd $GRAFT_REPO_ROOT
for sp in 1; do echo "SPLIT=$sp"; SB_ATTN_BWD_SPLIT=$sp timeout 300 python scratch/attn_bench.py 2>&1 | head -1; done > gpurun_out/bwd2.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "flash or attention" >> gpurun_out/bwd2.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q >> gpurun_out/bwd2.log 2>&1
