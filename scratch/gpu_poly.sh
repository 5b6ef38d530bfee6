cd $GRAFT_REPO_ROOT
for pl in 0 1 2; do echo "POLY=$pl"; SB_ATTN_POLY=$pl timeout 300 python scratch/attn_bench.py 2>&1 | head -2; done > gpurun_out/poly.log 2>&1
SB_ATTN_POLY=2 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "tcgen05_forward" >> gpurun_out/poly.log 2>&1
