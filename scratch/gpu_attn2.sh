cd $GRAFT_REPO_ROOT
timeout 300 python scratch/attn_bench.py > gpurun_out/attn2.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "flash or attention" >> gpurun_out/attn2.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q >> gpurun_out/attn2.log 2>&1
