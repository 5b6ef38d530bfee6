cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/t_attn.log 2>&1; echo "rc=$?" >> gpurun_out/t_attn.log
timeout 120 python scratch/attn_bench.py > gpurun_out/attn_bench.log 2>&1
timeout 120 python scratch/ts.py > gpurun_out/ts.log 2>&1
