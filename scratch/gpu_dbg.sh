cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/t_attn.log 2>&1; echo "rc=$?" >> gpurun_out/t_attn.log
for d in 0 7; do echo "dbg=$d"; SB_ATTN_DBG=$d timeout 120 python scratch/attn_bench.py 2>&1 | grep "engine cap 0: used 3 bwd"; done > gpurun_out/dbg.log 2>&1
