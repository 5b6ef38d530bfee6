cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/t_attn.log 2>&1; echo "rc=$?" >> gpurun_out/t_attn.log
for nt in 1 2; do echo "nt=$nt"; SB_ATTN_FWD_NT=$nt timeout 120 python scratch/attn_bench.py 2>&1 | grep "engine cap 0: used 3 fwd"; done > gpurun_out/dbg.log 2>&1
