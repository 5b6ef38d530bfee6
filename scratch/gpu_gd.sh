cd $GRAFT_REPO_ROOT
for d in 0 1 2 3; do echo "dbg=$d"; SB_GEMM_DBG=$d python scratch/gemm_bench.py 2>&1 | grep "dense1+gelu"; done > gpurun_out/gd.log
