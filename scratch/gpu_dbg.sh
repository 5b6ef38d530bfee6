cd $GRAFT_REPO_ROOT
for d in 0 1 2 3 4 5 7; do echo "dbg=$d"; SB_ATTN_DBG=$d timeout 120 python scratch/attn_bench.py 2>&1 | grep "engine cap 0: used 3 bwd"; done > gpurun_out/dbg.log 2>&1
