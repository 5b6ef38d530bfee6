cd $GRAFT_REPO_ROOT
for d in 0 5 13; do echo "DBG=$d"; SB_ATTN_DBG=$d SB_ATTN_FWD_NT=6 timeout 300 python scratch/attn_bench.py 2>&1 | head -1; done > gpurun_out/attn6d.log 2>&1
