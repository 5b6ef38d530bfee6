O=gpurun_out
timeout 300 python scratch/bwd_ab.py scratch/fav/nosplit.so@1 paper_2302_08005_b200/libslapo_b200.so@1 > $O/bwd_grp.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_causal_gpu.py -m gpu -x -q -p no:cacheprovider -k "attn or causal or bwd" > $O/grp_tests.log 2>&1
DBGS=0 SB_ATTN_TS=0 timeout 120 python scratch/ts7.py > $O/grp_ts.log 2>&1
