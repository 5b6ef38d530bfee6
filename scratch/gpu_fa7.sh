#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "attention or attn" > $O/fa7_t.log 2>&1; echo "rc=$?" >> $O/fa7_t.log
timeout 300 python scratch/attn_bench.py > $O/fa7_bench.log 2>&1
SB_ATTN_BWD=5 timeout 300 python scratch/attn_bench.py > $O/fa5_bench.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_nccl_gpu.py tests/test_fullsize_gpu.py -x -q -p no:cacheprovider > $O/fa7_par.log 2>&1; echo "rc=$?" >> $O/fa7_par.log
