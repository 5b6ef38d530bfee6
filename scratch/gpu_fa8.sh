#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -k "tcgen05_backward" -x -q -p no:cacheprovider > $O/fa8.log 2>&1; echo "rc=$?" >> $O/fa8.log
timeout 600 python -m pytest tests/test_causal_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider >> $O/fa8.log 2>&1; echo "rc=$?" >> $O/fa8.log
ATTN_CFG=8,1024,16,128 timeout 300 python scratch/attn_bench.py > $O/attn_bench128.log 2>&1
