#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
SB_PARITY_OUT=$O/parity timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_causal_gpu.py tests/test_kernels_gpu.py -k "decoder or causal or tcgen05_forward" -x -q -p no:cacheprovider > $O/dec.log 2>&1; echo "rc=$?" >> $O/dec.log
timeout 300 python scratch/attn_bench.py > $O/attn_bench.log 2>&1
ATTN_CFG=8,1024,16,128 timeout 300 python scratch/attn_bench.py > $O/attn_bench128.log 2>&1
