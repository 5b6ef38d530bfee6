#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
SB_PARITY_OUT=$O/parity timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_kernels_gpu.py tests/test_causal_gpu.py -x -q -p no:cacheprovider -k "t5 or tcgen05 or causal or decoder" > $O/cross.log 2>&1; echo "rc=$?" >> $O/cross.log
timeout 600 python profiles/bench_t5.py > $O/t5_bench2.json 2> $O/t5_bench2.err
