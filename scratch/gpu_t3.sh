#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_causal_gpu.py -x -q -p no:cacheprovider > $O/t3_kern.log 2>&1; echo "rc=$?" >> $O/t3_kern.log
timeout 300 python scratch/attn_bench.py > $O/attn_bench.log 2>&1
SB_PARITY_OUT=$O/parity timeout 1500 python -m pytest tests/test_cli.py tests/test_c3_parity_gpu.py -x -q -p no:cacheprovider -k "verify_train or depth" --durations=10 > $O/t3_new.log 2>&1; echo "rc=$?" >> $O/t3_new.log
