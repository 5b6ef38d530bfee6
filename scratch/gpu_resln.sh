#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
SB_PARITY_OUT=$O/parity timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_pipeline_train_gpu.py tests/test_parity_gpu.py tests/test_causal_gpu.py -x -q -p no:cacheprovider > $O/resln.log 2>&1; echo "rc=$?" >> $O/resln.log
timeout 600 python profiles/bench_c4.py > $O/c4_resln.json 2>&1
timeout 600 python profiles/bench_t5.py > $O/t5_resln.json 2>&1
