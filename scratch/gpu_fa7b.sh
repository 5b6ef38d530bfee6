#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "attention or attn" > $O/fa7_t.log 2>&1; echo "rc=$?" >> $O/fa7_t.log
timeout 300 python scratch/ts7.py > $O/ts7.log 2>&1
