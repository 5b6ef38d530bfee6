#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 300 python scratch/ts7.py > $O/ts7.log 2>&1
timeout 300 python -m pytest tests/test_nccl_gpu.py -x -q -p no:cacheprovider > $O/nccl_t.log 2>&1; echo "rc=$?" >> $O/nccl_t.log
