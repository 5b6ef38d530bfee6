#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 600 python -m pytest tests/test_abi_kernels_gpu.py tests/test_integration.py -q -p no:cacheprovider > $O/abi.log 2>&1; echo "rc=$?" >> $O/abi.log
