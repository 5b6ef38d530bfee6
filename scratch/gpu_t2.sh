#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests/test_nccl_gpu.py tests/test_parity_gpu.py tests/test_c3_parity_gpu.py -x -q -p no:cacheprovider > $O/t2.log 2>&1; echo "rc=$?" >> $O/t2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fa5_bwd" -s 1 -c 1 -o $O/bwd_r2a python profiles/ncu_targets.py > $O/ncu_bwd.log 2>&1
