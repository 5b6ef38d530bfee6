#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests/test_pipeline_train_gpu.py tests/test_pipeline.py -x -q -p no:cacheprovider > $O/pp.log 2>&1; echo "rc=$?" >> $O/pp.log
