#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_abi_kernels_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider > $O/r2c_tests.log 2>&1; echo "rc=$?" >> $O/r2c_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/r2c_bench$i.json 2>/dev/null; done
timeout 900 python profiles/bench_c4.py > $O/r2c_c4.json 2>&1
