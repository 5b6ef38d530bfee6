#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python profiles/bench_c4.py > $O/c4.json 2> $O/c4.err
timeout 900 python profiles/bench_c4.py --layers 24 --batch 16 > $O/c4_b16.json 2>> $O/c4.err
timeout 900 python bench.py --steps 10 --warmup 3 --profile --no-cpu-baseline > $O/bench_prof.json 2> $O/bench_prof.err
SB_PARITY_OUT=$O/parity timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
