#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
SB_PARITY_OUT=$O/parity timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1800 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/n1.out 2> $O/n1.err; echo "rc=$?" >> $O/n1.err
SB_ATTN_BWD=5 timeout 1800 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/n1_fa5.out 2> $O/n1_fa5.err
