#!/bin/bash
# one GPU session: tests, smoke, the driver's two bench commands, launch list
mkdir -p gpurun_out
O=gpurun_out
{ nvidia-smi; nproc; df -h /tmp .; } > $O/env.txt 2>&1
SB_PARITY_OUT=$O/parity timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
df -h /tmp . > $O/df_before.txt
timeout 1800 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref1.out 2> $O/ref1.err; echo "rc=$?" >> $O/ref1.err
df -h /tmp . > $O/df_mid.txt
timeout 1800 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/n1.out 2> $O/n1.err; echo "rc=$?" >> $O/n1.err
df -h /tmp . > $O/df_after.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1000 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_list.log 2>&1
