#!/bin/bash
# the driver's two bench commands, in its order, with wall clocks and disk checks
mkdir -p gpurun_out; O=gpurun_out
df -h /tmp . > $O/df_before.txt
t0=$(date +%s.%N)
timeout 1800 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref1.out 2> $O/ref1.err; echo "rc=$?" >> $O/ref1.err
t1=$(date +%s.%N)
df -h /tmp . > $O/df_mid.txt
timeout 1800 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/n1.out 2> $O/n1.err; echo "rc=$?" >> $O/n1.err
t2=$(date +%s.%N)
df -h /tmp . > $O/df_after.txt
echo "ref_wall $(echo "$t1 - $t0" | bc) ours_wall $(echo "$t2 - $t1" | bc)" > $O/walls.txt
timeout 300 python scratch/attn_bench.py > $O/attn_bench.log 2>&1
SB_ATTN_TS=1 timeout 120 python scratch/ts.py > $O/attn_ts.log 2>&1
