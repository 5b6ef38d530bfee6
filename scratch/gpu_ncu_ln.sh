#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ln_bwd_w|k_bias_partial_v|k_splitk_reduce|k_col_final" -s 200 -c 6 -o $O/prof_r2_lnb python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-graph > $O/ncu_lnb.log 2>&1
