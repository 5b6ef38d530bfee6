#!/bin/bash
# the driver's two bench commands + ncu full of the attention / keep-bit / LN kernels
mkdir -p gpurun_out; O=gpurun_out
bash scratch/gpu_bench.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fa6_fwd|k_fa7_bwd|k_dropout_mask_dual" -s 4 -c 4 -o $O/prof_r2a python profiles/ncu_targets.py > $O/ncu_r2a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ln_bwd_w|k_bdrln_fwd_w|k_bias_partial_v" -s 30 -c 3 -o $O/prof_r2a_ln python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-graph > $O/ncu_r2a_ln.log 2>&1
