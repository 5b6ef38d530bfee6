#!/bin/bash
# one GPU session: tests, bench, launch list, ncu full of the hot kernels
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --no-cpu-baseline --profile --steps 5 > gpurun_out/bench_prof.json 2> gpurun_out/bench_prof.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_gemm_tc|k_fa_fwd|k_fa_dkdv|k_fa_dq|k_dropout_mask" -c 6 -o gpurun_out/prof python profiles/ncu_targets.py > gpurun_out/ncu_full.log 2>&1
echo done
