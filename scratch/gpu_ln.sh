#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_ln.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ln.log
for nr in 1; do
SB_BDRLN_NR=$nr timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bdrln|k_ln_bwd" -c 12 --csv --log-file gpurun_out/ln_nr$nr.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --layers 2 > /dev/null 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ln.json 2> gpurun_out/bench_ln.err
echo done
