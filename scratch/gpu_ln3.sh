cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q > gpurun_out/pytest_ln.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ln.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_bdrln|k_ln_bwd" -c 12 --csv --log-file gpurun_out/ln3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --layers 2 > /dev/null 2>&1
