cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_kernels_gpu.py -x -q -k "not gemm" > gpurun_out/ln4.log 2>&1; echo "rc=$?" >> gpurun_out/ln4.log
M="--metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_bdrln|k_ln_bwd -c 24 --csv"
timeout 600 ncu $M --log-file gpurun_out/ln4_new.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --layers 4 > /dev/null 2>&1
cp paper_2302_08005_b200/libslapo_b200.so /tmp/new.so; cp scratch/var/lib_lnold.so paper_2302_08005_b200/libslapo_b200.so
timeout 600 ncu $M --log-file gpurun_out/ln4_old.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --layers 4 > /dev/null 2>&1
cp /tmp/new.so paper_2302_08005_b200/libslapo_b200.so
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ln4.json 2> gpurun_out/bench_ln4.err
