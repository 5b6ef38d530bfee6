cd $GRAFT_REPO_ROOT
for c in 0 1; do timeout 600 python bench.py --no-cpu-baseline --steps 5 --gemm-cap $c --profile > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
