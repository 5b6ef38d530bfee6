cd $GRAFT_REPO_ROOT
for p in 0.1 0.0; do timeout 600 python bench.py --no-cpu-baseline --steps 5 --p $p --profile > gpurun_out/bench_p$p.json 2> gpurun_out/bench_p$p.err; done
