cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/clk1.json 2> gpurun_out/clk1.err
timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/clk2.json 2> gpurun_out/clk2.err
