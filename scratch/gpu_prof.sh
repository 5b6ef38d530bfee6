cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bdrln_fwd_w|k_ln_bwd_w" -s 4 -c 2 -o gpurun_out/prof_ln python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --layers 2 > /dev/null 2>&1
