cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bdrln_fwd_w" -s 2 -c 1 -o gpurun_out/prof_bd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --layers 2 > /dev/null 2>&1
