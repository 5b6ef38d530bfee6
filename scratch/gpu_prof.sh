cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fa5_bwd" -c 1 -o gpurun_out/prof_bwd4 python profiles/ncu_targets.py > gpurun_out/ncu_b.log 2>&1
