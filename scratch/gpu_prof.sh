cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fa5_bwd" -c 1 -o gpurun_out/prof_bwd3 python profiles/ncu_targets.py > gpurun_out/ncu_attn.log 2>&1
