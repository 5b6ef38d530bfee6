cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gemm2|k_fa6_fwd|k_fa5_bwd|k_dropout_mask_dual" -s 8 -c 6 -o gpurun_out/prof_r1b python profiles/ncu_targets.py > gpurun_out/ncu_r1b.log 2>&1
