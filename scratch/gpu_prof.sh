cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemm" -c 4 -o gpurun_out/prof_gemm2 python scratch/gemm_one.py > gpurun_out/ncu_gemm.log 2>&1
