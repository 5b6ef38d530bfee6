cd $GRAFT_REPO_ROOT
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm_2sm_vs_1sm and tn_bias and tileN-256 or tcgen05_forward and 256" > gpurun_out/sanit_mem.log 2>&1; echo "rc=$?" >> gpurun_out/sanit_mem.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm_2sm_vs_1sm and nn_dgelu and tileN-256" > gpurun_out/sanit_race.log 2>&1; echo "rc=$?" >> gpurun_out/sanit_race.log
