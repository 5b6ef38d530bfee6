cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_causal_gpu.py tests/test_kernels_gpu.py -x -q -k "causal or attention or flash" > gpurun_out/causal.log 2>&1; echo "rc=$?" >> gpurun_out/causal.log
