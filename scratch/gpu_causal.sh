cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_causal_gpu.py -x -q > gpurun_out/causal.log 2>&1; echo "rc=$?" >> gpurun_out/causal.log
