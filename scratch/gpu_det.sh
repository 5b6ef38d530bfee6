cd $GRAFT_REPO_ROOT
for sp in 2 0 0; do echo "SPLITS=$sp"; SB_GEMM_SPLITS=$sp timeout 600 python -m pytest tests/test_fullsize_gpu.py -x -q -k determin 2>&1 | tail -3; done > gpurun_out/det.log 2>&1
