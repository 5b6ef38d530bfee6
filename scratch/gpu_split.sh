cd $GRAFT_REPO_ROOT
for sp in 0 1 2 3 4; do echo "SPLITS=$sp"; SB_GEMM_SPLITS=$sp timeout 300 python scratch/gemm_bench.py 2>&1 | grep wgrad; done > gpurun_out/split.log 2>&1
