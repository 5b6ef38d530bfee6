cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm" > gpurun_out/pairs.log 2>&1; echo "rc=$?" >> gpurun_out/pairs.log
timeout 200 python scratch/gemm_bench.py >> gpurun_out/pairs.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
SB_GEMM_PAIRS=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_t1.json 2> gpurun_out/bench_t1.err
