cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm" > gpurun_out/dgelu.log 2>&1; echo "rc=$?" >> gpurun_out/dgelu.log
timeout 200 python scratch/gemm_bench.py >> gpurun_out/dgelu.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_parity_gpu.py -x -q >> gpurun_out/dgelu.log 2>&1; echo "rc=$?" >> gpurun_out/dgelu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_dg.json 2> gpurun_out/bench_dg.err
