cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_causal_gpu.py tests/test_kernels_gpu.py -x -q -k "causal or attention or flash" > gpurun_out/causal6.log 2>&1; echo "rc=$?" >> gpurun_out/causal6.log
timeout 200 python scratch/attn_bench.py >> gpurun_out/causal6.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q >> gpurun_out/causal6.log 2>&1; echo "rc=$?" >> gpurun_out/causal6.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err
