O=gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm or forward or dgrad or wgrad" > $O/ragged_tests.log 2>&1
timeout 300 python scratch/lmhead_bench.py > $O/lmhead.log 2>&1
timeout 600 python3 profiles/bench_c4.py --batch 8 > $O/c4_ragged.json 2> $O/c4_ragged.err
timeout 600 python3 profiles/bench_t5.py > $O/t5_ragged.json 2> $O/t5_ragged.err
