O=gpurun_out
timeout 900 python -m pytest tests/test_abi_kernels_gpu.py tests/test_parity_gpu.py tests/test_decoder_gpu.py tests/test_kernels_gpu.py -m gpu -x -q > $O/ln5_tests.log 2>&1
timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/ln5_n1.json 2> $O/ln5_n1.err
timeout 600 python3 profiles/bench_c4.py --batch 8 > $O/ln5_c4.json 2> $O/ln5_c4.err
timeout 600 python3 profiles/bench_t5.py > $O/ln5_t5.json 2> $O/ln5_t5.err
