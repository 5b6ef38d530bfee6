O=gpurun_out
timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_abi_kernels_gpu.py tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider > $O/w8_tests.log 2>&1; echo "rc=$?" >> $O/w8_tests.log
timeout 600 python3 profiles/bench_c4.py --batch 8 > $O/c4_w8.json 2> $O/c4_w8.err
