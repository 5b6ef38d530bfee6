O=gpurun_out
timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_pipeline_train_gpu.py tests/test_abi_kernels_gpu.py -m gpu -x -q -p no:cacheprovider > $O/t5ln_tests.log 2>&1; echo "rc=$?" >> $O/t5ln_tests.log
for i in 1 2; do timeout 600 python3 profiles/bench_t5.py > $O/t5_ln$i.json 2> $O/t5_ln.err; done
