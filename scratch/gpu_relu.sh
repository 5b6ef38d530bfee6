O=gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_decoder_gpu.py tests/test_pipeline_train_gpu.py -m gpu -x -q -p no:cacheprovider -k "relu or t5 or gemm" > $O/relu_tests.log 2>&1; echo "rc=$?" >> $O/relu_tests.log
for i in 1 2; do timeout 600 python3 profiles/bench_t5.py > $O/t5_relu$i.json 2> $O/t5_relu.err; done
SB_RELU_FUSE=0 timeout 600 python3 profiles/bench_t5.py > $O/t5_norelu.json 2>> $O/t5_relu.err
