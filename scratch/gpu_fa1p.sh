O=gpurun_out
timeout 400 python scratch/fa_ab.py scratch/fav/fa_c4_p0.so paper_2302_08005_b200/libslapo_b200.so > $O/fa_ab2.log 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_causal_gpu.py tests/test_decoder_gpu.py tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider > $O/fa1p_tests.log 2>&1
timeout 600 python3 profiles/bench_c4.py --batch 8 > $O/c4_fa1p.json 2> $O/c4_fa1p.err
timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/n1_fa1p.json 2> $O/n1_fa1p.err
