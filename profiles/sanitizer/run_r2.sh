# round 2: the kernels added this round (hd-128 attention fwd/bwd, causal hd-128) and the
# pipeline executor, under compute-sanitizer memcheck / racecheck (one GPU)
cd $GRAFT_REPO_ROOT
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "tcgen05_forward and 128-2-128 or tcgen05_backward and 128" > gpurun_out/sanit_r2_mem.log 2>&1; echo "rc=$?" >> gpurun_out/sanit_r2_mem.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_causal_gpu.py tests/test_pipeline_train_gpu.py -x -q -p no:cacheprovider -k "128 or verify_equals" > gpurun_out/sanit_r2_mem2.log 2>&1; echo "rc=$?" >> gpurun_out/sanit_r2_mem2.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "tcgen05_backward and 128-2-128-0.0" > gpurun_out/sanit_r2_race.log 2>&1; echo "rc=$?" >> gpurun_out/sanit_r2_race.log
