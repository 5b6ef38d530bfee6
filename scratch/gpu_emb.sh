cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_emb" --csv --log-file gpurun_out/emb.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph --layers 2 > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
