cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "parity" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bdrln" -c 10 --csv --log-file gpurun_out/launches_ln.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
