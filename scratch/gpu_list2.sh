cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "dropout" > gpurun_out/pytest_tie.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tie.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 802 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_list.log 2>&1
