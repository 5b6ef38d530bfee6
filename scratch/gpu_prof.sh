cd $GRAFT_REPO_ROOT
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_gemm2|k_gemm_tc|k_splitk" --csv --log-file gpurun_out/gemm_traffic.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/gemm_traffic.log 2>&1
