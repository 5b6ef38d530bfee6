cp paper_2302_08005_b200/libslapo_b200.so /tmp/l.so
python scratch/ln_bench.py /tmp/l.so > gpurun_out/ln_wpr.log 2>&1
SB_LN_WPR=2 python scratch/ln_bench.py /tmp/l.so >> gpurun_out/ln_wpr.log 2>&1
