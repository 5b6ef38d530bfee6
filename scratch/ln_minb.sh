cp paper_2302_08005_b200/libslapo_b200.so /tmp/l.so
python scratch/ln_bench.py /tmp/l.so > gpurun_out/ln_minb2.log 2>&1
SB_LN_WPR=4 python scratch/ln_bench.py /tmp/l.so >> gpurun_out/ln_minb2.log 2>&1
