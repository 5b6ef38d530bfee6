O=gpurun_out
cp paper_2302_08005_b200/libslapo_b200.so /tmp/new.so
timeout 300 python scratch/ln_cmp.py scratch/fav/head.so /tmp/new.so > $O/lnpk.log 2>&1
timeout 300 python scratch/ln_bench.py scratch/fav/head.so /tmp/new.so scratch/fav/head.so /tmp/new.so >> $O/lnpk.log 2>&1
