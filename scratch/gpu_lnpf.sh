O=gpurun_out
timeout 300 python scratch/ln_cmp.py scratch/fav/head.so scratch/fav/pf2.so > $O/lnpf.log 2>&1
timeout 300 python scratch/ln_bench.py scratch/fav/head.so scratch/fav/pf2.so scratch/fav/head.so scratch/fav/pf2.so >> $O/lnpf.log 2>&1
