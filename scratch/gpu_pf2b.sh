O=gpurun_out
timeout 300 python scratch/ln_cmp.py scratch/fav/cur.so scratch/fav/pf2b.so > $O/pf2b.log 2>&1
timeout 300 python scratch/ln_bench.py scratch/fav/cur.so scratch/fav/pf2b.so scratch/fav/cur.so scratch/fav/pf2b.so >> $O/pf2b.log 2>&1
