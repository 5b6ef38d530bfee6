O=gpurun_out
timeout 300 python scratch/ln_cmp.py scratch/fav/cur.so scratch/fav/onewave.so > $O/onewave.log 2>&1
timeout 300 python scratch/ln_bench.py scratch/fav/cur.so scratch/fav/onewave.so scratch/fav/cur.so scratch/fav/onewave.so >> $O/onewave.log 2>&1
