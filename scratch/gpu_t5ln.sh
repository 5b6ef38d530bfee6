O=gpurun_out
timeout 300 python scratch/ln_cmp.py scratch/fav/cur.so scratch/fav/t5ln.so > $O/t5ln2.log 2>&1
timeout 300 python scratch/bdfw_bench.py scratch/fav/cur.so scratch/fav/t5ln.so >> $O/t5ln2.log 2>&1
timeout 300 python scratch/ln_bench.py scratch/fav/cur.so scratch/fav/t5ln.so >> $O/t5ln2.log 2>&1
