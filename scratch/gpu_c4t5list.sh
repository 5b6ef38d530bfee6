O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 1500 --csv --log-file $O/c4_launches.csv \
    python profiles/bench_c4.py --batch 8 --steps 2 --warmup 3 > $O/c4_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 1500 --csv --log-file $O/t5_launches.csv \
    python profiles/bench_t5.py --steps 2 > $O/t5_ncu.log 2>&1
