O=gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -p no:cacheprovider -k "gemm or wgrad" > $O/skr_tests.log 2>&1; echo "rc=$?" >> $O/skr_tests.log
cp paper_2302_08005_b200/libslapo_b200.so /tmp/new.so
for v in new cur new cur; do
  if [ $v = cur ]; then cp scratch/fav/cur.so paper_2302_08005_b200/libslapo_b200.so; else cp /tmp/new.so paper_2302_08005_b200/libslapo_b200.so; fi
  timeout 600 python3 profiles/bench_t5.py > $O/t5_skr.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/t5_skr.json')); print('T5 $v', round(d['ms_per_step'],2))" >> $O/skr_ab.log
  timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/n1_skr.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/n1_skr.json').read().strip().splitlines()[-1]); print('C3 $v', round(d['value'],1), round(d['ms_per_step'],2))" >> $O/skr_ab.log
done
cp /tmp/new.so paper_2302_08005_b200/libslapo_b200.so
