O=gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "bias_grad or c2_config or bf16" > $O/qkvb_tests.log 2>&1; echo "rc=$?" >> $O/qkvb_tests.log
timeout 300 python scratch/bwd_ab.py scratch/fav/head.so@1 paper_2302_08005_b200/libslapo_b200.so@1 > $O/qkvb_bwd.log 2>&1
cp paper_2302_08005_b200/libslapo_b200.so /tmp/new.so
for v in new head new head; do
  if [ $v = head ]; then cp scratch/fav/head.so paper_2302_08005_b200/libslapo_b200.so; else cp /tmp/new.so paper_2302_08005_b200/libslapo_b200.so; fi
  timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/n1_q.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/n1_q.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['gpu_launches'])" >> $O/qkvb_ab.log
done
cp /tmp/new.so paper_2302_08005_b200/libslapo_b200.so
