O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/biasepi_tests.log 2>&1; echo "rc=$?" >> $O/biasepi_tests.log
for f in 0 1 0 1; do SB_BIAS_EPI=$f timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/n1_be$f.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/n1_be$f.json').read().strip().splitlines()[-1]); print('SB_BIAS_EPI=$f', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['gpu_launches'])" >> $O/biasepi_ab.log; done
for f in 0 1; do SB_BIAS_EPI=$f timeout 600 python3 profiles/bench_c4.py --batch 8 > $O/c4_be$f.json 2>/dev/null; grep -o '"ms_per_step": [0-9.]*' $O/c4_be$f.json | sed "s/^/C4 SB_BIAS_EPI=$f /" >> $O/biasepi_ab.log; done
