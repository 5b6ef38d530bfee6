O=gpurun_out
for mb in -1 148 296 74 592 -1; do
  if [ "$mb" = "-1" ]; then extra=""; else extra="--mask-blocks $mb"; fi
  timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline $extra > $O/n1_mb.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/n1_mb.json').read().strip().splitlines()[-1]); print('mask-blocks $mb', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> $O/mb_ab.log
done
