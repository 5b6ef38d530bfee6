O=gpurun_out
for p in 0.1 0.0 0.1 0.0; do timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --p $p > $O/n1_p$p.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/n1_p$p.json').read().strip().splitlines()[-1]); print('p=$p', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['gpu_launches'])" >> $O/p0_ab.log; done
timeout 600 python3 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --profile > /dev/null 2> $O/prof_p01.err
timeout 600 python3 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --profile --p 0.0 > /dev/null 2> $O/prof_p00.err
