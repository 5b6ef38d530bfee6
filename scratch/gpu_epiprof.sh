O=gpurun_out
for f in 1 0 1 0; do SB_BIAS_EPI=$f timeout 600 python3 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --profile > /dev/null 2> $O/prof_epi$f.err; python - >> $O/epiprof.log <<PY
import json, re
t = open("$O/prof_epi$f.err").read()
j = json.loads(t[t.index("{"):t.rindex("}") + 1])
print("SB_BIAS_EPI=$f", {k: round(v, 3) for k, v in j.items() if k in ("FusedLinearGelu(bwd)", "FusedLinearResLN(bwd)", "gemm")})
PY
done
