import sys, re, numpy as np
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
C3 = dict(layers=24, hidden=1024, heads=16, vocab=30528, batch=8, seq=512, p=0.1)
m = sb.toy_bert(C3["layers"], C3["hidden"], C3["heads"], C3["vocab"], C3["batch"], C3["seq"], C3["p"])
s = sb.create_schedule(m, 1); s.load_script(recipes.tp_script(24, 1, ckpt_ratio=0.25)); a = s.apply()
x = m.random_inputs(11)
ref = None
N = int(sys.argv[1]) if len(sys.argv) > 1 else 12
for t in range(N):
    ex = sb.Executor(a, mode="train", seed=2024, world=1, dtype="bf16")
    out = ex.forward(x); g = ex.backward(); del ex
    if ref is None:
        ref = (out, g); continue
    bad = [k for k, v in ref[1].params.items() if not np.array_equal(v, g.params[k])]
    od = [i for i, (u, w) in enumerate(zip(ref[0], out)) if not np.array_equal(u, w)]
    layers = sorted({int(re.search(r"layer\.(\d+)\.", k).group(1)) for k in bad if "layer." in k})
    print(f"run {t}: outputs differ {od}; {len(bad)} grads differ; layers {layers[-3:] if layers else []}", flush=True)
    if bad:
        top = max(layers) if layers else None
        print("   in top layer:", [k for k in bad if top is not None and f"layer.{top}." in k])
        print("   non-layer:", [k for k in bad if "layer." not in k])
