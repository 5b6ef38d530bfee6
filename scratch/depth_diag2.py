import sys, numpy as np
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref
def rl2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel(); b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
L, H, heads, V = 4, 1024, 16, 30528
sched = recipes.tp_script(L, 1, ckpt_ratio=0.25)
r = ref.run("toy_bert", schedule=sched, layers=L, hidden=H, heads=heads, vocab=V, batch=1, seq=512, p=0.1, world=1, mode="train", seed=123, input_seed=9, timeout=3000)
w = r.outputs(0)[0]; gw = r.grads(0)
for dt in ("fp32", "bf16"):
    m = sb.toy_bert(L, H, heads, V, 1, 512, 0.1)
    s = sb.create_schedule(m, 1); s.load_script(sched)
    ex = sb.Executor(s.apply(), "train", 123, 1, dtype=dt)
    o = ex.forward(m.random_inputs(9))[0]; g = ex.backward().params
    print(dt, "out", rl2(o, w), {k: round(rl2(g[k], v), 4) for k, v in gw.items() if "weight" in k and ("dense" in k or "qkv" in k)}, flush=True)
