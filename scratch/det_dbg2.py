import sys, re, numpy as np, torch
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
C3 = dict(layers=int(sys.argv[1]) if len(sys.argv) > 1 else 24, hidden=1024, heads=16, vocab=30528, batch=8, seq=512, p=0.1)
L = C3["layers"]
def model(ck):
    m = sb.toy_bert(L, C3["hidden"], C3["heads"], C3["vocab"], C3["batch"], C3["seq"], C3["p"])
    s = sb.create_schedule(m, 1); s.load_script(recipes.tp_script(L, 1, ckpt_ratio=ck)); return m, s.apply()
def run(a, x):
    ex = sb.Executor(a, mode="train", seed=2024, world=1, dtype="bf16")
    out = ex.forward(x); g = ex.backward(); del ex
    return out, g
def poison(val):
    free, _ = torch.cuda.mem_get_info()
    t = torch.empty(int(free * 0.9) // 4, dtype=torch.int32, device="cuda")
    t.fill_(val); torch.cuda.synchronize(); del t; torch.cuda.empty_cache()
m, a0 = model(0.0)
x = m.random_inputs(11)
ref = run(a0, x)
_, a1 = model(0.25)
for val in (0, 0x7fc00000, 0x3f800000, -1, 0x7fc00000):
    poison(val)
    out, g = run(a1, x)
    bad = [k for k, v in ref[1].params.items() if not np.array_equal(v, g.params[k])]
    layers = sorted({int(re.search(r"layer\.(\d+)\.", k).group(1)) for k in bad if "layer." in k})
    nan = [k for k, v in g.params.items() if not np.isfinite(v).all()]
    print(f"poison {val:#x}: {len(bad)} grads differ (layers {layers[-4:]}); non-finite {len(nan)} {nan[:3]}", flush=True)
    top = max(layers) if layers else None
    if top is not None:
        print("   top:", [k.split('layer.')[1] for k in bad if f"layer.{top}." in k])
