import sys, numpy as np
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
L_ = sb.lib()
def rl2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel(); b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
def run(L, H, heads, V, S, dt, mode="train", B=1):
    m = sb.toy_bert(L, H, heads, V, B, S, 0.1)
    s = sb.create_schedule(m, 1); s.load_script(recipes.tp_script(L, 1, ckpt_ratio=0.25))
    ex = sb.Executor(s.apply(), mode, 123, 1, dtype=dt)
    o = ex.forward(m.random_inputs(9))[0]
    return o, ex.backward().params
for (L, H, heads, V, S) in [(4, 1024, 16, 30528, 512), (4, 1024, 16, 30528, 128), (4, 512, 8, 30528, 512), (4, 1024, 16, 64, 512), (4, 256, 4, 30528, 512)]:
    o32, g32 = run(L, H, heads, V, S, "fp32")
    res = []
    for eng in (0, 1):
        L_.sb_attn_set_engine(eng)
        o16, g16 = run(L, H, heads, V, S, "bf16")
        res.append((eng, L_.sb_attn_engine(0), rl2(o16, o32), rl2(g16['embeddings.weight'], g32['embeddings.weight'])))
    L_.sb_attn_set_engine(0)
    print(f"L{L} H{H} nh{heads} V{V} S{S}:", res, flush=True)
