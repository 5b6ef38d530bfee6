import sys, numpy as np
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref
def rl2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel(); b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
def run(L, H, heads, V, mode, dt, ck=0.25, S=512, B=1):
    m = sb.toy_bert(L, H, heads, V, B, S, 0.1)
    s = sb.create_schedule(m, 1); s.load_script(recipes.tp_script(L, 1, ckpt_ratio=ck))
    ex = sb.Executor(s.apply(), mode, 123, 1, dtype=dt)
    o = ex.forward(m.random_inputs(9))[0]
    return o, ex.backward().params
for (L, H, heads, V) in [(4, 1024, 16, 30528), (8, 1024, 16, 30528), (8, 256, 4, 64), (16, 256, 4, 64)]:
    for mode in ("verify", "train"):
        o32, g32 = run(L, H, heads, V, mode, "fp32")
        o16, g16 = run(L, H, heads, V, mode, "bf16")
        o16b, _ = run(L, H, heads, V, mode, "bf16", ck=0.0)
        print(f"L{L} H{H} {mode}: bf16 vs fp32 out {rl2(o16, o32):.3e}  grad(emb) {rl2(g16['embeddings.weight'], g32['embeddings.weight']):.3e}  bf16 ckpt vs none {rl2(o16b, o16):.3e}", flush=True)
        if H == 256:
            with ref.run("toy_bert", schedule=recipes.tp_script(L, 1, ckpt_ratio=0.25), layers=L, hidden=H, heads=heads, vocab=V, batch=1, seq=512, p=0.1, world=1, mode=mode, seed=123, input_seed=9) as r:
                w = r.outputs(0)[0]
                print(f"   vs ref: fp32 {rl2(o32, w):.3e} bf16 {rl2(o16, w):.3e}", flush=True)
