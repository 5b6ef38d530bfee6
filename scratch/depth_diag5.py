import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
Lb = sb.lib()
def rl2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel(); b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
def run(L, H, heads, V, S, dt, mode="train", B=1, world=1):
    m = sb.toy_bert(L, H, heads, V, B, S, 0.1)
    s = sb.create_schedule(m, world); s.load_script(recipes.tp_script(L, world, ckpt_ratio=0.25))
    ex = sb.Executor(s.apply(), mode, 123, world, dtype=dt)
    ex.forward(m.random_inputs(9))
    return ex.outputs_of_rank(0)[0], ex.backward_all_ranks()[0].params
for L in (1, 2, 4):
    o32, _ = run(L, 1024, 16, 30528, 512, "fp32")
    a, _ = run(L, 1024, 16, 30528, 512, "bf16")
    Lb.sb_attn_set_engine(1); b, _ = run(L, 1024, 16, 30528, 512, "bf16"); Lb.sb_attn_set_engine(0)
    c, _ = run(L, 1024, 16, 30528, 512, "bf16", world=2)
    Lb.sb_gemm_set_engine(1); d, _ = run(L, 1024, 16, 30528, 512, "bf16"); Lb.sb_gemm_set_engine(0)
    print(f"L{L}: tc vs fp32 {rl2(a,o32):.3e} | tc vs mma-attn {rl2(a,b):.3e} | tp1 vs tp2 {rl2(a,c):.3e} | gemm2 vs gemm1 {rl2(a,d):.3e}", flush=True)
