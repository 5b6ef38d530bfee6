import sys, re, numpy as np, torch
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
B = int(sys.argv[1]); W = int(sys.argv[2]); MODE = sys.argv[3]
L = 24
def model(ck):
    m = sb.toy_bert(L, 1024, 16, 30528, B, 512, 0.1)
    s = sb.create_schedule(m, W); s.load_script(recipes.tp_script(L, W, ckpt_ratio=ck)); return m, s.apply()
def run(a, x):
    ex = sb.Executor(a, mode=MODE, seed=77, world=W, dtype="bf16")
    out = ex.forward(x); g = ex.backward_all_ranks(); del ex
    return out, g
def poison(val):
    free, _ = torch.cuda.mem_get_info()
    t = torch.empty(int(free * 0.9) // 4, dtype=torch.int32, device="cuda")
    t.fill_(val); torch.cuda.synchronize(); del t; torch.cuda.empty_cache()
m, a0 = model(0.0)
x = m.random_inputs(5)
ref = run(a0, x)
_, a1 = model(0.25)
for val in (0, 0x7fc00000, 0x3f800000):
    poison(val)
    out, gs = run(a1, x)
    od = [i for i, (u, w) in enumerate(zip(ref[0], out)) if not np.array_equal(u, w)]
    nbad = 0; first = []
    for r in range(W):
        bad = [k for k, v in ref[1][r].params.items() if not np.array_equal(v, gs[r].params[k])]
        nbad += len(bad); first += bad[:3]
    print(f"B={B} W={W} {MODE} poison {val:#x}: outputs differ {od}; {nbad} grads differ {first}", flush=True)
