import sys, re, numpy as np
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
SPLIT1 = "trace encoder.layer\npipeline_split encoder.layer after=1\n"
cfg = dict(layers=4, hidden=32, heads=4, vocab=32, batch=4, seq=8, p=0.1)
m = sb.toy_bert(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])
def stage1(script):
    s = sb.create_schedule(m, 2); s.load_script(script + SPLIT1); return s.apply_pipeline().stages[1]
st_tp = stage1(recipes.tp_script(4, 2, fuse=False, shard_embeddings=False))
st_1 = stage1("")
print(st_tp.consumes, st_1.consumes)
rng = np.random.default_rng(0)
xs = [rng.normal(size=(4, 8, 32)) for _ in st_1.consumes]
e1 = sb.Executor(st_1.module, "verify", 123, 1); o1 = e1.forward(xs)[0]; g1 = e1.backward()
e2 = sb.Executor(st_tp.module, "verify", 123, 2); o2 = e2.forward(xs)[0]; g2 = e2.backward_all_ranks()
print("out", np.abs(o1 - o2).max())
for i in range(len(xs)):
    a = g1.inputs[i]; b0 = g2[0].inputs[i]; b1 = g2[1].inputs[i]
    print("input", i, "w1 vs r0", np.abs(a-b0).max()/np.abs(a).max(), "r0 vs r1", np.abs(b0-b1).max()/np.abs(a).max(), "r0+r1 vs w1", np.abs(a-(b0+b1)).max()/np.abs(a).max())
