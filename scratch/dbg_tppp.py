import sys, re, numpy as np
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
SPLIT1 = "trace encoder.layer\npipeline_split encoder.layer after=1\n"
cfg = dict(layers=4, hidden=32, heads=4, vocab=32, batch=4, seq=8, p=0.1)
for ck, micro, fuse, emb in [(0.25, 2, True, True), (0.0, 1, True, True), (0.0, 1, False, True), (0.0, 1, False, False)]:
    script = recipes.tp_script(4, 2, ckpt_ratio=ck, fuse=fuse, shard_embeddings=emb)
    m = sb.toy_bert(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])
    s = sb.create_schedule(m, 2); s.load_script(script + SPLIT1); plan = s.apply_pipeline()
    x = m.random_inputs(9)
    pe = sb.PipelineExecutor(plan, micro, "verify", 123, "fp32", tp=2)
    out = pe.forward(x); g = pe.backward()
    s2 = sb.create_schedule(m, 2); s2.load_script(script)
    ex = sb.Executor(s2.apply(), "verify", 123, 2); wo = ex.forward(x)[0]; want = [r.params for r in ex.backward_all_ranks()]
    print("cfg", ck, micro, fuse, emb, "out err", np.abs(out[0]-wo).max())
    for r in range(2):
        got = {}
        for st in range(2):
            for k, v in g[st*2+r].params.items(): got[re.sub(r"_p\d+(?=\.|$)", "", k)] = v
        errs = sorted(((np.abs(got[k]-want[r][k]).max()/max(np.abs(want[r][k]).max(),1e-9), k) for k in want[r]), reverse=True)[:4]
        print(" rank", r, [(f"{e:.2e}", k) for e, k in errs])
