import numpy as np, sys
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref
from tests.helpers import rel_err
cfg = dict(layers=2, hidden=256, heads=4, vocab=32, batch=8, seq=128, p=0.1)
for name, script, mode, fused in [
    ("plain-verify", "", "verify", True), ("plain-train", "", "train", True),
    ("c2-verify", recipes.c2_script(2), "verify", True), ("c2-train", recipes.c2_script(2), "train", True),
    ("flash-only-verify", recipes.c2_script(2, fuse=False), "verify", True),
    ("fuse-only-verify", recipes.c2_script(2, flash=False), "verify", True),
    ("seq64-flash", None, "verify", True)]:
    c = dict(cfg)
    if script is None:
        c["seq"] = 64; script = recipes.c2_script(2, fuse=False)
    m = sb.toy_bert(c["layers"], c["hidden"], c["heads"], c["vocab"], c["batch"], c["seq"], c["p"])
    s = sb.create_schedule(m, 1); s.load_script(script); ap = s.apply()
    ex = sb.Executor(ap, mode, 123, 1, fused=fused)
    o = ex.forward(m.random_inputs(9))[0]
    r = ref.run("toy_bert", schedule=script or None, world=1, mode=mode, seed=123, input_seed=9, backward=0, **c)
    print(name, rel_err(o, r.outputs(0)[0]), flush=True)
