import numpy as np, sys
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from oracle import ref
from tests.helpers import rel_err
def run(mode, **kw):
    c = dict(layers=1, hidden=32, heads=4, vocab=32, batch=2, seq=8, p=0.1); c.update(kw)
    m = sb.toy_bert(c["layers"], c["hidden"], c["heads"], c["vocab"], c["batch"], c["seq"], c["p"])
    x = m.random_inputs(9)
    o1 = sb.Executor(m, mode, 123, 1).forward(x)[0]
    o2 = sb.Executor(m, mode, 123, 1).forward(x)[0]
    r = ref.run("toy_bert", world=1, mode=mode, seed=123, input_seed=9, backward=0, **c)
    print(mode, kw, "err %.2e" % rel_err(o1, r.outputs(0)[0]), "repeat-identical", np.array_equal(o1, o2), flush=True)
for kw in [dict(), dict(hidden=256), dict(seq=128), dict(batch=8), dict(hidden=64), dict(hidden=128), dict(seq=64), dict(seq=65), dict(layers=2, hidden=256, batch=8, seq=128)]:
    for mode in ["verify", "train"]:
        run(mode, **kw)
