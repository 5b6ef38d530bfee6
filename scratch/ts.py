import os, sys, torch
sys.path.insert(0, '.')
exec(open('scratch/attn_bench.py').read().split("def t(")[0])
fwd(); torch.cuda.synchronize()
for d in ("0", "7"):
    os.environ["SB_ATTN_DBG"] = d
    bwd(); torch.cuda.synchronize()
    os.environ["SB_ATTN_TS"] = "1"
    print("dbg", d, file=sys.stderr)
    bwd(); torch.cuda.synchronize()
    del os.environ["SB_ATTN_TS"]
