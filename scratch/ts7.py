import os, sys, torch
sys.path.insert(0, '.')
exec(open('scratch/attn_bench.py').read().split("def t(")[0])
fwd(); torch.cuda.synchronize()
for d in os.environ.get("DBGS", "0,255").split(","):
    os.environ["SB_ATTN_DBG"] = d
    bwd(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(5): bwd()
    b.record(); torch.cuda.synchronize()
    print("dbg", d, "bwd us", a.elapsed_time(b) / 5 * 1000, file=sys.stderr, flush=True)
    os.environ["SB_ATTN_TS"] = "1"
    bwd(); torch.cuda.synchronize()
    del os.environ["SB_ATTN_TS"]
