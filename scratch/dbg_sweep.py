import os, sys, torch
sys.path.insert(0, '.')
exec(open('scratch/attn_bench.py').read().split("def t(")[0])
def tm(f, it=10):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1000
mask(); fwd(); torch.cuda.synchronize()
names = {1: "no-math", 2: "no-dQ", 4: "no-MMA", 8: "no-TMEM-ld", 16: "no-dS-smem", 32: "no-dKdV-out", 64: "no-TMEM-st"}
names[128] = 'no-loads'
for d in [0, 128, 1, 4, 1 | 4, 127, 127 | 128, 1 | 4 | 128, 2 | 16, 2 | 16 | 128] if os.environ.get('SWEEP', '1') == '1' else [0]:
    os.environ["SB_ATTN_DBG"] = str(d)
    desc = "+".join(v for k, v in names.items() if d & k) or "full"
    print(f"bwd dbg {d:3d} {desc:45s} {tm(bwd):7.1f} us", flush=True)
for d in ([0, 1, 4, 8, 1 | 4, 1 | 8] if os.environ.get('SWEEP', '1') == '1' else [0]):
    os.environ["SB_ATTN_DBG"] = str(d)
    print(f"fwd dbg {d:3d} {tm(fwd):7.1f} us", flush=True)
os.environ.pop("SB_ATTN_DBG")
p0 = 0.0
def fwd0(): L.sb_attn_fwd(P(q), P(k), P(v), P(o), 3*H, H, P(lse), B, S, nh, hd, hd**-0.5, 1, 2, 0.0, 1, None, None)
def bwd0(): L.sb_attn_bwd(P(q), P(k), P(v), P(o), 3*H, H, P(lse), P(do), P(g[..., :H]), P(g[..., H:2*H]), P(g[..., 2*H:]), P(delta), B, S, nh, hd, hd**-0.5, 1, 2, 0.0, 1, None, 0, None)
print(f"p=0: fwd {tm(fwd0):.1f} us bwd {tm(bwd0):.1f} us")
