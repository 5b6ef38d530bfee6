import ctypes, os, sys, torch
sys.path.insert(0, '.')
import paper_2302_08005_b200 as sb
from tests.test_kernels_gpu import L, P
B, S, nh, hd = (int(x) for x in os.environ.get("ATTN_CFG", "32,512,16,64").split(","))
p = 0.1
print('B,S,nh,hd', B, S, nh, hd)
H = nh * hd
qkv = (torch.randn(B, S, 3 * H, device="cuda") * 0.5).bfloat16()
q, k, v = qkv[..., :H], qkv[..., H:2*H], qkv[..., 2*H:]
o = torch.zeros(B, S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(B * nh * S, device="cuda"); delta = torch.empty(L.sb_attn_bwd_workspace(B, S, nh, hd), dtype=torch.uint8, device="cuda")
n = B * nh * S * S
bits = torch.zeros(2 * ((n + 31) // 32), dtype=torch.int32, device="cuda")
do = torch.randn(B, S, H, device="cuda").bfloat16(); g = torch.zeros_like(qkv)
def mask(): L.sb_attn_dropout_mask(P(bits), B, S, nh, 1, 2, p, None)
def fwd(): L.sb_attn_fwd(P(q), P(k), P(v), P(o), 3*H, H, P(lse), B, S, nh, hd, hd**-0.5, 1, 2, p, 1, P(bits), None)
def bwd(): L.sb_attn_bwd(P(q), P(k), P(v), P(o), 3*H, H, P(lse), P(do), P(g[..., :H]), P(g[..., H:2*H]), P(g[..., 2*H:]), P(delta), B, S, nh, hd, hd**-0.5, 1, 2, p, 1, P(bits), 0, None)
def t(f, it=10):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
unit = 2 * B * nh * S * S * hd / 1e12  # one S-sized GEMM in TFLOP
tm, tf, tb = t(mask), t(fwd), t(bwd)
print(f"mask {tm:.3f} ms  fwd {tf:.3f} ms ({2*unit/tf*1e3:.0f} TF/s)  bwd {tb:.3f} ms ({7*unit/tb*1e3:.0f} TF/s executed, {5*unit/tb*1e3:.0f} model)")
for eng in (0, 1):
    L.sb_attn_set_engine(eng)
    tf = t(fwd)
    print(f"engine cap {eng}: used {L.sb_attn_engine(0)} fwd {tf:.3f} ms ({2*unit/tf*1e3:.0f} TF/s)")
L.sb_attn_set_engine(0)
fwd()
for eng in (0, 1):
    L.sb_attn_set_engine(eng)
    tb = t(bwd)
    print(f"engine cap {eng}: used {L.sb_attn_engine(1)} bwd {tb:.3f} ms ({5*unit/tb*1e3:.0f} TF/s model)")
L.sb_attn_set_engine(0)
L.sb_attn_set_engine(0)
import tests.test_causal_gpu  # noqa: F401  (sets the _ex argtypes)
def fwdc(): L.sb_attn_fwd_ex(P(q), P(k), P(v), P(o), 3*H, H, P(lse), B, S, nh, hd, hd**-0.5, 1, 2, p, 1, P(bits), 1, None)
for eng in (0, 1):
    L.sb_attn_set_engine(eng)
    tf = t(fwdc)
    print(f"causal engine cap {eng}: used {L.sb_attn_engine(0)} fwd {tf:.3f} ms ({unit/tf*1e3:.0f} TF/s useful)")
L.sb_attn_set_engine(0)
def bwdc(): L.sb_attn_bwd_ex(P(q), P(k), P(v), P(o), 3*H, H, P(lse), P(do), P(g[..., :H]), P(g[..., H:2*H]), P(g[..., 2*H:]), P(delta), B, S, nh, hd, hd**-0.5, 1, 2, p, 1, P(bits), 0, 1, None)
fwdc()
for eng in (0, 1):
    L.sb_attn_set_engine(eng)
    tb = t(bwdc)
    print(f"causal engine cap {eng}: used {L.sb_attn_engine(1)} bwd {tb:.3f} ms ({2.5*unit/tb*1e3:.0f} TF/s useful)")
L.sb_attn_set_engine(0)
