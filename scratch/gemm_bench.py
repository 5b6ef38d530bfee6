import sys, torch
sys.path.insert(0, '.')
from tests.test_kernels_gpu import L, P
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
L.sb_gemm_set_workspace(P(ws), ws.numel())
T, H, F = 16384, 1024, 4096
def run(name, A, sA, B, sB, C, M, N, K, epi=0, aux=None, bias=None, acc=0):
    res = []
    for cap in (0, 1):
        L.sb_gemm_set_engine(cap)
        f = lambda: L.sb_gemm(P(A), 1, 0, sA[0], sA[1], P(B), 1, 0, sB[0], sB[1], P(C), 1 if C.dtype == torch.bfloat16 else 0, 0, C.stride(0), 1, 1, M, N, K, 1.0, acc, P(bias), epi, P(aux), None)
        f(); torch.cuda.synchronize()
        eng = L.sb_gemm_engine()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(20): f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        res.append(f"eng{eng} {ms*1000:7.1f} us {2*M*N*K/ms/1e9:6.0f} TF/s")
    L.sb_gemm_set_engine(0)
    print(f"{name:28s}", " | ".join(res), flush=True)
x = torch.randn(T, H, device="cuda").bfloat16(); h4 = torch.randn(T, F, device="cuda").bfloat16()
w_qkv = torch.randn(3 * H, H, device="cuda").bfloat16(); w1 = torch.randn(F, H, device="cuda").bfloat16(); w2 = torch.randn(H, F, device="cuda").bfloat16()
b3 = torch.randn(3 * H, device="cuda").bfloat16(); b4 = torch.randn(F, device="cuda").bfloat16()
y3 = torch.empty(T, 3 * H, device="cuda").bfloat16(); y4 = torch.empty(T, F, device="cuda").bfloat16(); pre = torch.empty_like(y4); y1 = torch.empty(T, H, device="cuda").bfloat16()
run("fwd qkv 16384x3072x1024", x, (H, 1), w_qkv, (1, H), y3, T, 3 * H, H, bias=b3)
run("fwd dense1+gelu 16384x4096x1024", x, (H, 1), w1, (1, H), y4, T, F, H, epi=1, aux=pre, bias=b4)
run("fwd dense2 16384x1024x4096", h4, (F, 1), w2, (1, F), y1, T, H, F)
g1 = torch.randn(T, H, device="cuda").bfloat16()
run("dgrad dense2 dgelu 16384x4096x1024", g1, (H, 1), w2, (F, 1), y4, T, F, H, epi=2, aux=pre)
run("dgrad dense1 16384x1024x4096", h4, (F, 1), w1, (H, 1), y1, T, H, F)
dw = torch.empty(F, H, device="cuda")
run("wgrad dense1 4096x1024x16384", h4, (1, F), x, (H, 1), dw, F, H, T)
dw2 = torch.empty(H, H, device="cuda")
run("wgrad out 1024x1024x16384", g1, (1, H), x, (H, 1), dw2, H, H, T)
