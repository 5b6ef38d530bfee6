import sys, torch
sys.path.insert(0, '.')
from tests.test_kernels_gpu import L, P
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L.sb_gemm_set_workspace(P(ws), ws.numel())
def run(name, A, sA, B, sB, C, M, N, K, acc=0):
    res = []
    for cap in (0, 1):
        L.sb_gemm_set_engine(cap)
        f = lambda: L.sb_gemm(P(A), 1, 0, sA[0], sA[1], P(B), 1, 0, sB[0], sB[1], P(C), 1 if C.dtype == torch.bfloat16 else 0, 0, C.stride(0), 1, 1, M, N, K, 1.0, acc, None, 0, None, None)
        f(); torch.cuda.synchronize()
        eng = L.sb_gemm_engine()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(10): f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        res.append(f"eng{eng} {ms*1000:8.1f} us {2*M*N*K/ms/1e9:6.0f} TF/s")
    L.sb_gemm_set_engine(0)
    print(f"{name:40s}", " | ".join(res), flush=True)
for (T, H, V, nm) in [(8192, 2048, 50304, "C4 lm_head"), (4096, 768, 32128, "T5 lm_head")]:
    x = torch.randn(T, H, device="cuda").bfloat16(); w = torch.randn(V, H, device="cuda").bfloat16()
    y = torch.empty(T, V, device="cuda").bfloat16()
    run(f"{nm} fwd {T}x{V}x{H}", x, (H, 1), w, (1, H), y, T, V, H)
    dx = torch.empty(T, H, device="cuda").bfloat16()
    run(f"{nm} dgrad {T}x{H}x{V}", y, (V, 1), w, (H, 1), dx, T, H, V)
    dw = torch.zeros(V, H, device="cuda")
    run(f"{nm} wgrad {V}x{H}x{T}", y, (1, V), x, (H, 1), dw, V, H, T, acc=1)
    del x, w, y, dx, dw
