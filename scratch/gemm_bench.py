import ctypes, sys, torch
sys.path.insert(0, '.')
from tests.test_kernels_gpu import L, P
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda"); L.sb_gemm_set_workspace(P(ws), ws.numel())
T, H = 16384, 1024
def run(name, M, N, K, kind, acc):
    if kind == "fwd":   A = torch.randn(M, K, device="cuda").bfloat16(); sA = (K, 1); B = torch.randn(N, K, device="cuda").bfloat16(); sB = (1, K); C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    if kind == "dgrad": A = torch.randn(M, K, device="cuda").bfloat16(); sA = (K, 1); B = torch.randn(K, N, device="cuda").bfloat16(); sB = (N, 1); C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    if kind == "wgrad": A = torch.randn(K, M, device="cuda").bfloat16(); sA = (1, M); B = torch.randn(K, N, device="cuda").bfloat16(); sB = (N, 1); C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    f = lambda: L.sb_gemm(P(A), 1, 0, sA[0], sA[1], P(B), 1, 0, sB[0], sB[1], P(C), 0 if C.dtype == torch.float32 else 1, 0, C.stride(0), 1, 1, M, N, K, 1.0, acc, None, 0, None, None)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True); a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize(); ms = a.elapsed_time(b) / 20
    print(f"{name:12s} {kind:6s} M={M:6d} N={N:5d} K={K:6d} acc={acc}: {ms*1e3:7.1f} us  {2*M*N*K/ms/1e9:6.0f} TF/s  engine={L.sb_gemm_engine()}")
for nm, o, i in [("qkv", 3*H, H), ("out", H, H), ("dense1", 4*H, H), ("dense2", H, 4*H)]:
    run(nm, T, o, i, "fwd", 0)
    run(nm, T, i, o, "dgrad", 1)
    run(nm, T, i, o, "dgrad", 0)
    run(nm, o, i, T, "wgrad", 1)
tt = torch.randn(8192, 8192, device="cuda").bfloat16(); 
a, b = torch.cuda.Event(True), torch.cuda.Event(True); torch.matmul(tt, tt); torch.cuda.synchronize(); a.record()
for _ in range(10): torch.matmul(tt, tt)
b.record(); torch.cuda.synchronize(); ms = a.elapsed_time(b)/10; print(f"cuBLAS 8192^3: {2*8192**3/ms/1e9:.0f} TF/s")
r = run("sq8192", 8192, 8192, 8192, "fwd", 0)
