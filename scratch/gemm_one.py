import sys, torch
sys.path.insert(0, '.')
from tests.test_kernels_gpu import L, P
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
L.sb_gemm_set_workspace(P(ws), ws.numel())
T, H, F = 16384, 1024, 4096
h4 = torch.randn(T, F, device="cuda").bfloat16(); w2 = torch.randn(H, F, device="cuda").bfloat16(); y1 = torch.empty(T, H, device="cuda").bfloat16()
for cap in (0, 1):
    L.sb_gemm_set_engine(cap)
    for _ in range(2):
        L.sb_gemm(P(h4), 1, 0, F, 1, P(w2), 1, 0, 1, F, P(y1), 1, 0, H, 1, 1, T, H, F, 1.0, 0, None, 0, None, None)
torch.cuda.synchronize()
