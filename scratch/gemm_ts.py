import os, sys, torch
sys.path.insert(0, '.')
from tests.test_kernels_gpu import L, P
T, H, F = 16384, 1024, 4096
h4 = torch.randn(T, F, device="cuda").bfloat16(); w2 = torch.randn(H, F, device="cuda").bfloat16(); y1 = torch.empty(T, H, device="cuda").bfloat16()
f = lambda: L.sb_gemm(P(h4), 1, 0, F, 1, P(w2), 1, 0, 1, F, P(y1), 1, 0, H, 1, 1, T, H, F, 1.0, 0, None, 0, None, None)
f(); f(); torch.cuda.synchronize()
os.environ["SB_GEMM_TS"] = "1"
f(); torch.cuda.synchronize()
