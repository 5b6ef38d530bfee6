"""One launch each of the hot kernels at BERT-large (C3) shapes, for
`ncu --set full` captures (profiles/README.md lists the commands)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_kernels_gpu import L, P  # noqa: E402

T, H, S, nh, hd, p = 16384, 1024, 512, 16, 64, 0.1
B = T // S
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
L.sb_gemm_set_workspace(P(ws), ws.numel())
# dense1 forward: y = gelu(x W^T + b), aux = pre-activation (FusedLinearGelu)
x = torch.randn(T, H, device="cuda").bfloat16()
w = torch.randn(4 * H, H, device="cuda").bfloat16()
b = torch.randn(4 * H, device="cuda").bfloat16()
y = torch.empty(T, 4 * H, device="cuda", dtype=torch.bfloat16)
pre = torch.empty_like(y)
for _ in range(2):
    L.sb_gemm(P(x), 1, 0, H, 1, P(w), 1, 0, 1, H, P(y), 1, 0, 4 * H, 1, 1, T, 4 * H, H, 1.0, 0, P(b), 1, P(pre), None)
# attention forward + backward (dropout p=0.1 from precomputed keep bits)
qkv = torch.randn(B, S, 3 * H, device="cuda").bfloat16()
q, k, v = qkv[..., :H], qkv[..., H:2 * H], qkv[..., 2 * H:]
o = torch.empty(B, S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * nh * S, device="cuda")
delta = torch.empty(L.sb_attn_bwd_workspace(B, S, nh, hd), dtype=torch.uint8, device="cuda")
n = B * nh * S * S
bits = torch.empty(2 * ((n + 31) // 32), dtype=torch.int32, device="cuda")
L.sb_attn_dropout_mask(P(bits), B, S, nh, 123, 1040, p, None)
do = torch.randn(B, S, H, device="cuda").bfloat16()
g = torch.zeros_like(qkv)
for _ in range(2):
    L.sb_attn_fwd(P(q), P(k), P(v), P(o), 3 * H, H, P(lse), B, S, nh, hd, hd ** -0.5, 123, 1040, p, 1, P(bits), None)
    L.sb_attn_bwd(P(q), P(k), P(v), P(o), 3 * H, H, P(lse), P(do), P(g[..., :H]), P(g[..., H:2 * H]), P(g[..., 2 * H:]),
                  P(delta), B, S, nh, hd, hd ** -0.5, 123, 1040, p, 1, P(bits), 0, None)
torch.cuda.synchronize()
print("ok")
