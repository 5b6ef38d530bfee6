"""One launch each of the hot kernels at BERT-large (C3) shapes, for
`ncu --set full` captures (profiles/README.md lists the commands): the 2-SM
tcgen05 GEMM (dense1 forward with the GeLU epilogue, dense2 forward, the
dense1 weight gradient), the keep-bit generator, and the tcgen05
flash-attention forward / backward (with its delta/lse prep)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_kernels_gpu import L, P  # noqa: E402

T, H, F, S, nh, hd, p = 16384, 1024, 4096, 512, 16, 64, 0.1
B = T // S
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
L.sb_gemm_set_workspace(P(ws), ws.numel())
x = torch.randn(T, H, device="cuda").bfloat16()
w1 = torch.randn(F, H, device="cuda").bfloat16()
b1 = torch.randn(F, device="cuda").bfloat16()
w2 = torch.randn(H, F, device="cuda").bfloat16()
y = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
pre = torch.empty_like(y)
y1 = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
dw = torch.empty(F, H, device="cuda")
for _ in range(2):
    # dense1 forward: y = gelu(x W1^T + b1), pre-activation side output (FusedLinearGelu)
    L.sb_gemm(P(x), 1, 0, H, 1, P(w1), 1, 0, 1, H, P(y), 1, 0, F, 1, 1, T, F, H, 1.0, 0, P(b1), 1, P(pre), None)
    # dense2 forward: y1 = gelu_out W2^T (K = 4096)
    L.sb_gemm(P(y), 1, 0, F, 1, P(w2), 1, 0, 1, F, P(y1), 1, 0, H, 1, 1, T, H, F, 1.0, 0, None, 0, None, None)
    # dense1 weight gradient: dW1 = g^T x (fp32 out, K = 16384 tokens)
    L.sb_gemm(P(y), 1, 0, 1, F, P(x), 1, 0, H, 1, P(dw), 0, 0, H, 1, 1, F, H, T, 1.0, 0, None, 0, None, None)
# attention forward + backward (dropout p=0.1 from precomputed dual-layout keep bits)
qkv = torch.randn(B, S, 3 * H, device="cuda").bfloat16()
q, k, v = qkv[..., :H], qkv[..., H:2 * H], qkv[..., 2 * H:]
o = torch.empty(B, S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * nh * S, device="cuda")
wsa = torch.empty(L.sb_attn_bwd_workspace(B, S, nh, hd), dtype=torch.uint8, device="cuda")
n = B * nh * S * S
bits = torch.empty(2 * ((n + 31) // 32), dtype=torch.int32, device="cuda")
do = torch.randn(B, S, H, device="cuda").bfloat16()
g = torch.zeros_like(qkv)
for _ in range(2):
    L.sb_attn_dropout_mask(P(bits), B, S, nh, 123, 1040, p, None)
    L.sb_attn_fwd(P(q), P(k), P(v), P(o), 3 * H, H, P(lse), B, S, nh, hd, hd ** -0.5, 123, 1040, p, 1, P(bits), None)
    L.sb_attn_bwd(P(q), P(k), P(v), P(o), 3 * H, H, P(lse), P(do), P(g[..., :H]), P(g[..., H:2 * H]), P(g[..., 2 * H:]),
                  P(wsa), B, S, nh, hd, hd ** -0.5, 123, 1040, p, 1, P(bits), 0, None)
torch.cuda.synchronize()
print("ok")
