import sys, torch
sys.path.insert(0, '.')
from tests.test_kernels_gpu import L, P
L.sb_set_mask_blocks.argtypes = [__import__('ctypes').c_int]
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda"); L.sb_gemm_set_workspace(P(ws), ws.numel())
T, H, F = 16384, 1024, 4096
B, S, nh = 32, 512, 16
x = torch.randn(T, H, device="cuda").bfloat16(); w1 = torch.randn(F, H, device="cuda").bfloat16(); y4 = torch.empty(T, F, device="cuda").bfloat16()
n = B * nh * S * S; bits = torch.empty(2 * n // 32, dtype=torch.int32, device="cuda")
s2 = torch.cuda.Stream(priority=0)
def gemm(): 
    for _ in range(8): L.sb_gemm(P(x), 1, 0, H, 1, P(w1), 1, 0, 1, H, P(y4), 1, 0, F, 1, 1, T, F, H, 1.0, 0, None, 0, None, None)
def mask(): L.sb_attn_dropout_mask(P(bits), B, S, nh, 1, 2, 0.1, torch.cuda.current_stream().cuda_stream)
def timed(f):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True); a.record(); f(); b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)
for mb in (0, 148, 296, 592):
    L.sb_set_mask_blocks(mb)
    tg = timed(gemm); tm = timed(mask)
    def both():
        ev = torch.cuda.Event(); ev.record()
        with torch.cuda.stream(s2):
            s2.wait_event(ev); mask()
        gemm()
        torch.cuda.current_stream().wait_stream(s2)
    tb = timed(both)
    print(f"mask_blocks {mb:4d}: gemm x8 {tg:.3f} ms  mask {tm:.3f} ms  both {tb:.3f} ms  (sum {tg+tm:.3f})", flush=True)
