# A/B of attention-backward builds / SB_ATTN_SPLIT: time, agreement with the first run, determinism
import ctypes as C, os, sys, torch
vp, i64 = C.c_void_p, C.c_int64
P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
runs = [x.split("@") for x in sys.argv[1:]]  # lib@SPLIT
for (B, S, nh, hd) in [(32, 512, 16, 64), (4, 512, 16, 64), (2, 256, 8, 64), (37, 512, 16, 64)]:
    H = nh * hd
    g = torch.Generator(device="cuda").manual_seed(2)
    qkv = (torch.randn(B, S, 3 * H, device="cuda", generator=g) * 0.5).bfloat16()
    q, k, v = qkv[..., :H], qkv[..., H:2 * H], qkv[..., 2 * H:]
    do = torch.randn(B, S, H, device="cuda", generator=g).bfloat16()
    n = B * nh * S * S
    bits = torch.zeros(2 * ((n + 31) // 32), dtype=torch.int32, device="cuda")
    ref = None
    for lib, sp in runs:
        os.environ["SB_ATTN_SPLIT"] = sp
        L = C.CDLL(lib)
        L.sb_attn_fwd.argtypes = [vp] * 4 + [i64, i64, vp] + [i64] * 4 + [C.c_float, C.c_uint64, C.c_uint64, C.c_double, C.c_int, vp, vp]
        L.sb_attn_bwd.argtypes = [vp] * 4 + [i64, i64] + [vp] * 6 + [i64] * 4 + [C.c_float, C.c_uint64, C.c_uint64, C.c_double, C.c_int, vp, C.c_int, vp]
        L.sb_attn_dropout_mask.argtypes = [vp, i64, i64, i64, C.c_uint64, C.c_uint64, C.c_double, vp]
        L.sb_attn_bwd_workspace.argtypes = [i64] * 4
        L.sb_attn_bwd_workspace.restype = C.c_size_t
        L.sb_attn_dropout_mask(P(bits), B, S, nh, 1, 2, 0.1, None)
        o = torch.zeros(B, S, H, device="cuda", dtype=torch.bfloat16)
        lse = torch.zeros(B * nh * S, device="cuda")
        L.sb_attn_fwd(P(q), P(k), P(v), P(o), 3 * H, H, P(lse), B, S, nh, hd, hd ** -0.5, 1, 2, 0.1, 1, P(bits), None)
        ws = torch.empty(L.sb_attn_bwd_workspace(B, S, nh, hd), dtype=torch.uint8, device="cuda")
        gq = torch.zeros_like(qkv)
        f = lambda: L.sb_attn_bwd(P(q), P(k), P(v), P(o), 3 * H, H, P(lse), P(do), P(gq[..., :H]), P(gq[..., H:2 * H]),
                                  P(gq[..., 2 * H:]), P(ws), B, S, nh, hd, hd ** -0.5, 1, 2, 0.1, 1, P(bits), 0, None)
        f(); torch.cuda.synchronize()
        first = gq.clone()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        best = 1e9
        for rep in range(3):
            a.record()
            for _ in range(10): f()
            b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 10 * 1000)
        det = bool(torch.equal(first, gq))
        if ref is None:
            ref = first.float(); cmp = "reference"
        else:
            d = (first.float() - ref).norm() / ref.norm()
            cmp = f"relL2 vs first {d.item():.2e} bitwise {bool(torch.equal(first.float(), ref))}"
        print(f"B{B} S{S} nh{nh}: {lib.split('/')[-1]:18s} split={sp}: {best:7.1f} us  deterministic {det}  {cmp}", flush=True)
