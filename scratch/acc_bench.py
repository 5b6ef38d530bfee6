# accumulate-epilogue A/B: libs given on the command line, same shapes, C += A B (fp32 and bf16 C)
import ctypes as C, sys, torch
vp, i64 = C.c_void_p, C.c_int64
P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
ref = {}
for name in sys.argv[1:]:
    L = C.CDLL(name)
    L.sb_gemm.argtypes = [vp, C.c_int, i64, i64, i64, vp, C.c_int, i64, i64, i64, vp, C.c_int, i64, i64, i64,
                          i64, i64, i64, i64, C.c_float, C.c_int, vp, C.c_int, vp, vp]
    L.sb_gemm_set_workspace.argtypes = [vp, C.c_size_t]
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L.sb_gemm_set_workspace(P(ws), ws.numel())
    for (M, N, K, f32) in [(32128, 768, 4096, 1), (50304, 2048, 8192, 1), (4096, 1024, 16384, 1), (1024, 1024, 16384, 1),
                           (16384, 1024, 1024, 0)]:
        g = torch.Generator(device="cuda").manual_seed(3)
        # wgrad-like: A = dY^T (MN-major), B = X
        a = torch.randn(K, M, device="cuda", generator=g).bfloat16(); b = torch.randn(K, N, device="cuda", generator=g).bfloat16()
        c0 = torch.randn(M, N, device="cuda", generator=g)
        c = c0.clone() if f32 else c0.bfloat16()
        f = lambda: L.sb_gemm(P(a), 1, 0, 1, M, P(b), 1, 0, N, 1, P(c), 0 if f32 else 1, 0, N, 1, 1, M, N, K, 1.0, 1, None, 0, None, None)
        f(); torch.cuda.synchronize()
        once = c.float().clone()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        key = (M, N, K, f32)
        if key not in ref:
            ref[key] = once; cmp = "reference"
        else:
            cmp = f"bitwise {bool(torch.equal(once, ref[key]))} maxdiff {(once - ref[key]).abs().max().item():.3e}"
        print(f"{name.split('/')[-1]:12s} {M}x{N}x{K} {'f32' if f32 else 'bf16'} acc: {ms*1000:8.1f} us {2*M*N*K/ms/1e9:6.0f} TF/s  {cmp}", flush=True)
