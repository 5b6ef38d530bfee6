import ctypes as c, sys, torch
vp, i64 = c.c_void_p, c.c_int64
P = lambda t: c.c_void_p(t.data_ptr()) if t is not None else None
for name in sys.argv[1:]:
    L = c.CDLL(name)
    L.sb_layernorm_fwd.argtypes = [vp] * 6 + [c.c_int, i64, i64, c.c_float, vp]
    L.sb_layernorm_bwd.argtypes = [vp] * 8 + [c.c_int, i64, i64, c.c_int, vp, vp]
    L.sb_bias_dropout_residual_ln_fwd.argtypes = [vp] * 9 + [c.c_int, i64, i64, c.c_float, c.c_uint64, c.c_uint64, c.c_double, vp]
    L.sb_bias_dropout_residual_ln_bwd.argtypes = [vp] * 10 + [c.c_int, i64, i64, c.c_uint64, c.c_uint64, c.c_double, vp, vp]
    for rows, n, mode in [(16384, 1024, 1), (16384, 1024, 0), (8192, 2048, 0), (8192, 2048, 1), (16384, 768, 1), (16384, 768, 0)]:
        x = torch.randn(rows, n, device="cuda").bfloat16(); g = torch.randn_like(x)
        gam = torch.ones(n, device="cuda").bfloat16(); bet = torch.zeros_like(gam)
        y, s = torch.empty_like(x), torch.empty_like(x)
        mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
        ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
        dg, db, dbi = (torch.empty(n, device="cuda") for _ in range(3))
        gx, gr = torch.empty_like(x), torch.empty_like(x)
        if mode == 1:
            L.sb_bias_dropout_residual_ln_fwd(P(x), P(bet), P(x), P(gam), P(bet), P(s), P(y), P(mean), P(rstd), 1, rows, n, 1e-5, 1, 2, 0.0, None)
            f = lambda: L.sb_bias_dropout_residual_ln_bwd(P(s), P(mean), P(rstd), P(gam), P(g), P(gr), P(gx), P(dbi), P(dg), P(db), 1, rows, n, 1, 2, 0.0, P(ws), None)
        else:
            L.sb_layernorm_fwd(P(x), P(gam), P(bet), P(y), P(mean), P(rstd), 1, rows, n, 1e-5, None)
            f = lambda: L.sb_layernorm_bwd(P(x), P(mean), P(rstd), P(gam), P(g), P(gx), P(dg), P(db), 1, rows, n, 1, P(ws), None)
        for _ in range(3): f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(50): f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 50
        nbytes = rows * n * 2 * (4 if mode == 1 else 4)  # mode1: sum, g in; gres, gpart out. mode0: x, g, gx(acc) in; gx out
        print(f"{name.split('/')[-1]} rows {rows} n {n} mode {mode}: {ms*1000:.1f} us  {nbytes/ms/1e9:.2f} TB/s (incl. col finish)")
