# LayerNorm-backward builds: outputs compared (first lib = reference), then timed (ln_bench)
import ctypes as c, sys, torch
vp, i64 = c.c_void_p, c.c_int64
P = lambda t: c.c_void_p(t.data_ptr()) if t is not None else None
res = {}
for name in sys.argv[1:]:
    L = c.CDLL(name)
    L.sb_layernorm_fwd.argtypes = [vp] * 6 + [c.c_int, i64, i64, c.c_float, vp]
    L.sb_layernorm_bwd.argtypes = [vp] * 8 + [c.c_int, i64, i64, c.c_int, vp, vp]
    L.sb_bias_dropout_residual_ln_fwd.argtypes = [vp] * 9 + [c.c_int, i64, i64, c.c_float, c.c_uint64, c.c_uint64, c.c_double, vp]
    L.sb_bias_dropout_residual_ln_bwd.argtypes = [vp] * 10 + [c.c_int, i64, i64, c.c_uint64, c.c_uint64, c.c_double, vp, vp]
    for rows, n, mode in [(16384, 1024, 1), (16384, 1024, 0), (8192, 2048, 0), (8192, 2048, 1), (16384, 768, 1), (16384, 768, 0), (4096, 768, 1)]:
        g0 = torch.Generator(device="cuda").manual_seed(5)
        x = torch.randn(rows, n, device="cuda", generator=g0).bfloat16(); g = torch.randn(rows, n, device="cuda", generator=g0).bfloat16()
        gam = (1 + 0.1 * torch.randn(n, device="cuda", generator=g0)).bfloat16(); bet = torch.zeros_like(gam)
        y, s = torch.empty_like(x), torch.empty_like(x)
        mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
        ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
        dg, db, dbi = (torch.zeros(n, device="cuda") for _ in range(3))
        gx, gr = torch.zeros_like(x), torch.zeros_like(x)
        if mode == 1:
            L.sb_bias_dropout_residual_ln_fwd(P(x), P(bet), P(x), P(gam), P(bet), P(s), P(y), P(mean), P(rstd), 1, rows, n, 1e-5, 1, 2, 0.0, None)
            L.sb_bias_dropout_residual_ln_bwd(P(s), P(mean), P(rstd), P(gam), P(g), P(gr), P(gx), P(dbi), P(dg), P(db), 1, rows, n, 1, 2, 0.0, P(ws), None)
        else:
            L.sb_layernorm_fwd(P(x), P(gam), P(bet), P(y), P(mean), P(rstd), 1, rows, n, 1e-5, None)
            L.sb_layernorm_bwd(P(x), P(mean), P(rstd), P(gam), P(g), P(gx), P(dg), P(db), 1, rows, n, 1, P(ws), None)
        torch.cuda.synchronize()
        out = [gx.float(), gr.float(), dg, db, dbi]
        key = (rows, n, mode)
        if key not in res:
            res[key] = out
            print(name.split('/')[-1], key, "reference")
        else:
            errs = [((a - b).norm() / max(b.norm().item(), 1e-30)).item() for a, b in zip(out, res[key])]
            bit = [bool(torch.equal(a, b)) for a, b in zip(out, res[key])]
            print(name.split('/')[-1], key, "relL2 gx/gres/dgamma/dbeta/dbias", ["%.1e" % e for e in errs], "bitwise", bit)
