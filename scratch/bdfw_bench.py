# bias+dropout+residual+LN forward builds: outputs compared (first lib = reference) and timed
import ctypes as c, sys, torch
vp, i64 = c.c_void_p, c.c_int64
P = lambda t: c.c_void_p(t.data_ptr()) if t is not None else None
ref = {}
for name in sys.argv[1:]:
    L = c.CDLL(name)
    L.sb_bias_dropout_residual_ln_fwd.argtypes = [vp] * 9 + [c.c_int, i64, i64, c.c_float, c.c_uint64, c.c_uint64, c.c_double, vp]
    for rows, n in [(16384, 1024), (8192, 2048), (16384, 768), (4096, 768)]:
        g0 = torch.Generator(device="cuda").manual_seed(5)
        x = torch.randn(rows, n, device="cuda", generator=g0).bfloat16(); r = torch.randn(rows, n, device="cuda", generator=g0).bfloat16()
        bias = torch.randn(n, device="cuda", generator=g0).bfloat16()
        gam = (1 + 0.1 * torch.randn(n, device="cuda", generator=g0)).bfloat16(); bet = (0.1 * torch.randn(n, device="cuda", generator=g0)).bfloat16()
        y, s = torch.empty_like(x), torch.empty_like(x)
        mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
        f = lambda: L.sb_bias_dropout_residual_ln_fwd(P(x), P(bias), P(r), P(gam), P(bet), P(s), P(y), P(mean), P(rstd), 1, rows, n, 1e-5, 1, 2, 0.0, None)
        f(); torch.cuda.synchronize()
        out = [y.float(), s.float(), mean.clone(), rstd.clone()]
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(50): f()
        b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) / 50 * 1000
        key = (rows, n)
        if key not in ref:
            ref[key] = out; cmp = "reference"
        else:
            cmp = "bitwise " + str([bool(torch.equal(p, q)) for p, q in zip(out, ref[key])]) + " relL2 " + str(["%.1e" % ((p - q).norm() / q.norm()).item() for p, q in zip(out, ref[key])])
        print(f"{name.split('/')[-1]:10s} rows {rows} n {n}: {us:6.1f} us  {rows*n*2*4/us/1e6:.2f} TB/s  {cmp}", flush=True)
