"""The kernel-level C-ABI entry points SURVEY.md §8(b) lists (LayerNorm backward,
bias+dropout+residual+LN backward, bias+GeLU forward/backward, embedding
forward/backward, all-reduce) against torch fp32 references of the reference's
formulas (proj/src/executor.cpp), called directly through ctypes."""
import ctypes

import numpy as np
import pytest

import paper_2302_08005_b200 as sb

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
L = sb.lib()
c = ctypes
vp, i64, f32p = c.c_void_p, c.c_int64, c.c_void_p
L.sb_layernorm_fwd.argtypes = [vp] * 6 + [c.c_int, i64, i64, c.c_float, vp]
L.sb_layernorm_bwd.argtypes = [vp] * 8 + [c.c_int, i64, i64, c.c_int, vp, vp]
L.sb_layernorm_bwd_workspace.argtypes = [i64, i64]
L.sb_layernorm_bwd_workspace.restype = c.c_size_t
L.sb_bias_dropout_residual_ln_fwd.argtypes = [vp] * 9 + [c.c_int, i64, i64, c.c_float, c.c_uint64, c.c_uint64,
                                                         c.c_double, vp]
L.sb_bias_dropout_residual_ln_bwd.argtypes = [vp] * 10 + [c.c_int, i64, i64, c.c_uint64, c.c_uint64, c.c_double, vp, vp]
L.sb_bias_dropout_residual_ln_bwd_workspace.argtypes = [i64, i64]
L.sb_bias_dropout_residual_ln_bwd_workspace.restype = c.c_size_t
L.sb_dropout_mask.argtypes = [vp, i64, c.c_uint64, c.c_uint64, c.c_double, vp]
L.sb_bias_gelu_fwd.argtypes = [vp] * 4 + [c.c_int, i64, i64, vp]
L.sb_bias_gelu_bwd.argtypes = [vp] * 4 + [c.c_int, i64, i64, vp, vp]
L.sb_bias_gelu_bwd_workspace.argtypes = [i64, i64]
L.sb_bias_gelu_bwd_workspace.restype = c.c_size_t
L.sb_embedding_fwd.argtypes = [vp, i64, vp, c.c_int, i64, i64, i64, i64, vp, vp]
L.sb_embedding_bwd.argtypes = [vp, i64, vp, c.c_int, i64, i64, i64, i64, vp, vp, vp]
L.sb_embedding_bwd_workspace.argtypes = [i64, i64]
L.sb_embedding_bwd_workspace.restype = c.c_size_t
L.sb_allreduce_local.argtypes = [vp, vp, c.c_int, c.c_int, i64, c.c_int, vp]
P = lambda t: c.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
DT = {torch.float32: 0, torch.bfloat16: 1}


def close(got, want, tol):
    err = (got.float() - want.float()).abs().max().item() / max(want.float().abs().max().item(), 1e-6)
    assert err < tol, err


def ws(nbytes):
    return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")


def _gelu(x):  # the reference's tanh form (executor.cpp:177-181)
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


@pytest.mark.parametrize("dtype,n", [(torch.float32, 96), (torch.bfloat16, 1024), (torch.bfloat16, 2048)])
def test_layernorm_backward(dtype, n):
    rows = 300
    g_ = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(rows, n, device="cuda", generator=g_).to(dtype)
    gamma = (1 + 0.1 * torch.randn(n, device="cuda", generator=g_)).to(dtype)
    beta = (0.1 * torch.randn(n, device="cuda", generator=g_)).to(dtype)
    gy = torch.randn(rows, n, device="cuda", generator=g_).to(dtype)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    assert L.sb_layernorm_fwd(P(x), P(gamma), P(beta), P(y), P(mean), P(rstd), DT[dtype], rows, n, 1e-5, None) == 0
    gx = torch.zeros_like(x)
    dg = torch.empty(n, device="cuda")
    db = torch.empty(n, device="cuda")
    w = ws(L.sb_layernorm_bwd_workspace(rows, n))
    assert L.sb_layernorm_bwd(P(x), P(mean), P(rstd), P(gamma), P(gy), P(gx), P(dg), P(db), DT[dtype], rows, n, 0, P(w),
                              None) == 0, L.sb_last_error()
    xr = x.float().requires_grad_()
    gr = gamma.float().requires_grad_()
    br = beta.float().requires_grad_()
    torch.nn.functional.layer_norm(xr, (n,), gr, br, 1e-5).backward(gy.float())
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    close(gx, xr.grad, tol)
    close(dg, gr.grad, tol)
    close(db, br.grad, tol)


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_bias_dropout_residual_ln_backward(p):
    rows, n, dtype = 256, 1024, torch.bfloat16
    g_ = torch.Generator(device="cuda").manual_seed(2)
    part = torch.randn(rows, n, device="cuda", generator=g_).to(dtype)
    bias = (0.1 * torch.randn(n, device="cuda", generator=g_)).to(dtype)
    res = torch.randn(rows, n, device="cuda", generator=g_).to(dtype)
    gamma = torch.ones(n, device="cuda", dtype=dtype)
    beta = torch.zeros(n, device="cuda", dtype=dtype)
    s, y = torch.empty_like(part), torch.empty_like(part)
    mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    assert L.sb_bias_dropout_residual_ln_fwd(P(part), P(bias), P(res), P(gamma), P(beta), P(s), P(y), P(mean), P(rstd),
                                             1, rows, n, 1e-5, 5, 77, p, None) == 0, L.sb_last_error()
    bits = torch.zeros((rows * n + 31) // 32, dtype=torch.int32, device="cuda")
    assert L.sb_dropout_mask(P(bits), rows * n, 5, 77, p, None) == 0
    keep = ((bits.view(-1, 1) >> torch.arange(32, device="cuda").view(1, -1)) & 1).view(-1)[:rows * n].view(rows, n).bool()
    gy = torch.randn(rows, n, device="cuda", generator=g_).to(dtype)
    gres, gpart = torch.empty_like(part), torch.empty_like(part)
    dbias, dg, db = (torch.empty(n, device="cuda") for _ in range(3))
    w = ws(L.sb_bias_dropout_residual_ln_bwd_workspace(rows, n))
    assert L.sb_bias_dropout_residual_ln_bwd(P(s), P(mean), P(rstd), P(gamma), P(gy), P(gres), P(gpart), P(dbias), P(dg),
                                             P(db), 1, rows, n, 5, 77, p, P(w), None) == 0, L.sb_last_error()
    pr = part.float().requires_grad_()
    br = bias.float().requires_grad_()
    rr = res.float().requires_grad_()
    z = pr + br
    if p > 0:
        z = torch.where(keep, z / (1 - p), torch.zeros_like(z))
    torch.nn.functional.layer_norm(z + rr, (n,), None, None, 1e-5).backward(gy.float())
    close(gres, rr.grad, 2e-2)
    close(gpart, pr.grad, 2e-2)
    close(dbias, br.grad, 2e-2)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_bias_gelu(dtype):
    rows, n = 200, 768
    g_ = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(rows, n, device="cuda", generator=g_).to(dtype)
    b = (0.5 * torch.randn(n, device="cuda", generator=g_)).to(dtype)
    y, pre = torch.empty_like(x), torch.empty_like(x)
    assert L.sb_bias_gelu_fwd(P(x), P(b), P(y), P(pre), DT[dtype], rows, n, None) == 0, L.sb_last_error()
    xr = x.float().requires_grad_()
    br = b.float().requires_grad_()
    ref = _gelu(xr + br)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    close(y, ref.detach(), tol)
    gy = torch.randn(rows, n, device="cuda", generator=g_).to(dtype)
    gx = torch.empty_like(x)
    db = torch.empty(n, device="cuda")
    w = ws(L.sb_bias_gelu_bwd_workspace(rows, n))
    assert L.sb_bias_gelu_bwd(P(pre), P(gy), P(gx), P(db), DT[dtype], rows, n, P(w), None) == 0, L.sb_last_error()
    ref.backward(gy.float())
    close(gx, xr.grad, 10 * tol)
    close(db, br.grad, 10 * tol)


@pytest.mark.parametrize("row0,local", [(0, 50), (25, 25)])
def test_embedding_fwd_bwd(row0, local):
    """vocab-parallel shard [row0, row0 + local) of a 50-row table; ids are f64 normals
    rounded half away from zero, mod vocab (executor.cpp:14-17)"""
    V, dim, n_ids = 50, 64, 500
    ids = torch.from_numpy(np.random.default_rng(4).normal(0, 30, n_ids)).cuda()
    table = torch.randn(local, dim, device="cuda").bfloat16()
    out = torch.empty(n_ids, dim, device="cuda", dtype=torch.bfloat16)
    assert L.sb_embedding_fwd(P(ids), n_ids, P(table), 1, dim, V, row0, local, P(out), None) == 0, L.sb_last_error()
    rows = torch.from_numpy(np.mod(np.where(ids.cpu().numpy() >= 0, np.floor(ids.cpu().numpy() + 0.5),
                                            np.ceil(ids.cpu().numpy() - 0.5)).astype(np.int64), V)).cuda()
    own = (rows >= row0) & (rows < row0 + local)
    want = torch.zeros(n_ids, dim, device="cuda")
    want[own] = table.float()[rows[own] - row0]
    assert torch.equal(out.float(), want)
    g = torch.randn(n_ids, dim, device="cuda").bfloat16()
    gt = torch.zeros(local, dim, device="cuda")
    w = ws(L.sb_embedding_bwd_workspace(n_ids, dim))
    assert L.sb_embedding_bwd(P(ids), n_ids, P(g), 1, dim, V, row0, local, P(gt), P(w), None) == 0, L.sb_last_error()
    ref = torch.zeros(local, dim, device="cuda", dtype=torch.float64)
    ref.index_add_(0, rows[own] - row0, g.double()[own])
    close(gt, ref, 1e-5)


def test_allreduce_local():
    R, n = 4, 10000
    bufs = [torch.randn(n, device="cuda") for _ in range(R)]
    want = sum(b.double() for b in bufs)
    srcs = (c.c_void_p * R)(*[b.data_ptr() for b in bufs])
    outs = [torch.empty(n, device="cuda") for _ in range(R)]
    dsts = (c.c_void_p * R)(*[o.data_ptr() for o in outs])
    assert L.sb_allreduce_local(srcs, dsts, R, 0, n, 0, None) == 0, L.sb_last_error()
    torch.cuda.synchronize()
    for o in outs:
        close(o, want, 1e-6)
        assert torch.equal(o, outs[0])


def test_nvtx_tracing_runs(tmp_path):
    """SB_NVTX=1 wraps every plan op in an NVTX range (no tool attached: no-ops); the step's
    results are unchanged"""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2302_08005_b200 as sb\n"
            "m = sb.toy_bert(2, 32, 4, 32, 2, 8, 0.1); ex = sb.Executor(m, 'train', 1, 1)\n"
            "o = ex.forward(m.random_inputs(3))[0]; g = ex.backward().params\n"
            "print(float(np.abs(o).sum()) + sum(float(np.abs(v).sum()) for v in g.values()))\n") % os.path.dirname(
        os.path.dirname(os.path.abspath(__file__)))
    out = [subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                          env=dict(os.environ, SB_NVTX=v)) for v in ("0", "1")]
    assert all(r.returncode == 0 for r in out), [r.stderr for r in out]
    assert out[0].stdout == out[1].stdout
