"""Kernel-level GPU checks through the C ABI: the tcgen05 GEMM against a
torch fp32 reference for all three Linear operand layouts and every epilogue,
and the attention kernels against a torch fp32 reference of the same math."""
import ctypes

import numpy as np
import pytest

import paper_2302_08005_b200 as sb

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
L = sb.lib()
L.sb_gemm.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                      ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                      ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_float, ctypes.c_int,
                      ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
L.sb_gemm_set_workspace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.sb_gemm_set_engine.argtypes = [ctypes.c_int]
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
DT = {torch.float32: 0, torch.bfloat16: 1}


def gemm(A, sA, B, sB, C, M, N, K, acc=False, bias=None, gelu=False, aux=None, epi=None, cap=0):
    """C (+)= A B through the C ABI; epi: 0 none, 1 gelu (+aux pre-activation), 2 dgelu(aux); cap: engine cap."""
    L.sb_gemm_set_engine(cap)
    try:
        rc = L.sb_gemm(P(A), DT[A.dtype], 0, sA[0], sA[1], P(B), DT[B.dtype], 0, sB[0], sB[1], P(C), DT[C.dtype], 0,
                       C.stride(0), 1, 1, M, N, K, 1.0, int(acc), P(bias), (1 if gelu else 0) if epi is None else epi,
                       P(aux), None)
    finally:
        L.sb_gemm_set_engine(0)
    assert rc == 0, L.sb_last_error()
    torch.cuda.synchronize()
    return L.sb_gemm_engine()


@pytest.fixture(scope="module", autouse=True)
def workspace():
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    L.sb_gemm_set_workspace(P(ws), ws.numel())
    yield ws
    L.sb_gemm_set_workspace(None, 0)


def close(got, want, tol=2e-2):
    err = (got.float() - want).abs().max().item() / max(want.abs().max().item(), 1e-6)
    assert err < tol, err


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 512, 192), (512, 768, 1024), (384, 256, 320)])
def test_forward_tn(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    w = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, device="cuda", generator=g).bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    eng = gemm(x, (K, 1), w, (1, K), y, M, N, K, bias=b)
    assert eng in (1, 2), "tcgen05 path not taken"
    close(y, x.float() @ w.float().T + b.float())


def test_forward_gelu_epilogue_and_aux():
    M, N, K = 256, 512, 256
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    b = torch.randn(N, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    pre = torch.empty_like(y)
    assert gemm(x, (K, 1), w, (1, K), y, M, N, K, bias=b, gelu=True, aux=pre) in (1, 2)
    ref = x.float() @ w.float().T + b.float()
    close(pre, ref)
    close(y, torch.nn.functional.gelu(ref, approximate="tanh"))


@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (512, 1024, 768)])
def test_dgrad_nn_accumulate(M, N, K):
    g = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(K, N, device="cuda").bfloat16()  # W is (out=K, in=N)
    dx = torch.randn(M, N, device="cuda").bfloat16()
    want = dx.float() + g.float() @ w.float()
    assert gemm(g, (K, 1), w, (N, 1), dx, M, N, K, acc=True) in (1, 2)  # B(k,n) = W[k][n]: sBk=N, sBn=1
    close(dx, want)


@pytest.mark.parametrize("O,I,T", [(256, 256, 512), (1024, 1024, 4096), (384, 512, 8192)])
def test_wgrad_nt_fp32_splitk(O, I, T):
    gy = torch.randn(T, O, device="cuda").bfloat16()
    x = torch.randn(T, I, device="cuda").bfloat16()
    dw = torch.randn(O, I, device="cuda", dtype=torch.float32)
    want = dw + gy.float().T @ x.float()
    # A(m=o, k=t) = gy[t][o]: sAm=1, sAk=O ; B(k=t, n=i) = x[t][i]: sBk=I, sBn=1
    assert gemm(gy, (1, O), x, (I, 1), dw, O, I, T, acc=True) in (1, 2)
    close(dw, want, 1e-2)


def test_tc_matches_simt_engine():
    M, N, K = 256, 256, 128
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    y1 = torch.empty(M, N, device="cuda", dtype=torch.float32)
    y2 = torch.empty_like(y1)
    assert gemm(x, (K, 1), w, (1, K), y1, M, N, K) in (1, 2)
    L.sb_gemm_force_simt(1)
    try:
        assert gemm(x, (K, 1), w, (1, K), y2, M, N, K) == 0
    finally:
        L.sb_gemm_force_simt(0)
    assert (y1 - y2).abs().max().item() < 1e-3 * y2.abs().max().item()


def _gemm_engine(cap, *a, **k):
    return gemm(*a, cap=cap, **k)


@pytest.fixture(params=[0, 128, 256], ids=["tileN-auto", "tileN-128", "tileN-256"])
def tile_n(request):
    L.sb_gemm_set_tile_n.argtypes = [ctypes.c_int]
    L.sb_gemm_set_tile_n(request.param)
    yield request.param
    L.sb_gemm_set_tile_n(0)


@pytest.mark.parametrize("layout", ["tn", "tn_bias", "tn_gelu", "nn", "nn_acc", "nn_dgelu", "nt_f32", "nt_f32_acc",
                                    "nt_splitk"])
def test_gemm_2sm_vs_1sm(layout, tile_n):
    """The 2-SM cta_group::2 kernel (engine 2, TMA-store epilogue) against the 1-SM kernel and fp32 torch,
    every operand layout / epilogue the executor uses, at shapes that need several tiles per cluster."""
    M, N, K = 1024, 768, 512
    outs = {}
    for cap in (0, 1):
        g = torch.Generator(device="cuda").manual_seed(3)  # same inputs for both engines
        rnd = lambda *sh: torch.randn(*sh, device="cuda", generator=g)  # noqa: E731
        if layout.startswith("tn"):
            x, w, b = rnd(M, K).bfloat16(), rnd(N, K).bfloat16(), rnd(N).bfloat16()
            y = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
            pre = torch.zeros_like(y) if layout == "tn_gelu" else None
            e = _gemm_engine(cap, x, (K, 1), w, (1, K), y, M, N, K, bias=b if layout != "tn" else None,
                             gelu=layout == "tn_gelu", aux=pre)
            ref = x.float() @ w.float().T + (b.float() if layout != "tn" else 0)
            outs[cap] = (y, pre)
            if layout == "tn_gelu":
                close(pre, ref)
                ref = torch.nn.functional.gelu(ref, approximate="tanh")
            close(y, ref)
        elif layout.startswith("nn"):
            gy, w = rnd(M, K).bfloat16(), rnd(K, N).bfloat16()
            base = rnd(M, N).bfloat16()
            dx = base.clone() if layout == "nn_acc" else torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
            aux = rnd(M, N).bfloat16() if layout == "nn_dgelu" else None
            if aux is not None:
                e = _gemm_engine(cap, gy, (K, 1), w, (N, 1), dx, M, N, K, epi=2, aux=aux)
                a = aux.float()
                t = torch.tanh(0.7978845608028654 * (a + 0.044715 * a ** 3))
                dg = 0.5 * (1 + t) + 0.5 * a * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * a * a)
                close(dx, (gy.float() @ w.float()) * dg)
            else:
                e = _gemm_engine(cap, gy, (K, 1), w, (N, 1), dx, M, N, K, acc=layout == "nn_acc")
                close(dx, (base.float() if layout == "nn_acc" else 0) + gy.float() @ w.float())
            outs[cap] = (dx, None)
        else:
            T = 4096 if layout == "nt_splitk" else K
            gy, x = rnd(T, M).bfloat16(), rnd(T, N).bfloat16()
            base = rnd(M, N)
            dw = base.clone() if layout.endswith("acc") else torch.zeros(M, N, device="cuda")
            e = _gemm_engine(cap, gy, (1, M), x, (N, 1), dw, M, N, T, acc=layout.endswith("acc"))
            close(dw, (base if layout.endswith("acc") else 0) + gy.float().T @ x.float(), 1e-2)
            outs[cap] = (dw, None)
        assert e == (2 if cap == 0 else 1), (layout, cap, e)
    assert (outs[0][0].float() - outs[1][0].float()).abs().max().item() <= 2e-2 * outs[1][0].float().abs().max().item()


@pytest.mark.parametrize("layout", ["tn", "tn_bias", "nn", "nt_f32", "nt_f32_acc"])
def test_gemm_4cta_multicast(layout):
    """K >= 4096 with an even number of 256-wide N tiles takes the 4-CTA cluster variant
    (two CTA pairs multicasting their shared A block): against the 1-SM kernel and torch."""
    M, N, K = 1024, 1024, 4096
    outs = {}
    for cap in (0, 1):
        g = torch.Generator(device="cuda").manual_seed(5)
        rnd = lambda *sh: torch.randn(*sh, device="cuda", generator=g)  # noqa: E731
        if layout.startswith("tn"):
            x, w, b = rnd(M, K).bfloat16(), rnd(N, K).bfloat16(), rnd(N).bfloat16()
            y = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
            e = _gemm_engine(cap, x, (K, 1), w, (1, K), y, M, N, K, bias=b if layout == "tn_bias" else None)
            close(y, x.float() @ w.float().T + (b.float() if layout == "tn_bias" else 0))
            outs[cap] = y
        elif layout == "nn":
            gy, w = rnd(M, K).bfloat16(), rnd(K, N).bfloat16()
            dx = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
            e = _gemm_engine(cap, gy, (K, 1), w, (N, 1), dx, M, N, K)
            close(dx, gy.float() @ w.float())
            outs[cap] = dx
        else:
            gy, x = rnd(K, M).bfloat16(), rnd(K, N).bfloat16()
            base = rnd(M, N)
            dw = base.clone() if layout.endswith("acc") else torch.zeros(M, N, device="cuda")
            e = _gemm_engine(cap, gy, (1, M), x, (N, 1), dw, M, N, K, acc=layout.endswith("acc"))
            close(dw, (base if layout.endswith("acc") else 0) + gy.float().T @ x.float(), 1e-2)
            outs[cap] = dw
        assert e == (2 if cap == 0 else 1), (layout, cap, e)
    assert (outs[0].float() - outs[1].float()).abs().max().item() <= 2e-2 * outs[1].float().abs().max().item()


@pytest.mark.parametrize("M,N,K", [(1056, 800, 512), (1152, 640, 256), (544, 800, 4096), (32, 96, 128)])
@pytest.mark.parametrize("layout", ["tn_bias", "tn_gelu", "nn_acc", "nn_dgelu", "nt_f32", "nt_f32_acc", "nt_splitk"])
def test_gemm_2sm_ragged_tiles(layout, M, N, K):
    """M, N multiples of 32 but not of the 256-wide tile (GPT-Neo's vocab 50304, T5's 32128): the
    2-SM kernel's last tiles are ragged (TMA zero-fill on loads, clipped stores, the direct bias /
    pre-activation / accumulate / split-K accesses skip the chunks past the edge) — against fp32
    torch, with guard bands around C checking nothing is written past the edge"""
    if layout == "nt_splitk":
        M, N, K = min(M, 288), 160, 4096  # few tiles, long K: split-K partials
    g = torch.Generator(device="cuda").manual_seed(11)
    rnd = lambda *sh: torch.randn(*sh, device="cuda", generator=g)  # noqa: E731
    f32 = layout.startswith("nt")
    # C inside a larger buffer (row stride N + 64, 32 extra rows): the band must stay untouched
    big = torch.full((M + 32, N + 64), 7.0, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    C = big[:M, :N]
    if layout.startswith("tn"):
        x, w, b = rnd(M, K).bfloat16(), rnd(N, K).bfloat16(), rnd(N).bfloat16()
        C.zero_()
        # (the pre-activation shares C's row stride)
        pre = torch.zeros(M + 32, N + 64, device="cuda", dtype=torch.bfloat16)[:M, :N] if layout == "tn_gelu" else None
        e = gemm(x, (K, 1), w, (1, K), C, M, N, K, bias=b, gelu=layout == "tn_gelu", aux=pre)
        ref = x.float() @ w.float().T + b.float()
        if pre is not None:
            close(pre, ref)
            ref = torch.nn.functional.gelu(ref, approximate="tanh")
    elif layout.startswith("nn"):
        gy, w = rnd(M, K).bfloat16(), rnd(K, N).bfloat16()
        if layout == "nn_acc":
            C.copy_(rnd(M, N).bfloat16())
            base = C.float().clone()
            e = gemm(gy, (K, 1), w, (N, 1), C, M, N, K, acc=True)
            ref = base + gy.float() @ w.float()
        else:
            C.zero_()
            aux = torch.zeros(M + 32, N + 64, device="cuda", dtype=torch.bfloat16)[:M, :N]
            aux.copy_(rnd(M, N).bfloat16())
            e = gemm(gy, (K, 1), w, (N, 1), C, M, N, K, epi=2, aux=aux)
            a = aux.float()
            t = torch.tanh(0.7978845608028654 * (a + 0.044715 * a ** 3))
            ref = (gy.float() @ w.float()) * (0.5 * (1 + t) + 0.5 * a * (1 - t * t) * 0.7978845608028654 *
                                              (1 + 3 * 0.044715 * a * a))
    else:
        gy, x = rnd(K, M).bfloat16(), rnd(K, N).bfloat16()
        acc = layout == "nt_f32_acc"
        if acc:
            C.copy_(rnd(M, N))
        else:
            C.zero_()
        base = C.clone()
        e = gemm(gy, (1, M), x, (N, 1), C, M, N, K, acc=acc)
        ref = (base if acc else 0) + gy.float().T @ x.float()
    assert e == 2, (layout, M, N, K, e)
    close(C, ref, 1e-2 if f32 else 2e-2)
    assert bool((big[M:] == 7).all()) and bool((big[:, N:] == 7).all()), "written past the ragged edge"


@pytest.mark.parametrize("cap", [0, 1, 2])
def test_gemm_relu_epilogues(cap):
    """The folded ReLU (T5's wi -> relu -> wo, lower.cpp fuse_linear_relu): epilogue 3 writes
    max(x W^T + b, 0); epilogue 4 writes (g W) * (a > 0) for the activation a — on the 2-SM,
    1-SM and SIMT engines, against fp32 torch."""
    M, N, K = 512, 768, 256
    g = torch.Generator(device="cuda").manual_seed(13)
    x, w, b = (torch.randn(M, K, device="cuda", generator=g).bfloat16(), torch.randn(N, K, device="cuda", generator=g).bfloat16(),
               torch.randn(N, device="cuda", generator=g).bfloat16())
    y = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    if cap == 2:
        L.sb_gemm_force_simt(1)
    try:
        e = gemm(x, (K, 1), w, (1, K), y, M, N, K, bias=b, epi=3, cap=min(cap, 1))
        close(y, torch.relu(x.float() @ w.float().T + b.float()))
        gy, w2 = torch.randn(M, K, device="cuda", generator=g).bfloat16(), torch.randn(K, N, device="cuda", generator=g).bfloat16()
        a = torch.randn(M, N, device="cuda", generator=g).bfloat16()
        dx = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        e2 = gemm(gy, (K, 1), w2, (N, 1), dx, M, N, K, epi=4, aux=a, cap=min(cap, 1))
        close(dx, (gy.float() @ w2.float()) * (a.float() > 0))
    finally:
        L.sb_gemm_force_simt(0)
    assert e == e2 == (2 - cap), (e, e2)


# ------------------------------------------------------------------ attention
L.sb_attn_fwd.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p] + \
    [ctypes.c_int64] * 4 + [ctypes.c_float, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_void_p]
L.sb_attn_bwd.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 6 + \
    [ctypes.c_int64] * 4 + [ctypes.c_float, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
L.sb_dropout_mask.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                              ctypes.c_void_p]
ES, NS = 123, 1040


def _attn_case(B, S, nh, hd, p, qscale=0.5, seed=0):
    """FusedQKV-layout (B, S, 3H) input consumed in place + dual-layout keep bits."""
    H = nh * hd
    g = torch.Generator(device="cuda").manual_seed(seed)
    qkv = (torch.randn(B, S, 3 * H, device="cuda", generator=g) * 0.5).bfloat16()
    qkv[..., :H] = (qkv[..., :H].float() * (qscale / 0.5)).bfloat16()
    n = B * nh * S * S
    bits = torch.zeros(2 * ((n + 31) // 32), dtype=torch.int32, device="cuda")
    if p > 0:
        assert L.sb_attn_dropout_mask(P(bits), B, S, nh, ES, NS, p, None) == 0
    return qkv, bits


def _keep(bits, B, S, nh):
    n = B * nh * S * S
    idx = torch.arange(n, device="cuda")
    return ((bits[idx // 32] >> (idx % 32)) & 1).bool().reshape(B, nh, S, S)


def _attn_fwd(qkv, bits, B, S, nh, hd, p, engine):
    H = nh * hd
    o = torch.full((B, S, H), float("nan"), device="cuda", dtype=torch.bfloat16)
    lse = torch.full((B * nh * S,), float("nan"), device="cuda")
    L.sb_attn_set_engine(engine)
    try:
        rc = L.sb_attn_fwd(P(qkv[..., :H]), P(qkv[..., H:2 * H]), P(qkv[..., 2 * H:]), P(o), 3 * H, H, P(lse), B, S, nh,
                           hd, hd ** -0.5, ES, NS, p, 1, P(bits) if p > 0 else None, None)
        assert rc == 0, L.sb_last_error()
        torch.cuda.synchronize()
        used = L.sb_attn_engine(0)
    finally:
        L.sb_attn_set_engine(0)
    return o, lse, used


def _attn_bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, engine, g=None):
    """g given: accumulate into it (acc_mask 7); else overwrite a garbage-filled buffer (acc_mask 0)."""
    H = nh * hd
    acc = 7 if g is not None else 0
    g = torch.full_like(qkv, 1e4) if g is None else g
    ws = torch.empty(L.sb_attn_bwd_workspace(B, S, nh, hd), dtype=torch.uint8, device="cuda")
    L.sb_attn_set_engine(engine)
    try:
        rc = L.sb_attn_bwd(P(qkv[..., :H]), P(qkv[..., H:2 * H]), P(qkv[..., 2 * H:]), P(o), 3 * H, H, P(lse), P(do),
                           P(g[..., :H]), P(g[..., H:2 * H]), P(g[..., 2 * H:]), P(ws), B, S, nh, hd, hd ** -0.5, ES,
                           NS, p, 1, P(bits) if p > 0 else None, acc, None)
        assert rc == 0, L.sb_last_error()
        torch.cuda.synchronize()
        used = L.sb_attn_engine(1)
    finally:
        L.sb_attn_set_engine(0)
    return g, used


def _attn_ref(qkv, bits, B, S, nh, hd, p, do=None):
    """torch fp32 reference of the same math (+ autograd gradients of q, k, v when do is given)."""
    H = nh * hd
    q, k, v = (qkv[..., i * H:(i + 1) * H].float().reshape(B, S, nh, hd).transpose(1, 2).requires_grad_()
               for i in range(3))
    s = q @ k.transpose(-1, -2) * hd ** -0.5
    lse = torch.logsumexp(s, -1).reshape(-1)
    pr = torch.softmax(s, -1)
    if p > 0:
        pr = torch.where(_keep(bits, B, S, nh), pr / (1 - p), torch.zeros_like(pr))
    o = (pr @ v).transpose(1, 2).reshape(B, S, H)
    grads = None
    if do is not None:
        o.backward(do.float())
        grads = [t.grad.transpose(1, 2).reshape(B, S, H) for t in (q, k, v)]
    return o.detach(), lse.detach(), grads


def test_attention_dropout_mask_dual_layout():
    B, S, nh, p = 2, 256, 3, 0.1
    n = B * nh * S * S
    dual = torch.zeros(2 * n // 32, dtype=torch.int32, device="cuda")
    nat = torch.zeros(n // 32, dtype=torch.int32, device="cuda")
    assert L.sb_attn_dropout_mask(P(dual), B, S, nh, ES, NS, p, None) == 0
    assert L.sb_dropout_mask(P(nat), n, ES, NS, p, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(dual[:n // 32], nat)  # natural half: the reference's bits exactly
    keep = _keep(dual, B, S, nh)
    keep_t = _keep(dual[n // 32:], B, S, nh)
    assert torch.equal(keep_t, keep.transpose(-1, -2))


@pytest.mark.parametrize("B,S,nh,hd,p", [(2, 128, 4, 64, 0.0), (2, 256, 2, 64, 0.1), (1, 128, 2, 128, 0.1)])
def test_flash_attention_tensor_core(B, S, nh, hd, p):
    """mma.sync kernels (engine 2) vs a torch fp32 reference."""
    H = nh * hd
    qkv, bits = _attn_case(B, S, nh, hd, p)
    o, lse, used = _attn_fwd(qkv, bits, B, S, nh, hd, p, 1)
    assert used == 2
    do = (torch.randn(B, S, H, device="cuda") * 0.5).bfloat16()
    ref, _, grads = _attn_ref(qkv, bits, B, S, nh, hd, p, do)
    close(o, ref)
    g, used = _attn_bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, 1)
    assert used == 2
    for i in range(3):
        close(g[..., i * H:(i + 1) * H], grads[i], 3e-2)


@pytest.mark.parametrize("B,S,nh,hd,p,qscale", [(2, 128, 4, 64, 0.0, 0.5), (2, 256, 2, 64, 0.1, 0.5),
                                                 (1, 384, 2, 64, 0.1, 0.5), (2, 512, 16, 64, 0.1, 0.5),
                                                 (1, 512, 2, 64, 0.1, 4.0), (1, 1024, 2, 64, 0.0, 3.0),
                                                 (2, 128, 2, 128, 0.0, 0.5), (2, 256, 4, 128, 0.1, 0.5),
                                                 (1, 1024, 16, 128, 0.1, 3.0)])
def test_flash_attention_tcgen05_forward(B, S, nh, hd, p, qscale):
    """tcgen05/TMEM forward (engine 3; head_dim 64: four CTAs per SM, 128: two, with
    two-panel Q/K/V tiles and M128 N128 PV MMAs) vs a torch fp32 reference and vs the
    mma.sync kernel; qscale > 1 makes logits large enough to exercise the lazy
    running-max rescale."""
    qkv, bits = _attn_case(B, S, nh, hd, p, qscale)
    o5, lse5, used = _attn_fwd(qkv, bits, B, S, nh, hd, p, 0)
    assert used == 3, "tcgen05 attention path not taken"
    ref, lse_ref, _ = _attn_ref(qkv, bits, B, S, nh, hd, p)
    close(o5, ref)
    assert (lse5 - lse_ref).abs().max().item() < 2e-3 * max(1.0, lse_ref.abs().max().item())
    o2, lse2, used2 = _attn_fwd(qkv, bits, B, S, nh, hd, p, 1)
    assert used2 == 2
    close(o5, o2.float(), 1e-2)


@pytest.mark.parametrize("B,S,nh,hd,p,qscale", [(2, 128, 4, 64, 0.0, 0.5), (2, 256, 2, 64, 0.1, 0.5),
                                                 (1, 384, 2, 64, 0.1, 0.5), (2, 512, 16, 64, 0.1, 0.5),
                                                 (1, 512, 2, 64, 0.1, 3.0), (1, 128, 2, 128, 0.0, 0.5),
                                                 (2, 256, 2, 128, 0.1, 0.5), (1, 1024, 4, 128, 0.1, 3.0)])
def test_flash_attention_tcgen05_backward(B, S, nh, hd, p, qscale):
    """tcgen05 backward (engine 3: TS/SS MMAs, ordered fp32 dQ accumulation) vs torch autograd
    of the fp32 reference, vs the mma.sync backward, accumulate mode, and run-to-run bitwise equality."""
    H = nh * hd
    qkv, bits = _attn_case(B, S, nh, hd, p, qscale)
    o, lse, _ = _attn_fwd(qkv, bits, B, S, nh, hd, p, 0)
    do = (torch.randn(B, S, H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)) * 0.5).bfloat16()
    _, _, grads = _attn_ref(qkv, bits, B, S, nh, hd, p, do)
    g5, used = _attn_bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, 0)
    assert used == 3, "tcgen05 attention backward not taken"
    for i in range(3):
        close(g5[..., i * H:(i + 1) * H], grads[i], 3e-2)
    g2, used2 = _attn_bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, 1)
    assert used2 == 2
    for i in range(3):
        close(g5[..., i * H:(i + 1) * H], g2[..., i * H:(i + 1) * H].float(), 2e-2)
    g5b, _ = _attn_bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, 0)
    assert torch.equal(g5, g5b)  # deterministic (no float atomics)
    base = (torch.randn_like(qkv.float()) * 0.1).bfloat16()
    gacc, _ = _attn_bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, 0, g=base.clone())
    close(gacc, base.float() + g5.float(), 2e-2)
