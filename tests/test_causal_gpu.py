"""Causal attention core (the first piece of C4's decoder blocks).

The reference's op set has no mask op (proj/src/shape_inference.cpp:10-16); causal
parity is pinned end to end against the documented oracle extension (oracle/causal_ext.py,
tests/test_decoder_gpu.py, tests/test_causal_oracle_cpu.py). The checks here are
(1) the kernels through the C ABI (`sb_attn_fwd_ex` / `sb_attn_bwd_ex`, SB_ATTN_CAUSAL)
against a torch fp32 causal reference with the same keep bits, on both engines that take
the flag (mma.sync, SIMT), and (2) at the executor level, the defining property of a
causal stack: outputs at positions < t do not depend on inputs at positions >= t.
"""
import ctypes
import json

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from tests.helpers import compare_grads
from tests.test_kernels_gpu import ES, NS, L, P, _attn_case, _keep, close

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CAUSAL = 1
L.sb_attn_fwd_ex.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p] + \
    [ctypes.c_int64] * 4 + [ctypes.c_float, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
L.sb_attn_bwd_ex.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 6 + \
    [ctypes.c_int64] * 4 + [ctypes.c_float, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]


def _fwd(qkv, bits, B, S, nh, hd, p, cap, flags=CAUSAL):
    H = nh * hd
    o = torch.full((B, S, H), float("nan"), device="cuda", dtype=torch.bfloat16)
    lse = torch.full((B * nh * S,), float("nan"), device="cuda")
    L.sb_attn_set_engine(cap)
    try:
        rc = L.sb_attn_fwd_ex(P(qkv[..., :H]), P(qkv[..., H:2 * H]), P(qkv[..., 2 * H:]), P(o), 3 * H, H, P(lse),
                              B, S, nh, hd, hd ** -0.5, ES, NS, p, 1, P(bits) if p > 0 else None, flags, None)
        assert rc == 0, L.sb_last_error()
        torch.cuda.synchronize()
        used = L.sb_attn_engine(0)
    finally:
        L.sb_attn_set_engine(0)
    return o, lse, used


def _bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, cap):
    H = nh * hd
    g = torch.full_like(qkv, 1e4)
    ws = torch.empty(L.sb_attn_bwd_workspace(B, S, nh, hd), dtype=torch.uint8, device="cuda")
    L.sb_attn_set_engine(cap)
    try:
        rc = L.sb_attn_bwd_ex(P(qkv[..., :H]), P(qkv[..., H:2 * H]), P(qkv[..., 2 * H:]), P(o), 3 * H, H, P(lse),
                              P(do), P(g[..., :H]), P(g[..., H:2 * H]), P(g[..., 2 * H:]), P(ws), B, S, nh, hd,
                              hd ** -0.5, ES, NS, p, 1, P(bits) if p > 0 else None, 0, CAUSAL, None)
        assert rc == 0, L.sb_last_error()
        torch.cuda.synchronize()
        used = L.sb_attn_engine(1)
    finally:
        L.sb_attn_set_engine(0)
    return g, used


def _causal_ref(qkv, bits, B, S, nh, hd, p, do):
    """torch fp32: softmax over keys j <= i, then the reference's dropout (keep / (1-p))."""
    H = nh * hd
    q, k, v = (qkv[..., i * H:(i + 1) * H].float().reshape(B, S, nh, hd).transpose(1, 2).requires_grad_()
               for i in range(3))
    s = q @ k.transpose(-1, -2) * hd ** -0.5
    s = s.masked_fill(torch.ones(S, S, dtype=torch.bool, device="cuda").triu(1), float("-inf"))
    lse = torch.logsumexp(s, -1).reshape(-1)
    pr = torch.softmax(s, -1)
    if p > 0:
        pr = torch.where(_keep(bits, B, S, nh), pr / (1 - p), torch.zeros_like(pr))
    o = (pr @ v).transpose(1, 2).reshape(B, S, H)
    o.backward(do.float())
    return o.detach(), lse.detach(), [t.grad.transpose(1, 2).reshape(B, S, H) for t in (q, k, v)]


@pytest.mark.parametrize("cap,engine", [(0, 2), (1, 2), (2, 1)])
@pytest.mark.parametrize("B,S,nh,hd,p", [(2, 128, 2, 64, 0.0), (1, 256, 2, 64, 0.1), (1, 256, 2, 128, 0.1),
                                         (2, 512, 4, 64, 0.1), (1, 128, 2, 128, 0.0), (2, 512, 2, 128, 0.1)])
def test_causal_attention_kernels(cap, engine, B, S, nh, hd, p):
    """cap 0 (best available): the tcgen05 forward (k_fa6_fwd: diagonal chunks masked, later
    chunks skipped) and backward (k_fa7_bwd<true>: key block j visits query blocks i >= j only,
    the diagonal block masked in the softmax warps) where they fit (hd 64, S % 128 == 0)."""
    H = nh * hd
    qkv, bits = _attn_case(B, S, nh, hd, p, qscale=1.0)
    do = (torch.randn(B, S, H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)) * 0.5).bfloat16()
    ref, lse_ref, grads = _causal_ref(qkv, bits, B, S, nh, hd, p, do)
    o, lse, used = _fwd(qkv, bits, B, S, nh, hd, p, cap)
    assert used == (3 if cap == 0 else engine)  # tcgen05 forward: k_fa6_fwd<causal, hd>
    close(o, ref)
    assert (lse - lse_ref).abs().max().item() < 2e-3 * max(1.0, lse_ref.abs().max().item())
    g, used = _bwd(qkv, o, lse, do, bits, B, S, nh, hd, p, cap)
    assert used == (3 if cap == 0 else engine)  # tcgen05 backward: k_fa7_bwd<causal> (hd 64) / k_fa8_bwd (128)
    for i in range(3):
        close(g[..., i * H:(i + 1) * H], grads[i], 3e-2)
    # the first query row attends to key 0 alone: o[:, 0] = v[:, 0] (x keep / (1-p))
    v0 = qkv[:, 0, 2 * H:].float()
    if p == 0:
        assert (o[:, 0].float() - v0).abs().max().item() < 1e-2


@pytest.mark.parametrize("S,hd", [(100, 64), (72, 32)])
def test_causal_ragged_sequence_uses_simt(S, hd):
    """S % 64 != 0 (or head_dim outside {64, 128}): the tensor-core engines decline and the
    SIMT kernels take the causal call, tile edges included."""
    B, nh, H = 2, 2, 2 * hd
    qkv, bits = _attn_case(B, S, nh, hd, 0.0, qscale=1.0)
    do = (torch.randn(B, S, H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)) * 0.5).bfloat16()
    ref, lse_ref, grads = _causal_ref(qkv, bits, B, S, nh, hd, 0.0, do)
    o, lse, used = _fwd(qkv, bits, B, S, nh, hd, 0.0, 0)
    assert used == 1
    close(o, ref)
    assert (lse - lse_ref).abs().max().item() < 2e-3 * max(1.0, lse_ref.abs().max().item())
    g, used = _bwd(qkv, o, lse, do, bits, B, S, nh, hd, 0.0, 0)
    assert used == 1
    for i in range(3):
        close(g[..., i * H:(i + 1) * H], grads[i], 3e-2)


def test_causal_flag_is_not_a_noop_and_bad_flags_fail():
    B, S, nh, hd = 1, 128, 2, 64
    qkv, bits = _attn_case(B, S, nh, hd, 0.0)
    oc, _, usedc = _fwd(qkv, bits, B, S, nh, hd, 0.0, 0)
    on, _, used = _fwd(qkv, bits, B, S, nh, hd, 0.0, 0, flags=0)
    assert usedc == 3 and used == 3 and not torch.equal(oc, on)
    o2, _, used2 = _fwd(qkv, bits, B, S, nh, hd, 0.0, 1)  # mma.sync: same math, other engine
    assert used2 == 2
    close(oc, o2.float(), 1e-2)
    H = nh * hd
    o = torch.empty(B, S, H, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * nh * S, device="cuda")
    rc = L.sb_attn_fwd_ex(P(qkv[..., :H]), P(qkv[..., H:2 * H]), P(qkv[..., 2 * H:]), P(o), 3 * H, H, P(lse),
                          B, S, nh, hd, hd ** -0.5, ES, NS, 0.0, 1, None, 2, None)
    assert rc != 0 and b"flags" in L.sb_last_error()


def _causal_model(hidden, heads, seq, batch, p):
    m = sb.toy_bert(2, hidden, heads, 64, batch, seq, p)
    s = sb.create_schedule(m, 1)
    s.load_script(recipes.c2_script(2))
    j = json.loads(s.apply().to_json())

    def walk(d):
        if isinstance(d, dict):
            if d.get("kind") == "EfficientAttention":
                d["attrs"]["causal"] = 1
            for v in d.values():
                walk(v)
        elif isinstance(d, list):
            for v in d:
                walk(v)
    walk(j)
    return m, sb.Model.from_json(json.dumps(j))


@pytest.mark.parametrize("dtype,hidden,heads,seq", [("fp32", 32, 4, 16), ("bf16", 256, 4, 128)])
def test_causal_executor_prefix_property(dtype, hidden, heads, seq):
    """Changing the ids at positions >= t leaves every output at positions < t bitwise
    unchanged (verify mode; deterministic kernels), while the non-causal model's change;
    the train-mode backward through the causal cores runs and is finite."""
    m, cm = _causal_model(hidden, heads, seq, 2, 0.1)
    x = m.random_inputs(5)
    x2 = [a.copy() for a in x]
    t = seq // 2
    x2[0][:, t:] = (x2[0][:, t:] + 7) % 64
    ex = sb.Executor(cm, "verify", 123, 1, dtype=dtype)
    a, b = ex.forward(x)[0], ex.forward(x2)[0]
    assert np.array_equal(a[:, :t], b[:, :t])
    assert not np.array_equal(a[:, t:], b[:, t:])
    s = sb.create_schedule(m, 1)
    s.load_script(recipes.c2_script(2))
    nc = sb.Executor(s.apply(), "verify", 123, 1, dtype=dtype)
    assert not np.array_equal(nc.forward(x)[0][:, :t], nc.forward(x2)[0][:, :t])
    tr = sb.Executor(cm, "train", 123, 1, dtype=dtype)
    tr.forward(x)
    g = tr.backward()
    assert all(np.isfinite(v).all() for v in g.params.values())


def test_causal_composed_path_matches_fused():
    """fused=False runs a causal EfficientAttention as the reference graph with the
    oracle extension's causal softmax; it agrees with the flash path (fp32, train)."""
    m, cm = _causal_model(32, 4, 16, 2, 0.1)
    x = m.random_inputs(5)
    res = []
    for fused in (False, True):
        ex = sb.Executor(cm, "train", 123, 1, dtype="fp32", fused=fused)
        out = ex.forward(x)[0]
        res.append((out, ex.backward().params))
    (o0, g0), (o1, g1) = res
    assert np.abs(o0 - o1).max() <= 1e-4 * np.abs(o1).max()
    compare_grads(g0, g1, 1e-4)  # (the analytically-zero key bias normalised by its QKV-bias group)
