"""CPU restatement of the reference's hot path in numpy (f64) —
TEST INFRASTRUCTURE, not product code.

Pinned against the compiled reference (oracle/_ref/slapo_ref_driver) by
tests/test_oracle_cpu.py and by the committed golden vectors in tests/golden/.

Covers: the counter RNG (proj/include/slapo/rng.hpp:16-46), parameter init and
shard maps (proj/src/module.cpp:412-498, via the C restatement
oracle/rng_oracle.c so glibc log/cos match bit-for-bit), and the toy_bert
forward + reverse-mode backward with loss = sum(outputs)
(proj/src/executor.cpp:80-202, 637-806, 1122-1462; fixture structure
proj/tests/support/fixtures.cpp:11-133), unscheduled, world 1.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

M64 = (1 << 64) - 1
HERE = os.path.dirname(os.path.abspath(__file__))


# ------------------------------------------------------------------ RNG (rng.hpp:16-38)
def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def hash_combine(a: int, b: int) -> int:
    return splitmix64(a ^ ((b + 0x9E3779B97F4A7C15 + ((a << 6) & M64) + (a >> 2)) & M64))


def _np_splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def uniform01_array(seed: int, stream: int, n: int) -> np.ndarray:
    """uniform01(seed, stream, i) for i in [0, n) (rng.hpp:35-38), vectorised."""
    s = np.uint64(hash_combine(seed, stream))
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _np_splitmix64(s ^ (i + np.uint64(0x9E3779B97F4A7C15) + (s << np.uint64(6)) + (s >> np.uint64(2))))
    h = _np_splitmix64(h)
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def keep_mask(exec_seed: int, node_seed: int, p: float, n: int) -> np.ndarray:
    """apply_dropout keep test (executor.cpp:788-803)."""
    return uniform01_array(hash_combine(exec_seed, node_seed), 0xD0, n) >= p


_crng = None


def _c():
    global _crng
    if _crng is None:
        _crng = ctypes.CDLL(os.path.join(HERE, "_ref", "librefrng.so"))
        _crng.oracle_init_plain.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int,
                                            ctypes.c_uint64, ctypes.c_int]
        _crng.oracle_random_tensor.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_uint64,
                                               ctypes.c_uint64, ctypes.c_int]
    return _crng


def init_plain(shape, kind: str, seed: int, f32: bool = False) -> np.ndarray:
    """init_plain (module.cpp:412-431): normal = 0.1*normal01(seed, 0x9a7a, i)."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    k = {"normal": 0, "uniform": 1, "zeros": 2, "ones": 3}[kind]
    _c().oracle_init_plain(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, k, seed, int(f32))
    return out.reshape(shape)


def random_tensor(shape, seed: int, stream: int = 0, f32: bool = False) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    _c().oracle_random_tensor(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, seed, stream, int(f32))
    return out.reshape(shape)


def slice_axis(full: np.ndarray, axis: int, world: int, rank: int) -> np.ndarray:
    """slice_axis (module.cpp:435-461)."""
    part = full.shape[axis] // world
    return np.take(full, np.arange(rank * part, (rank + 1) * part), axis=axis)


def slice_blocks(full: np.ndarray, axis: int, world: int, rank: int, blocks: int) -> np.ndarray:
    """blockwise init_param_rank (module.cpp:463-498)."""
    group = full.shape[axis] // blocks
    part = group // world
    idx = np.concatenate([np.arange(b * group + rank * part, b * group + (rank + 1) * part) for b in range(blocks)])
    return np.take(full, idx, axis=axis)


def embedding_row(raw: np.ndarray, V: int) -> np.ndarray:
    """llround(raw) mod V (executor.cpp:14-17); llround rounds half away from zero."""
    r = np.where(raw >= 0, np.floor(raw + 0.5), np.ceil(raw - 0.5)).astype(np.int64)
    return np.mod(r, V)


# ------------------------------------------------------------ toy_bert forward/backward
@dataclass
class BertCfg:
    layers: int = 2
    hidden: int = 8
    heads: int = 2
    vocab: int = 28
    batch: int = 4
    seq: int = 4
    p: float = 0.1


C_GELU, A_GELU = 0.7978845608028654, 0.044715


def gelu(x):
    return 0.5 * x * (1.0 + np.tanh(C_GELU * (x + A_GELU * x ** 3)))


def gelu_grad(x):
    t = np.tanh(C_GELU * (x + A_GELU * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * C_GELU * (1 + 3 * A_GELU * x * x)


def toy_bert_params(c: BertCfg):
    """Fixture seeds (SURVEY.md Appendix C / fixtures.cpp:79-133)."""
    H, F = c.hidden, 4 * c.hidden
    P = {"embeddings.weight": init_plain((c.vocab, H), "normal", 7)}
    for i in range(c.layers):
        L = 1000 + 977 * i
        pre = f"encoder.layer.{i}."
        for j, n in enumerate(("query", "key", "value")):
            P[pre + f"attention.qkv.{n}.weight"] = init_plain((H, H), "normal", L + 10 * j)
            P[pre + f"attention.qkv.{n}.bias"] = np.zeros(H)
        P[pre + "attention.output.dense.weight"] = init_plain((H, H), "normal", L + 50)
        P[pre + "attention.output.dense.bias"] = np.zeros(H)
        P[pre + "attention.output.norm.gamma"] = np.ones(H)
        P[pre + "attention.output.norm.beta"] = np.zeros(H)
        P[pre + "ffn.dense1.weight"] = init_plain((F, H), "normal", L + 100)
        P[pre + "ffn.dense1.bias"] = np.zeros(F)
        P[pre + "ffn.dense2.weight"] = init_plain((H, F), "normal", L + 110)
        P[pre + "ffn.dense2.bias"] = np.zeros(H)
        P[pre + "ffn.norm.gamma"] = np.ones(H)
        P[pre + "ffn.norm.beta"] = np.zeros(H)
    P["pooler.dense.weight"] = init_plain((H, H), "normal", 31)
    P["pooler.dense.bias"] = np.zeros(H)
    return P


class _Tape:
    def __init__(self):
        self.ops = []


def _ln_fwd(x, g, b, eps=1e-5):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * inv
    return g * xh + b, (xh, inv)


def _ln_bwd(gy, g, cache):
    xh, inv = cache
    gh = gy * g
    gx = inv * (gh - gh.mean(-1, keepdims=True) - xh * (gh * xh).mean(-1, keepdims=True))
    dg = (gy * xh).reshape(-1, xh.shape[-1]).sum(0)
    db = gy.reshape(-1, xh.shape[-1]).sum(0)
    return gx, dg, db


def toy_bert_step(c: BertCfg, ids: np.ndarray, exec_seed: int, train: bool = True):
    """Forward + backward (loss = sum of outputs) of the unscheduled toy_bert at
    world 1. Returns (output, grads: dotted path -> array)."""
    P = toy_bert_params(c)
    B, S, H, nh = c.batch, c.seq, c.hidden, c.heads
    hd = H // nh
    T = B * S
    G = {k: np.zeros_like(v) for k, v in P.items()}

    def drop(x, node_seed):
        if not train or c.p <= 0:
            return x, None
        keep = keep_mask(exec_seed, node_seed, c.p, x.size).reshape(x.shape)
        return np.where(keep, x / (1 - c.p), 0.0), keep

    rows = embedding_row(ids.reshape(-1), c.vocab)
    emb = P["embeddings.weight"][rows].reshape(B, S, H)
    x = emb
    caches = []
    for i in range(c.layers):
        L = 1000 + 977 * i
        pre = f"encoder.layer.{i}."
        lin = lambda v, n: v @ P[pre + n + ".weight"].T + P[pre + n + ".bias"]  # noqa: E731
        q, k, v = (lin(x, f"attention.qkv.{n}") for n in ("query", "key", "value"))
        heads = lambda t: t.reshape(B, S, nh, hd).transpose(0, 2, 1, 3)  # noqa: E731
        qh, kh, vh = heads(q), heads(k), heads(v)
        s = (qh @ kh.transpose(0, 1, 3, 2)) * (1.0 / math.sqrt(hd))
        s = s - s.max(-1, keepdims=True)
        e = np.exp(s)
        pr = e / e.sum(-1, keepdims=True)
        prd, keep_a = drop(pr, L + 40)
        ctxh = prd @ vh
        ctx = ctxh.transpose(0, 2, 1, 3).reshape(B, S, H)
        d = lin(ctx, "attention.output.dense")
        dd, keep_o = drop(d, L + 51)
        a, ln1 = _ln_fwd(dd + x, P[pre + "attention.output.norm.gamma"], P[pre + "attention.output.norm.beta"])
        h1 = lin(a, "ffn.dense1")
        act = gelu(h1)
        h2 = lin(act, "ffn.dense2")
        y, ln2 = _ln_fwd(h2 + a, P[pre + "ffn.norm.gamma"], P[pre + "ffn.norm.beta"])
        caches.append((x, qh, kh, vh, pr, keep_a, ctx, keep_o, a, ln1, h1, act, ln2))
        x = y
    z = x + emb
    pd_ = z @ P["pooler.dense.weight"].T + P["pooler.dense.bias"]
    out = gelu(pd_)

    # ---- backward, loss = sum(out)
    g_pd = gelu_grad(pd_)
    G["pooler.dense.weight"] += g_pd.reshape(T, H).T @ z.reshape(T, H)
    G["pooler.dense.bias"] += g_pd.reshape(T, H).sum(0)
    gz = g_pd @ P["pooler.dense.weight"]
    gx = gz.copy()
    g_emb = gz.copy()
    for i in reversed(range(c.layers)):
        pre = f"encoder.layer.{i}."
        x_in, qh, kh, vh, pr, keep_a, ctx, keep_o, a, ln1, h1, act, ln2 = caches[i]
        gsum2, dg, db = _ln_bwd(gx, P[pre + "ffn.norm.gamma"], ln2)
        G[pre + "ffn.norm.gamma"] += dg
        G[pre + "ffn.norm.beta"] += db
        ga = gsum2.copy()
        G[pre + "ffn.dense2.weight"] += gsum2.reshape(T, H).T @ act.reshape(T, -1)
        G[pre + "ffn.dense2.bias"] += gsum2.reshape(T, H).sum(0)
        gact = gsum2 @ P[pre + "ffn.dense2.weight"]
        gh1 = gact * gelu_grad(h1)
        G[pre + "ffn.dense1.weight"] += gh1.reshape(T, -1).T @ a.reshape(T, H)
        G[pre + "ffn.dense1.bias"] += gh1.reshape(T, -1).sum(0)
        ga += gh1 @ P[pre + "ffn.dense1.weight"]
        gsum1, dg, db = _ln_bwd(ga, P[pre + "attention.output.norm.gamma"], ln1)
        G[pre + "attention.output.norm.gamma"] += dg
        G[pre + "attention.output.norm.beta"] += db
        gx_in = gsum1.copy()
        gd = np.where(keep_o, gsum1 / (1 - c.p), 0.0) if keep_o is not None else gsum1
        G[pre + "attention.output.dense.weight"] += gd.reshape(T, H).T @ ctx.reshape(T, H)
        G[pre + "attention.output.dense.bias"] += gd.reshape(T, H).sum(0)
        gctx = (gd @ P[pre + "attention.output.dense.weight"]).reshape(B, S, nh, hd).transpose(0, 2, 1, 3)
        prd = np.where(keep_a, pr / (1 - c.p), 0.0) if keep_a is not None else pr
        gvh = prd.transpose(0, 1, 3, 2) @ gctx
        gprd = gctx @ vh.transpose(0, 1, 3, 2)
        gpr = np.where(keep_a, gprd / (1 - c.p), 0.0) if keep_a is not None else gprd
        gs = pr * (gpr - (gpr * pr).sum(-1, keepdims=True))
        gs *= 1.0 / math.sqrt(hd)
        gqh = gs @ kh
        gkh = gs.transpose(0, 1, 3, 2) @ qh
        merge = lambda t: t.transpose(0, 2, 1, 3).reshape(B, S, H)  # noqa: E731
        for n, gh in (("query", gqh), ("key", gkh), ("value", gvh)):
            gm = merge(gh)
            G[pre + f"attention.qkv.{n}.weight"] += gm.reshape(T, H).T @ x_in.reshape(T, H)
            G[pre + f"attention.qkv.{n}.bias"] += gm.reshape(T, H).sum(0)
            gx_in += gm @ P[pre + f"attention.qkv.{n}.weight"]
        gx = gx_in
    g_emb += gx
    np.add.at(G["embeddings.weight"], rows, g_emb.reshape(T, H))
    return out, G
