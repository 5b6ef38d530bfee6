"""The documented causal oracle extension (oracle/causal_ext.py)
and the decoder model family's interop with the reference (CPU only).

* The patched reference executor is the reference on every model without the
  new attr: bitwise-identical dumps to the unpatched driver (toy_bert, train).
* Its causal softmax is pinned against an independent numpy f64 restatement of
  the GPT-Neo-style decoder forward (verify mode) and backward (loss = sum of
  outputs), built from the parameters the reference itself materialised.
* The decoder built here (``gpt_neo``) is loadable by the reference
  (slapo-model-v1), and the decoder recipe applies to a byte-identical model on
  both sides (TP 1 and 2).
"""
import math
import os

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref
from oracle.slapo_oracle import gelu, gelu_grad

pytestmark = pytest.mark.skipif(not os.path.exists(ref.DRIVER_CAUSAL), reason="causal oracle not built")

NEO = dict(layers=2, hidden=16, heads=2, vocab=24, batch=2, seq=8, p=0.1)


def _neo(cfg=NEO):
    return sb.gpt_neo(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])


def _write(tmp, name, text):
    p = os.path.join(tmp, name)
    with open(p, "w") as f:
        f.write(text)
    return p


def test_causal_driver_is_the_reference_without_the_attr(tmp_path):
    kw = dict(layers=2, hidden=16, heads=2, vocab=24, batch=2, seq=8, p=0.1, mode="train", dump_params=1)
    script = recipes.c2_script(2, checkpoint_layers=[1])
    with ref.run("toy_bert", schedule=script, **kw) as a, ref.run("toy_bert", schedule=script, causal=True, **kw) as b:
        for x, y in zip(a.outputs(0), b.outputs(0)):
            assert np.array_equal(x, y)
        ga, gb = a.grads(0), b.grads(0)
        assert ga.keys() == gb.keys()
        for k in ga:
            assert np.array_equal(ga[k], gb[k]), k


def _ln(x, g, b, eps=1e-5):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * inv
    return g * xh + b, (xh, inv)


def _ln_bwd(gy, g, cache):
    xh, inv = cache
    gh = gy * g
    gx = inv * (gh - gh.mean(-1, keepdims=True) - xh * (gh * xh).mean(-1, keepdims=True))
    return gx, (gy * xh).reshape(-1, xh.shape[-1]).sum(0), gy.reshape(-1, xh.shape[-1]).sum(0)


def neo_step(P, ids, cfg):
    """numpy f64 restatement of the gpt_neo decoder (verify mode, no dropout):
    forward and backward with loss = sum(outputs). Causal softmax: query q sees keys k <= q."""
    B, S, H, nh, V = cfg["batch"], cfg["seq"], cfg["hidden"], cfg["heads"], cfg["vocab"]
    hd = H // nh
    T = B * S
    G = {k: np.zeros_like(v) for k, v in P.items()}
    raw = ids.reshape(-1)
    rows = np.mod(np.where(raw >= 0, np.floor(raw + 0.5), np.ceil(raw - 0.5)).astype(np.int64), V)
    x = P["wte.weight"][rows].reshape(B, S, H)
    mask = np.triu(np.ones((S, S), dtype=bool), 1)
    caches = []
    for i in range(cfg["layers"]):
        pre = f"h.{i}."
        h1, c1 = _ln(x, P[pre + "ln_1.gamma"], P[pre + "ln_1.beta"])
        q, k, v = (h1 @ P[pre + f"attn.qkv.{n}.weight"].T for n in ("query", "key", "value"))
        heads = lambda t: t.reshape(B, S, nh, hd).transpose(0, 2, 1, 3)  # noqa: E731
        qh, kh, vh = heads(q), heads(k), heads(v)
        s = (qh @ kh.transpose(0, 1, 3, 2)) * (1.0 / math.sqrt(hd))
        s = np.where(mask, -np.inf, s)
        e = np.exp(s - s.max(-1, keepdims=True))
        pr = e / e.sum(-1, keepdims=True)
        ctx = (pr @ vh).transpose(0, 2, 1, 3).reshape(B, S, H)
        a = ctx @ P[pre + "attn.out_proj.weight"].T + P[pre + "attn.out_proj.bias"]
        r = a + x
        h2, c2 = _ln(r, P[pre + "ln_2.gamma"], P[pre + "ln_2.beta"])
        f1 = h2 @ P[pre + "mlp.c_fc.weight"].T + P[pre + "mlp.c_fc.bias"]
        act = gelu(f1)
        m = act @ P[pre + "mlp.c_proj.weight"].T + P[pre + "mlp.c_proj.bias"]
        caches.append((x, c1, h1, qh, kh, vh, pr, ctx, c2, h2, f1, act))
        x = m + r
    hf, cf = _ln(x, P["ln_f.gamma"], P["ln_f.beta"])
    out = hf @ P["lm_head.weight"].T
    G["lm_head.weight"] = np.ones((T, V)).T @ hf.reshape(T, H)
    ghf = np.ones_like(out) @ P["lm_head.weight"]
    gx, G["ln_f.gamma"], G["ln_f.beta"] = _ln_bwd(ghf, P["ln_f.gamma"], cf)
    for i in reversed(range(cfg["layers"])):
        pre = f"h.{i}."
        x_in, c1, h1, qh, kh, vh, pr, ctx, c2, h2, f1, act = caches[i]
        gm = gx  # d(out)/dm and the residual r
        G[pre + "mlp.c_proj.weight"] = gm.reshape(T, H).T @ act.reshape(T, -1)
        G[pre + "mlp.c_proj.bias"] = gm.reshape(T, H).sum(0)
        gf1 = (gm @ P[pre + "mlp.c_proj.weight"]) * gelu_grad(f1)
        G[pre + "mlp.c_fc.weight"] = gf1.reshape(T, -1).T @ h2.reshape(T, H)
        G[pre + "mlp.c_fc.bias"] = gf1.reshape(T, -1).sum(0)
        gh2 = gf1 @ P[pre + "mlp.c_fc.weight"]
        gr_ln, G[pre + "ln_2.gamma"], G[pre + "ln_2.beta"] = _ln_bwd(gh2, P[pre + "ln_2.gamma"], c2)
        gr = gx + gr_ln
        G[pre + "attn.out_proj.weight"] = gr.reshape(T, H).T @ ctx.reshape(T, H)
        G[pre + "attn.out_proj.bias"] = gr.reshape(T, H).sum(0)
        gctx = (gr @ P[pre + "attn.out_proj.weight"]).reshape(B, S, nh, hd).transpose(0, 2, 1, 3)
        gvh = pr.transpose(0, 1, 3, 2) @ gctx
        gpr = gctx @ vh.transpose(0, 1, 3, 2)
        gs = pr * (gpr - (gpr * pr).sum(-1, keepdims=True)) * (1.0 / math.sqrt(hd))
        gqh, gkh = gs @ kh, gs.transpose(0, 1, 3, 2) @ qh
        merge = lambda t: t.transpose(0, 2, 1, 3).reshape(B, S, H)  # noqa: E731
        gh1 = 0.0
        for n, g in (("query", gqh), ("key", gkh), ("value", gvh)):
            gg = merge(g)
            G[pre + f"attn.qkv.{n}.weight"] = gg.reshape(T, H).T @ h1.reshape(T, H)
            gh1 = gh1 + gg @ P[pre + f"attn.qkv.{n}.weight"]
        gx_ln, G[pre + "ln_1.gamma"], G[pre + "ln_1.beta"] = _ln_bwd(gh1, P[pre + "ln_1.gamma"], c1)
        gx = gr + gx_ln
    gw = np.zeros_like(P["wte.weight"])
    np.add.at(gw, rows, gx.reshape(T, H))
    G["wte.weight"] = gw
    return out, G


def test_causal_oracle_matches_numpy_decoder(tmp_path):
    """verify mode: outputs and every gradient of the patched reference on gpt_neo
    equal the numpy f64 restatement (1e-10 relative)."""
    tmp = str(tmp_path)
    mj = _write(tmp, "neo.json", _neo().to_json())
    with ref.run(model_json=mj, causal=True, mode="verify", dump_params=1) as r:
        P = r.params(0)
        ids = r.inputs()[0]
        out, G = neo_step(P, ids, NEO)
        want = r.outputs(0)[0]
        assert np.abs(out - want).max() <= 1e-10 * np.abs(want).max()
        gr = r.grads(0)
        assert set(gr) == set(G), sorted(set(gr) ^ set(G))
        for k, v in gr.items():
            assert np.abs(G[k] - v).max() <= 1e-10 * max(np.abs(v).max(), 1e-12), k
    # and the mask is real: the unpatched reference (no mask) gives different outputs
    with ref.run(model_json=mj, mode="verify", backward=0) as r0:
        assert np.abs(r0.outputs(0)[0] - want).max() > 1e-3 * np.abs(want).max()


@pytest.mark.parametrize("world", [1, 2])
def test_decoder_recipe_applies_identically(tmp_path, world):
    """gpt_neo written here, loaded by the reference; the decoder recipe
    (FusedQKV + TP + causal EfficientAttention + bias+GeLU fusion + checkpoint)
    gives byte-identical post-apply JSON on both sides."""
    tmp = str(tmp_path)
    m = _neo()
    mj = _write(tmp, "neo.json", m.to_json())
    script = recipes.neo_script(NEO["layers"], world, checkpoint_layers=[0])
    sch = _write(tmp, "neo.sch", script)
    out = os.path.join(tmp, "ref")
    os.makedirs(out)
    ref.run(model_json=mj, causal=True, schedule=sch, world=world, outdir=out, backward=0, mode="verify").close()
    s = sb.create_schedule(m, world)
    s.load_script(script)
    mine = s.apply().to_json()
    assert mine == open(os.path.join(out, "model.json")).read()
    assert '"causal": 1' in mine and "EfficientAttention" in mine


T5 = dict(enc_layers=2, dec_layers=2, hidden=32, heads=4, vocab=32, batch=2, enc_seq=12, dec_seq=8, p=0.1)


def _t5():
    c = T5
    return sb.t5(c["enc_layers"], c["dec_layers"], c["hidden"], c["heads"], c["vocab"], c["batch"], c["enc_seq"],
                 c["dec_seq"], c["p"])


@pytest.mark.parametrize("world", [1, 2])
def test_t5_recipe_applies_identically(tmp_path, world):
    """the encoder-decoder (cross-attention, shared embedding, two id inputs) loads into
    the reference and its recipe applies to byte-identical JSON; replacing the
    cross-attention core violates R4 on both sides (q and k/v shapes differ)"""
    tmp = str(tmp_path)
    m = _t5()
    mj = _write(tmp, "t5.json", m.to_json())
    script = recipes.t5_script(2, 2, world, checkpoint=["encoder.block.0", "decoder.block.1"])
    sch = _write(tmp, "t5.sch", script)
    out = os.path.join(tmp, "ref")
    os.makedirs(out)
    ref.run(model_json=mj, causal=True, schedule=sch, world=world, outdir=out, backward=0, mode="verify").close()
    s = sb.create_schedule(m, world)
    s.load_script(script)
    assert s.apply().to_json() == open(os.path.join(out, "model.json")).read()
    bad = _write(tmp, "bad.sch", "replace decoder.block.0.cross_attn.core with EfficientAttention\n")
    with pytest.raises(RuntimeError, match="R4"):
        ref.run(model_json=mj, causal=True, schedule=bad, outdir=out, backward=0, mode="verify")
    s = sb.create_schedule(m, 1)
    s.load_script(open(bad).read())
    with pytest.raises(sb.SlapoError, match="R4"):
        s.apply()
