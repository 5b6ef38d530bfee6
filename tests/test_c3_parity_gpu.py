"""X1: parity at the benchmarked configuration (BASELINE.json configs[2], C3).

The scheduled BERT-large recipe — FusedQKV, shard+sync, EfficientAttention, the
all_reduce-including fusions, vocab-parallel embeddings, checkpoint — at full
BERT-large width (H 1024, 16 heads, hd 64, F 4096, S 512, V 30528) in bf16 on
the sm_100a kernels (2-SM tcgen05 GEMM, tcgen05 flash attention at S=512,
vectorised fused LayerNorm, vocab-parallel embedding), against the reference
executor itself (oracle/_ref/slapo_ref_driver: the reference's proj/src compiled
by oracle/Makefile, f64) on the same seeds, inputs and schedule script.
Reference entry points: Executor::forward + backward_all_ranks
(proj/src/executor.cpp:285-381), run under run_sharded semantics for TP=2.

Depth is what the CPU reference can afford (L <= 2 at this
width, ~70 s per layer-step on one core); B=1 so the CPU runs finish in minutes.
All reference runs of this module start together in a module fixture (one
process per run, each single-threaded) and overlap each other.

Checked per rank: every output, the loss (sum of outputs, executor.cpp:355-362)
and every parameter gradient. Metric: relL2 per tensor (the
analytically-zero key-bias gradient normalised by its QKV-bias group). The
measured errors are written to $SB_PARITY_OUT (committed as
profiles/r2_bf16_parity.json) and the tolerances below are derived from them
(DESIGN.md §2).
"""
import json
import os
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref
from tests.helpers import BF16_GRAD_TOL, BF16_LOSS_TOL, BF16_OUT_TOL, group_scale, rel_err, rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle not built")]

C3W = dict(hidden=1024, heads=16, vocab=30528, batch=1, seq=512, p=0.1)
# (layers, world, mode, checkpoint ratio)
CASES = [(1, 1, "train", 1.0), (1, 2, "train", 1.0), (1, 1, "verify", 0.0), (1, 2, "verify", 0.0),
         (2, 1, "train", 0.5), (2, 2, "train", 0.5), (2, 1, "verify", 0.0), (2, 2, "verify", 0.0)]



def _name(c):
    L, world, mode, ck = c
    return f"L{L}_tp{world}_{mode}"


def _script(c):
    L, world, _, ck = c
    return recipes.tp_script(L, world, ckpt_ratio=ck)


@pytest.fixture(scope="module")
def ref_runs():
    tmp = tempfile.TemporaryDirectory(prefix="sb_c3ref_")

    def one(c):
        L, world, mode, _ = c
        d = os.path.join(tmp.name, _name(c))
        os.makedirs(d)
        return _name(c), ref.run("toy_bert", schedule=_script(c), outdir=d, layers=L, world=world, mode=mode,
                                 seed=123, input_seed=9, timeout=3000, **C3W)

    with ThreadPoolExecutor(len(CASES)) as pool:
        runs = dict(pool.map(one, CASES))
    yield runs
    tmp.cleanup()


def _record(name, rec):
    out = os.environ.get("SB_PARITY_OUT")
    if not out:
        return
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"c3_{name}.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)


@pytest.mark.parametrize("case", CASES, ids=_name)
def test_c3_width_bf16_vs_reference(case, ref_runs):
    L, world, mode, _ = case
    r = ref_runs[_name(case)]
    m = sb.toy_bert(L, C3W["hidden"], C3W["heads"], C3W["vocab"], C3W["batch"], C3W["seq"], C3W["p"])
    s = sb.create_schedule(m, world)
    s.load_script(_script(case))
    ex = sb.Executor(s.apply(), mode, 123, world, dtype="bf16")
    ex.forward(m.random_inputs(9))
    engines = dict(gemm=sb.lib().sb_gemm_engine(), attn_fwd=sb.lib().sb_attn_engine(0))
    grads = ex.backward_all_ranks()
    engines["attn_bwd"] = sb.lib().sb_attn_engine(1)
    assert engines == dict(gemm=2, attn_fwd=3, attn_bwd=3), engines
    assert ex.collective_invocations() == r.meta["collectives_total"]

    rec = {"case": _name(case), "layers": L, "world": world, "mode": mode, **C3W, "ranks": []}
    worst_out = worst_loss = 0.0
    worst_grad = (0.0, None)
    for rank in range(world):
        outs = ex.outputs_of_rank(rank)
        want = r.outputs(rank)
        assert len(outs) == len(want)
        e_out = max(rel_l2(g, w) for g, w in zip(outs, want))
        e_out_inf = max(rel_err(g, w) for g, w in zip(outs, want))
        loss_g = sum(float(np.asarray(o, dtype=np.float64).sum()) for o in outs)
        loss_w = sum(float(w.sum()) for w in want)
        e_loss = abs(loss_g - loss_w) / abs(loss_w)
        gw = r.grads(rank)
        got = grads[rank].params
        assert set(got) == set(gw), sorted(set(got) ^ set(gw))
        per = {}
        for k, w in gw.items():
            gs = group_scale(k, gw)
            if gs is not None:
                e = float(np.abs(np.asarray(got[k]).ravel() - np.asarray(w).ravel()).max() / gs)
            else:
                e = rel_l2(got[k], w)
            per[k] = e
            if e > worst_grad[0]:
                worst_grad = (e, f"r{rank}:{k}")
        rec["ranks"].append({"rank": rank, "out_rel_l2": e_out, "out_rel_inf": e_out_inf, "loss": loss_g,
                             "loss_ref": loss_w, "loss_rel": e_loss, "grad_rel_l2": per})
        worst_out = max(worst_out, e_out)
        worst_loss = max(worst_loss, e_loss)
    rec.update(worst_out=worst_out, worst_loss=worst_loss, worst_grad=worst_grad[0], worst_grad_name=worst_grad[1],
               engines=engines)
    _record(_name(case), rec)
    assert worst_out <= BF16_OUT_TOL, f"output relL2 {worst_out:.3e}"
    assert worst_loss <= BF16_LOSS_TOL, f"loss rel {worst_loss:.3e}"
    assert worst_grad[0] <= BF16_GRAD_TOL, f"gradient {worst_grad[1]}: {worst_grad[0]:.3e}"


# ---------------------------------------------------------------- depth scaling
# The CPU reference affords L <= 2 at this width, so the bf16 error's growth with
# depth is measured against this repo's fp32 path (SIMT fp32 GEMMs / attention,
# itself equal to the reference within 1e-5 relative wherever the reference runs:
# 1.6e-5 at BERT-large width, L = 4, train mode; tests/test_parity_gpu.py for the
# rest) on the full-width model at L = 2, 8 and 24, in verify mode. The measured
# errors go to $SB_PARITY_OUT (profiles/r2_bf16_parity.json) and set the stated
# depth rule in DESIGN.md §2.
#
# Train mode is different: with the reference's initialisation (weights
# 0.1·N(0,1), a gain of 3.2 per Linear at H = 1024, so the attention softmax is
# close to one-hot) and dropout on, the step amplifies any rounding difference by
# ~1.7x per layer: two bf16 implementations that differ only in the attention
# kernel (tcgen05 vs mma.sync) disagree with each other by as much as either does
# with fp32 (profiles/r2_bf16_parity.json). So in train mode the bf16-vs-fp32
# deviation is checked against that sensitivity floor instead of a fixed number.
DEPTH_TOL = {2: (2e-2, 2e-3, 5e-2), 8: (3e-2, 3e-3, 1.2e-1), 24: (5e-2, 5e-3, 3e-1)}


def _depth_run(layers, dtype, mode, attn_engine=0):
    m = sb.toy_bert(layers, C3W["hidden"], C3W["heads"], C3W["vocab"], C3W["batch"], C3W["seq"], C3W["p"])
    s = sb.create_schedule(m, 1)
    s.load_script(recipes.tp_script(layers, 1, ckpt_ratio=0.25))
    sb.lib().sb_attn_set_engine(attn_engine)
    try:
        ex = sb.Executor(s.apply(), mode, 123, 1, dtype=dtype)
        outs = ex.forward(m.random_inputs(9))
        return outs, ex.backward().params
    finally:
        sb.lib().sb_attn_set_engine(0)


def _errors(a, b):
    (oa, ga), (ob, gb) = a, b
    e_out = max(rel_l2(x, y) for x, y in zip(oa, ob))
    la = sum(float(np.asarray(o, dtype=np.float64).sum()) for o in oa)
    lb = sum(float(np.asarray(o, dtype=np.float64).sum()) for o in ob)
    per = {}
    for k, w in gb.items():
        gs = group_scale(k, gb)
        per[k] = (float(np.abs(np.asarray(ga[k]).ravel() - np.asarray(w).ravel()).max() / gs) if gs is not None
                  else rel_l2(ga[k], w))
    worst = max(per.items(), key=lambda kv: kv[1])
    return e_out, abs(la - lb) / abs(lb), worst, per


@pytest.mark.parametrize("layers", sorted(DEPTH_TOL))
def test_c3_width_bf16_vs_fp32_by_depth_verify(layers):
    e_out, e_loss, worst, per = _errors(_depth_run(layers, "bf16", "verify"), _depth_run(layers, "fp32", "verify"))
    _record(f"depth_L{layers}_verify_bf16_vs_fp32", {"layers": layers, **C3W, "mode": "verify", "out_rel_l2": e_out,
                                                      "loss_rel": e_loss, "worst_grad": worst[1],
                                                      "worst_grad_name": worst[0], "grad_rel_l2": per})
    t_out, t_loss, t_grad = DEPTH_TOL[layers]
    assert e_out <= t_out, e_out
    assert e_loss <= t_loss, e_loss
    assert worst[1] <= t_grad, worst


@pytest.mark.parametrize("layers", [2, 4])
def test_c3_width_bf16_train_at_sensitivity_floor(layers):
    """Train mode: bf16 (tcgen05 attention) vs fp32 is within 2x (+1e-3) of bf16
    (tcgen05) vs bf16 (mma.sync attention) — rounding noise amplified by the model,
    not a systematic deviation of one kernel."""
    f32 = _depth_run(layers, "fp32", "train")
    tc = _depth_run(layers, "bf16", "train", attn_engine=0)
    mma = _depth_run(layers, "bf16", "train", attn_engine=1)
    e32 = _errors(tc, f32)
    efl = _errors(tc, mma)
    _record(f"depth_L{layers}_train_sensitivity", {"layers": layers, **C3W, "mode": "train",
                                                    "bf16_vs_fp32": {"out": e32[0], "loss": e32[1], "worst_grad": e32[2][1]},
                                                    "bf16_tcgen05_vs_bf16_mma": {"out": efl[0], "loss": efl[1],
                                                                                 "worst_grad": efl[2][1]}})
    assert e32[0] <= 2 * efl[0] + 1e-3, (e32[0], efl[0])
    assert e32[2][1] <= 2 * efl[2][1] + 1e-3, (e32[2], efl[2])
