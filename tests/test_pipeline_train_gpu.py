"""Pipeline-parallel training step (f1; csrc/host/pipeline_exec.cpp) against the
reference executor.

The reference's run_pipeline (proj/src/executor.cpp:1531-1579) is forward-only;
its training-step semantics follow from it: micro-batch m of every stage runs
the stage module with the executor seed on micro-batch-shaped tensors, and the
loss is the sum of all outputs. So
  * verify mode (no dropout): the pipelined gradients equal the reference's
    full-batch gradients of the unsplit model (sum over micro-batches of a
    per-sample model);
  * train mode: they equal the sum over micro-batches of the reference's
    gradients of the unsplit model run on that micro-batch (same seed, same
    micro-batch-local dropout indices as run_pipeline's stages).
Stage parameters carry the partitioner's names (encoder_p0.layer_p0.0...); they
map back to the model's by dropping the _p<k> suffixes.
"""
import re

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref
from tests.helpers import BF16_GRAD_TOL, BF16_OUT_TOL, compare_grads, rel_err, rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="oracle not built")]

SPLIT1 = "trace encoder.layer\npipeline_split encoder.layer after=1\n"
SPLIT02 = "trace encoder.layer\npipeline_split encoder.layer after=0\npipeline_split encoder.layer after=2\n"


def _plan(cfg, script):
    m = sb.toy_bert(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])
    s = sb.create_schedule(m, 2)  # pipeline_split needs a distributed world (R2); stages run at world 1
    s.load_script(script)
    return m, s.apply_pipeline()


def _merged(stage_grads):
    out = {}
    for g in stage_grads:
        for k, v in g.params.items():
            name = re.sub(r"_p\d+(?=\.|$)", "", k)
            assert name not in out, name
            out[name] = v
    return out


def _ref_grads(cfg, mode, seed, input_seed, micro=1, x=None, dtype="f64", schedule=None):
    """reference gradients of the unsplit model: full batch (micro=1) or the sum over
    micro-batches of runs on each micro-batch's inputs"""
    if micro == 1:
        with ref.run("toy_bert", schedule=schedule, mode=mode, seed=seed, input_seed=input_seed, dtype=dtype,
                     **cfg) as r:
            return r.outputs(0), r.grads(0)
    per = cfg["batch"] // micro
    tot, outs = None, []
    for mb in range(micro):
        c = dict(cfg, batch=per)
        with ref.run("toy_bert", mode=mode, seed=seed, inputs=[x[mb * per:(mb + 1) * per]], dtype=dtype, **c) as r:
            g = r.grads(0)
            outs.append(r.outputs(0)[0])
        tot = g if tot is None else {k: tot[k] + g[k] for k in tot}
    return [np.concatenate(outs, 0)], tot


CFG = dict(layers=4, hidden=32, heads=4, vocab=32, batch=4, seq=8, p=0.1)


@pytest.mark.parametrize("script,micro", [(SPLIT1, 1), (SPLIT1, 2), (SPLIT02, 4)])
def test_pipeline_step_verify_equals_full_batch(script, micro):
    m, plan = _plan(CFG, script)
    x = m.random_inputs(9)
    pe = sb.PipelineExecutor(plan, micro, "verify", 123, "fp32")
    out = pe.forward(x)
    grads = _merged(pe.backward())
    want_out, want = _ref_grads(CFG, "verify", 123, 9)
    assert rel_err(out[0], want_out[0]) <= 1e-4
    compare_grads(grads, {k: v.ravel() for k, v in want.items()}, 1e-4)


@pytest.mark.parametrize("micro", [1, 2])
def test_pipeline_step_train_equals_micro_batch_sum(micro):
    m, plan = _plan(CFG, SPLIT1)
    x = m.random_inputs(9)
    pe = sb.PipelineExecutor(plan, micro, "train", 123, "fp32")
    out = pe.forward(x)
    grads = _merged(pe.backward())
    want_out, want = _ref_grads(CFG, "train", 123, 9, micro, x[0])
    assert rel_err(out[0], want_out[0]) <= 1e-4
    compare_grads(grads, {k: v.ravel() for k, v in want.items()}, 1e-4)
    # a second step (stashes, seeds and accumulators reused) gives the same gradients
    pe.forward(x)
    again = _merged(pe.backward())
    for k in grads:
        assert np.array_equal(grads[k], again[k]), k


def test_pipeline_step_bf16_tcgen05():
    """C2's fused + flash-attention schedule split in two stages, bf16 on the tcgen05
    kernels, 2 micro-batches, verify mode vs the reference's full batch"""
    cfg = dict(layers=2, hidden=256, heads=4, vocab=64, batch=8, seq=128, p=0.1)
    m, plan = _plan(cfg, recipes.c2_script(2) + SPLIT1.replace("after=1", "after=0"))
    x = m.random_inputs(9)
    pe = sb.PipelineExecutor(plan, 2, "verify", 123, "bf16")
    out = pe.forward(x)
    grads = _merged(pe.backward())
    assert sb.lib().sb_attn_engine(1) == 3 and sb.lib().sb_gemm_engine() == 2
    want_out, want = _ref_grads(cfg, "verify", 123, 9, schedule=recipes.c2_script(2))  # (fused module names)
    assert rel_l2(out[0], want_out[0]) <= BF16_OUT_TOL
    compare_grads(grads, {k: v.ravel() for k, v in want.items()}, BF16_GRAD_TOL, rel_l2)


def test_pipeline_timing_and_errors():
    m, plan = _plan(CFG, SPLIT02)
    pe = sb.PipelineExecutor(plan, 2, "train", 1, "fp32")
    with pytest.raises(sb.SlapoError):
        pe.backward()  # before any forward
    x = m.random_inputs(3)
    pe.forward(x)
    g0 = _merged(pe.backward())
    assert pe.time_steps(2, use_graph=False) > 0
    assert pe.time_steps(3) > 0  # the step captured into a CUDA graph and replayed
    pe.forward(x)  # eager again after the replays: identical gradients
    g1 = _merged(pe.backward())
    for k in g0:
        assert np.array_equal(g0[k], g1[k]), k
    with pytest.raises(sb.SlapoError, match="micro-batches"):
        sb.PipelineExecutor(plan, 3, "train", 1, "fp32")  # batch 4 is not divisible by 3
    with pytest.raises(sb.SlapoError, match="one device per stage"):
        sb.PipelineExecutor(plan, 2, "train", 1, "fp32", devices=[0])


@pytest.mark.parametrize("mode", ["verify", "train"])
def test_pipeline_with_tensor_parallel_stages(mode):
    """C5's TP x PP shape on one GPU ('pin each stage's TP with
    run_sharded, and the composition at world 1, separately'): the TP=2 recipe split into
    2 stages, each on 2 lockstep tensor-parallel ranks, 2 micro-batches. Per rank, the
    gradients equal the unsplit TP=2 executor's (pinned against the reference's
    run_sharded by tests/test_parity_gpu.py): verify — on the full batch; train — summed
    over unsplit runs on each micro-batch (run_pipeline's per-chunk semantics)."""
    cfg = dict(layers=4, hidden=32, heads=4, vocab=32, batch=4, seq=8, p=0.1)
    script = recipes.tp_script(4, 2, ckpt_ratio=0.25)
    m, plan = _plan(cfg, script + SPLIT1)
    x = m.random_inputs(9)
    pe = sb.PipelineExecutor(plan, 2, mode, 123, "fp32", tp=2)
    out = pe.forward(x)
    g = pe.backward()
    assert len(g) == 2 * 2
    got = [_merged([g[st * 2 + r] for st in range(2)]) for r in range(2)]
    micro = 1 if mode == "verify" else 2
    per = cfg["batch"] // micro
    want, wout = None, []
    for mb in range(micro):
        mm = sb.toy_bert(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], per, cfg["seq"], cfg["p"])
        s = sb.create_schedule(mm, 2)
        s.load_script(script)
        ex = sb.Executor(s.apply(), mode, 123, 2)
        wout.append(ex.forward([x[0][mb * per:(mb + 1) * per]])[0])
        gm = [r.params for r in ex.backward_all_ranks()]
        want = gm if want is None else [{k: a[k] + b[k] for k in a} for a, b in zip(want, gm)]
    assert rel_err(out[0], np.concatenate(wout, 0)) <= 1e-4
    for r in range(2):
        compare_grads(got[r], want[r], 1e-4)


@pytest.mark.parametrize("tp", [1, 2])
def test_t5_pipeline_step(tp):
    """C5 as an encoder-decoder: the T5-style model (t5_script at TP tp) split inside the
    encoder into 2 stages (the decoder's ids are consumed by stage 1), 2 micro-batches, verify
    mode; per rank the gradients equal the unsplit executor's (TP 1: the reference's)"""
    import os
    cfg = dict(enc_layers=2, dec_layers=2, hidden=32, heads=4, vocab=32, batch=4, enc_seq=24, dec_seq=16)
    # (untied tables: a tied one would be used by both segments, which the partitioner rejects)
    m = sb.t5(cfg["enc_layers"], cfg["dec_layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"],
              cfg["enc_seq"], cfg["dec_seq"], 0.1, tie_embeddings=False)
    script = recipes.t5_script(2, 2, tp, tied=False)
    s = sb.create_schedule(m, 2)
    s.load_script(script + "trace encoder.block\npipeline_split encoder.block after=0\n")
    plan = s.apply_pipeline()
    assert len(plan.stages) == 2
    x = m.random_inputs(9)
    pe = sb.PipelineExecutor(plan, 2, "verify", 123, "fp32", tp=tp)
    out = pe.forward(x)
    g = pe.backward()
    s2 = sb.create_schedule(m, tp)
    s2.load_script(script)
    ex = sb.Executor(s2.apply(), "verify", 123, tp)
    wout = ex.forward(x)[0]
    want = [r.params for r in ex.backward_all_ranks()]
    assert rel_err(out[0], wout) <= 1e-4
    for r in range(tp):
        compare_grads(_merged([g[st * tp + r] for st in range(2)]), want[r], 1e-4)
