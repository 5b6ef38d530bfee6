"""GPU parity of the decoder model family (f2, BASELINE.json configs[3]):
``gpt_neo`` (pre-LN blocks, causal self-attention) through the B200 executor
(C ABI) against the documented causal oracle extension (oracle/causal_ext.py:
the reference executor with a `causal` softmax attr, pinned against a numpy
restatement in tests/test_causal_oracle_cpu.py), same seeds / inputs / schedule.

Tolerances as for the encoder: fp32 1e-4 per tensor
(||a-b||_inf/||b||_inf) on outputs, loss and every gradient; bf16 relL2 2e-2
outputs, 5e-2 gradients, and 2e-3 on the loss taken relative to sum|logits|
(the logits have both signs, so their plain sum cancels; the condition number
sum|o| / |sum o| is recorded with the errors).
"""
import json
import os

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref
from tests.helpers import BF16_GRAD_TOL, BF16_LOSS_TOL, BF16_OUT_TOL, rel_l2
from tests.test_parity_gpu import check

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not os.path.exists(ref.DRIVER_CAUSAL), reason="causal oracle not built")]


def run_both(tmp, cfg, script, world, mode="train", dtype="fp32", seed=123, input_seed=9):
    m = sb.gpt_neo(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])
    mj = os.path.join(tmp, "neo.json")
    with open(mj, "w") as f:
        f.write(m.to_json())
    s = sb.create_schedule(m, world)
    if script:
        s.load_script(script)
    ex = sb.Executor(s.apply(), mode, seed, world, dtype=dtype)
    ex.forward(m.random_inputs(input_seed))
    outs = [ex.outputs_of_rank(r) for r in range(world)]
    grads = ex.backward_all_ranks()
    r = ref.run(model_json=mj, causal=True, schedule=script or None, world=world, mode=mode, seed=seed,
                input_seed=input_seed)
    return ex, outs, grads, r


SMALL = dict(layers=2, hidden=32, heads=2, vocab=32, batch=2, seq=16, p=0.1)


@pytest.mark.parametrize("mode", ["train", "verify"])
def test_decoder_unscheduled_fp32(tmp_path, mode):
    """the composed causal attention core (causal softmax kernel) and pre-LN blocks"""
    _, outs, grads, r = run_both(str(tmp_path), SMALL, "", 1, mode)
    check(outs, grads, r, 1, 1e-4, 1e-4)


@pytest.mark.parametrize("world", [1, 2])
def test_decoder_recipe_fp32(tmp_path, world):
    """FusedQKV (bias-free) + TP shard/sync + causal EfficientAttention + bias+GeLU
    fusion + a checkpointed block, at TP 1 and 2 (local placement)"""
    script = recipes.neo_script(SMALL["layers"], world, checkpoint_layers=[1])
    ex, outs, grads, r = run_both(str(tmp_path), SMALL, script, world)
    check(outs, grads, r, world, 1e-4, 1e-4)
    assert ex.collective_invocations() == r.meta["collectives_total"]


@pytest.mark.parametrize("heads,seq", [(4, 128), (2, 128), (4, 256)])
def test_decoder_recipe_bf16(tmp_path, heads, seq):
    """bf16 on the tensor-core paths: head_dim 64 runs the tcgen05 causal flash
    attention (k_fa6_fwd<true> / k_fa7_bwd<true>), head_dim 128 the mma.sync one"""
    cfg = dict(layers=2, hidden=256, heads=heads, vocab=64, batch=2, seq=seq, p=0.1)
    script = recipes.neo_script(2, 1, checkpoint_layers=[0])
    _, outs, grads, r = run_both(str(tmp_path), cfg, script, 1, dtype="bf16")
    check(outs, grads, r, 1, BF16_OUT_TOL, BF16_GRAD_TOL, metric=rel_l2, tol_loss=BF16_LOSS_TOL,
          record=f"decoder_bf16_h256_nh{heads}_s{seq}", loss_l1=True)
    if heads == 4:
        assert sb.lib().sb_attn_engine(0) == 3 and sb.lib().sb_attn_engine(1) == 3


def test_decoder_prefix_independence(tmp_path):
    """causality end to end: outputs of the first S/2 positions do not change when
    the second half of every sequence changes (verify mode, bf16 tcgen05 path)"""
    cfg = dict(layers=2, hidden=256, heads=4, vocab=64, batch=2, seq=128, p=0.0)
    m = sb.gpt_neo(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])
    s = sb.create_schedule(m, 1)
    s.load_script(recipes.neo_script(2, 1))
    ex = sb.Executor(s.apply(), "verify", 5, 1, dtype="bf16")
    ids = m.random_inputs(3)[0]
    a = ex.forward([ids])[0]
    ids2 = ids.copy()
    ids2[:, 64:] = np.random.default_rng(0).normal(size=ids2[:, 64:].shape)
    b = ex.forward([ids2])[0]
    assert np.array_equal(a[:, :64], b[:, :64])
    assert not np.array_equal(a[:, 64:], b[:, 64:])


T5 = dict(enc_layers=2, dec_layers=2, hidden=32, heads=4, vocab=32, batch=2, enc_seq=24, dec_seq=16, p=0.1)


def run_t5(tmp, cfg, script, world, mode="train", dtype="fp32", seed=123, input_seed=9):
    m = sb.t5(cfg["enc_layers"], cfg["dec_layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"],
              cfg["enc_seq"], cfg["dec_seq"], cfg["p"])
    mj = os.path.join(tmp, "t5.json")
    with open(mj, "w") as f:
        f.write(m.to_json())
    s = sb.create_schedule(m, world)
    if script:
        s.load_script(script)
    ex = sb.Executor(s.apply(), mode, seed, world, dtype=dtype)
    ex.forward(m.random_inputs(input_seed))
    outs = [ex.outputs_of_rank(r) for r in range(world)]
    grads = ex.backward_all_ranks()
    r = ref.run(model_json=mj, causal=True, schedule=script or None, world=world, mode=mode, seed=seed,
                input_seed=input_seed)
    return ex, outs, grads, r


@pytest.mark.parametrize("mode", ["train", "verify"])
def test_t5_unscheduled_fp32(tmp_path, mode):
    """encoder-decoder with cross-attention (S_dec x S_enc scores), causal decoder
    self-attention, a shared embedding used twice, two id inputs"""
    _, outs, grads, r = run_t5(str(tmp_path), T5, "", 1, mode)
    check(outs, grads, r, 1, 1e-4, 1e-4)


@pytest.mark.parametrize("world", [1, 2])
def test_t5_recipe_fp32(tmp_path, world):
    """the cross-attention cores stay composed in the schedule (R4) and are lowered to the
    flash kernels by their graph (S_dec != S_enc); the activation ledger still follows the
    reference's accounting of the composed graph"""
    script = recipes.t5_script(2, 2, world, checkpoint=["encoder.block.0", "decoder.block.1"])
    ex, outs, grads, r = run_t5(str(tmp_path), T5, script, world)
    check(outs, grads, r, world, 1e-4, 1e-4)
    assert ex.collective_invocations() == r.meta["collectives_total"]
    assert ex.ledger() == r.meta["ledger_bytes"]
    assert ex.describe()["kinds"].get("FlashAttn", 0) == 2 + 2 + 2  # encoder self, decoder self and cross cores


def test_t5_cross_core_composed_switch(tmp_path):
    """SB_ATTN_CORE_FLASH=0 keeps the composed cross-attention graph; both agree"""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2302_08005_b200 as sb\n"
            "m = sb.t5(2, 2, 32, 4, 32, 2, 24, 16, 0.1); ex = sb.Executor(m, 'train', 5, 1)\n"
            "o = ex.forward(m.random_inputs(3))[0]; g = ex.backward().params\n"
            "np.save(sys.argv[1], np.concatenate([o.ravel()] + [g[k].ravel() for k in sorted(g)]))\n"
            "print(ex.ledger())\n") % root
    res = []
    for v in ("1", "0"):
        f = str(tmp_path / f"r{v}.npy")
        r = subprocess.run([sys.executable, "-c", code, f], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, SB_ATTN_CORE_FLASH=v))
        assert r.returncode == 0, r.stderr
        res.append((np.load(f), r.stdout.strip()))
    (a, la), (b, lb) = res
    assert la == lb  # same ledger
    assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()


def test_t5_recipe_bf16(tmp_path):
    cfg = dict(T5, hidden=256, heads=4, vocab=64, enc_seq=256, dec_seq=128)
    script = recipes.t5_script(2, 2, 1, checkpoint=["decoder.block.0"])
    _, outs, grads, r = run_t5(str(tmp_path), cfg, script, 1, dtype="bf16")
    check(outs, grads, r, 1, BF16_OUT_TOL, BF16_GRAD_TOL, metric=rel_l2, tol_loss=BF16_LOSS_TOL,
          record="t5_bf16_h256_enc256_dec128", loss_l1=True)


def test_residual_stream_fusion(tmp_path):
    """pre-LN blocks: out_proj / mlp.c_proj -> dropout -> residual add -> next LayerNorm run as
    one FusedLinearResLN whose sum is also the residual stream (lower.cpp
    fuse_residual_stream); SB_RESLN_FUSE=0 keeps the separate ops — same results"""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2302_08005_b200 as sb\n"
            "m = sb.gpt_neo(2, 32, 2, 32, 2, 16, 0.1); ex = sb.Executor(m, 'train', 5, 1)\n"
            "o = ex.forward(m.random_inputs(3))[0]; g = ex.backward().params\n"
            "np.save(sys.argv[1], np.concatenate([o.ravel()] + [g[k].ravel() for k in sorted(g)]))\n"
            "print(json.dumps(ex.describe()['kinds']))\n") % root
    res = []
    for v in ("1", "0"):
        f = str(tmp_path / f"r{v}.npy")
        r = subprocess.run([sys.executable, "-c", code, f], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, SB_RESLN_FUSE=v))
        assert r.returncode == 0, r.stderr
        res.append((np.load(f), json.loads(r.stdout.strip().splitlines()[-1])))
    (a, ka), (b, kb) = res
    # per block: attn.out_proj + ln_2 and mlp.c_proj + the next LayerNorm (block 1's ln_1, then ln_f)
    assert ka.get("FusedLinearResLN", 0) == 4 and kb.get("FusedLinearResLN", 0) == 0, (ka, kb)
    assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()


def test_t5_relu_fold(tmp_path):
    """T5's feed-forward wi -> relu -> wo: the ReLU runs in wi's GEMM epilogue and its backward
    in wo's dgrad epilogue (lower.cpp fuse_linear_relu); SB_RELU_FUSE=0 keeps the separate op —
    fp32: the same outputs and gradients up to rounding; no Relu op left in the fused plan."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2302_08005_b200 as sb\n"
            "m = sb.t5(2, 2, 32, 4, 32, 2, 24, 16, 0.1); ex = sb.Executor(m, 'train', 5, 1)\n"
            "o = ex.forward(m.random_inputs(3))[0]; g = ex.backward().params\n"
            "np.save(sys.argv[1], np.concatenate([o.ravel()] + [g[k].ravel() for k in sorted(g)]))\n"
            "print(json.dumps(ex.describe()['kinds']))\n") % root
    res = []
    for v in ("1", "0"):
        f = str(tmp_path / f"r{v}.npy")
        r = subprocess.run([sys.executable, "-c", code, f], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, SB_RELU_FUSE=v))
        assert r.returncode == 0, r.stderr
        res.append((np.load(f), json.loads(r.stdout.strip().splitlines()[-1])))
    (a, ka), (b, kb) = res
    assert ka.get("Relu", 0) == 0 and kb.get("Relu", 0) == 4, (ka, kb)  # 2 encoder + 2 decoder blocks
    assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()
