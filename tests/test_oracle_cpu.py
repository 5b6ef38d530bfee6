"""Pin the CPU oracle (oracle/slapo_oracle.py, numpy + the C restatement of the
RNG) against golden vectors produced by the reference's own executor
(tests/golden/make_golden.py), and pin the host boundary (schedule apply,
param materialisation, host plan / activation ledger) against the same
fixtures. CPU only; nothing here reads /root/reference."""
import json
import os

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from oracle import slapo_oracle as so
from paper_2302_08005_b200 import recipes

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
HAVE_C = os.path.exists(os.path.join(os.path.dirname(so.__file__), "_ref", "librefrng.so"))


def load(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def model_of(meta):
    if meta["model"] == "fig3c":
        return sb.fig3c_exact()
    return sb.toy_bert(meta["layers"], meta["hidden"], meta["heads"], meta["vocab"], meta["batch"], meta["seq"], meta["p"])


def test_rng_bit_exact():
    z = np.load(os.path.join(GOLD, "rng.npz"))
    s = int(z["stream"][0])
    assert s == so.hash_combine(123, 1040)
    got = so.uniform01_array(s, 0xD0, 4096)
    assert got.tobytes() == z["uniform01"].tobytes()


@pytest.mark.skipif(not HAVE_C, reason="oracle C restatement not built (make -C oracle)")
def test_oracle_param_init_bit_exact():
    z, meta = load("toy_train")
    params = so.toy_bert_params(so.BertCfg(meta["layers"], meta["hidden"], meta["heads"], meta["vocab"], meta["batch"],
                                           meta["seq"], meta["p"]))
    for k, v in params.items():
        assert v.tobytes() == z[f"param/0/{k}"].tobytes(), k
    assert so.random_tensor((meta["batch"], meta["seq"]), 9, 0).tobytes() == z["input/0"].tobytes()


@pytest.mark.skipif(not HAVE_C, reason="oracle C restatement not built (make -C oracle)")
@pytest.mark.parametrize("case", ["toy_train", "toy_verify"])
def test_numpy_oracle_matches_reference(case):
    z, meta = load(case)
    c = so.BertCfg(meta["layers"], meta["hidden"], meta["heads"], meta["vocab"], meta["batch"], meta["seq"], meta["p"])
    out, grads = so.toy_bert_step(c, z["input/0"], meta["seed"], train=meta["mode"] == "train")
    assert np.abs(out - z["out/0/0"]).max() <= 1e-12 * max(1.0, np.abs(z["out/0/0"]).max())
    for k, g in grads.items():
        w = z[f"grad/0/{k}"]
        assert np.abs(g - w).max() <= 1e-10 * max(1.0, np.abs(w).max()), k


def test_boundary_param_values_match_golden():
    for case in ("toy_train", "toy_tp2"):
        z, meta = load(case)
        m = model_of(meta)
        s = sb.create_schedule(m, meta["world"])
        if meta["schedule"]:
            s.load_script(meta["schedule"])
        a = s.apply()
        # the post-apply model is structurally the reference's
        assert a.structurally_equal(sb.Model.from_json(bytes(z["model_json"]).decode()))
        for key in z.files:
            if key.startswith("param/"):
                _, rank, name = key.split("/", 2)
                assert a.param_values(name, int(rank)).tobytes() == z[key].ravel().tobytes(), key


@pytest.mark.parametrize("case", ["toy_train", "toy_c2", "toy_verify"])
def test_host_plan_ledger_matches_reference(case):
    z, meta = load(case)
    m = model_of(meta)
    s = sb.create_schedule(m, meta["world"])
    if meta["schedule"]:
        s.load_script(meta["schedule"])
    plan = sb.plan_summary(s.apply(), meta["mode"], meta["seed"], meta["world"])
    assert plan["ledger_bytes"] == meta["ledger_bytes"]


def test_known_answer_fig3c_partials_plan():
    # proj/tests/executor_test.cpp:88-121: with sync, one collective in forward
    m = sb.fig3c_exact()
    s = sb.create_schedule(m, 2)
    s.at("wa").shard(["weight"], 0)
    s.at("wb").shard(["weight"], 1)
    s.at("wb").sync("forward")
    p = sb.plan_summary(s.apply(), "verify", 0, 2, 0)
    assert p["collectives_fwd"] == 1
    assert [sb.fig3c_exact().param_values("wa.weight").tolist()] == [[1, 0, 0, 1, 1, 1, -1, 0]]


def test_tp_plans_are_lockstep_and_bias_rank0_only():
    m = sb.toy_bert(layers=2, hidden=32, heads=4, vocab=32, batch=2, seq=8)
    s = sb.create_schedule(m, 4)
    s.load_script(recipes.tp_script(2, 4))
    a = s.apply()
    plans = [sb.plan_summary(a, "train", 1, 4, r) for r in range(4)]
    assert len({p["structure"] for p in plans}) == 1
    # row-parallel biases are added before the reduce on rank 0 only (executor.cpp:645) — except
    # inside a fused Linear->all_reduce->...->LayerNorm region, where the whole bias is added once
    # after the reduce on every rank (identical sum)
    assert plans[0]["bias_added"] == plans[1]["bias_added"]


def test_c3_plan_shape():
    m = sb.toy_bert(layers=4, hidden=64, heads=4, vocab=64, batch=2, seq=16)
    s = sb.create_schedule(m, 1)
    s.load_script(recipes.tp_script(4, 1, ckpt_ratio=0.25))
    p = sb.plan_summary(s.apply(), "train", 123, 1, 0, "bf16")
    assert p["kinds"]["FlashAttn"] == 4
    assert p["kinds"]["FusedLinearResLN"] == 8
    assert p["kinds"]["FusedLinearGelu"] == 4
    assert p["gelu_folded"] == 4  # every dense1 GeLU backward folded into dense2's dgrad
    assert p["regions"] == 1
