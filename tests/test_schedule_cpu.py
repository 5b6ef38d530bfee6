"""Host boundary parity (CPU): the schedule API applied here produces the same
post-apply ModuleDef as the reference's Schedule::apply, and parameter /
shard-map materialisation is bit-identical."""
import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes
from oracle import ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle driver not built")

TOY = dict(layers=2, hidden=32, heads=4, vocab=32, batch=2, seq=8, p=0.1)


def ours(script, world, dtype="f64", **cfg):
    c = dict(TOY)
    c.update(cfg)
    m = sb.toy_bert(c["layers"], c["hidden"], c["heads"], c["vocab"], c["batch"], c["seq"], c["p"])
    if dtype == "f32":
        m.to_f32()
    s = sb.create_schedule(m, world)
    if script:
        s.load_script(script)
    return m, s.apply()


@pytest.mark.parametrize("name,script,world", [
    ("default", "", 1),
    ("c2", recipes.c2_script(2, checkpoint_layers=[1]), 1),
    ("tp2", recipes.tp_script(2, 2, ckpt_ratio=0.5), 2),
    ("tp4", recipes.tp_script(2, 4), 4),
    ("tp1", recipes.tp_script(2, 1, ckpt_ratio=0.5), 1),
    ("bert_tp_demo", open("/dev/null").read() or
     "replace encoder.layer.*.attention.qkv with FusedQKV\n"
     "shard encoder.layer.*.attention.qkv weight,bias axis=0\n"
     "shard encoder.layer.*.attention.output.dense weight,bias axis=1\n"
     "sync encoder.layer.*.attention.output.dense type=forward\n"
     "shard embeddings weight axis=0\nsync embeddings type=both\n", 2),
])
def test_apply_matches_reference(name, script, world):
    _, applied = ours(script, world)
    r = ref.run("toy_bert", schedule=script or None, world=world, backward=0, **TOY)
    theirs = sb.Model.from_json(r.model_json())
    assert applied.structurally_equal(theirs), name
    # and the JSON round trip of ours is stable
    assert sb.Model.from_json(applied.to_json()).structurally_equal(applied)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_param_materialisation_bit_exact(world):
    script = recipes.tp_script(2, world) if world > 1 else recipes.c2_script(2)
    _, applied = ours(script, world)
    r = ref.run("toy_bert", schedule=script, world=world, backward=0, dump_params=1, **TOY)
    for rank in range(world):
        want = r.params(rank)
        assert len(want) > 20
        for name, w in want.items():
            got = applied.param_values(name, rank)
            assert got.tobytes() == w.ravel().tobytes(), (rank, name)


def test_f32_param_rounding_bit_exact():
    _, applied = ours("", 1, dtype="f32")
    r = ref.run("toy_bert", world=1, backward=0, dump_params=1, dtype="f32", **TOY)
    for name, w in r.params(0).items():
        assert applied.param_values(name, 0).tobytes() == w.ravel().tobytes(), name


def test_random_inputs_bit_exact():
    m, _ = ours("", 1)
    r = ref.run("toy_bert", world=1, backward=0, input_seed=9, **TOY)
    assert m.random_inputs(9)[0].tobytes() == r.inputs()[0].tobytes()


def test_rule_errors():
    m = sb.toy_bert(layers=1)
    s = sb.create_schedule(m, 2)
    with pytest.raises(sb.RuleError) as e:
        s.at("encoder.layer.0.attention.output.dense").sync("forward")
    assert e.value.rule == "R1"
    with pytest.raises(sb.RuleError) as e:
        s.at("encoder.layer.0.ffn").fuse("nope")
    assert e.value.rule == "R3"
    odd = sb.tp_two_linear(8, 6, 4)
    s3 = sb.create_schedule(odd, 4)
    with pytest.raises(sb.RuleError) as e:
        s3.at("a").shard(["weight"], 0)
    assert e.value.rule == "R5"
    with pytest.raises(sb.SlapoError):
        s.at("encoder.layer.0.attention.core").replace("FusedQKV")


def test_fuse_warns_when_pattern_matches_nothing():
    # after sync(forward) the 4-node pattern no longer matches
    m = sb.toy_bert(layers=1, hidden=16, heads=4, vocab=16)
    s = sb.create_schedule(m, 2)
    s.load_script(recipes.tp_script(1, 2, fuse=False, flash=False, shard_embeddings=False))
    s.at("encoder.layer.0.attention.output").trace(flatten=True)
    s.define_pattern("bdrln", recipes.pattern_res_ln(False, True))
    s.set_eager = None
    applied = s.apply()  # deferred script records replay cleanly
    assert applied is not None
    s2 = sb.create_schedule(applied, 2)
    s2.at("encoder.layer.0.attention.output").trace(flatten=True)
    s2.define_pattern("bdrln", recipes.pattern_res_ln(False, True))
    s2.define_pattern("ar_bdrln", recipes.pattern_res_ln(True, True))
    n0 = s2.num_warnings()
    s2.at("encoder.layer.0.attention.output").fuse("bdrln")
    assert s2.num_warnings() == n0 + 1
    s2.at("encoder.layer.0.attention.output").fuse("ar_bdrln")
    assert s2.num_warnings() == n0 + 1
