"""Pipeline stages: the stage plan materialised from
pipeline_split annotations against the reference's partitioner
(proj/src/pipeline.cpp build_pipeline_plan) — byte-identical stage modules and
stage I/O — and the GPipe forward (run_pipeline, executor.cpp:1531-1579) of the
stages on the GPU against the reference's run_pipeline."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import dump, recipes
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle driver not built (make -C oracle)")

SCRIPTS = {
    "after1": "trace encoder.layer\npipeline_split encoder.layer after=1\n",
    "after0_2": "trace encoder.layer\npipeline_split encoder.layer after=0\npipeline_split encoder.layer after=2\n",
    "tp_after1": None,  # TP=2 recipe + a split (combos_test.cpp:70-86)
}


def _script(name, layers=4, world=2):
    if name == "tp_after1":
        return recipes.tp_script(layers, world) + "trace encoder.layer\npipeline_split encoder.layer after=1\n"
    return SCRIPTS[name]


def _ref_stages(tmp, name, layers=4, world=2):
    sch = os.path.join(tmp, "pp.sch")
    with open(sch, "w") as f:
        f.write(_script(name, layers, world))
    ref.run("toy_bert", schedule=sch, outdir=tmp, layers=layers, world=world, mode="verify", backward=0, dtype="f32",
            hidden=8, heads=2, vocab=28)
    lines = open(os.path.join(tmp, "stages.txt")).read().splitlines()
    ins = lines[0].split()[1:]
    outs = lines[1].split()[1:]
    stages = []
    for ln in lines[2:]:
        t = ln.split()
        c, p = t.index("consumes"), t.index("produces")
        stages.append((t[c + 1:p], t[p + 1:]))
    return sch, ins, outs, stages


@needs_ref
@pytest.mark.parametrize("name", list(SCRIPTS))
def test_stage_plan_identical_to_reference(tmp_path, name):
    tmp = str(tmp_path)
    sch, ins, outs, stages = _ref_stages(tmp, name)
    m = sb.Model.from_json(open(os.path.join(tmp, "original.json")).read())
    s = sb.create_schedule(m, 2)
    s.load_script(open(sch).read())
    plan = s.apply_pipeline()
    assert plan.model_inputs == ins and plan.model_outputs == outs
    assert len(plan.stages) == len(stages)
    for i, (st, (c, p)) in enumerate(zip(plan.stages, stages)):
        assert st.consumes == c and st.produces == p
        assert st.module.to_json() == open(os.path.join(tmp, f"stage{i}.json")).read()


def test_stage_plan_errors():
    m = sb.toy_bert(layers=2)
    s = sb.create_schedule(m, 2)
    with pytest.raises(sb.SlapoError):
        s.apply_pipeline()  # no pipeline_split annotations


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("name,micro,mode", [("after1", 1, "verify"), ("after0_2", 2, "verify"),
                                             ("after1", 2, "train"), ("tp_after1", 1, "verify")])
def test_run_pipeline_matches_reference(tmp_path, name, micro, mode):
    """`run` of a split model: every stage on the GPU, GPipe micro-batches,
    against the reference's run_pipeline on the same inputs and seed."""
    tmp = str(tmp_path)
    sch, *_ = _ref_stages(tmp, name)
    model_json = os.path.join(tmp, "original.json")
    ref_out = os.path.join(tmp, "ref.sld")
    r = subprocess.run([ref.DRIVER, "--model_json", model_json, "--schedule", sch, "--world", "2", "--seed", "31",
                        "--mode", mode, "--micro", str(micro), "--cli_run", ref_out], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    mine = os.path.join(tmp, "mine.sld")
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "paper_2302_08005_b200", "run", model_json, sch, "--seed", "31",
                        "--world-size", "2", "--mode", mode, "--micro-batches", str(micro), "--dump", mine],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr
    a, b = dump.read_tensor_dump(mine), dump.read_tensor_dump(ref_out)
    assert len(a) == len(b)
    for (x, dx), (y, dy) in zip(a, b):
        assert dx == dy and x.shape == y.shape
        assert np.abs(x - y).max() / np.abs(y).max() < 1e-4


@pytest.mark.gpu
def test_run_pipeline_composes_to_the_model():
    """Stage-wise execution reproduces the unsplit model (pipeline_test.cpp:78-110's
    composition property) on the GPU, with 1 and 4 micro-batches."""
    m = sb.toy_bert(layers=4, batch=4).to_f32()
    x = m.random_inputs(3)
    whole = sb.Executor(m, mode="verify", seed=5).forward(x)
    s = sb.create_schedule(m, 2)
    s.load_script(SCRIPTS["after0_2"])
    plan = s.apply_pipeline()
    assert len(plan.stages) == 3
    for micro in (1, 4):
        got = sb.run_pipeline(plan, x, micro, "verify", 5)
        for g, w in zip(got, whole):
            assert g.shape == w.shape
            assert np.abs(g - w).max() <= 1e-5 * max(1.0, np.abs(w).max())
