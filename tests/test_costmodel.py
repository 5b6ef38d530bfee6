"""Cost model and tuner against the reference's own
implementation (proj/src/costmodel.cpp, proj/src/tuner.cpp) run by the oracle
driver (`--estimate`, `--tune`), on the same post-apply models."""
import json
import os
import subprocess

import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import costmodel as cm
from paper_2302_08005_b200 import recipes
from oracle import ref

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle driver not built (make -C oracle)")

CASES = [  # (layers, hidden, heads, schedule, world, batch, constants, memory)
    (2, 8, 2, None, 1, 0, None, 16 * 1024 ** 3),
    (2, 8, 2, None, 1, 16, (1e15, 7.75e11, 1.3e-6, 2.0), 16 * 1024 ** 3),
    (3, 16, 4, "tp", 2, 0, None, 16 * 1024 ** 3),
    (3, 16, 4, "tp", 4, 12, (0.97e15, 7.75e11, 1.3e-6, 2.0), 16 * 1024 ** 3),
    (2, 8, 2, "ckpt", 1, 8, None, 16 * 1024 ** 3),
    (2, 8, 2, "c2", 1, 0, None, 16 * 1024 ** 3),
    (2, 8, 2, None, 1, 64, None, 200000),  # oom
]


def _schedule_text(kind, layers, world):
    if kind == "tp":
        return recipes.tp_script(layers, world)
    if kind == "ckpt":
        return "checkpoint encoder.layer.0\n"
    if kind == "c2":
        return open(sb.schedule_path("c2_fuse_flash.sch")).read()
    return ""


def _mine(layers, hidden, heads, kind, world):
    m = sb.toy_bert(layers=layers, hidden=hidden, heads=heads, vocab=32)
    text = _schedule_text(kind, layers, world)
    if not text:
        return m
    s = sb.create_schedule(m, world)
    s.load_script(text)
    return s.apply()


def _ref_estimate(tmp, layers, hidden, heads, kind, world, batch, consts, mem, extra=()):
    args = [ref.DRIVER, "--model", "toy_bert", "--layers", str(layers), "--hidden", str(hidden), "--heads", str(heads),
            "--vocab", "32", "--world", str(world), "--est_batch", str(batch), "--est_mem", str(mem), *extra]
    text = _schedule_text(kind, layers, world)
    if text:
        p = os.path.join(tmp, "s.sch")
        with open(p, "w") as f:
            f.write(text)
        args += ["--schedule", p]
    if consts:
        args += ["--est_consts", ",".join(repr(c) for c in consts)]
    r = subprocess.run(args + ["--estimate", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    return "\n".join(lines[:-1]) + "\n", json.loads(lines[-1])


@needs_ref
@pytest.mark.parametrize("case", CASES, ids=[f"{c[3]}-w{c[4]}-b{c[5]}" for c in CASES])
def test_estimate_matches_reference(tmp_path, case):
    layers, hidden, heads, kind, world, batch, consts, mem = case
    text, want = _ref_estimate(str(tmp_path), *case)
    c = cm.CostConstants(*consts) if consts else None
    got = cm.estimate(_mine(layers, hidden, heads, kind, world), batch=batch, world_size=world,
                      device_memory_bytes=mem, constants=c)
    for k in ("flops", "recompute_flops", "launches", "collective_bytes", "param_bytes", "activation_bytes",
              "peak_memory_bytes"):
        assert getattr(got, k) == want[k], k
    assert got.oom == bool(want["oom"])
    assert got.step_time_s == want["step_time_s"]
    assert got.throughput_samples_per_s == want["throughput_samples_per_s"]
    assert got.to_text() == text  # CostReport::to_text


@needs_ref
@pytest.mark.parametrize("ratio", [0.0, 0.34, 0.5, 1.0])
def test_checkpoint_ratio_matches_reference(tmp_path, ratio):
    m = sb.toy_bert(layers=3, hidden=8, heads=2, vocab=32)
    assert m.apply_checkpoint_ratio("encoder.layer", ratio) == int(ratio * 3)
    _, want = _ref_estimate(str(tmp_path), 3, 8, 2, None, 1, 0, None, 16 * 1024 ** 3,
                            extra=("--ckpt_container", "encoder.layer", "--ckpt_ratio", repr(ratio)))
    got = cm.estimate(m)
    assert (got.recompute_flops, got.activation_bytes) == (want["recompute_flops"], want["activation_bytes"])
    with pytest.raises(sb.SlapoError):
        m.apply_checkpoint_ratio("encoder.nope", 0.5)


def _space(b0):
    return cm.Space([cm.Var("batch", [b0 * f // 4 for f in (1, 2, 4, 8, 16)]),
                     cm.Var("ckpt", [0.0, 0.25, 0.5, 0.75, 1.0])])


def _objective(layers, mem):
    base = sb.toy_bert(layers=layers, hidden=8, heads=2, vocab=32).to_json()

    def build(a):
        m = sb.Model.from_json(base)
        m.apply_checkpoint_ratio("encoder.layer", a["ckpt"])
        return m
    return cm.estimate_objective(build, device_memory_bytes=mem, constants=cm.CostConstants())


@needs_ref
@pytest.mark.parametrize("algo,seed,restarts", [("exhaustive", 0, 1), ("cd", 3, 3), ("cd", 11, 1), ("cd", 99, 5)])
def test_tuner_matches_reference(algo, seed, restarts):
    """Same trial sequence, objectives and best as the reference's tuner with the
    cost-model objective of `slapo tune` (batch x checkpoint-ratio polygon)."""
    layers, b0, mem = 4, 8, 400000
    r = subprocess.run([ref.DRIVER, "--model", "toy_bert", "--layers", str(layers), "--vocab", "32",
                        "--tune", algo, "--ckpt_container", "encoder.layer", "--est_batch", str(b0),
                        "--tune_seed", str(seed), "--tune_restarts", str(restarts), "--est_mem", str(mem)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    want = [ln.split() for ln in r.stdout.splitlines()]
    obj = _objective(layers, mem)
    res = (cm.exhaustive(_space(b0), obj) if algo == "exhaustive"
           else cm.coordinate_descent(_space(b0), obj, seed, restarts))
    got = [["trial", repr(t.assignment["batch"]), repr(t.assignment["ckpt"]), t.objective] for t in res.trials]
    wt = [w for w in want if w[0] == "trial"]
    assert len(got) == len(wt)
    for g, w in zip(got, wt):
        assert float(g[1]) == float(w[1]) and float(g[2]) == float(w[2]) and g[3] == float(w[3])
    best = [w for w in want if w[0] == "best"][0]
    assert (res.best.assignment["batch"], res.best.assignment["ckpt"], res.best.objective) == \
        (float(best[1]), float(best[2]), float(best[3]))
    assert res.all_zero == (best[5] == "1")


def test_tuner_semantics():
    """tuner.hpp:52-71 on small spaces: lexicographic enumeration, first-wins ties,
    polygon candidates, constraints, empty feasible sets."""
    sp = cm.Space([cm.Var("a", [1, 2, 3]), cm.Var("b", lambda pre: [pre["a"], 2 * pre["a"]], when=lambda x: x["b"] < 6)],
                  constraints=[lambda x: x["a"] + x["b"] != 4])
    feas = cm.enumerate_space(sp)
    assert feas == [{"a": 1.0, "b": 1.0}, {"a": 1.0, "b": 2.0}, {"a": 2.0, "b": 4.0}, {"a": 3.0, "b": 3.0}]
    res = cm.exhaustive(sp, lambda x: (1.0, None))
    assert res.best.assignment == {"a": 1.0, "b": 1.0} and len(res.trials) == 4 and not res.all_zero
    assert cm.is_feasible(sp, {"a": 2.0, "b": 4.0}) and not cm.is_feasible(sp, {"a": 2.0, "b": 2.0})
    cd = cm.coordinate_descent(sp, lambda x: (x["a"] * 10 + x["b"], None), seed=5, restarts=2)
    assert cd.best.objective == max(t.objective for t in cd.trials)  # each restart ends at its path's max
    assert len({tuple(sorted(t.assignment.items())) for t in cd.trials}) == len(cd.trials)  # memoised
    assert cm.exhaustive(sp, lambda x: (0.0, None)).all_zero
    with pytest.raises(ValueError):
        cm.exhaustive(cm.Space([cm.Var("a", [1])], constraints=[lambda x: False]), lambda x: (1.0, None))
    with pytest.raises(ValueError):
        cm.enumerate_space(cm.Space([cm.Var("a", [1]), cm.Var("a", [2])]))


@pytest.mark.gpu
def test_measured_tuning_loop():
    """The tuner driving measured step times on the GPU (toy BERT, batch x ratio):
    every trial runs, the measured best is feasible and the calibrated cost
    model's ranking is reported beside it."""
    base = sb.toy_bert(layers=4, hidden=64, heads=4, vocab=64, batch=4, seq=32).to_json()

    def build(a):
        m = sb.Model.from_json(base)
        m.apply_checkpoint_ratio("encoder.layer", a["ckpt"])
        return m
    sp = cm.Space([cm.Var("ckpt", [0.0, 0.5, 1.0])])
    res = cm.exhaustive(sp, cm.measured_objective(build, batch_var="none", steps=3, warmup=2, dtype="fp32"))
    assert len(res.trials) == 3 and all(t.objective > 0 for t in res.trials)
    est = cm.exhaustive(sp, cm.estimate_objective(build, batch_var="none"))
    assert est.best.assignment["ckpt"] == 0.0  # the model charges recompute, never rewards it without OOM
