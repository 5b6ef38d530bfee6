"""The `slapo` CLI surface: `apply` output, SLD1 dumps,
`run` and `verify` against the reference's own CLI semantics
(proj/tools/slapo_main.cpp) as reproduced by the oracle driver
(oracle/ref_driver.cpp `--cli_run`, linking the reference's dump.cpp /
executor.cpp)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import dump, recipes
from paper_2302_08005_b200.cli import derive_seed
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle driver not built (make -C oracle)")


def _cli(*args, timeout=600):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    return subprocess.run([sys.executable, "-m", "paper_2302_08005_b200", *map(str, args)], capture_output=True,
                          text=True, timeout=timeout, env=env)


def _ref_model(tmp, world=2, layers=2, dtype="f32", p=0.1):
    """original.json + the reference's post-apply model.json for the TP recipe."""
    sch = os.path.join(tmp, "tp.sch")
    with open(sch, "w") as f:
        f.write(recipes.tp_script(layers, world))
    heads = max(2, world)
    ref.run("toy_bert", schedule=sch, outdir=tmp, layers=layers, dtype=dtype, world=world, p=p, mode="verify",
            backward=0, hidden=4 * heads, heads=heads, vocab=28 if world < 4 else 32)
    return os.path.join(tmp, "original.json"), sch


def _ref_cli_run(tmp, model_json, sch, world, seed, mode, name):
    out = os.path.join(tmp, name)
    args = [ref.DRIVER, "--model_json", model_json, "--world", str(world), "--seed", str(seed), "--mode", mode,
            "--cli_run", out]
    if sch:
        args += ["--schedule", sch]
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return out, r.stdout


def test_derive_seed_matches_reference_rng():
    """derive_seed (rng.hpp:28-32) restated in the CLI equals the host library's."""
    from oracle import slapo_oracle as so
    for seed in (0, 1, 123, 2 ** 63 + 5):
        h = so.splitmix64(seed)
        for c in b"cli-input":
            h = so.hash_combine(h, c)
        assert derive_seed(seed, "cli-input") == h


def test_sld1_write_read(tmp_path):
    a = np.arange(24, dtype=np.float64).reshape(2, 3, 4) / 7
    b = np.array([1.5, -2.25])
    p = str(tmp_path / "x.sld")
    dump.write_tensor_dump(p, [(a, "f64"), (b, "f32")])
    back = dump.read_tensor_dump(p)
    assert back[0][1] == "f64" and np.array_equal(back[0][0], a)
    assert back[1][1] == "f32" and np.array_equal(back[1][0], b.astype(np.float32))
    raw = open(p, "rb").read()
    assert raw[:4] == b"SLD1" and len(raw) == 8 + (4 + 24 + 1 + 24 * 8) + (4 + 8 + 1 + 2 * 4)
    with pytest.raises(ValueError):
        open(str(tmp_path / "bad.sld"), "wb").write(b"SBT1\0\0\0\0")
        dump.read_tensor_dump(str(tmp_path / "bad.sld"))


@needs_ref
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_sld1_bytes_identical_to_reference(tmp_path, dtype):
    """A dump written by the reference's write_tensor_dump (dump.cpp:29-48), read
    and re-written here, is byte-for-byte the same file."""
    tmp = str(tmp_path)
    model_json, sch = _ref_model(tmp, world=2, dtype=dtype)
    out, text = _ref_cli_run(tmp, model_json, sch, 2, 5, "verify", "ref.sld")
    tensors = dump.read_tensor_dump(out)
    assert tensors and all(dt == dtype for _, dt in tensors)
    dump.write_tensor_dump(os.path.join(tmp, "re.sld"), tensors)
    assert open(out, "rb").read() == open(os.path.join(tmp, "re.sld"), "rb").read()
    # the text form printed per output (dump.cpp:72-88)
    lines = [ln for ln in text.splitlines() if ln.startswith("tensor ")]
    assert lines == [dump.format_tensor_text(t, dt) for t, dt in tensors]


@needs_ref
@pytest.mark.parametrize("world", [1, 2, 4])
def test_cli_apply_json_identical_to_reference(tmp_path, world):
    """`apply` writes the post-apply model: byte-for-byte the JSON the reference
    writes for the same model and TP recipe (save_model, model_io.cpp:225)."""
    tmp = str(tmp_path)
    model_json, sch = _ref_model(tmp, world=world)
    mine = os.path.join(tmp, "mine.json")
    r = _cli("apply", model_json, sch, "--world-size", world, "--out", mine)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "wrote " + mine
    assert open(mine).read() == open(os.path.join(tmp, "model.json")).read()


@needs_ref
def test_cli_inspect_and_errors(tmp_path):
    tmp = str(tmp_path)
    model_json, sch = _ref_model(tmp, world=2)
    r = _cli("inspect", os.path.join(tmp, "model.json"))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "toy_bert: composite"
    assert any("FusedQKV" in ln and "[shard axis=0 world=2]" in ln for ln in lines)
    assert any("[fused]" in ln for ln in lines)
    assert _cli("bogus").returncode == 1  # usage (slapo_main.cpp:14)
    # an illegal schedule exits with the rule-violation code (slapo_main.cpp:15, 58-67)
    bad = os.path.join(tmp, "bad.sch")
    with open(bad, "w") as f:
        f.write("shard encoder.layer.0.attention.qkv.query weight axis=0\n")
    r = _cli("apply", model_json, bad, "--world-size", 3)
    assert r.returncode in (2, 4), (r.returncode, r.stderr)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("world,mode", [(1, "verify"), (2, "verify"), (2, "train")])
def test_cli_run_matches_reference_dump(tmp_path, world, mode):
    """`run --dump` on the GPU vs the reference's `slapo run --dump` (same model
    JSON, script, seed, mode): the SLD1 dumps agree to the fp32 tolerance
    (north star: 1e-4 relative, ||a-b||_inf / ||b||_inf)."""
    tmp = str(tmp_path)
    model_json, sch = _ref_model(tmp, world=world)
    ref_out, _ = _ref_cli_run(tmp, model_json, sch if world > 1 else "", world, 17, mode, "ref.sld")
    mine = os.path.join(tmp, "mine.sld")
    args = ["run", model_json] + ([sch] if world > 1 else []) + ["--seed", 17, "--world-size", world, "--mode", mode,
                                                                 "--dump", mine]
    r = _cli(*args)
    assert r.returncode == 0, r.stderr
    a, b = dump.read_tensor_dump(mine), dump.read_tensor_dump(ref_out)
    assert len(a) == len(b)
    for (x, dx), (y, dy) in zip(a, b):
        assert dx == dy and x.shape == y.shape
        assert np.abs(x - y).max() / np.abs(y).max() < 1e-4
    r = _cli("diff", mine, ref_out, "--atol", 1e-4, "--rtol", 1.0)
    assert r.returncode == 0 and "pass          true" in r.stdout, r.stdout


@pytest.mark.gpu
@needs_ref
def test_cli_verify_tp_recipe(tmp_path):
    """`verify`: unscheduled vs TP-2-scheduled toy BERT on the GPU, EquivalenceReport text."""
    tmp = str(tmp_path)
    model_json, sch = _ref_model(tmp, world=2)
    r = _cli("verify", model_json, sch, "--world-size", 2, "--trials", 3, "--atol", 1e-4, "--rtol", 1.0)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    assert lines[0].split() == ["trials", "3"] and lines[5].startswith("pass          true")
    assert float(lines[1].split()[1]) < 1e-4


@needs_ref
def test_cli_estimate_matches_reference(tmp_path):
    """`estimate MODEL SCRIPT --batch B`: CostReport::to_text of the reference's estimate."""
    tmp = str(tmp_path)
    model_json, sch = _ref_model(tmp, world=2)
    r = subprocess.run([ref.DRIVER, "--model_json", model_json, "--schedule", sch, "--world", "2", "--est_batch", "8",
                        "--estimate", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    want = "\n".join(r.stdout.strip().splitlines()[:-1]) + "\n"
    got = _cli("estimate", model_json, sch, "--world-size", 2, "--batch", 8)
    assert got.returncode == 0, got.stderr
    assert got.stdout == want


def _ref_cli_train(tmp, model_json, sch, world, seed, mode, name):
    """The reference executor's training step with `slapo run`'s seeds, dumped per rank
    as SLD1 outputs / gradients (oracle/ref_driver.cpp --cli_train)."""
    out = os.path.join(tmp, name)
    os.makedirs(out, exist_ok=True)
    args = [ref.DRIVER, "--model_json", model_json, "--world", str(world), "--seed", str(seed), "--mode", mode,
            "--cli_train", out]
    if sch:
        args += ["--schedule", sch]
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("world,mode,dtype", [(1, "train", "fp32"), (2, "train", "fp32"), (2, "verify", "fp32"),
                                              (2, "train", "bf16")])
def test_cli_verify_train_against_reference(tmp_path, world, mode, dtype):
    """`verify-train`: one scheduled training step on the GPU — every rank's outputs,
    loss and parameter gradients — against the reference executor's dump of the same
    step. fp32 at the north star's 1e-4; bf16 at the stated bf16 tolerances."""
    tmp = str(tmp_path)
    model_json, sch = _ref_model(tmp, world=world, dtype="f32")
    refdir = _ref_cli_train(tmp, model_json, sch, world, 23, mode, "ref_train")
    tol = ["--tol-out", 2e-2, "--tol-loss", 2e-3, "--tol-grad", 5e-2] if dtype == "bf16" else []
    r = _cli("verify-train", model_json, sch, "--reference", refdir, "--world-size", world, "--seed", 23, "--mode",
             mode, "--dtype", dtype, *tol)
    assert r.returncode == 0, r.stdout + r.stderr
    rep = dict(ln.split(None, 1) for ln in r.stdout.splitlines())
    assert rep["pass"].strip() == "true" and int(rep["ranks"]) == world and int(rep["gradients"]) > 10
    # a corrupted reference gradient is caught (exit code 3, the numeric-failure code)
    names = open(os.path.join(refdir, "grads.r0.names")).read().split()
    gs = dump.read_tensor_dump(os.path.join(refdir, "grads.r0.sld1"))
    k = names.index(next(n for n in names if n.endswith("dense.weight")))
    bad = [(t.copy(), d) for t, d in gs]
    bad[k][0].reshape(-1)[0] += 10 * np.abs(bad[k][0]).max()
    dump.write_tensor_dump(os.path.join(refdir, "grads.r0.sld1"), bad)
    r = _cli("verify-train", model_json, sch, "--reference", refdir, "--world-size", world, "--seed", 23, "--mode",
             mode, "--dtype", dtype, *tol)
    assert r.returncode == 3 and "pass          false" in r.stdout, r.stdout + r.stderr
    assert names[k] in r.stdout
