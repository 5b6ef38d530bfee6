"""Command-line surface of the reference's `slapo` tool for the B200 executor
(proj/tools/slapo_main.cpp): `inspect`, `apply`, `run`, `verify` and `estimate` with the
reference's arguments, outputs and exit codes, plus `diff` to compare two SLD1
dumps (e.g. one written by the reference's `slapo run --dump`).

    python -m paper_2302_08005_b200 inspect MODEL.json
    python -m paper_2302_08005_b200 apply   MODEL.json SCRIPT [--world-size N] [--out OUT.json]
    python -m paper_2302_08005_b200 run     MODEL.json [SCRIPT] [--seed S] [--world-size N] [--micro-batches M]
                                            [--mode verify|train] [--dump OUT.sld] [--dtype fp32|bf16]
    python -m paper_2302_08005_b200 verify  MODEL.json SCRIPT [--world-size N] [--seed S]
                                            [--trials T] [--atol A] [--rtol R]
    python -m paper_2302_08005_b200 verify-train MODEL.json [SCRIPT] --reference DIR [--world-size N] [--seed S]
                                            [--mode train|verify] [--dtype fp32|bf16] [--tol-out/--tol-loss/--tol-grad X]
    python -m paper_2302_08005_b200 estimate MODEL.json [SCRIPT] [--world-size N] [--batch B] [--b200]
    python -m paper_2302_08005_b200 diff    A.sld B.sld [--atol A] [--rtol R]

`run` and `verify` execute on the GPU through the C ABI (there is no CPU
path); `inspect`, `apply` and `diff` are host-only.
"""
from __future__ import annotations

import argparse
import json
import sys
from typing import List, Optional

import numpy as np

from . import dump as _dump

# exit codes (slapo_main.cpp:13-17)
EXIT_OK, EXIT_USAGE, EXIT_RULE, EXIT_NUMERIC, EXIT_INTERNAL = 0, 1, 2, 3, 4

_M64 = (1 << 64) - 1


# seed derivation (proj/include/slapo/rng.hpp:16-32): host-side arithmetic of the CLI
def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _hash_combine(a: int, b: int) -> int:
    return _splitmix64(a ^ ((b + 0x9E3779B97F4A7C15 + ((a << 6) & _M64) + (a >> 2)) & _M64))


def derive_seed(seed: int, label: str) -> int:
    h = _splitmix64(seed & _M64)
    for c in label.encode():
        h = _hash_combine(h, c)
    return h


def _read(path: str) -> str:
    with open(path, "rb") as f:
        return f.read().decode()


def _load_model(path: str):
    from . import Model
    return Model.from_json(_read(path))


def _input_dtype(model_json: dict) -> str:
    """dtype of the first declared input of the root forward (f64 unless marked f32)."""
    for node in model_json.get("modules", {}).get("forward", []):
        if node.get("kind") == "input":
            return str(node.get("attrs", {}).get("dtype", "f64"))
    return "f64"


def _apply(model, script_path: Optional[str], world: int):
    from . import RuleError, create_schedule
    sch = create_schedule(model, world)
    if script_path:
        sch.load_script(_read(script_path))
    try:
        return sch.apply()
    except RuleError as e:  # validate_and_apply (slapo_main.cpp:58-67)
        print(str(e), file=sys.stderr)
        sys.exit(EXIT_RULE)


# print_tree (slapo_main.cpp:38-50) over the slapo-model-v1 JSON
def _print_tree(m: dict, name: str, depth: int) -> None:
    line = "  " * depth + name + ": " + str(m.get("kind", ""))
    for p in m.get("params", []):
        line += "  " + p["name"] + _dump.spec_text(p.get("shape", []), p.get("dtype", "f64"))
        sh = p.get("shard")
        if sh:
            line += "[shard axis=%d world=%d]" % (int(sh.get("axis", 0)), int(sh.get("world_size", 1)))
    attrs = m.get("attrs", {})
    if attrs.get("checkpoint") in (True, 1, "true"):
        line += "  [checkpoint]"
    if attrs.get("fused") in (True, 1, "true"):
        line += "  [fused]"
    print(line)
    for sub, sm in m.get("submodules", {}).items():
        _print_tree(sm, sub, depth + 1)


def cmd_inspect(a) -> int:
    d = json.loads(_read(a.model))
    _print_tree(d["modules"], d.get("name", ""), 0)
    return EXIT_OK


def cmd_apply(a) -> int:
    model = _load_model(a.model)
    res = _apply(model, a.script, a.world_size)
    out = a.out or a.model + ".out.json"
    with open(out, "w") as f:
        f.write(res.to_json())
    print("wrote " + out)
    return EXIT_OK


def cmd_estimate(a) -> int:
    """cmd_estimate (slapo_main.cpp:146-166): the cost model of the (scheduled) model."""
    from . import costmodel
    model = _load_model(a.model)
    if a.script and _has_stages(a.script):
        raise NotImplementedError("estimate_pipeline is not built (pipeline stages: DESIGN.md §8)")
    target = _apply(model, a.script, a.world_size) if a.script else model
    c = costmodel.B200_CONSTANTS if a.b200 else costmodel.CostConstants()
    mem = costmodel.B200_MEMORY_BYTES if a.b200 else 16 * 1024 ** 3
    r = costmodel.estimate(target, batch=a.batch, world_size=a.world_size, device_memory_bytes=mem, constants=c)
    print(r.to_text(), end="")
    return EXIT_OK


def cli_inputs(model, seed: int) -> List[np.ndarray]:
    """default_inputs (slapo_main.cpp:69-76): random_tensor(spec_i, derive_seed(seed, "cli-input"), i)."""
    from . import lib, _check  # noqa: F401
    import ctypes as _c
    s = derive_seed(seed, "cli-input")
    res = []
    for i, shape in enumerate(model.input_shapes()):
        n = int(np.prod(shape)) if shape else 1
        arr = np.empty(n, dtype=np.float64)
        nn = _c.c_size_t()
        _check(lib().sb_model_random_input(model._h, i, s, i, arr.ctypes.data_as(_c.POINTER(_c.c_double)), n,
                                           _c.byref(nn)))
        res.append(arr.reshape(shape))
    return res


def _run_outputs(model, inputs, world: int, mode: str, seed: int, dtype: str) -> List[np.ndarray]:
    from . import Executor
    ex = Executor(model, mode=mode, seed=seed, world=world, dtype=dtype)
    return ex.forward(inputs)


def _has_stages(script_path: Optional[str]) -> bool:
    return bool(script_path) and any(ln.split()[:1] == ["pipeline_split"] for ln in _read(script_path).splitlines())


def cmd_run(a) -> int:
    from . import create_schedule, run_pipeline
    model = _load_model(a.model)
    dt = _input_dtype(json.loads(_read(a.model)))
    inputs = cli_inputs(model, a.seed)
    if _has_stages(a.script):  # cmd_run's run_pipeline branch (slapo_main.cpp:180-182)
        sch = create_schedule(model, a.world_size)
        sch.load_script(_read(a.script))
        outs = run_pipeline(sch.apply_pipeline(), inputs, max(a.micro_batches, 1), a.mode, derive_seed(a.seed, "run"),
                            a.dtype)
    else:
        target = _apply(model, a.script, a.world_size) if a.script else model
        outs = _run_outputs(target, inputs, a.world_size if a.script else 1, a.mode, derive_seed(a.seed, "run"),
                            a.dtype)
    for o in outs:
        print(_dump.format_tensor_text(o, dt))
    if a.dump:
        _dump.write_tensor_dump(a.dump, [(o, dt) for o in outs])
        print("dumped %d tensors to %s" % (len(outs), a.dump))
    return EXIT_OK


def _diff(ref: List[np.ndarray], got: List[np.ndarray]):
    """DiffAccum (proj/src/verifier.cpp:61-80)."""
    if len(ref) != len(got):
        raise ValueError("output arity differs between the two modules")
    max_abs = max_rel = 0.0
    for i, (x, y) in enumerate(zip(ref, got)):
        x = np.asarray(x, dtype=np.float64).reshape(-1)
        y = np.asarray(y, dtype=np.float64).reshape(-1)
        if x.size != y.size:
            raise ValueError(f"output {i} sizes differ")
        d = np.abs(x - y)
        if d.size:
            max_abs = max(max_abs, float(d.max()))
            den = np.maximum(np.abs(x), np.abs(y))
            nz = den > 0
            if nz.any():
                max_rel = max(max_rel, float((d[nz] / den[nz]).max()))
    return max_abs, max_rel


def _report(trials: int, max_abs: float, max_rel: float, atol: float, rtol: float, ok: bool, vacuous: bool) -> str:
    """EquivalenceReport::to_text (proj/src/verifier.cpp:14-24)."""
    g = lambda v: "%g" % v  # noqa: E731 - ostream default formatting
    return ("trials        %d\nmax_abs_diff  %s\nmax_rel_diff  %s\natol          %s\nrtol          %s\n"
            "pass          %s%s\nnote          sampled, not proven\n" %
            (trials, g(max_abs), g(max_rel), g(atol), g(rtol), "true" if ok else "false",
             " (vacuous)" if vacuous else ""))


def cmd_verify(a) -> int:
    """verify_end_to_end (proj/src/verifier.cpp:169-205): per trial, inputs
    random_tensor(spec_i, hash_combine(seed', trial), i) with seed' =
    derive_seed(seed, "verify"); the unscheduled and the scheduled model run in
    verify mode (no dropout) on the GPU and the max abs / rel differences are
    compared with atol / rtol."""
    from . import Executor
    import ctypes as _c
    from . import lib, _check
    model = _load_model(a.model)
    res = _apply(model, a.script, a.world_size)
    vseed = derive_seed(a.seed, "verify")
    if a.trials == 0:
        print(_report(0, 0.0, 0.0, a.atol, a.rtol, True, True), end="")
        return EXIT_OK
    ref_ex = Executor(model, mode="verify", seed=vseed, world=1, dtype=a.dtype)
    got_ex = Executor(res, mode="verify", seed=vseed, world=a.world_size, dtype=a.dtype)
    max_abs = max_rel = 0.0
    for t in range(a.trials):
        s = _hash_combine(vseed, t)
        inputs = []
        for i, shape in enumerate(model.input_shapes()):
            n = int(np.prod(shape)) if shape else 1
            arr = np.empty(n, dtype=np.float64)
            nn = _c.c_size_t()
            _check(lib().sb_model_random_input(model._h, i, s, i, arr.ctypes.data_as(_c.POINTER(_c.c_double)), n,
                                               _c.byref(nn)))
            inputs.append(arr.reshape(shape))
        ma, mr = _diff(ref_ex.forward(inputs), got_ex.forward(inputs))
        max_abs, max_rel = max(max_abs, ma), max(max_rel, mr)
    ok = max_abs <= a.atol and max_rel <= a.rtol
    print(_report(a.trials, max_abs, max_rel, a.atol, a.rtol, ok, False), end="")
    return EXIT_OK if ok else EXIT_NUMERIC


def grad_error(name: str, got: np.ndarray, want: np.ndarray, grads: dict) -> float:
    """Per-tensor normalised max error ||a-b||_inf / ||b||_inf (SURVEY.md Appendix A.5:
    the verifier's elementwise max_rel breaks on gradients). An analytically-zero
    gradient (the key-bias of a softmax attention: shift invariance) is normalised by
    its layer's query-bias gradient instead of by its own round-off-sized norm."""
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    if got.shape != want.shape:
        raise ValueError(f"gradient {name}: {got.size} vs {want.size} elements")
    scale = float(np.abs(want).max(initial=0.0))
    if name.endswith("key.bias"):
        q = grads.get(name[: -len("key.bias")] + "query.bias")
        if q is not None:
            scale = float(np.abs(np.asarray(q)).max(initial=0.0))
    return float(np.abs(got - want).max(initial=0.0)) / max(scale, 1e-30)


def cmd_verify_train(a) -> int:
    """The random-input verifier extended to one training step (
    verify_end_to_end, proj/src/verifier.cpp:169-205, compares forward outputs only):
    the scheduled model runs forward + backward_all_ranks on the GPU with `slapo run`'s
    inputs and seeds (slapo_main.cpp:69-82: inputs random_tensor(spec_i,
    derive_seed(seed, "cli-input"), i), executor seed derive_seed(seed, "run")), and
    every rank's outputs, loss (sum of outputs, executor.cpp:355-362) and parameter
    gradients are checked against the reference executor's dump of the same step
    (--reference DIR: outputs.r<R>.sld1, grads.r<R>.sld1 + grads.r<R>.names, SLD1
    tensor dumps written by the reference's write_tensor_dump, dump.cpp:29).
    Metrics: per-tensor ||a-b||_inf/||b||_inf for outputs and gradients (Appendix A.5),
    |loss - loss_ref| / |loss_ref| for the loss."""
    import os
    from . import Executor
    model = _load_model(a.model)
    target = _apply(model, a.script, a.world_size) if a.script else model
    world = a.world_size if a.script else 1
    inputs = cli_inputs(model, a.seed)
    ex = Executor(target, mode=a.mode, seed=derive_seed(a.seed, "run"), world=world, dtype=a.dtype)
    ex.forward(inputs)
    gm = ex.backward_all_ranks()
    worst_out = worst_loss = worst_grad = 0.0
    worst_name = ""
    n_grads = 0
    for r in range(world):
        want = [t for t, _ in _dump.read_tensor_dump(os.path.join(a.reference, "outputs.r%d.sld1" % r))]
        got = ex.outputs_of_rank(r)
        if len(want) != len(got):
            raise ValueError("rank %d: %d outputs vs %d in the reference dump" % (r, len(got), len(want)))
        for g, w in zip(got, want):
            worst_out = max(worst_out, grad_error("", g, w, {}))
        lg = sum(float(np.asarray(o, dtype=np.float64).sum()) for o in got)
        lw = sum(float(np.asarray(w, dtype=np.float64).sum()) for w in want)
        worst_loss = max(worst_loss, abs(lg - lw) / max(abs(lw), 1e-30))
        names = _read(os.path.join(a.reference, "grads.r%d.names" % r)).split()
        gw = [t for t, _ in _dump.read_tensor_dump(os.path.join(a.reference, "grads.r%d.sld1" % r))]
        if len(names) != len(gw):
            raise ValueError("rank %d: %d gradient names for %d tensors" % (r, len(names), len(gw)))
        want_g = dict(zip(names, gw))
        got_g = gm[r].params
        if set(want_g) != set(got_g):
            raise ValueError("rank %d: gradient sets differ: %s" % (r, sorted(set(want_g) ^ set(got_g))))
        for k, w in want_g.items():
            e = grad_error(k, got_g[k], w, want_g)
            n_grads += 1
            if e > worst_grad:
                worst_grad, worst_name = e, "r%d:%s" % (r, k)
    ok = worst_out <= a.tol_out and worst_loss <= a.tol_loss and worst_grad <= a.tol_grad
    g = lambda v: "%g" % v  # noqa: E731 - ostream default formatting
    print("ranks         %d\noutputs_err   %s\nloss_rel_err  %s\ngradients     %d\nworst_grad    %s %s\n"
          "tol_out       %s\ntol_loss      %s\ntol_grad      %s\npass          %s\n" %
          (world, g(worst_out), g(worst_loss), n_grads, g(worst_grad), worst_name or "-", g(a.tol_out),
           g(a.tol_loss), g(a.tol_grad), "true" if ok else "false"), end="")
    return EXIT_OK if ok else EXIT_NUMERIC


def cmd_diff(a) -> int:
    ra = [t for t, _ in _dump.read_tensor_dump(a.a)]
    rb = [t for t, _ in _dump.read_tensor_dump(a.b)]
    ma, mr = _diff(ra, rb)
    ok = ma <= a.atol and mr <= a.rtol
    print(_report(1, ma, mr, a.atol, a.rtol, ok, False), end="")
    return EXIT_OK if ok else EXIT_NUMERIC


def main(argv: Optional[List[str]] = None) -> int:
    p = argparse.ArgumentParser(prog="python -m paper_2302_08005_b200",
                                description="slapo CLI surface on the B200 executor")
    sp = p.add_subparsers(dest="cmd", required=True)
    q = sp.add_parser("inspect")
    q.add_argument("model")
    q = sp.add_parser("apply")
    q.add_argument("model")
    q.add_argument("script")
    q.add_argument("--world-size", type=int, default=1)
    q.add_argument("--out", default="")
    q = sp.add_parser("run")
    q.add_argument("model")
    q.add_argument("script", nargs="?", default="")
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--world-size", type=int, default=1)
    q.add_argument("--mode", choices=["verify", "train"], default="verify")
    q.add_argument("--dump", default="")
    q.add_argument("--micro-batches", type=int, default=1)
    q.add_argument("--dtype", choices=["fp32", "bf16"], default="fp32")
    q = sp.add_parser("verify")
    q.add_argument("model")
    q.add_argument("script")
    q.add_argument("--world-size", type=int, default=1)
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--trials", type=int, default=10)
    q.add_argument("--atol", type=float, default=1e-4)
    q.add_argument("--rtol", type=float, default=1e-3)
    q.add_argument("--dtype", choices=["fp32", "bf16"], default="fp32")
    q = sp.add_parser("verify-train")
    q.add_argument("model")
    q.add_argument("script", nargs="?", default="")
    q.add_argument("--reference", required=True, help="directory with the reference's per-rank SLD1 dumps")
    q.add_argument("--world-size", type=int, default=1)
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--mode", choices=["verify", "train"], default="train")
    q.add_argument("--dtype", choices=["fp32", "bf16"], default="fp32")
    # defaults: the north star's fp32 bar; bf16 runs pass the stated bf16 tolerances
    q.add_argument("--tol-out", type=float, default=1e-4)
    q.add_argument("--tol-loss", type=float, default=1e-4)
    q.add_argument("--tol-grad", type=float, default=1e-4)
    q = sp.add_parser("estimate")
    q.add_argument("model")
    q.add_argument("script", nargs="?", default="")
    q.add_argument("--world-size", type=int, default=1)
    q.add_argument("--batch", type=int, default=0)
    q.add_argument("--b200", action="store_true", help="B200-calibrated constants and 180 GB instead of the defaults")
    q = sp.add_parser("diff")
    q.add_argument("a")
    q.add_argument("b")
    q.add_argument("--atol", type=float, default=1e-4)
    q.add_argument("--rtol", type=float, default=1e-3)
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    try:
        return {"inspect": cmd_inspect, "apply": cmd_apply, "run": cmd_run, "verify": cmd_verify,
                "verify-train": cmd_verify_train, "estimate": cmd_estimate, "diff": cmd_diff}[a.cmd](a)
    except SystemExit:
        raise
    except Exception as e:  # noqa: BLE001 - the CLI's internal-error exit
        print("error: %s" % e, file=sys.stderr)
        return EXIT_INTERNAL
