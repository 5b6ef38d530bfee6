"""Cost model and tuner.

* ``estimate`` — the reference's analytical step-time / memory model
  (proj/include/slapo/costmodel.hpp, proj/src/costmodel.cpp) computed by the
  host library (``host/step_model.cpp``) over a scheduled model, through the
  C ABI (``sb_estimate``).
* ``B200_CONSTANTS`` — its constants calibrated on this pool's B200s (the
  measured in-step GEMM rate, launch cost and NVLink 5 bandwidth).
* ``exhaustive`` / ``coordinate_descent`` — the reference's tuner
  (proj/include/slapo/tuner.hpp, proj/src/tuner.cpp) over plain candidate
  lists: a variable is (name, candidates[, when]) where ``candidates`` may be a
  callable of the prefix assignment and ``when`` a predicate of the prefix plus
  the variable's value (the polygon spaces of the reference's Expr language);
  constraints are predicates of the full assignment. Same enumeration order,
  seeded RNG, memoisation and tie-breaks.
* ``measured_objective`` — the paper's tuning loop on the device: build the
  scheduled model at (batch, checkpoint ratio), time steps on the GPU.
"""
from __future__ import annotations

import ctypes as _c
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import Model, _check, _lib

_M64 = (1 << 64) - 1


@dataclass
class CostConstants:
    device_flops_per_s: float = 1e12
    link_bytes_per_s: float = 1e10
    kernel_launch_overhead_s: float = 1e-6
    optimizer_state_multiplier: float = 2.0


# Calibrated on one B200 of this pool (round 1, bench.py at C3, power-capped SM clock
# 1.64-1.80 GHz): in-step achieved rate of the tcgen05 GEMMs that carry 98% of the
# model's flops (970 TF/s), the per-kernel cost of a CUDA-graph replayed step beyond
# its math (1.3 us, 802 kernels), NVLink 5 peer bandwidth (775 GB/s measured on the
# B300 sibling, B300_MICROARCH.md; one GPU here), Adam moments, 180 GB HBM3e.
B200_CONSTANTS = CostConstants(device_flops_per_s=0.97e15, link_bytes_per_s=775e9, kernel_launch_overhead_s=1.3e-6,
                               optimizer_state_multiplier=2.0)
B200_MEMORY_BYTES = 180 * 10 ** 9


@dataclass
class CostReport:
    step_time_s: float
    flops: int
    recompute_flops: int
    launches: int
    collective_bytes: int
    param_bytes: int
    activation_bytes: int
    peak_memory_bytes: int
    oom: bool
    throughput_samples_per_s: float
    text: str = field(repr=False, default="")

    def to_text(self) -> str:
        return self.text


def estimate(model: Model, batch: int = 0, world_size: int = 1, device_memory_bytes: int = 16 * 1024 ** 3,
             constants: Optional[CostConstants] = None) -> CostReport:
    c = constants or CostConstants()
    cv = (_c.c_double * 4)(c.device_flops_per_s, c.link_bytes_per_s, c.kernel_launch_overhead_s,
                           c.optimizer_state_multiplier)
    ints = (_c.c_int64 * 8)()
    reals = (_c.c_double * 2)()
    need = _c.c_size_t()
    _check(_lib.sb_estimate(model._h, batch, world_size, device_memory_bytes, cv, ints, reals, None, 0,
                            _c.byref(need)))
    buf = _c.create_string_buffer(need.value)
    _check(_lib.sb_estimate(model._h, batch, world_size, device_memory_bytes, cv, ints, reals, buf, need.value,
                            _c.byref(need)))
    return CostReport(reals[0], ints[0], ints[1], ints[2], ints[3], ints[4], ints[5], ints[6], bool(ints[7]),
                      reals[1], buf.value.decode())


# ----------------------------------------------------------------------- tuner
@dataclass
class Var:
    name: str
    candidates: object  # list of values, or callable(prefix: dict) -> list
    when: Optional[Callable[[dict], bool]] = None


@dataclass
class Space:
    vars: List[Var]
    constraints: List[Callable[[dict], bool]] = field(default_factory=list)


@dataclass
class Trial:
    assignment: Dict[str, float]
    objective: float
    report: object = None


@dataclass
class TunerResult:
    best: Trial
    trials: List[Trial]
    all_zero: bool


def _key(a: dict) -> Tuple:
    return tuple(sorted(a.items()))  # std::map<std::string, double> ordering


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


class _Rng:  # tuner.cpp:30-39
    def __init__(self, seed: int):
        self.state = _splitmix64((seed ^ 0x7454756E65) & _M64)

    def below(self, n: int) -> int:
        self.state = _splitmix64(self.state)
        return self.state % n


def _validate(space: Space) -> None:  # tuner.cpp:13-20
    if not space.vars:
        raise ValueError("search space has no variables")
    seen = set()
    for v in space.vars:
        if not callable(v.candidates) and not v.candidates:
            raise ValueError(f"variable '{v.name}' has no candidates")
        if v.name in seen:
            raise ValueError(f"duplicate variable '{v.name}'")
        seen.add(v.name)


def var_candidates(space: Space, i: int, prefix: dict) -> List[float]:  # tuner.cpp:43-57
    v = space.vars[i]
    raw = v.candidates(prefix) if callable(v.candidates) else v.candidates
    out: List[float] = []
    for val in raw:
        val = float(val)
        if v.when is not None and not v.when({**prefix, v.name: val}):
            continue
        if val in out:
            raise ValueError(f"variable '{v.name}' has duplicate candidate {val}")
        out.append(val)
    return out


def is_feasible(space: Space, a: dict) -> bool:  # tuner.cpp:59-70
    prefix: dict = {}
    for i, v in enumerate(space.vars):
        if v.name not in a or a[v.name] not in var_candidates(space, i, prefix):
            return False
        prefix[v.name] = a[v.name]
    return all(c(a) for c in space.constraints)


def enumerate_space(space: Space) -> List[dict]:  # tuner.cpp:74-96
    _validate(space)
    out: List[dict] = []

    def rec(i: int, prefix: dict) -> None:
        if i == len(space.vars):
            if all(c(prefix) for c in space.constraints):
                out.append(dict(prefix))
            return
        for val in var_candidates(space, i, prefix):
            prefix[space.vars[i].name] = val
            rec(i + 1, prefix)
            del prefix[space.vars[i].name]

    rec(0, {})
    return out


Objective = Callable[[dict], Tuple[float, object]]


def exhaustive(space: Space, objective: Objective) -> TunerResult:  # tuner.cpp:98-115
    feasible = enumerate_space(space)
    if not feasible:
        raise ValueError("search space has an empty feasible set")
    trials: List[Trial] = []
    best = None
    for a in feasible:
        obj, rep = objective(a)
        trials.append(Trial(a, obj, rep))
        if best is None or obj > best.objective:
            best = trials[-1]
    return TunerResult(best, trials, all(t.objective == 0.0 for t in trials))


def coordinate_descent(space: Space, objective: Objective, seed: int, restarts: int = 3) -> TunerResult:
    """tuner.cpp:117-180: seeded random feasible start, dimensions swept in a seeded
    random order (Fisher-Yates), best candidate per dimension, until a full sweep
    brings no improvement; `restarts` starts; memoised evaluations."""
    feasible = enumerate_space(space)
    if not feasible:
        raise ValueError("search space has an empty feasible set")
    rng = _Rng(seed)
    trials: List[Trial] = []
    memo: Dict[Tuple, Trial] = {}

    def evaluate(a: dict) -> float:
        k = _key(a)
        if k not in memo:
            obj, rep = objective(dict(a))
            memo[k] = Trial(dict(a), obj, rep)
            trials.append(memo[k])
        return memo[k].objective

    best: Optional[Trial] = None
    for _ in range(max(restarts, 1)):
        current = dict(feasible[rng.below(len(feasible))])
        cur_obj = evaluate(current)
        dims = list(range(len(space.vars)))
        for i in range(len(dims), 1, -1):
            j = rng.below(i)
            dims[i - 1], dims[j] = dims[j], dims[i - 1]
        improved = True
        while improved:
            improved = False
            for d in dims:
                name = space.vars[d].name
                prefix = {space.vars[i].name: current[space.vars[i].name] for i in range(d)}
                best_val, best_obj = current[name], cur_obj
                for cand in var_candidates(space, d, prefix):
                    if cand == current[name]:
                        continue
                    probe = dict(current)
                    probe[name] = cand
                    if not is_feasible(space, probe):
                        continue
                    obj = evaluate(probe)
                    if obj > best_obj:
                        best_obj, best_val = obj, cand
                if best_val != current[name]:
                    current[name] = best_val
                    cur_obj = best_obj
                    improved = True
        if best is None or cur_obj > best.objective or (cur_obj == best.objective and _key(current) < _key(best.assignment)):
            best = Trial(dict(current), cur_obj, memo[_key(current)].report)
    return TunerResult(best, trials, all(t.objective == 0.0 for t in trials))


# ------------------------------------------------------------- model-level loops
def estimate_objective(build: Callable[[dict], Model], batch_var: str = "batch", world_size: int = 1,
                       device_memory_bytes: int = B200_MEMORY_BYTES,
                       constants: Optional[CostConstants] = None) -> Objective:
    """cmd_tune's objective (slapo_main.cpp:218-252) with the cost model: the
    scheduled model for an assignment, estimated at its batch; 0 when it OOMs."""
    def f(a: dict):
        m = build(a)
        r = estimate(m, batch=int(a.get(batch_var, 0)), world_size=world_size,
                     device_memory_bytes=device_memory_bytes, constants=constants or B200_CONSTANTS)
        return (0.0 if r.oom else r.throughput_samples_per_s), r
    return f


def measured_objective(build: Callable[[dict], Model], batch_var: str = "batch", steps: int = 3, warmup: int = 2,
                       dtype: str = "bf16", p: float = 0.1) -> Objective:
    """The tuner driving measured step times: samples/s of `steps` CUDA-graph
    replayed training steps of the scheduled model on the current GPU (0 on
    device OOM)."""
    import numpy as np
    from . import Executor, SlapoError

    def f(a: dict):
        m = build(a)
        try:
            ex = Executor(m, mode="train", seed=1, dtype=dtype)
            ex.upload_inputs(m.random_inputs(7))
            for _ in range(warmup):
                ex.step()
            ex.synchronize()
            ms = ex.time_steps(steps)
        except SlapoError as e:
            if "out of memory" in str(e).lower():
                return 0.0, None
            raise
        batch = int(a.get(batch_var, m.input_shapes()[0][0]))
        del ex
        return batch / (ms / steps * 1e-3), {"ms_per_step": ms / steps}
    return f


def fit_device_rate(points: Sequence[Tuple[CostReport, float]], constants: Optional[CostConstants] = None) -> CostConstants:
    """Calibrate `device_flops_per_s` from measured steps: least squares of
    measured_s - launch/comm terms = W / rate over (report, measured seconds)
    points, W = 3 * flops + recompute_flops (finish(), costmodel.cpp:236-240)."""
    c = constants or B200_CONSTANTS
    num = den = 0.0
    for r, t in points:
        w = 3.0 * r.flops + r.recompute_flops
        rest = t - 3.0 * r.launches * c.kernel_launch_overhead_s - r.collective_bytes / c.link_bytes_per_s
        num += w * w
        den += w * rest
    return CostConstants(num / den, c.link_bytes_per_s, c.kernel_launch_overhead_s, c.optimizer_state_multiplier)


def bert_large_builder(layers: int = 24, seq: int = 512, world: int = 1, p: float = 0.1):
    """C3's scheduled model (bench.py) at an assignment {batch, ckpt}."""
    from . import create_schedule, recipes, toy_bert

    def build(a: dict) -> Model:
        m = toy_bert(layers, 1024, 16, 30528, int(a["batch"]), seq, p)
        s = create_schedule(m, world)
        s.load_script(recipes.tp_script(layers, world, ckpt_ratio=float(a["ckpt"])))
        return s.apply()
    return build
