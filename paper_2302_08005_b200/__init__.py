"""B200-native executor for Slapo's scheduled forward+backward step.

Python mirror of the reference's C++ interface, bound to the C ABI of
``libslapo_b200.so`` (include/slapo_b200.h):

* models: ``toy_bert``, ``gpt_neo`` (f2), ``tp_two_linear``, ``fig3c_exact``, ``ffn_stack``
  (proj/tests/support/fixtures.hpp:21-38), ``Model.from_json`` (model_io.hpp:16);
* ``create_schedule`` / ``Schedule`` with ``at``, ``trace``, ``replace``, ``shard``,
  ``sync``, ``checkpoint``, ``define_pattern``, ``fuse``, ``pipeline_split``,
  ``find``, ``load_script``, ``apply`` (proj/include/slapo/schedule.hpp:65-111);
* ``Executor(model, mode, seed, world)`` with ``forward``, ``outputs_of_rank``,
  ``backward``, ``backward_all_ranks``, ``ledger``, ``collective_invocations``,
  ``set_nan_guard`` (proj/include/slapo/executor.hpp:37-63).

There is no CPU fallback: importing this package without the built library
raises, and every executor call runs the sm_100a kernels.
"""
from __future__ import annotations

import ctypes
import json
import weakref
import os
import sys
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslapo_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the B200 executor)")

_lib = ctypes.CDLL(LIB_PATH)

_c = ctypes
_P = _c.c_void_p
_i64 = _c.c_int64
_u64 = _c.c_uint64
_dp = _c.POINTER(_c.c_double)


def _sig(name, *argtypes):
    f = getattr(_lib, name)
    f.argtypes = list(argtypes)
    f.restype = _c.c_int
    return f


_lib.sb_last_error.restype = _c.c_char_p
for _n, _a in {
    "sb_model_toy_bert": (_c.c_int, _i64, _i64, _i64, _i64, _i64, _c.c_double, _c.POINTER(_P)),
    "sb_model_gpt_neo": (_c.c_int, _i64, _i64, _i64, _i64, _i64, _c.c_double, _c.POINTER(_P)),
    "sb_pipeline_executor_create": (_P, _c.c_int, _c.c_int, _u64, _c.c_int, _c.POINTER(_c.c_int), _c.c_int,
                                    _c.POINTER(_P)),
    "sb_pipeline_executor_create_tp": (_P, _c.c_int, _c.c_int, _c.c_int, _u64, _c.c_int, _c.POINTER(_c.c_int),
                                       _c.c_int, _c.POINTER(_P)),
    "sb_pipeline_executor_create_dist": (_P, _c.c_int, _c.c_int, _c.c_int, _u64, _c.c_int, _c.c_int, _c.c_int,
                                         _c.c_int, _c.c_char_p, _c.c_char_p, _c.POINTER(_P)),
    "sb_pipeline_program": (_P, _c.c_int, _c.c_int, _c.c_int, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_pipeline_executor_forward": (_P, _c.POINTER(_dp), _c.c_int),
    "sb_pipeline_executor_num_outputs": (_P, _c.POINTER(_c.c_int)),
    "sb_pipeline_executor_output": (_P, _c.c_int, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t), _c.POINTER(_i64),
                                    _c.POINTER(_c.c_int)),
    "sb_pipeline_executor_backward": (_P,),
    "sb_pipeline_executor_num_grads": (_P, _c.c_int, _c.POINTER(_c.c_int)),
    "sb_pipeline_executor_grad_name": (_P, _c.c_int, _c.c_int, _c.c_char_p, _c.c_size_t),
    "sb_pipeline_executor_grad": (_P, _c.c_int, _c.c_char_p, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_pipeline_executor_num_input_grads": (_P, _c.c_int, _c.POINTER(_c.c_int)),
    "sb_pipeline_executor_input_grad": (_P, _c.c_int, _c.c_int, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_pipeline_executor_time_steps": (_P, _c.c_int, _c.POINTER(_c.c_float)),
    "sb_pipeline_executor_time_steps_ex": (_P, _c.c_int, _c.c_int, _c.POINTER(_c.c_float)),
    "sb_pipeline_executor_free": (_P,),
    "sb_model_t5": (_c.c_int, _c.c_int, _i64, _i64, _i64, _i64, _i64, _i64, _c.c_double, _c.POINTER(_P)),
    "sb_model_t5_ex": (_c.c_int, _c.c_int, _i64, _i64, _i64, _i64, _i64, _i64, _c.c_double, _c.c_int,
                       _c.POINTER(_P)),
    "sb_model_tp_two_linear": (_i64, _i64, _i64, _c.POINTER(_P)),
    "sb_model_fig3c": (_c.POINTER(_P),),
    "sb_model_ffn_stack": (_c.c_int, _i64, _i64, _c.POINTER(_P)),
    "sb_model_from_json": (_c.c_char_p, _c.POINTER(_P)),
    "sb_model_to_json": (_P, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_model_to_f32": (_P,),
    "sb_model_equal": (_P, _P, _c.POINTER(_c.c_int)),
    "sb_model_free": (_P,),
    "sb_estimate": (_P, _i64, _c.c_int, _i64, _dp, _c.POINTER(_i64), _dp, _c.c_char_p, _c.c_size_t,
                    _c.POINTER(_c.c_size_t)),
    "sb_model_apply_checkpoint_ratio": (_P, _c.c_char_p, _c.c_double, _c.POINTER(_c.c_int)),
    "sb_model_num_inputs": (_P, _c.POINTER(_c.c_int)),
    "sb_model_input_shape": (_P, _c.c_int, _c.POINTER(_i64), _c.POINTER(_c.c_int)),
    "sb_model_random_input": (_P, _c.c_int, _u64, _u64, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_model_param_values": (_P, _c.c_char_p, _c.c_int, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_schedule_create": (_P, _c.c_int, _c.POINTER(_P)),
    "sb_schedule_at": (_P, _c.c_char_p, _c.POINTER(_P)),
    "sb_schedule_trace": (_P, _c.c_int, _c.c_char_p),
    "sb_schedule_replace": (_P, _c.c_char_p, _c.c_char_p),
    "sb_schedule_shard": (_P, _c.c_char_p, _c.c_int),
    "sb_schedule_sync": (_P, _c.c_char_p),
    "sb_schedule_checkpoint": (_P, _c.c_char_p),
    "sb_schedule_define_pattern": (_P, _c.c_char_p, _c.c_char_p),
    "sb_schedule_fuse": (_P, _c.c_char_p, _c.c_char_p),
    "sb_schedule_pipeline_split": (_P, _c.c_char_p),
    "sb_schedule_find": (_P, _c.c_char_p, _c.POINTER(_c.c_int)),
    "sb_schedule_load_script": (_P, _c.c_char_p),
    "sb_schedule_num_warnings": (_P, _c.POINTER(_c.c_int)),
    "sb_schedule_apply": (_P, _c.POINTER(_P)),
    "sb_schedule_free": (_P,),
    "sb_schedule_apply_pipeline": (_P, _c.POINTER(_P)),
    "sb_pipeline_num_stages": (_P, _c.POINTER(_c.c_int)),
    "sb_pipeline_stage": (_P, _c.c_int, _c.POINTER(_P)),
    "sb_pipeline_stage_io": (_P, _c.c_int, _c.c_int, _c.c_char_p, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_pipeline_free": (_P,),
    "sb_executor_create": (_P, _c.c_int, _u64, _c.c_int, _c.c_int, _c.c_int, _c.POINTER(_P)),
    "sb_nccl_unique_id": (_P,),
    "sb_executor_create_nccl": (_P, _c.c_int, _u64, _c.c_int, _c.c_int, _P, _c.c_int, _c.c_int, _c.POINTER(_P)),
    "sb_executor_free": (_P,),
    "sb_executor_set_nan_guard": (_P, _c.c_int),
    "sb_executor_forward": (_P, _c.POINTER(_dp), _c.c_int),
    "sb_executor_num_outputs": (_P, _c.c_int, _c.POINTER(_c.c_int)),
    "sb_executor_output": (_P, _c.c_int, _c.c_int, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t), _c.POINTER(_i64),
                           _c.POINTER(_c.c_int)),
    "sb_executor_backward": (_P,),
    "sb_executor_num_grads": (_P, _c.c_int, _c.POINTER(_c.c_int)),
    "sb_executor_grad_name": (_P, _c.c_int, _c.c_int, _c.c_char_p, _c.c_size_t),
    "sb_executor_grad": (_P, _c.c_int, _c.c_char_p, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_executor_input_grad": (_P, _c.c_int, _c.c_int, _dp, _c.c_size_t, _c.POINTER(_c.c_size_t)),
    "sb_executor_ledger": (_P, _c.POINTER(_i64)),
    "sb_executor_collectives": (_P, _c.POINTER(_i64)),
    "sb_executor_upload_inputs": (_P, _c.POINTER(_dp), _c.c_int),
    "sb_executor_step": (_P, _c.c_int),
    "sb_executor_step_loss": (_P, _c.c_int, _c.POINTER(_c.c_float)),
    "sb_executor_synchronize": (_P,),
    "sb_executor_stream": (_P, _c.POINTER(_P)),
    "sb_executor_describe": (_P, _c.c_char_p, _c.c_size_t),
    "sb_executor_profile": (_P, _c.c_char_p, _c.c_size_t),
    "sb_executor_device_bytes": (_P, _c.POINTER(_i64)),
    "sb_executor_time_steps": (_P, _c.c_int, _c.c_int, _c.POINTER(_c.c_float)),
    "sb_executor_kernels_per_step": (_P, _c.POINTER(_c.c_int)),
    "sb_executor_time_e2e": (_P, _c.c_int, _c.POINTER(_dp), _c.c_int, _c.c_int, _c.POINTER(_c.c_float),
                             _c.POINTER(_c.c_float)),
    "sb_gemm_force_simt": (_c.c_int,),
    "sb_dropout_mask": (_P, _i64, _u64, _u64, _c.c_double, _P),
    "sb_attn_dropout_mask": (_P, _i64, _i64, _i64, _u64, _u64, _c.c_double, _P),
    "sb_attn_set_engine": (_c.c_int,),
    "sb_attn_engine": (_c.c_int,),
    "sb_attn_bwd_workspace": (_i64, _i64, _i64, _i64),
}.items():
    _sig(_n, *_a)
_lib.sb_gemm_engine.restype = _c.c_int
_lib.sb_attn_engine.restype = _c.c_int
_lib.sb_attn_bwd_workspace.restype = _c.c_size_t


class SlapoError(RuntimeError):
    """slapo::Error (proj/include/slapo/attrs.hpp:21-24)."""


class RuleError(SlapoError):
    """slapo::RuleError R1..R5 (proj/include/slapo/schedule.hpp:27-35)."""

    def __init__(self, msg: str):
        super().__init__(msg)
        self.rule = msg.split(":", 1)[0]


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.sb_last_error().decode()
    if rc == 2:
        raise RuleError(msg)
    raise SlapoError(msg)


def lib() -> ctypes.CDLL:
    return _lib


# ------------------------------------------------------------------- models
class Model:
    """A ModuleDef handle (proj/include/slapo/module.hpp:88-124)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:  # (at interpreter exit the module may be gone)
            _lib.sb_model_free(self._h)
            self._h = None

    @staticmethod
    def _make(fn, *args) -> "Model":
        h = _P()
        _check(fn(*args, _c.byref(h)))
        return Model(h)

    @staticmethod
    def from_json(text: str) -> "Model":
        return Model._make(_lib.sb_model_from_json, text.encode())

    def to_json(self) -> str:
        need = _c.c_size_t()
        _check(_lib.sb_model_to_json(self._h, None, 0, _c.byref(need)))
        buf = _c.create_string_buffer(need.value)
        _check(_lib.sb_model_to_json(self._h, buf, need.value, _c.byref(need)))
        return buf.value.decode()

    def to_f32(self) -> "Model":
        _check(_lib.sb_model_to_f32(self._h))
        return self

    def structurally_equal(self, other: "Model") -> bool:
        eq = _c.c_int()
        _check(_lib.sb_model_equal(self._h, other._h, _c.byref(eq)))
        return bool(eq.value)

    def input_shapes(self) -> List[List[int]]:
        n = _c.c_int()
        _check(_lib.sb_model_num_inputs(self._h, _c.byref(n)))
        out = []
        for i in range(n.value):
            dims = (_i64 * 16)()
            nd = _c.c_int(16)
            _check(_lib.sb_model_input_shape(self._h, i, dims, _c.byref(nd)))
            out.append([dims[k] for k in range(nd.value)])
        return out

    def random_inputs(self, seed: int) -> List[np.ndarray]:
        """random_tensor(spec_i, seed, stream=i) for every declared input."""
        res = []
        for i, shape in enumerate(self.input_shapes()):
            n = int(np.prod(shape)) if shape else 1
            a = np.empty(n, dtype=np.float64)
            nn = _c.c_size_t()
            _check(_lib.sb_model_random_input(self._h, i, seed, i, a.ctypes.data_as(_dp), n, _c.byref(nn)))
            res.append(a.reshape(shape))
        return res

    def apply_checkpoint_ratio(self, container: str, ratio: float) -> int:
        """Flag the first floor(ratio * L) children of `container` as checkpointed (costmodel.cpp:310-324)."""
        n = _c.c_int()
        _check(_lib.sb_model_apply_checkpoint_ratio(self._h, container.encode(), ratio, _c.byref(n)))
        return n.value

    def param_values(self, dotted: str, rank: int = 0) -> np.ndarray:
        """init_param_rank(param, rank): bit-exact host materialisation."""
        nn = _c.c_size_t()
        _check(_lib.sb_model_param_values(self._h, dotted.encode(), rank, None, 0, _c.byref(nn)))
        a = np.empty(nn.value, dtype=np.float64)
        _check(_lib.sb_model_param_values(self._h, dotted.encode(), rank, a.ctypes.data_as(_dp), nn.value,
                                          _c.byref(nn)))
        return a


def toy_bert(layers=24, hidden=8, heads=2, vocab=28, batch=4, seq=4, dropout_p=0.1) -> Model:
    return Model._make(_lib.sb_model_toy_bert, layers, hidden, heads, vocab, batch, seq, dropout_p)


def gpt_neo(layers=24, hidden=8, heads=2, vocab=28, batch=4, seq=4, dropout_p=0.1) -> Model:
    """GPT-Neo-style pre-LN causal decoder (f2, BASELINE.json configs[3]); no reference
    fixture exists — its oracle is the documented causal extension (oracle/causal_ext.py)."""
    return Model._make(_lib.sb_model_gpt_neo, layers, hidden, heads, vocab, batch, seq, dropout_p)


def t5(enc_layers=2, dec_layers=2, hidden=8, heads=2, vocab=28, batch=4, enc_seq=4, dec_seq=4,
       dropout_p=0.1, tie_embeddings=True) -> Model:
    """T5-style encoder-decoder with cross-attention (f2, BASELINE.json configs[4]); two id
    inputs (encoder, decoder); oracle: the causal extension (oracle/causal_ext.py).
    tie_embeddings=False: separate encoder / decoder tables (needed to pipeline_split it)."""
    return Model._make(_lib.sb_model_t5_ex, enc_layers, dec_layers, hidden, heads, vocab, batch, enc_seq, dec_seq,
                       dropout_p, int(tie_embeddings))


def tp_two_linear(hidden=8, inner=16, batch=4) -> Model:
    return Model._make(_lib.sb_model_tp_two_linear, hidden, inner, batch)


def fig3c_exact() -> Model:
    return Model._make(_lib.sb_model_fig3c)


def ffn_stack(n=24, hidden=4, batch=2) -> Model:
    return Model._make(_lib.sb_model_ffn_stack, n, hidden, batch)


# ----------------------------------------------------------------- schedule
def _graph_json(pattern) -> str:
    return pattern if isinstance(pattern, str) else json.dumps(pattern)


class Schedule:
    """Handle into the schedule tree (proj/include/slapo/schedule.hpp:60-111)."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:  # (at interpreter exit the module may be gone)
            _lib.sb_schedule_free(self._h)
            self._h = None

    def at(self, path: str) -> "Schedule":
        h = _P()
        _check(_lib.sb_schedule_at(self._h, path.encode(), _c.byref(h)))
        return Schedule(h, self)

    def __getitem__(self, path: str) -> "Schedule":
        return self.at(path)

    def trace(self, flatten: bool = False, leaves: Sequence[str] = ()) -> None:
        _check(_lib.sb_schedule_trace(self._h, int(flatten), ",".join(leaves).encode()))

    def replace(self, library: str, pattern: Optional[str] = None) -> None:
        _check(_lib.sb_schedule_replace(self._h, library.encode(), pattern.encode() if pattern else None))

    def shard(self, params: Sequence[str] | str, axis: int) -> None:
        if isinstance(params, str):
            params = [params]
        _check(_lib.sb_schedule_shard(self._h, ",".join(params).encode(), axis))

    def sync(self, type: str) -> None:  # noqa: A002 - the reference's argument name
        _check(_lib.sb_schedule_sync(self._h, type.encode()))

    def checkpoint(self, pattern: Optional[str] = None) -> None:
        _check(_lib.sb_schedule_checkpoint(self._h, pattern.encode() if pattern else None))

    def define_pattern(self, name: str, graph) -> None:
        _check(_lib.sb_schedule_define_pattern(self._h, name.encode(), _graph_json(graph).encode()))

    def fuse(self, pattern: str, backend: str = "composed") -> None:
        _check(_lib.sb_schedule_fuse(self._h, pattern.encode(), backend.encode()))

    def pipeline_split(self, after_child: str) -> None:
        _check(_lib.sb_schedule_pipeline_split(self._h, after_child.encode()))

    def find(self, glob: str) -> int:
        n = _c.c_int()
        _check(_lib.sb_schedule_find(self._h, glob.encode(), _c.byref(n)))
        return n.value

    def load_script(self, text: str) -> None:
        _check(_lib.sb_schedule_load_script(self._h, text.encode()))

    def num_warnings(self) -> int:
        n = _c.c_int()
        _check(_lib.sb_schedule_num_warnings(self._h, _c.byref(n)))
        return n.value

    def apply_pipeline(self) -> "PipelinePlan":
        """apply() with pipeline_split annotations: the stage plan (ApplyResult::stages)."""
        h = _P()
        _check(_lib.sb_schedule_apply_pipeline(self._h, _c.byref(h)))
        try:
            n = _c.c_int()
            _check(_lib.sb_pipeline_num_stages(h, _c.byref(n)))

            def names(i, which):
                need = _c.c_size_t()
                _check(_lib.sb_pipeline_stage_io(h, i, which, None, 0, _c.byref(need)))
                buf = _c.create_string_buffer(need.value)
                _check(_lib.sb_pipeline_stage_io(h, i, which, buf, need.value, _c.byref(need)))
                return [x for x in buf.value.decode().split("\n") if x]
            stages = []
            for i in range(n.value):
                mh = _P()
                _check(_lib.sb_pipeline_stage(h, i, _c.byref(mh)))
                stages.append(PipelineStage(Model(mh), names(i, 0), names(i, 1)))
            plan = PipelinePlan(stages, names(-1, 0), names(-1, 1))
        except BaseException:
            _lib.sb_pipeline_free(h)
            raise
        plan._h = h  # kept for PipelineExecutor; freed with the plan
        weakref.finalize(plan, _lib.sb_pipeline_free, h)
        return plan

    def apply(self) -> Model:
        h = _P()
        _check(_lib.sb_schedule_apply(self._h, _c.byref(h)))
        return Model(h)


@dataclass
class PipelineStage:
    module: Model
    consumes: List[str]
    produces: List[str]


@dataclass
class PipelinePlan:
    """slapo::PipelineStagePlan (proj/include/slapo/pipeline.hpp:14-27)."""
    stages: List[PipelineStage]
    model_inputs: List[str]
    model_outputs: List[str]
    _h: object = field(default=None, repr=False, compare=False)


def create_schedule(model: Model, world_size: int = 1) -> Schedule:
    h = _P()
    _check(_lib.sb_schedule_create(model._h, world_size, _c.byref(h)))
    return Schedule(h)


def schedule_path(name: str) -> str:
    return os.path.join(_HERE, "schedules", name)


# ----------------------------------------------------------------- executor
@dataclass
class GradientMap:
    """slapo::GradientMap (proj/include/slapo/executor.hpp:27-30)."""
    params: Dict[str, np.ndarray] = field(default_factory=dict)
    inputs: List[np.ndarray] = field(default_factory=list)


_DTYPES = {"fp32": 0, "f32": 0, "float32": 0, "bf16": 1, "bfloat16": 1}


class Executor:
    """slapo::Executor on B200 (proj/include/slapo/executor.hpp:37-63).

    ``world`` ranks of a sharded model run in lockstep on the current device
    (collectives are device-side rank-ascending sums, the reference's
    simulator semantics); ``nccl=(rank, unique_id)`` instead makes this process
    one rank of a one-process-per-GPU job with NCCL collectives.
    """

    def __init__(self, model: Model, mode: str = "train", seed: int = 0, world: int = 1, dtype: str = "fp32",
                 fused: bool = True, nccl: Optional[tuple] = None):
        h = _P()
        train = 1 if mode == "train" else 0
        if mode not in ("train", "verify"):
            raise ValueError("mode must be 'train' or 'verify'")
        dt = _DTYPES[dtype]
        self.world = world
        self.nccl_rank = None
        if nccl is None:
            _check(_lib.sb_executor_create(model._h, train, seed, world, dt, int(fused), _c.byref(h)))
        else:
            rank, uid = nccl
            _pin_nccl()
            ub = _c.create_string_buffer(bytes(uid), 128)
            _check(_lib.sb_executor_create_nccl(model._h, train, seed, world, rank, ub, dt, int(fused), _c.byref(h)))
            self.nccl_rank = rank
        self._h = h
        self._shapes = model.input_shapes()
        self._pinned = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:  # (at interpreter exit the module may be gone)
            _lib.sb_executor_free(self._h)
            self._h = None

    def _in_ptrs(self, inputs: Sequence[np.ndarray]):
        arrs = [np.ascontiguousarray(np.asarray(x, dtype=np.float64)) for x in inputs]
        for a, s in zip(arrs, self._shapes):
            if a.size != (int(np.prod(s)) if s else 1):
                raise SlapoError(f"input of size {a.size} does not match declared shape {s}")
        ptrs = (_dp * len(arrs))(*[a.ctypes.data_as(_dp) for a in arrs])
        return arrs, ptrs

    def set_nan_guard(self, on: bool) -> None:
        _check(_lib.sb_executor_set_nan_guard(self._h, int(on)))

    def forward(self, inputs: Sequence[np.ndarray]) -> List[np.ndarray]:
        arrs, ptrs = self._in_ptrs(inputs)
        _check(_lib.sb_executor_forward(self._h, ptrs, len(arrs)))
        return self.outputs_of_rank(self.nccl_rank or 0)

    def outputs_of_rank(self, rank: int) -> List[np.ndarray]:
        n = _c.c_int()
        _check(_lib.sb_executor_num_outputs(self._h, rank, _c.byref(n)))
        outs = []
        for i in range(n.value):
            nn = _c.c_size_t()
            dims = (_i64 * 16)()
            nd = _c.c_int(16)
            _check(_lib.sb_executor_output(self._h, rank, i, None, 0, _c.byref(nn), dims, _c.byref(nd)))
            a = np.empty(nn.value, dtype=np.float64)
            _check(_lib.sb_executor_output(self._h, rank, i, a.ctypes.data_as(_dp), nn.value, _c.byref(nn), dims,
                                           _c.byref(nd)))
            outs.append(a.reshape([dims[k] for k in range(nd.value)]))
        return outs

    def _grad_map(self, rank: int) -> GradientMap:
        n = _c.c_int()
        _check(_lib.sb_executor_num_grads(self._h, rank, _c.byref(n)))
        gm = GradientMap()
        buf = _c.create_string_buffer(4096)
        for i in range(n.value):
            _check(_lib.sb_executor_grad_name(self._h, rank, i, buf, 4096))
            name = buf.value
            nn = _c.c_size_t()
            _check(_lib.sb_executor_grad(self._h, rank, name, None, 0, _c.byref(nn)))
            a = np.empty(nn.value, dtype=np.float64)
            _check(_lib.sb_executor_grad(self._h, rank, name, a.ctypes.data_as(_dp), nn.value, _c.byref(nn)))
            gm.params[name.decode()] = a
        for i in range(len(self._shapes)):
            nn = _c.c_size_t()
            _check(_lib.sb_executor_input_grad(self._h, rank, i, None, 0, _c.byref(nn)))
            a = np.empty(nn.value, dtype=np.float64)
            _check(_lib.sb_executor_input_grad(self._h, rank, i, a.ctypes.data_as(_dp), nn.value, _c.byref(nn)))
            gm.inputs.append(a)
        return gm

    def backward_all_ranks(self) -> List[GradientMap]:
        _check(_lib.sb_executor_backward(self._h))
        ranks = [self.nccl_rank] if self.nccl_rank is not None else range(self.world)
        return [self._grad_map(r) for r in ranks]

    def backward(self) -> GradientMap:
        return self.backward_all_ranks()[0]

    def ledger(self) -> int:
        v = _i64()
        _check(_lib.sb_executor_ledger(self._h, _c.byref(v)))
        return v.value

    def collective_invocations(self) -> int:
        v = _i64()
        _check(_lib.sb_executor_collectives(self._h, _c.byref(v)))
        return v.value

    # -- device-resident stepping (bench.py) --
    def upload_inputs(self, inputs: Sequence[np.ndarray]) -> None:
        arrs, ptrs = self._in_ptrs(inputs)
        _check(_lib.sb_executor_upload_inputs(self._h, ptrs, len(arrs)))

    def step(self, use_graph: bool = True) -> None:
        _check(_lib.sb_executor_step(self._h, int(use_graph)))

    def step_loss(self, use_graph: bool = True) -> float:
        v = _c.c_float()
        _check(_lib.sb_executor_step_loss(self._h, int(use_graph), _c.byref(v)))
        return v.value

    def synchronize(self) -> None:
        _check(_lib.sb_executor_synchronize(self._h))

    def time_steps(self, steps: int, use_graph: bool = True) -> float:
        """Device milliseconds of `steps` back-to-back fwd+bwd steps (CUDA events)."""
        v = _c.c_float()
        _check(_lib.sb_executor_time_steps(self._h, steps, int(use_graph), _c.byref(v)))
        return v.value

    def time_e2e(self, steps: int, inputs: Sequence[np.ndarray], use_graph: bool = True):
        """(device ms, last loss) of `steps` end-to-end steps: H2D of `inputs`
        (pass pinned host arrays for async DMA), fwd+bwd, D2H of the loss."""
        arrs = [np.asarray(x) for x in inputs]
        for a in arrs:
            assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
        ptrs = (_dp * len(arrs))(*[a.ctypes.data_as(_dp) for a in arrs])
        ms, loss = _c.c_float(), _c.c_float()
        _check(_lib.sb_executor_time_e2e(self._h, steps, ptrs, len(arrs), int(use_graph), _c.byref(ms),
                                         _c.byref(loss)))
        return ms.value, loss.value

    def kernels_per_step(self) -> int:
        v = _c.c_int()
        _check(_lib.sb_executor_kernels_per_step(self._h, _c.byref(v)))
        return v.value

    def stream(self) -> int:
        s = _P()
        _check(_lib.sb_executor_stream(self._h, _c.byref(s)))
        return s.value or 0

    def describe(self) -> dict:
        buf = _c.create_string_buffer(1 << 16)
        _check(_lib.sb_executor_describe(self._h, buf, 1 << 16))
        return json.loads(buf.value.decode())

    def profile(self) -> dict:
        buf = _c.create_string_buffer(1 << 16)
        _check(_lib.sb_executor_profile(self._h, buf, 1 << 16))
        return json.loads(buf.value.decode())

    def device_bytes(self) -> int:
        v = _i64()
        _check(_lib.sb_executor_device_bytes(self._h, _c.byref(v)))
        return v.value


_lib.sb_plan_describe.argtypes = [_P, _c.c_int, _u64, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_char_p, _c.c_size_t]
_lib.sb_plan_describe.restype = _c.c_int


def plan_summary(model: Model, mode: str = "train", seed: int = 0, world: int = 1, rank: int = 0,
                 dtype: str = "fp32", fused: bool = True) -> dict:
    """Host-only lowering of one rank's device plan (no GPU): op kinds,
    checkpoint regions, activation ledger, forward collective count."""
    buf = _c.create_string_buffer(1 << 20)
    _check(_lib.sb_plan_describe(model._h, 1 if mode == "train" else 0, seed, world, rank, _DTYPES[dtype], int(fused),
                                 buf, 1 << 20))
    return json.loads(buf.value.decode())


def _pin_nccl() -> None:
    """One NCCL per process: when torch (torch.distributed) is in this process, make
    the executor dlopen the NCCL torch ships (nvidia/nccl/lib) instead of whatever
    libnccl.so.2 the loader would find first (the system copy may be another version)."""
    if os.environ.get("SB_NCCL_LIB") or "torch" not in sys.modules:
        return
    try:
        import nvidia.nccl  # noqa: F401  (the wheel torch's libtorch_cuda links against)
        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                os.environ["SB_NCCL_LIB"] = p
                return
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    _pin_nccl()
    buf = _c.create_string_buffer(128)
    _check(_lib.sb_nccl_unique_id(buf))
    return buf.raw


def run_forward(model: Model, inputs, mode="verify", seed=0, **kw) -> List[np.ndarray]:
    """run_forward (proj/include/slapo/executor.hpp:66)."""
    return Executor(model, mode, seed, 1, **kw).forward(inputs)


def run_backward(model: Model, inputs, mode="verify", seed=0, **kw) -> GradientMap:
    """run_backward (proj/include/slapo/executor.hpp:70)."""
    ex = Executor(model, mode, seed, 1, **kw)
    ex.forward(inputs)
    return ex.backward()


def run_sharded(model: Model, inputs, world_size: int, mode="verify", seed=0, **kw) -> List[np.ndarray]:
    """run_sharded (proj/include/slapo/executor.hpp:74)."""
    if world_size < 2:
        raise SlapoError("run_sharded requires world_size > 1")
    return Executor(model, mode, seed, world_size, **kw).forward(inputs)


def run_pipeline(plan: PipelinePlan, inputs, micro_batches: int = 1, mode: str = "verify", seed: int = 0,
                 dtype: str = "fp32") -> List[np.ndarray]:
    """GPipe forward of a stage plan on the GPU (run_pipeline, proj/src/executor.cpp:1531-1579):
    the batch is cut into `micro_batches` slices along dim 0; for each micro-batch
    the stages run in order, every stage on the device through its own executor,
    its inputs bound by name from the model inputs and earlier stages' outputs;
    the model outputs are concatenated along dim 0 in micro-batch order."""
    if micro_batches < 1:
        raise SlapoError("micro_batches must be >= 1")
    if len(inputs) != len(plan.model_inputs):
        raise SlapoError(f"pipeline expects {len(plan.model_inputs)} inputs")
    def micro_module(m: Model) -> Model:
        # the executor plans from declared input shapes: a stage runs on 1/micro of the batch
        if micro_batches == 1:
            return m
        d = json.loads(m.to_json())
        for node in d["modules"].get("forward", []):
            if node.get("kind") == "input":
                shape = node["attrs"]["shape"]
                if shape[0] % micro_batches:
                    raise SlapoError(f"batch dimension {shape[0]} not divisible into {micro_batches} micro-batches")
                shape[0] //= micro_batches
        return Model.from_json(json.dumps(d))

    execs = [Executor(micro_module(st.module), mode=mode, seed=seed, dtype=dtype) for st in plan.stages]
    chunks = []
    for c in range(micro_batches):
        env = {}
        for name, x in zip(plan.model_inputs, inputs):
            x = np.asarray(x)
            if micro_batches > 1:
                if x.shape[0] % micro_batches:
                    raise SlapoError(f"batch dimension {x.shape[0]} not divisible into {micro_batches} micro-batches")
                per = x.shape[0] // micro_batches
                x = x[c * per:(c + 1) * per]
            env[name] = x
        for st, ex in zip(plan.stages, execs):
            missing = [n for n in st.consumes if n not in env]
            if missing:
                raise SlapoError(f"pipeline stage consumes unknown value '{missing[0]}'")
            outs = ex.forward([env[n] for n in st.consumes])
            if len(outs) != len(st.produces):
                raise SlapoError(f"pipeline stage produced {len(outs)} values, expected {len(st.produces)}")
            env.update(zip(st.produces, outs))
        chunks.append([env[n] for n in plan.model_outputs])
    if micro_batches == 1:
        return chunks[0]
    return [np.concatenate([ch[o] for ch in chunks], axis=0) for o in range(len(plan.model_outputs))]


class PipelineExecutor:
    """Pipeline-parallel training step over a stage plan (f1; csrc/host/pipeline_exec.hpp):
    GPipe with re-materialisation, one executor per stage on `devices[stage]` (default:
    the current device), stage-boundary values stashed per micro-batch and moved
    device-to-device (peer copies over NVLink between devices), the backward of
    sum(outputs) seeded stage by stage with the consumers' input gradients, parameter
    gradients summed over micro-batches. The forward is run_pipeline's (proj/src/
    executor.cpp:1531-1579): every micro-batch of a stage runs with the executor seed
    on micro-batch-shaped tensors."""

    def __init__(self, plan: PipelinePlan, micro_batches: int = 1, mode: str = "train", seed: int = 0,
                 dtype: str = "fp32", devices: Optional[Sequence[int]] = None, fused: bool = True, tp: int = 1,
                 dist: Optional[tuple] = None):
        """dist = (rank, world, pp_uid, tp_uid): one process per (stage, tp rank), rank = stage * tp +
        tp_rank, world = stages * tp; pp_uid (128 bytes, the same on every rank) names the pipeline
        communicator, tp_uid (the same on the tp ranks of one stage; None for tp == 1) the stage's."""
        if plan._h is None:
            raise SlapoError("PipelineExecutor needs a plan from Schedule.apply_pipeline()")
        self._plan = plan
        self.micro_batches = micro_batches
        devs = None
        if devices is not None:
            if len(devices) != len(plan.stages):
                raise SlapoError("one device per stage")
            devs = (_c.c_int * len(devices))(*devices)
        h = _P()
        self.dist = dist
        if dist is not None:
            _pin_nccl()
            rank, world, pp_uid, tp_uid = dist
            _check(_lib.sb_pipeline_executor_create_dist(plan._h, micro_batches, tp, int(mode == "train"), seed,
                                                         _DTYPES[dtype], int(fused), rank, world, pp_uid, tp_uid,
                                                         _c.byref(h)))
        else:
            _check(_lib.sb_pipeline_executor_create_tp(plan._h, micro_batches, tp, int(mode == "train"), seed,
                                                       _DTYPES[dtype], devs, int(fused), _c.byref(h)))
        self.tp = tp
        self._h = h
        weakref.finalize(self, _lib.sb_pipeline_executor_free, h)

    def forward(self, inputs: Sequence[np.ndarray]) -> List[np.ndarray]:
        arrs = [np.ascontiguousarray(np.asarray(x, dtype=np.float64)) for x in inputs]
        ptrs = (_dp * len(arrs))(*[a.ctypes.data_as(_dp) for a in arrs])
        _check(_lib.sb_pipeline_executor_forward(self._h, ptrs, len(arrs)))
        n = _c.c_int()
        _check(_lib.sb_pipeline_executor_num_outputs(self._h, _c.byref(n)))
        outs = []
        for i in range(n.value):
            nn = _c.c_size_t()
            dims = (_i64 * 16)()
            nd = _c.c_int(16)
            _check(_lib.sb_pipeline_executor_output(self._h, i, None, 0, _c.byref(nn), dims, _c.byref(nd)))
            a = np.empty(nn.value, dtype=np.float64)
            _check(_lib.sb_pipeline_executor_output(self._h, i, a.ctypes.data_as(_dp), nn.value, _c.byref(nn), dims,
                                                    _c.byref(nd)))
            outs.append(a.reshape([dims[k] for k in range(nd.value)]))
        return outs

    def backward(self) -> List[GradientMap]:
        """Per stage (and tensor-parallel rank: slot stage * tp + rank): parameter
        gradients (stage-local names) and the gradients of the model inputs the stage
        consumes."""
        _check(_lib.sb_pipeline_executor_backward(self._h))
        res = []
        buf = _c.create_string_buffer(4096)
        for st in range(1 if self.dist is not None else len(self._plan.stages) * self.tp):
            gm = GradientMap()
            n = _c.c_int()
            _check(_lib.sb_pipeline_executor_num_grads(self._h, st, _c.byref(n)))
            for i in range(n.value):
                _check(_lib.sb_pipeline_executor_grad_name(self._h, st, i, buf, 4096))
                name = buf.value
                nn = _c.c_size_t()
                _check(_lib.sb_pipeline_executor_grad(self._h, st, name, None, 0, _c.byref(nn)))
                a = np.empty(nn.value, dtype=np.float64)
                _check(_lib.sb_pipeline_executor_grad(self._h, st, name, a.ctypes.data_as(_dp), nn.value, _c.byref(nn)))
                gm.params[name.decode()] = a
            _check(_lib.sb_pipeline_executor_num_input_grads(self._h, st, _c.byref(n)))
            for i in range(n.value):
                nn = _c.c_size_t()
                _check(_lib.sb_pipeline_executor_input_grad(self._h, st, i, None, 0, _c.byref(nn)))
                a = np.empty(nn.value, dtype=np.float64)
                _check(_lib.sb_pipeline_executor_input_grad(self._h, st, i, a.ctypes.data_as(_dp), nn.value,
                                                            _c.byref(nn)))
                gm.inputs.append(a)
            res.append(gm)
        return res

    def time_steps(self, steps: int, use_graph: bool = True) -> float:
        """device ms of `steps` training steps; use_graph: captured once into a CUDA graph
        (stages on one device) and replayed"""
        ms = _c.c_float()
        _check(_lib.sb_pipeline_executor_time_steps_ex(self._h, steps, int(use_graph), _c.byref(ms)))
        return ms.value


def pipeline_program(plan: PipelinePlan, micro_batches: int, tp: int, rank: int):
    """The transfer program a distributed pipeline rank executes (csrc/host/pipeline_exec.hpp
    pipe_program): [(kind, micro_batch, index, peer, value, numel)]."""
    if plan._h is None:
        raise SlapoError("pipeline_program needs a plan from Schedule.apply_pipeline()")
    need = _c.c_size_t()
    _check(_lib.sb_pipeline_program(plan._h, micro_batches, tp, rank, None, 0, _c.byref(need)))
    buf = _c.create_string_buffer(need.value)
    _check(_lib.sb_pipeline_program(plan._h, micro_batches, tp, rank, buf, need.value, _c.byref(need)))
    out = []
    for ln in buf.value.decode().splitlines():
        k, m, i, p, v, n = ln.split()
        out.append((k, int(m), int(i), int(p), v, int(n)))
    return out
