"""Schedule recipes for the BASELINE configs, as schedule scripts.

The same script text drives this executor (``Schedule.load_script``) and the
reference oracle (``load_schedule_script``, proj/src/script.cpp:74), so both
apply the identical primitive log.

* ``c2_script``: .replace(EfficientAttention) + .fuse of bias+dropout+residual+LN,
  bias+GeLU and bias+residual+LN (+ optional checkpoint) — BASELINE configs[1].
* ``tp_script``: Megatron tensor parallelism exactly as SURVEY.md §8(d):
  FusedQKV sharded blockwise on axis 0 + sync backward, attention.output.dense
  axis 1 + sync forward, ffn.dense1 axis 0 + sync backward, ffn.dense2 axis 1 +
  sync forward, vocab-parallel embeddings + sync both; then EfficientAttention,
  the all_reduce-including fusion patterns and
  checkpointing of the first ``ckpt_ratio * layers`` layers — BASELINE configs[2].
"""
from __future__ import annotations

import json


def _node(i, kind, **kw):
    d = {"id": i, "kind": kind}
    d.update(kw)
    return d


def pattern_linear_gelu():
    return [_node(0, "input"), _node(1, "call_module", target="Linear", args=[0]),
            _node(2, "call_op", op="gelu", args=[1]), _node(3, "output", args=[2])]


def pattern_res_ln(all_reduce: bool, dropout: bool):
    """Linear -> [all_reduce] -> [Dropout] -> add(., residual) -> LayerNorm."""
    nodes = [_node(0, "input"), _node(1, "input"), _node(2, "call_module", target="Linear", args=[0])]
    cur, nid = 2, 3
    if all_reduce:
        nodes.append(_node(nid, "call_op", op="all_reduce", args=[cur]))
        cur, nid = nid, nid + 1
    if dropout:
        nodes.append(_node(nid, "call_module", target="Dropout", args=[cur]))
        cur, nid = nid, nid + 1
    nodes.append(_node(nid, "call_op", op="add", args=[cur, 1]))
    nodes.append(_node(nid + 1, "call_module", target="LayerNorm", args=[nid]))
    nodes.append(_node(nid + 2, "output", args=[nid + 1]))
    return nodes


def _pattern_block(name, nodes):
    return f"pattern {name} {{\n  {json.dumps(nodes)}\n}}\n"


def fusion_lines(layers: int, all_reduce: bool, backend: str = "composed") -> str:
    s = _pattern_block("bdrln", pattern_res_ln(all_reduce, True))
    s += _pattern_block("bias_gelu", pattern_linear_gelu())
    s += _pattern_block("brln", pattern_res_ln(all_reduce, False))
    for i in range(layers):
        lp = f"encoder.layer.{i}"
        s += f"trace {lp}.attention.output flatten=true\n"
        s += f"fuse {lp}.attention.output at bdrln backend={backend}\n"
        s += f"trace {lp}.ffn flatten=true\n"
        s += f"fuse {lp}.ffn at bias_gelu backend={backend}\n"
        s += f"fuse {lp}.ffn at brln backend={backend}\n"
    return s


def c2_script(layers: int, checkpoint_layers=(), flash: bool = True, fuse: bool = True) -> str:
    s = "# BASELINE configs[1]: replace(EfficientAttention) + fuse + checkpoint\n"
    if flash:
        s += "".join(f"replace encoder.layer.{i}.attention.core with EfficientAttention\n" for i in range(layers))
    if fuse:
        s += fusion_lines(layers, all_reduce=False)
    s += "".join(f"checkpoint encoder.layer.{i}\n" for i in checkpoint_layers)
    return s


def tp_script(layers: int, world: int, fuse: bool = True, flash: bool = True, ckpt_ratio: float = 0.0,
              fused_qkv: bool = True, shard_embeddings: bool = True) -> str:
    s = f"# Megatron TP={world} recipe (SURVEY.md §8(d) verified order)\n"
    for i in range(layers):
        lp = f"encoder.layer.{i}"
        if fused_qkv:
            s += f"replace {lp}.attention.qkv with FusedQKV\n"
        if world > 1:
            if fused_qkv:
                s += f"shard {lp}.attention.qkv weight,bias axis=0\n"
                s += f"sync {lp}.attention.qkv type=backward\n"
            s += f"shard {lp}.attention.output.dense weight,bias axis=1\n"
            s += f"sync {lp}.attention.output.dense type=forward\n"
            s += f"shard {lp}.ffn.dense1 weight,bias axis=0\n"
            s += f"sync {lp}.ffn.dense1 type=backward\n"
            s += f"shard {lp}.ffn.dense2 weight,bias axis=1\n"
            s += f"sync {lp}.ffn.dense2 type=forward\n"
        if flash:
            s += f"replace {lp}.attention.core with EfficientAttention\n"
    if fuse:
        s += fusion_lines(layers, all_reduce=world > 1)
    if world > 1 and shard_embeddings:
        s += "shard embeddings weight axis=0\nsync embeddings type=both\n"
    for i in range(int(ckpt_ratio * layers)):
        s += f"checkpoint encoder.layer.{i}\n"
    return s


def neo_script(layers: int, world: int = 1, flash: bool = True, fuse: bool = True, fused_qkv: bool = True,
               checkpoint_layers=(), shard_embeddings: bool = True) -> str:
    """The decoder recipe (f2, BASELINE.json configs[3]) for ``gpt_neo``: FusedQKV
    (bias-free, sharded blockwise on axis 0 + sync backward), out_proj axis 1 + sync
    forward, mlp.c_fc axis 0 + sync backward, mlp.c_proj axis 1 + sync forward,
    vocab-parallel wte + sync both; the causal core replaced by EfficientAttention
    (its ``causal`` attr is copied, library.cpp:106-113); bias+GeLU fused in the MLP;
    selective checkpointing of ``checkpoint_layers``."""
    s = f"# GPT-Neo-style decoder recipe, TP={world}\n"
    for i in range(layers):
        lp = f"h.{i}"
        if fused_qkv:
            s += f"replace {lp}.attn.qkv with FusedQKV\n"
        if world > 1:
            if fused_qkv:
                s += f"shard {lp}.attn.qkv weight axis=0\n"
                s += f"sync {lp}.attn.qkv type=backward\n"
            s += f"shard {lp}.attn.out_proj weight,bias axis=1\n"
            s += f"sync {lp}.attn.out_proj type=forward\n"
            s += f"shard {lp}.mlp.c_fc weight,bias axis=0\n"
            s += f"sync {lp}.mlp.c_fc type=backward\n"
            s += f"shard {lp}.mlp.c_proj weight,bias axis=1\n"
            s += f"sync {lp}.mlp.c_proj type=forward\n"
        if flash:
            s += f"replace {lp}.attn.core with EfficientAttention\n"
    if fuse:
        s += _pattern_block("bias_gelu", pattern_linear_gelu())
        for i in range(layers):
            s += f"trace h.{i}.mlp flatten=true\n"
            s += f"fuse h.{i}.mlp at bias_gelu backend=composed\n"
    if world > 1 and shard_embeddings:
        s += "shard wte weight axis=0\nsync wte type=both\n"
    s += "".join(f"checkpoint h.{i}\n" for i in checkpoint_layers)
    return s


def t5_script(enc_layers: int, dec_layers: int, world: int = 1, flash: bool = True, fused_qkv: bool = True,
              checkpoint=(), shard_embeddings: bool = True, tied: bool = True) -> str:
    """The encoder-decoder recipe (f2, BASELINE.json configs[4]) for ``t5``: self-attention
    as FusedQKV (sharded blockwise on axis 0 + sync backward), cross-attention query / key /
    value Linears sharded on axis 0 with sync backward (the key / value SyncGrads sum the
    encoder output's gradient contributions), out_proj / mlp.wo row-parallel + sync forward,
    mlp.wi column-parallel + sync backward, the shared vocab-parallel embedding + sync both;
    every self-attention core replaced by EfficientAttention (the decoder's keeps its causal
    attr; the cross-attention core cannot be — rule R4, q and k/v shapes differ — and runs as
    the composed reference graph); checkpointing of the listed blocks ("encoder.block.0", ...)."""
    s = f"# T5-style encoder-decoder recipe, TP={world}\n"

    def self_attn(p):
        nonlocal s
        if fused_qkv:
            s += f"replace {p}.qkv with FusedQKV\n"
        if world > 1:
            if fused_qkv:
                s += f"shard {p}.qkv weight axis=0\nsync {p}.qkv type=backward\n"
            s += f"shard {p}.out_proj weight,bias axis=1\nsync {p}.out_proj type=forward\n"
        if flash:
            s += f"replace {p}.core with EfficientAttention\n"

    def mlp(p):
        nonlocal s
        if world > 1:
            s += f"shard {p}.wi weight,bias axis=0\nsync {p}.wi type=backward\n"
            s += f"shard {p}.wo weight,bias axis=1\nsync {p}.wo type=forward\n"

    for i in range(enc_layers):
        self_attn(f"encoder.block.{i}.attn")
        mlp(f"encoder.block.{i}.mlp")
    for i in range(dec_layers):
        p = f"decoder.block.{i}"
        self_attn(f"{p}.self_attn")
        if world > 1:
            for n in ("query", "key", "value"):
                s += f"shard {p}.cross_attn.{n} weight axis=0\nsync {p}.cross_attn.{n} type=backward\n"
            s += f"shard {p}.cross_attn.out_proj weight,bias axis=1\nsync {p}.cross_attn.out_proj type=forward\n"
        # (the cross-attention core stays the composed reference graph: replacing it with
        # EfficientAttention violates rule R4 — its q and k/v specs differ, S_dec vs S_enc)
        mlp(f"{p}.mlp")
    if world > 1 and shard_embeddings:
        for e in (("shared",) if tied else ("enc_embed", "dec_embed")):
            s += f"shard {e} weight axis=0\nsync {e} type=both\n"
    s += "".join(f"checkpoint {c}\n" for c in checkpoint)
    return s
