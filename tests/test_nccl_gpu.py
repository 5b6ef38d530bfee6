"""The one-process-per-GPU NCCL executor (sb_executor_create_nccl) and the
capture-safe NaN guard.

* world 1: an NCCL communicator of one rank with the one-rank collectives kept
  (LowerOptions::keep_collectives), so ncclCommInitRank, in-place ncclAllReduce on
  the executor stream and on the high-priority communication stream, the
  chunked forward all-reduce overlap and the early backward all-reduce all run,
  eagerly and captured in a CUDA graph. A one-rank all-reduce is an exact copy,
  so outputs and every gradient must be bitwise equal to the plain executor's.
* world 2 (skipped unless two GPUs are visible): two processes, one per GPU,
  against the lockstep world-2 executor (which tests/test_parity_gpu.py checks
  against the reference's run_sharded).
* NaN guard (reference executor.cpp:308-316,845; executor_test.cpp:318-329):
  a NaN input raises "NaN produced by" at the producing op, eagerly and from a
  graph replay.
"""
import numpy as np
import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes

pytestmark = pytest.mark.gpu

CFG = dict(layers=2, hidden=256, heads=4, vocab=64, batch=2, seq=256, p=0.1)


def _model_sched(world, ckpt=0.5, cfg=CFG):
    m = sb.toy_bert(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])
    s = sb.create_schedule(m, world)
    s.load_script(recipes.tp_script(cfg["layers"], world, ckpt_ratio=ckpt))
    return m, s.apply()


def _assert_same(ex_a, ex_b, rank_a=0, rank_b=0):
    oa, ob = ex_a.outputs_of_rank(rank_a), ex_b.outputs_of_rank(rank_b)
    assert len(oa) == len(ob)
    for a, b in zip(oa, ob):
        assert np.array_equal(a, b), np.abs(a - b).max()
    ga, gb = ex_a._grad_map(rank_a).params, ex_b._grad_map(rank_b).params
    assert set(ga) == set(gb)
    for k in ga:
        assert np.array_equal(ga[k], gb[k]), (k, np.abs(ga[k] - gb[k]).max())


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_nccl_world1_bitwise_equal_to_local(dtype):
    m, applied = _model_sched(1)
    x = m.random_inputs(9)
    plain = sb.Executor(applied, "train", 123, 1, dtype=dtype)
    plain.forward(x)
    plain.backward_all_ranks()
    nc = sb.Executor(applied, "train", 123, 1, dtype=dtype, nccl=(0, sb.nccl_unique_id()))
    nc.forward(x)
    nc.backward_all_ranks()
    _assert_same(plain, nc)
    # the NCCL executor counts one more collective per kept SyncGrad (the reference
    # inserts none at world 1); the forward all_reduce count is the same
    assert nc.collective_invocations() >= plain.collective_invocations()
    # captured: NCCL calls on the executor and communication streams inside a CUDA graph
    nc.upload_inputs(x)
    nc.step(use_graph=True)
    nc.step(use_graph=True)
    nc.synchronize()
    _assert_same(plain, nc)
    plain.upload_inputs(x)
    plain.step(use_graph=True)
    plain.synchronize()
    _assert_same(plain, nc)


def test_nccl_world1_chunked_forward_allreduce_bf16():
    """Rows divisible into >= 2 chunks of 256: the row-parallel GEMM / all-reduce /
    LayerNorm-tail pipeline runs chunked (fused_res_ln_overlapped)."""
    cfg = dict(CFG, batch=4, seq=256)  # 1024 rows -> 4 chunks of 256
    m, applied = _model_sched(1, cfg=cfg)
    x = m.random_inputs(9)
    plain = sb.Executor(applied, "train", 123, 1, dtype="bf16")
    plain.forward(x)
    plain.backward_all_ranks()
    nc = sb.Executor(applied, "train", 123, 1, dtype="bf16", nccl=(0, sb.nccl_unique_id()))
    nc.forward(x)
    nc.backward_all_ranks()
    assert sb.lib().sb_gemm_engine() == 2
    _assert_same(plain, nc)


def _worker(rank, uid, q):
    import torch
    torch.cuda.set_device(rank)
    m, applied = _model_sched(2)
    ex = sb.Executor(applied, "train", 123, 2, dtype="bf16", nccl=(rank, uid))
    outs = ex.forward(m.random_inputs(9))
    g = ex.backward()
    q.put((rank, outs, g.params, ex.collective_invocations()))


@pytest.mark.skipif(not __import__("torch").cuda.is_available() or __import__("torch").cuda.device_count() < 2,
                    reason="needs two GPUs (one process per GPU)")
def test_nccl_two_processes_match_lockstep():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = sb.nccl_unique_id()
    ps = [ctx.Process(target=_worker, args=(r, uid, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        r, outs, grads, coll = q.get(timeout=600)
        res[r] = (outs, grads, coll)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, applied = _model_sched(2)
    lock = sb.Executor(applied, "train", 123, 2, dtype="bf16")
    lock.forward(m.random_inputs(9))
    lg = lock.backward_all_ranks()
    for r in range(2):
        outs, grads, coll = res[r]
        assert coll == lock.collective_invocations()
        for a, b in zip(outs, lock.outputs_of_rank(r)):
            # NCCL's reduction order differs from the rank-ascending device sum
            assert np.linalg.norm(a - b) <= 1e-2 * np.linalg.norm(b)
        for k, v in lg[r].params.items():
            assert np.linalg.norm(grads[k] - v) <= 2e-2 * max(np.linalg.norm(v), 1e-30), k


def _single_gelu(dtype="f32"):
    """single_op_model("gelu", {spec}) of executor_test.cpp:318-329 as slapo-model-v1 JSON."""
    import json
    d = {"format": "slapo-model-v1", "name": "gelu", "modules": {"kind": "composite", "submodules": {}, "forward": [
        {"id": 0, "kind": "input", "attrs": {"dtype": dtype, "shape": [2]}},
        {"id": 1, "kind": "call_op", "op": "gelu", "args": [0]},
        {"id": 2, "kind": "output", "args": [1]}]}}
    return sb.Model.from_json(json.dumps(d))


def test_nan_guard_eager_and_graph():
    m = _single_gelu()
    x = [np.array([1.0, np.nan])]
    quiet = sb.Executor(m, "verify", 0, 1)
    quiet.forward(x)
    guarded = sb.Executor(m, "verify", 0, 1)
    guarded.set_nan_guard(True)
    with pytest.raises(sb.SlapoError, match="NaN produced by op 'Gelu' on rank 0"):
        guarded.forward(x)
    ok = sb.Executor(m, "verify", 0, 1)
    ok.set_nan_guard(True)
    ok.forward([np.array([1.0, 2.0])])
    # inside a captured graph: counted on the device, reported after the replay
    g2 = sb.Executor(m, "train", 0, 1)
    g2.set_nan_guard(True)
    g2.upload_inputs(x)
    with pytest.raises(sb.SlapoError, match="NaN produced by"):
        g2.step(use_graph=True)
