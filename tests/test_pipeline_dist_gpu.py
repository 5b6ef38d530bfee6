"""The distributed pipeline step (one process per stage x tp rank, NCCL send/recv of the
stage I/O, csrc/host/pipeline_exec.cpp) against the single-process PipelineExecutor on the
same plan: outputs and every gradient. Needs one GPU per rank — skipped on this pool's
one-GPU boxes; the transfer programs themselves are checked on CPU
(tests/test_pipeline_program_cpu.py: simulation + gloo)."""
import os

import numpy as np
import pytest

import paper_2302_08005_b200 as sb

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
SPLIT = "trace encoder.layer\npipeline_split encoder.layer after=1\n"


def _plan():
    m = sb.toy_bert(4, 32, 4, 32, 4, 8, 0.1)
    s = sb.create_schedule(m, 2)
    s.load_script(SPLIT)
    return m, s.apply_pipeline()


def _worker(rank, world, uid, q):
    try:
        torch.cuda.set_device(rank)
        m, plan = _plan()
        pe = sb.PipelineExecutor(plan, 2, "train", 123, "fp32", dist=(rank, world, uid, None))
        out = pe.forward(m.random_inputs(9))
        g = pe.backward()[0].params
        q.put((rank, [o.tolist() for o in out], {k: v.tolist() for k, v in g.items()}))
    except BaseException as e:
        q.put((rank, repr(e), None))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (one process per pipeline stage)")
def test_distributed_pipeline_matches_single_process():
    import torch.multiprocessing as mp
    m, plan = _plan()
    local = sb.PipelineExecutor(plan, 2, "train", 123, "fp32")
    want_out = local.forward(m.random_inputs(9))
    want = local.backward()
    uid = sb.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, uid, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, out, g = q.get(timeout=300)
        assert g is not None, out
        res[r] = (out, g)
    for p in procs:
        p.join(timeout=60)
    got_out = np.asarray(res[1][0][0])  # the last stage produces the model output
    assert np.abs(got_out.reshape(want_out[0].shape) - want_out[0]).max() <= 1e-6 * np.abs(want_out[0]).max()
    for st in range(2):
        for k, v in want[st].params.items():
            assert np.allclose(np.asarray(res[st][1][k]), v, rtol=0, atol=1e-6 * max(np.abs(v).max(), 1e-9)), k
