"""Host-side logic of the distributed pipeline step (one process per stage x tp rank,
csrc/host/pipeline_exec.hpp pipe_program): the per-rank transfer programs pair up and
cannot deadlock. Checked by simulation under rendezvous semantics (a send completes
only together with the matching receive, the strictest NCCL behaviour) and by running
the programs over real blocking point-to-point transfers (torch.distributed gloo, one
process per rank, world up to 6) with payloads that identify (micro-batch, value)."""
import os

import pytest

import paper_2302_08005_b200 as sb
from paper_2302_08005_b200 import recipes

SPLITS = {
    "2 stages": "trace encoder.layer\npipeline_split encoder.layer after=1\n",
    "3 stages, pass-through": "trace encoder.layer\npipeline_split encoder.layer after=0\n"
                              "pipeline_split encoder.layer after=2\n",
}


def _plan(split, tp):
    m = sb.toy_bert(4, 32, 4, 32, 4, 8, 0.1)
    s = sb.create_schedule(m, max(2, tp))
    s.load_script((recipes.tp_script(4, tp) if tp > 1 else "") + SPLITS[split])
    return s.apply_pipeline()


def _programs(plan, micro, tp):
    world = len(plan.stages) * tp
    return [sb.pipeline_program(plan, micro, tp, r) for r in range(world)]


def simulate(progs):
    """Rendezvous semantics: returns the number of matched transfers; raises on a
    mismatch or a deadlock."""
    pc = [0] * len(progs)
    matched = 0
    while True:
        progressed = False
        done = True
        for r, prog in enumerate(progs):
            if pc[r] >= len(prog):
                continue
            done = False
            k, m, i, peer, v, n = prog[pc[r]]
            if k.endswith("_run"):
                pc[r] += 1
                progressed = True
                continue
            if pc[peer] >= len(progs[peer]):
                continue
            pk, pm, pi, ppeer, pv, pn = progs[peer][pc[peer]]
            want = k.replace("send", "X").replace("recv", "send").replace("X", "recv")
            if pk == want and ppeer == r:
                assert (pm, pv, pn) == (m, v, n), f"rank {r} {prog[pc[r]]} paired with rank {peer} {progs[peer][pc[peer]]}"
                assert k[:3] == pk[:3]
                pc[r] += 1
                pc[peer] += 1
                matched += 1
                progressed = True
        if done:
            return matched
        assert progressed, f"deadlock at {[(r, progs[r][pc[r]] if pc[r] < len(progs[r]) else None) for r in range(len(progs))]}"


@pytest.mark.parametrize("split", list(SPLITS))
@pytest.mark.parametrize("micro", [1, 2, 4])
@pytest.mark.parametrize("tp", [1, 2])
def test_programs_pair_up_without_deadlock(split, micro, tp):
    plan = _plan(split, tp)
    progs = _programs(plan, micro, tp)
    n = simulate(progs)
    sends = sum(1 for p in progs for s in p if s[0].endswith("send"))
    assert n == sends > 0
    # every rank runs each micro-batch exactly once forward and once backward
    for p in progs:
        assert [s[1] for s in p if s[0] == "fwd_run"] == list(range(micro))
        assert [s[1] for s in p if s[0] == "bwd_run"] == list(reversed(range(micro)))
    # transfers only between ranks of equal tensor-parallel rank
    for r, p in enumerate(progs):
        assert all(s[3] % tp == r % tp for s in p if s[3] >= 0)


def _gloo_worker(rank, world, port, progs, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        names = sorted({s[4] for p in progs for s in p if s[4] != "-"})
        code = {n: i for i, n in enumerate(names)}
        for k, m, i, peer, v, n in progs[rank]:
            tag = 1000 * m + code.get(v, 0)
            if k.endswith("send"):
                dist.send(torch.full((n,), float(tag) + (0.5 if k.startswith("bwd") else 0.0)), dst=peer)
            elif k.endswith("recv"):
                t = torch.empty(n)
                dist.recv(t, src=peer)
                want = float(tag) + (0.5 if k.startswith("bwd") else 0.0)
                assert bool((t == want).all()), (rank, k, m, v, float(t[0]), want)
        q.put((rank, "ok"))
    except BaseException as e:  # report, do not hang the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split,tp,micro", [("3 stages, pass-through", 1, 3), ("2 stages", 2, 2),
                                            ("3 stages, pass-through", 2, 2)])
def test_programs_run_over_blocking_p2p(split, tp, micro):
    import socket

    import torch.multiprocessing as mp
    plan = _plan(split, tp)
    progs = _programs(plan, micro, tp)
    world = len(progs)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, progs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res
