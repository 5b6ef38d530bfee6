"""N>1 host path on CPU with torch.distributed (gloo, world_size 2): the
one-process-per-GPU launch applies the same schedule in every process, each
rank materialises only its own shards and lowers its own device plan. Checks
(1) shards of every TP-sharded parameter (incl. the blockwise FusedQKV layout
and the vocab-parallel embedding) reassemble the unsharded parameter,
(2) the per-rank plans are structurally identical (lockstep collectives), and
(3) the NCCL unique id made on rank 0 reaches every rank intact."""
import os
import socket
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2302_08005_b200 as sb
        from paper_2302_08005_b200 import recipes
        cfg = dict(layers=2, hidden=32, heads=4, vocab=32, batch=2, seq=8)
        m = sb.toy_bert(**cfg)
        s = sb.create_schedule(m, world)
        s.load_script(recipes.tp_script(2, world, ckpt_ratio=0.5))
        a = s.apply()
        errors = []
        # (1) shards reassemble the full parameters
        # (sharded path after the fusions moved children, path in the unfused model)
        names = [("encoder.layer.0.attention.qkv.weight",) * 2, ("encoder.layer.0.attention.qkv.bias",) * 2,
                 ("encoder.layer.1.attention.output.fused_bdrln_0.dense.weight",
                  "encoder.layer.1.attention.output.dense.weight"),
                 ("encoder.layer.0.ffn.fused_bias_gelu_0.dense1.weight", "encoder.layer.0.ffn.dense1.weight"),
                 ("encoder.layer.1.ffn.fused_brln_0.dense2.weight", "encoder.layer.1.ffn.dense2.weight"),
                 ("embeddings.weight",) * 2]
        full_m = sb.toy_bert(**cfg)
        fs = sb.create_schedule(full_m, 1)
        fs.load_script("".join(f"replace encoder.layer.{i}.attention.qkv with FusedQKV\n" for i in range(2)))
        full = fs.apply()
        H = cfg["hidden"]
        for name, full_name in names:
            mine = torch.tensor(a.param_values(name, rank))
            parts = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)
            want = full.param_values(full_name, 0)
            if "qkv" in name:  # blockwise: [q_r0 q_r1 | k_r0 k_r1 | v_r0 v_r1] along rows
                rows = 3 * H
                inner = want.size // rows
                blocks = [p.numpy().reshape(3, -1, inner) for p in parts]
                got = np.concatenate([np.concatenate([b[k] for b in blocks]) for k in range(3)]).ravel()
            elif "dense.weight" in name or "dense2" in name:  # axis 1
                got = np.concatenate([p.numpy().reshape(H, -1) for p in parts], axis=1).ravel()
            else:  # axis 0
                got = np.concatenate([p.numpy() for p in parts])
            if got.tobytes() != want.tobytes():
                errors.append(name)
        # (2) identical plan structure on every rank
        plan = sb.plan_summary(a, "train", 123, world, rank)
        sig = torch.tensor([zlib.crc32(plan["structure"].encode()), plan["ops"], plan["regions"]], dtype=torch.int64)
        sigs = [torch.zeros_like(sig) for _ in range(world)]
        dist.all_gather(sigs, sig)
        if any(not torch.equal(x, sigs[0]) for x in sigs):
            errors.append("plan structure differs across ranks")
        # (3) NCCL unique id broadcast (bytes only; no GPU needed)
        try:
            uid = torch.tensor(list(sb.nccl_unique_id() if rank == 0 else bytes(128)), dtype=torch.uint8)
            dist.broadcast(uid, 0)
            got_uid = bytes(uid.numpy().tobytes())
            ref_uid = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(ref_uid, uid)
            if any(bytes(x.numpy().tobytes()) != got_uid for x in ref_uid):
                errors.append("nccl unique id mismatch")
        except sb.SlapoError as e:  # NCCL library not loadable on this host
            if "NCCL" not in str(e):
                raise
        q.put((rank, errors))
    finally:
        dist.destroy_process_group()


def test_two_process_gloo_tp_host_path():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = [q.get(timeout=10) for _ in range(world)]
    for p in procs:
        assert p.exitcode == 0
    for rank, errors in results:
        assert not errors, (rank, errors)
