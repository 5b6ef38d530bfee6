"""Oracle runner — TEST INFRASTRUCTURE ONLY (never imported by the product).

Runs the reference executor compiled from /root/reference/proj by
oracle/Makefile (`oracle/_ref/slapo_ref_driver`, a static binary that also
travels to the GPU box) and reads back its dumps (format in ref_driver.cpp).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use it.
"""
from __future__ import annotations

import json
import os
import shutil
import struct
import subprocess
import tempfile
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "_ref", "slapo_ref_driver")
# the documented causal extension (oracle/causal_ext.py): the reference executor with a
# `causal` attr on softmax; identical to DRIVER on models without that attr
DRIVER_CAUSAL = os.path.join(HERE, "_ref", "slapo_ref_driver_causal")


def available() -> bool:
    return os.path.exists(DRIVER)


def read_dump(path: str) -> Dict[str, np.ndarray]:
    out: Dict[str, np.ndarray] = {}
    with open(path, "rb") as f:
        data = f.read()
    assert data[:4] == b"SBT1", path
    off = 4
    (n,) = struct.unpack_from("<I", data, off)
    off += 4
    for _ in range(n):
        (ln,) = struct.unpack_from("<I", data, off)
        off += 4
        name = data[off:off + ln].decode()
        off += ln
        (rank,) = struct.unpack_from("<I", data, off)
        off += 4
        dims = struct.unpack_from("<%dq" % rank, data, off)
        off += 8 * rank
        cnt = int(np.prod(dims)) if rank else 1
        arr = np.frombuffer(data, dtype="<f8", count=cnt, offset=off).copy()
        off += 8 * cnt
        out[name] = arr.reshape(dims)
    return out


def write_dump(path: str, tensors) -> None:
    """SBT1 (ref_driver.cpp write_dump): [(name, array)], f64."""
    with open(path, "wb") as f:
        f.write(b"SBT1" + struct.pack("<I", len(tensors)))
        for name, a in tensors:
            a = np.ascontiguousarray(np.asarray(a, dtype="<f8"))
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)) + nb + struct.pack("<I", a.ndim) + struct.pack("<%dq" % a.ndim, *a.shape))
            f.write(a.tobytes())


class RefRun:
    """Dumps of one oracle run. A temporary dump directory (no `outdir` given to
    `run`) is owned by this object and removed with it (`close()` / GC / `with`):
    full-width runs dump hundreds of MB (the embedding gradient alone is 250 MB at
    BERT-large width), so nothing may accumulate under /tmp."""

    def __init__(self, outdir: str, meta: dict, owned: bool = False):
        self.dir = outdir
        self.meta = meta
        self._owned = owned

    def close(self):
        if self._owned and self.dir and os.path.isdir(self.dir):
            shutil.rmtree(self.dir, ignore_errors=True)
        self._owned = False

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def outputs(self, rank: int = 0):
        d = read_dump(os.path.join(self.dir, "outputs.bin"))
        return [d[k] for k in sorted(d) if k.startswith(f"r{rank}:out")]

    def grads(self, rank: int = 0) -> Dict[str, np.ndarray]:
        d = read_dump(os.path.join(self.dir, "grads.bin"))
        p = f"r{rank}:"
        return {k[len(p):]: v for k, v in d.items() if k.startswith(p) and not k[len(p):].startswith("@input")}

    def input_grads(self, rank: int = 0):
        d = read_dump(os.path.join(self.dir, "grads.bin"))
        p = f"r{rank}:@input"
        return [d[k] for k in sorted(d) if k.startswith(p)]

    def params(self, rank: int = 0) -> Dict[str, np.ndarray]:
        d = read_dump(os.path.join(self.dir, "params.bin"))
        p = f"r{rank}:"
        return {k[len(p):]: v for k, v in d.items() if k.startswith(p)}

    def inputs(self):
        d = read_dump(os.path.join(self.dir, "inputs.bin"))
        return [d[k] for k in sorted(d)]

    def model_json(self) -> str:
        with open(os.path.join(self.dir, "model.json")) as f:
            return f.read()


def run(model: str = "toy_bert", schedule: Optional[str] = None, outdir: Optional[str] = None, timeout: int = 600,
        causal: bool = False, inputs=None, **kw) -> RefRun:
    """kw: layers, hidden, heads, vocab, batch, seq, p, dtype, world, mode, seed, input_seed,
    backward, dump_params, tp_hidden, tp_inner, tp_batch, repeat, model_json (path).
    causal=True runs the causal extension's driver (needed for decoder models);
    inputs: explicit model inputs (arrays in declared order) instead of random_tensor ones."""
    drv = DRIVER_CAUSAL if causal else DRIVER
    if not os.path.exists(drv):
        raise RuntimeError(f"oracle driver missing: build it with `make -C oracle` ({drv})")
    owned = outdir is None
    outdir = outdir or tempfile.mkdtemp(prefix="sbref_")
    args = [drv, "--model", model, "--out", outdir]
    sched_file = None
    if schedule:
        if os.path.exists(schedule):
            sched_file = schedule
        else:
            sched_file = os.path.join(outdir, "schedule.sch")
            with open(sched_file, "w") as f:
                f.write(schedule)
        args += ["--schedule", sched_file]
    for k, v in kw.items():
        args += ["--" + k, str(v)]
    if inputs is not None:
        ipath = os.path.join(outdir, "given_inputs.bin")
        write_dump(ipath, [(f"input{i}", a) for i, a in enumerate(inputs)])
        args += ["--inputs", ipath]
    try:
        r = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
        if r.returncode != 0:
            raise RuntimeError(f"oracle failed ({r.returncode}): {r.stderr.strip()}")
        meta = json.loads(r.stdout.strip().splitlines()[-1])
    except BaseException:
        if owned:
            shutil.rmtree(outdir, ignore_errors=True)
        raise
    return RefRun(outdir, meta, owned)


def time_step(model: str = "toy_bert", schedule: Optional[str] = None, timeout: int = 3600, cpu: Optional[int] = None,
              **kw) -> dict:
    """One forward()+backward_all_ranks() of the reference executor WITHOUT any dump
    (no --out: the driver writes nothing, ref_driver.cpp:289), optionally pinned to
    host core `cpu` (the reference is single-threaded). Returns the driver's meta
    line (fwd_s, bwd_s, collectives, ledger)."""
    if not available():
        raise RuntimeError(f"oracle driver missing: build it with `make -C oracle` ({DRIVER})")
    args = [DRIVER, "--model", model]
    if schedule:
        if not os.path.exists(schedule):
            raise ValueError("time_step takes a schedule file path")
        args += ["--schedule", schedule]
    for k, v in kw.items():
        args += ["--" + k, str(v)]
    if cpu is not None and shutil.which("taskset"):
        args = ["taskset", "-c", str(cpu)] + args
    r = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"oracle failed ({r.returncode}): {r.stderr.strip()}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def uniform01_probe(stream_seed: int, n: int) -> np.ndarray:
    with tempfile.TemporaryDirectory(prefix="sbrng_") as outdir:
        r = subprocess.run([DRIVER, "--probe_rng", f"{stream_seed},{n}", "--out", outdir], capture_output=True,
                           text=True)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
        return read_dump(os.path.join(outdir, "rng.bin"))["uniform01"]
