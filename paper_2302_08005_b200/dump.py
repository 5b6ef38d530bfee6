"""SLD1 tensor dumps and the CLI's tensor text form.

Restates the reference's dump format (proj/src/dump.cpp:29-70,
proj/include/slapo/dump.hpp:12-15): little-endian, magic 'SLD1' (u32
0x31444C53), u32 tensor count, then per tensor u32 rank, i64 dims[rank], u8
dtype tag (0 = f32, 1 = f64) and the raw values. ``format_tensor_text``
follows dump.cpp:72-88 (the text `slapo run` prints per output), with the
TensorSpec form of proj/src/tensor.cpp:15-24.
"""
from __future__ import annotations

import struct
from typing import List, Sequence, Tuple

import numpy as np

MAGIC = 0x31444C53  # 'SLD1'


def write_tensor_dump(path: str, tensors: Sequence[Tuple[np.ndarray, str]]) -> None:
    """tensors: (values, dtype) pairs, dtype 'f32' or 'f64' (the TensorSpec dtype)."""
    with open(path, "wb") as f:
        f.write(struct.pack("<II", MAGIC, len(tensors)))
        for a, dt in tensors:
            a = np.asarray(a)
            f.write(struct.pack("<I", a.ndim))
            f.write(struct.pack("<%dq" % a.ndim, *a.shape))
            if dt == "f32":
                f.write(b"\x00")
                f.write(np.ascontiguousarray(a, dtype="<f4").tobytes())
            elif dt == "f64":
                f.write(b"\x01")
                f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())
            else:
                raise ValueError(f"dtype must be 'f32' or 'f64', got {dt!r}")


def read_tensor_dump(path: str) -> List[Tuple[np.ndarray, str]]:
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 8 or struct.unpack_from("<I", data, 0)[0] != MAGIC:
        raise ValueError(f"'{path}' is not a slapo tensor dump (bad format header)")
    (count,) = struct.unpack_from("<I", data, 4)
    off, out = 8, []
    for _ in range(count):
        (rank,) = struct.unpack_from("<I", data, off)
        off += 4
        dims = list(struct.unpack_from("<%dq" % rank, data, off))
        off += 8 * rank
        tag = data[off]
        off += 1
        n = int(np.prod(dims)) if dims else 1
        dt, np_dt, sz = ("f32", "<f4", 4) if tag == 0 else ("f64", "<f8", 8)
        if off + n * sz > len(data):
            raise ValueError(f"truncated tensor dump '{path}'")
        a = np.frombuffer(data, dtype=np_dt, count=n, offset=off).reshape(dims).astype(np.float64)
        off += n * sz
        out.append((a, dt))
    return out


def spec_text(shape: Sequence[int], dtype: str) -> str:
    return "(" + ",".join(str(int(d)) for d in shape) + "):" + dtype


def format_tensor_text(a: np.ndarray, dtype: str) -> str:
    a = np.asarray(a, dtype=np.float64)
    flat = a.reshape(-1)
    parts = []
    for i, v in enumerate(flat):
        if i == 16 and flat.size > 20:
            parts.append(f"... {flat.size - i} more")
            break
        parts.append("%.17g" % float(v))
    return "tensor " + spec_text(a.shape, dtype) + " [" + ", ".join(parts) + "]"
