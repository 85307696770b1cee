"""ACSENV1 — the binary environment format of oracle/ref_tool (eval mode).

TEST INFRASTRUCTURE ONLY.  Mirrors satcc's Environment
(proj/include/satcc/interp.hpp:51-54): name-ordered scalars and arrays; ints
are int64 (Scalar::i is long long), doubles binary64.

    "ACSENV1\\0"
    u32 n_scalars; n x { u32 len, name, u8 type (0 int / 1 double), 8-byte value }
    u32 n_arrays;  n x { u32 len, name, u8 type, u32 ndim, i64 dims[ndim],
                         prod(dims) x 8-byte values }
"""
from __future__ import annotations

import struct
from typing import Dict, Tuple

import numpy as np

MAGIC = b"ACSENV1\0"


def write_env(path: str, scalars: Dict[str, Tuple[str, float]], arrays: Dict[str, np.ndarray]) -> None:
    """scalars: name -> ('int'|'double', value); arrays: int or float ndarrays."""
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(scalars)))
        for name in sorted(scalars):
            ty, v = scalars[name]
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)) + nb)
            if ty == "int":
                f.write(struct.pack("<Bq", 0, int(v)))
            else:
                f.write(struct.pack("<Bd", 1, float(v)))
        f.write(struct.pack("<I", len(arrays)))
        for name in sorted(arrays):
            a = arrays[name]
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)) + nb)
            is_int = np.issubdtype(a.dtype, np.integer)
            f.write(struct.pack("<BI", 0 if is_int else 1, a.ndim))
            f.write(struct.pack(f"<{a.ndim}q", *a.shape))
            f.write(np.ascontiguousarray(a, dtype=np.int64 if is_int else np.float64).tobytes())


def read_env(path: str):
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:8] == MAGIC, "bad ACSENV1 magic"
    off = 8
    scalars, arrays = {}, {}

    def take(fmt):
        nonlocal off
        v = struct.unpack_from(fmt, buf, off)
        off += struct.calcsize(fmt)
        return v

    (ns,) = take("<I")
    for _ in range(ns):
        (ln,) = take("<I")
        name = buf[off:off + ln].decode()
        off += ln
        (ty,) = take("<B")
        scalars[name] = ("int", take("<q")[0]) if ty == 0 else ("double", take("<d")[0])
    (na,) = take("<I")
    for _ in range(na):
        (ln,) = take("<I")
        name = buf[off:off + ln].decode()
        off += ln
        ty, nd = take("<BI")
        dims = take(f"<{nd}q")
        n = int(np.prod(dims))
        dt = np.int64 if ty == 0 else np.float64
        arrays[name] = np.frombuffer(buf, dtype=dt, count=n, offset=off).reshape(dims).copy()
        off += 8 * n
    return scalars, arrays
