"""On-disk formats of the ranking output (serialize.py:14-38 in the reference).

``write_ranking_csv`` orders the vertices on the device (``pr_rank_order``:
score descending, ties by original id) and writes the rows natively with the
reference's exact bytes (``csv.writer`` line ends, scores as Python
``repr(float)``).  The binary vector format is a little-endian int64 length
followed by float64 values.
"""

from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from . import _lib


def _ids(g, n: int):
    ids = getattr(g, "original_ids", None)
    if ids is None:
        return None
    ids = np.ascontiguousarray(ids, np.int64)
    if ids.shape != (n,):
        raise ValueError("original_ids must have one entry per vertex")
    return ids


def ranking_order(values, g=None, k: int | None = None) -> np.ndarray:
    """Indices of ``values`` by score descending, ties by original id
    ascending (serialize.py:16), the first ``k`` of them (all by default)."""
    v = np.ascontiguousarray(values, np.float64)
    n = int(v.size)
    k = n if k is None else max(0, min(int(k), n))
    ids = _ids(g, n) if g is not None else None
    out = np.empty(max(k, 1), np.int64)
    ctx = _lib.context()
    _lib.check(_lib.load().pr_rank_order(ctx.handle, _lib.ptr(v), _lib.ptr(ids), n, k, _lib.ptr(out)),
               "rank_order")
    return out[:k]


def write_ranking_csv(vec, g, path) -> None:
    """Scores sorted descending, ties broken by original id ascending (serialize.py:14-21)."""
    v = np.ascontiguousarray(vec.values, np.float64)
    ids = _ids(g, int(v.size))
    ctx = _lib.context()
    _lib.check(_lib.load().pr_write_ranking_csv(ctx.handle, _lib.ptr(v), _lib.ptr(ids), int(v.size),
                                                 os.fsencode(os.fspath(path))), "write_ranking_csv")


def format_score(value: float) -> str:
    """The CSV score text: Python repr(float), produced by the library."""
    buf = ctypes.create_string_buffer(40)
    n = _lib.load().pr_format_score(float(value), buf)
    return buf.raw[:n].decode()


def write_vector_binary(vec, path) -> None:
    """Little-endian int64 length followed by the float64 values (serialize.py:24-29)."""
    values = np.asarray(vec.values, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<q", values.size))
        fh.write(values.tobytes())


def read_vector_binary(path) -> np.ndarray:
    """serialize.py:32-38 (raises ValueError on a truncated file)."""
    with open(path, "rb") as fh:
        (n,) = struct.unpack("<q", fh.read(8))
        data = np.frombuffer(fh.read(8 * n), dtype="<f8")
    if data.size != n:
        raise ValueError(f"truncated vector file: expected {n} values, got {data.size}")
    return data.astype(np.float64)
