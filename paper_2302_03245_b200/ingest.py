"""Edge-list ingest (graph.py:180-259 ``load_edge_list``) on the device.

The text is parsed and remapped by ``pr_graph_load_edge_list``
(``csrc/ingest.cu``): one thread per line, then a dense remap of the ids in
order of first appearance over the interleaved (src, dst) sequence, then the
device ``from_edges``.  When the device parser meets a line outside the plain
"src dst" grammar it returns PR_ERR_FORMAT; the text is then read on the host
the way the reference reads it -- the same pandas call, and on failure a
line-by-line pass that reports the offending line (graph.py:180-198,
220-236) -- and the parsed ids go through the same device remap
(``pr_graph_from_raw_ids``).  Valid input therefore never leaves the device
path, and malformed input raises the reference's ``GraphFormatError``
messages.
"""

from __future__ import annotations

import ctypes
import io
import os

import numpy as np

from . import _lib
from .graph import DeviceGraph, Graph


class GraphFormatError(ValueError):
    """Raised when an edge-list stream cannot be parsed into a graph (graph.py:17-18)."""


def _read_source(source) -> tuple[bytes, str]:
    # graph.py:211-219: a path, bytes, or a binary/text stream
    if isinstance(source, (str, os.PathLike)):
        name = os.path.splitext(os.path.basename(os.fspath(source)))[0]
        with open(source, "rb") as fh:
            return fh.read(), name
    data = source.read() if hasattr(source, "read") else source
    if isinstance(data, str):
        data = data.encode()
    return bytes(data), "graph"


def _line_parse(text: str) -> tuple[np.ndarray, np.ndarray]:
    """Line-by-line reading that names the first bad line (graph.py:180-198)."""
    src, dst = [], []
    for lineno, line in enumerate(text.splitlines(), start=1):
        body = line.strip()
        if not body or body.startswith("#"):
            continue
        fields = body.split()
        if len(fields) != 2:
            raise GraphFormatError(f"line {lineno}: expected 'src dst', got {body!r}")
        try:
            a, b = int(fields[0]), int(fields[1])
        except ValueError:
            raise GraphFormatError(f"line {lineno}: non-integer vertex id in {body!r}") from None
        if a < 0 or b < 0:
            raise GraphFormatError(f"line {lineno}: negative vertex id in {body!r}")
        src.append(a)
        dst.append(b)
    return np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64)


def _host_parse(data: bytes) -> tuple[np.ndarray, np.ndarray]:
    """The reference's reading of a stream (graph.py:220-236): pandas' C
    tokenizer on whitespace-separated int64 columns with '#' comments, and on
    any failure the line-by-line pass for the error position."""
    text = data.decode("utf-8", errors="replace")
    try:
        import pandas as pd

        frame = pd.read_csv(io.StringIO(text), sep=r"\s+", comment="#", header=None, dtype=np.int64,
                            engine="c")
        if frame.shape[1] != 2:
            raise GraphFormatError("expected two columns")
        src = frame[0].to_numpy(dtype=np.int64)
        dst = frame[1].to_numpy(dtype=np.int64)
        if src.size and (src.min() < 0 or dst.min() < 0):
            raise GraphFormatError("negative vertex id")
    except Exception:
        src, dst = _line_parse(text)
    return src, dst


def load_edge_list(source, name: str | None = None) -> Graph:
    """Load a whitespace-separated "src dst" edge list (graph.py:201-259).

    Ids may be arbitrary non-negative integers; they are remapped to [0, n) in
    order of first appearance (interleaved source/target order) and kept as
    ``original_ids``.  Duplicate edges are dropped, self-loops kept; a stream
    with no edges raises ``GraphFormatError``.
    """
    data, inferred = _read_source(source)
    ctx = _lib.context()
    L = _lib.load()
    h = ctypes.c_void_p()
    raw_dev = ctypes.c_int64(0)
    rc = L.pr_graph_load_edge_list(ctx.handle, data, len(data), ctypes.byref(h), ctypes.byref(raw_dev))
    raw = int(raw_dev.value)
    if rc == _lib.PR_ERR_FORMAT:
        src, dst = _host_parse(data)
        if src.size == 0:
            raise GraphFormatError("empty graph: no edges found")
        src = np.ascontiguousarray(src, np.int64)
        dst = np.ascontiguousarray(dst, np.int64)
        rc = L.pr_graph_from_raw_ids(ctx.handle, _lib.ptr(src), _lib.ptr(dst), int(src.size), ctypes.byref(h))
        raw = int(src.size)
    _lib.check(rc, "load_edge_list")
    dev = DeviceGraph(h, ctx)
    g = Graph(dev, raw, name=name or inferred)
    g._orig_on_device = True
    return g
