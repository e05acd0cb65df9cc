"""Device-resident graph core (CSR + CSC on the B200).

Mirrors the reference's graph API (``graph.py:21-110, 133-177, 274-378``):
``Graph``, ``VertexClassification``, ``IFP2Graph``, ``from_edges``,
``classify``, ``dangling_target_counts``, ``preprocess_ifp2``.  The arrays
live in HBM (int32 column indices, int64 offsets) and are built there by
the K1-K3 kernels; the reference-layout numpy views (int64) are exported
lazily on first attribute access, so reference-style tests and harness code
keep working.  Any object with the reference Graph's array attributes can
be passed where a ``Graph`` is expected; it is uploaded once and cached.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib


class DeviceGraph:
    """Owner of one ``pr_graph`` handle."""

    def __init__(self, handle, ctx: _lib.Context):
        self.handle = handle
        self.ctx = ctx
        n, m = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().pr_graph_info(handle, ctypes.byref(n), ctypes.byref(m)))
        self.n, self.m = int(n.value), int(m.value)
        self._counts = None
        self._ifp2 = None
        self._pending_out_targets = None   # host out_targets not yet on the device
        self.h2d_bytes = 0                 # bytes copied host -> device so far

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().pr_graph_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- constructors
    @classmethod
    def from_edges(cls, n: int, src: np.ndarray, dst: np.ndarray, ctx=None) -> "DeviceGraph":
        ctx = ctx or _lib.context()
        h = ctypes.c_void_p()
        _lib.check(_lib.load().pr_graph_from_edges(ctx.handle, int(n), _lib.ptr(src), _lib.ptr(dst),
                                                   int(src.size), ctypes.byref(h)), "from_edges")
        return cls(h, ctx)

    @classmethod
    def upload(cls, g, ctx=None, lazy_out_targets: bool = True) -> "DeviceGraph":
        """Upload a reference-layout graph.  With ``lazy_out_targets`` only the
        in-adjacency and ``out_offsets`` are copied: the fast engines rebuild
        the out-adjacency of their own vertex layout on the device, and
        ``out_targets`` follows on the first call that needs the original one
        (classify, IFP2 exports, exact mode, export)."""
        ctx = ctx or _lib.context()
        arrs = {k: np.ascontiguousarray(getattr(g, k), dtype=np.int64)
                for k in ("out_offsets", "out_targets", "in_offsets", "in_sources")}
        lazy = lazy_out_targets and int(g.m) > 0
        h = ctypes.c_void_p()
        _lib.check(_lib.load().pr_graph_upload(ctx.handle, int(g.n), int(g.m), _lib.ptr(arrs["out_offsets"]),
                                               None if lazy else _lib.ptr(arrs["out_targets"]),
                                               _lib.ptr(arrs["in_offsets"]), _lib.ptr(arrs["in_sources"]),
                                               ctypes.byref(h)), "upload")
        dev = cls(h, ctx)
        dev.h2d_bytes = dev._copied_bytes()
        if lazy:
            dev._pending_out_targets = arrs["out_targets"]
        return dev

    def need_out_targets(self) -> None:
        """Copy the original out_targets to the device if the upload deferred them."""
        a = self._pending_out_targets
        if a is not None:
            _lib.check(_lib.load().pr_graph_attach_out_targets(self.handle, _lib.ptr(a)), "attach_out_targets")
            self.h2d_bytes = self._copied_bytes()
            self._pending_out_targets = None

    def _copied_bytes(self) -> int:
        """Bytes the library copied host -> device for this graph (the int64
        index arrays partly travel narrowed to int32, hostio.cu)."""
        b = ctypes.c_int64()
        _lib.check(_lib.load().pr_graph_h2d_bytes(self.handle, ctypes.byref(b)), "h2d_bytes")
        return int(b.value)

    @classmethod
    def rmat(cls, scale: int, edge_factor: int, a=0.57, b=0.19, c=0.19, seed: int = 0, ctx=None):
        ctx = ctx or _lib.context()
        h = ctypes.c_void_p()
        _lib.check(_lib.load().pr_graph_rmat(ctx.handle, int(scale), int(edge_factor), a, b, c, int(seed),
                                             ctypes.byref(h)), "rmat")
        return cls(h, ctx)

    # -- exports
    def export(self) -> dict:
        self.need_out_targets()
        n, m = self.n, self.m
        out = {"out_offsets": np.zeros(n + 1, np.int64), "out_targets": np.zeros(max(m, 1), np.int64),
               "in_offsets": np.zeros(n + 1, np.int64), "in_sources": np.zeros(max(m, 1), np.int64)}
        _lib.check(_lib.load().pr_graph_export(self.handle, *[_lib.ptr(out[k]) for k in
                                                              ("out_offsets", "out_targets", "in_offsets",
                                                               "in_sources")]), "export")
        out["out_targets"] = out["out_targets"][:m]
        out["in_sources"] = out["in_sources"][:m]
        return out

    def classify(self) -> _lib.ClassCounts:
        if self._counts is None:
            self.need_out_targets()
            c = _lib.ClassCounts()
            _lib.check(_lib.load().pr_classify(self.handle, ctypes.byref(c)), "classify")
            self._counts = c
        return self._counts

    def classify_export(self) -> dict:
        c = self.classify()
        out = {k: np.zeros(max(getattr(c, k), 1), np.int64)
               for k in ("dangling", "unreferenced", "weak_dangling", "weak_unreferenced")}
        _lib.check(_lib.load().pr_classify_export(self.handle, *[_lib.ptr(out[k]) for k in
                                                                 ("dangling", "unreferenced", "weak_dangling",
                                                                  "weak_unreferenced")]), "classify_export")
        return {k: v[:getattr(c, k)] for k, v in out.items()}

    def dangling_target_counts(self) -> np.ndarray:
        out = np.zeros(self.n, np.int64)
        _lib.check(_lib.load().pr_dangling_target_counts(self.handle, _lib.ptr(out)), "dtc")
        return out

    def preprocess_ifp2(self) -> _lib.Ifp2Counts:
        if self._ifp2 is None:
            c = _lib.Ifp2Counts()
            _lib.check(_lib.load().pr_preprocess_ifp2(self.handle, ctypes.byref(c)), "preprocess_ifp2")
            self._ifp2 = c
        return self._ifp2

    def ifp2_export(self) -> dict:
        self.need_out_targets()
        c = self.preprocess_ifp2()
        n = self.n
        out = {"live_offsets": np.zeros(n + 1, np.int64), "live_targets": np.zeros(max(c.live_edges, 1), np.int64),
               "live_degree": np.zeros(n, np.int64), "dangling_ids": np.zeros(max(c.dangling, 1), np.int64),
               "source_offsets": np.zeros(c.dangling + 1, np.int64),
               "source_ids": np.zeros(max(c.source_edges, 1), np.int64)}
        keys = ("live_offsets", "live_targets", "live_degree", "dangling_ids", "source_offsets", "source_ids")
        _lib.check(_lib.load().pr_ifp2_export(self.handle, *[_lib.ptr(out[k]) for k in keys]), "ifp2_export")
        out["live_targets"] = out["live_targets"][:c.live_edges]
        out["dangling_ids"] = out["dangling_ids"][:c.dangling]
        out["source_ids"] = out["source_ids"][:c.source_edges]
        return out

    # -- engines
    def run(self, algorithm: str, mode: str, damping: float, threshold: float, max_rounds: int,
            converged_scope: int, push_switch: float = 0.0, host_loop: bool = False, want_state: bool = False,
            on_round=None, row_cap: int = 1 << 16, values_out: np.ndarray | None = None):
        """One solve through pr_run; returns (values, rows, result, reserved, pending)."""
        n = self.n
        if mode == "exact":
            self.need_out_targets()
        # PUSHRANK_HOST_LOOP=1 launches the same kernels round by round from
        # the host (ncu cannot profile kernel nodes of conditional graphs)
        host_loop = host_loop or os.environ.get("PUSHRANK_HOST_LOOP", "0") == "1"
        params = _lib.RunParams(algorithm=_lib.ALGO[algorithm], mode=_lib.MODE[mode], damping=float(damping),
                                threshold=float(threshold), max_rounds=int(max_rounds),
                                push_switch=float(push_switch), converged_scope=int(converged_scope),
                                host_loop=int(bool(host_loop)))
        cb = None
        if on_round is not None:
            def _cb(_user, t, r_ptr, h_ptr):
                r = np.ctypeslib.as_array(r_ptr, shape=(n,))
                h = np.ctypeslib.as_array(h_ptr, shape=(n,))
                r.flags.writeable = False
                h.flags.writeable = False
                on_round(int(t), r, h)
            cb = _lib.ROUND_CB(_cb)
            params.on_round = cb
        # page-locked output: the D2H copy runs at link speed (a pageable
        # destination goes through driver staging at ~5 GB/s)
        if values_out is not None:
            values = values_out
        elif os.environ.get("PUSHRANK_PINNED_OUT", "1") != "0":
            values = _lib.pinned_empty(n)
        else:
            values = np.empty(n, np.float64)
        reserved = np.empty(n, np.float64) if want_state else None
        pending = np.empty(n, np.float64) if want_state else None
        rows = np.zeros(row_cap, _lib.ROUND_DTYPE)
        res = _lib.RunResult()
        rc = _lib.load().pr_run(self.handle, ctypes.byref(params), _lib.ptr(values), _lib.ptr(reserved),
                                _lib.ptr(pending), _lib.ptr(rows), int(row_cap), ctypes.byref(res))
        _lib.check(rc, "run")
        return values, rows[: min(res.rows, row_cap)].copy(), res, reserved, pending

    def power(self, damping: float, iterations: int, tolerance: float, threshold: float,
              personalization=None, on_iterate=None):
        n = self.n
        pi = np.empty(n, np.float64)
        cap = max(int(iterations), 1)
        deltas = np.zeros(cap, np.float64)
        conv = np.zeros(cap, np.int64)
        p = None if personalization is None else np.ascontiguousarray(personalization, np.float64)
        res = _lib.RunResult()
        L = _lib.load()
        if on_iterate is None:
            rc = L.pr_power(self.handle, float(damping), int(iterations), float(tolerance), float(threshold),
                            _lib.ptr(p), _lib.ptr(pi), _lib.ptr(deltas), _lib.ptr(conv), ctypes.byref(res))
        else:
            def _cb(_user, k, pi_ptr):
                view = np.ctypeslib.as_array(pi_ptr, shape=(n,))
                view.flags.writeable = False
                return 1 if on_iterate(int(k), view) else 0
            cb = _lib.POWER_CB(_cb)
            rc = L.pr_power_observed(self.handle, float(damping), int(iterations), float(tolerance),
                                     float(threshold), _lib.ptr(p), _lib.ptr(pi), _lib.ptr(deltas),
                                     _lib.ptr(conv), cb, None, ctypes.byref(res))
        _lib.check(rc, "power")
        k = int(res.rounds)
        return pi, deltas[:k].copy(), conv[:k].copy(), res


class Graph:
    """Directed graph with out- and in-adjacency resident on the device.

    Same attributes as the reference ``Graph`` (graph.py:21-42); the int64
    numpy arrays are exported from the device on first access.
    ``out_degree`` is the original out-degree and stays the push-weight
    denominator for both engines.
    """

    def __init__(self, dev: DeviceGraph, raw_edge_count: int, name: str = "graph", original_ids=None):
        self.dev = dev
        self.n = dev.n
        self.m = dev.m
        self.raw_edge_count = int(raw_edge_count)
        self.name = name
        self._orig = None if original_ids is None else np.asarray(original_ids, np.int64)
        self._orig_on_device = False   # load_edge_list keeps the id table on the device
        self._arrays = None

    def _export(self) -> dict:
        if self._arrays is None:
            a = self.dev.export()
            a["out_degree"] = np.diff(a["out_offsets"])
            a["in_degree"] = np.diff(a["in_offsets"])
            self._arrays = a
        return self._arrays

    out_offsets = property(lambda self: self._export()["out_offsets"])
    out_targets = property(lambda self: self._export()["out_targets"])
    out_degree = property(lambda self: self._export()["out_degree"])
    in_offsets = property(lambda self: self._export()["in_offsets"])
    in_sources = property(lambda self: self._export()["in_sources"])
    in_degree = property(lambda self: self._export()["in_degree"])

    @property
    def original_ids(self) -> np.ndarray:
        if self._orig is None and self._orig_on_device:
            out = np.empty(self.n, np.int64)
            _lib.check(_lib.load().pr_graph_original_ids(self.dev.handle, _lib.ptr(out)), "original_ids")
            self._orig = out
        return self._orig if self._orig is not None else np.arange(self.n, dtype=np.int64)

    def out_neighbors(self, v: int) -> np.ndarray:
        return self.out_targets[self.out_offsets[v]: self.out_offsets[v + 1]]

    def in_neighbors(self, v: int) -> np.ndarray:
        return self.in_sources[self.in_offsets[v]: self.in_offsets[v + 1]]

    def edge_set(self) -> set[tuple[int, int]]:
        src = np.repeat(np.arange(self.n), np.diff(self.out_offsets))
        return set(zip(src.tolist(), self.out_targets.tolist()))

    def validate(self) -> None:
        if self.n < 1:
            raise ValueError("graph must have at least one vertex")
        off = self.out_offsets
        if off.shape[0] != self.n + 1 or off[-1] != self.m:
            raise ValueError("out_offsets inconsistent with n/m")
        if np.any(np.diff(off) < 0):
            raise ValueError("out_offsets must be non-decreasing")
        if self.m and (self.out_targets.min() < 0 or self.out_targets.max() >= self.n):
            raise ValueError("edge target out of range")


def device_graph(g) -> DeviceGraph:
    """The DeviceGraph behind ``g`` (uploading a reference-style graph once)."""
    if isinstance(g, Graph):
        return g.dev
    if isinstance(g, IFP2Graph):
        return device_graph(g.base)
    dev = getattr(g, "_pr_device_graph", None)
    if dev is None:
        dev = DeviceGraph.upload(g)
        try:
            setattr(g, "_pr_device_graph", dev)
        except AttributeError:
            pass
    return dev


@dataclass
class VertexClassification:
    """Structural vertex classes (graph.py:68-89); sorted int64 id arrays."""

    dangling: np.ndarray
    unreferenced: np.ndarray
    weak_dangling: np.ndarray
    weak_unreferenced: np.ndarray
    dangling_edge_count: int
    peel_rounds: int = 0

    def dangling_mask(self, n: int) -> np.ndarray:
        mask = np.zeros(n, dtype=bool)
        mask[self.dangling] = True
        return mask


@dataclass
class StatsRow:
    """Dataset summary row (graph.py:113-127): counts and dangling structure."""

    name: str
    n: int
    m: int
    dangling_vertices: int
    dangling_edges: int
    avg_degree: float
    raw_edge_count: int

    def as_csv_row(self) -> list:
        return [self.name, self.n, self.m, self.dangling_vertices, self.dangling_edges, f"{self.avg_degree:.6g}"]


def stats(g, cls: VertexClassification) -> StatsRow:
    """Summary counts of a graph and its classification (graph.py:321-331);
    the counts come from the device classification, no host arrays."""
    return StatsRow(name=g.name, n=int(g.n), m=int(g.m), dangling_vertices=int(len(cls.dangling)),
                    dangling_edges=int(cls.dangling_edge_count), avg_degree=g.m / g.n,
                    raw_edge_count=int(g.raw_edge_count))


class IFP2Graph:
    """Graph split for two-phase pushing (graph.py:92-110), on the device.

    ``live_*`` is the CSR restricted to non-dangling targets (row order kept),
    ``source_*`` the sources of each dangling vertex (ascending).
    """

    def __init__(self, base, counts: _lib.Ifp2Counts, dangling_edge_count: int):
        self.base = base
        self.dev = device_graph(base)
        self.live_edges = int(counts.live_edges)
        self.dangling_edge_count = int(dangling_edge_count)
        self._arrays = None

    def _export(self) -> dict:
        if self._arrays is None:
            self._arrays = self.dev.ifp2_export()
        return self._arrays

    live_offsets = property(lambda self: self._export()["live_offsets"])
    live_targets = property(lambda self: self._export()["live_targets"])
    live_degree = property(lambda self: self._export()["live_degree"])
    dangling_ids = property(lambda self: self._export()["dangling_ids"])
    source_offsets = property(lambda self: self._export()["source_offsets"])
    source_ids = property(lambda self: self._export()["source_ids"])


def from_edges(n: int, src, dst, name: str = "graph", original_ids=None, raw_edge_count: int | None = None) -> Graph:
    """K1 on the device: dedup (src, dst) pairs (self-loops kept), CSR sorted
    by (src, dst), CSC ascending source within a target (graph.py:133-177)."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    if src.shape != dst.shape:
        raise ValueError("source and target arrays must have equal length")
    if n < 1:
        raise ValueError("graph must have at least one vertex")
    raw = int(src.shape[0]) if raw_edge_count is None else int(raw_edge_count)
    if src.shape[0] and (src.min() < 0 or dst.min() < 0 or max(src.max(), dst.max()) >= n):
        raise ValueError("vertex id out of range")
    dev = DeviceGraph.from_edges(int(n), src, dst)
    return Graph(dev, raw, name=name, original_ids=original_ids)


def classify(g) -> VertexClassification:
    """K2 on the device: base dangling/unreferenced sets and the joint weak
    peel (graph.py:274-318), frontier-based with atomic counters."""
    dev = device_graph(g)
    c = dev.classify()
    arrays = dev.classify_export()
    return VertexClassification(dangling=arrays["dangling"], unreferenced=arrays["unreferenced"],
                                weak_dangling=arrays["weak_dangling"],
                                weak_unreferenced=arrays["weak_unreferenced"],
                                dangling_edge_count=int(c.dangling_edge_count), peel_rounds=int(c.peel_rounds))


def dangling_target_counts(g, cls: VertexClassification | None = None) -> np.ndarray:
    """Per-vertex count of out-edges into dangling vertices (graph.py:334-340)."""
    return device_graph(g).dangling_target_counts()


def preprocess_ifp2(g, cls: VertexClassification) -> IFP2Graph:
    """K3 on the device: live CSR + dangling-source CSR (graph.py:343-378)."""
    dev = device_graph(g)
    counts = dev.preprocess_ifp2()
    m_d = int(counts.source_edges) if cls is None else int(cls.dangling_edge_count)
    return IFP2Graph(g, counts, m_d)
