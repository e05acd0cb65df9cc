"""CPU oracle for the pushrank IFP1/IFP2 hot path.

TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured or
shipped.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package; the
product package ``paper_2302_03245_b200`` never does and has no CPU path.

Two layers:
  * ``oracle.c`` (loaded here via ctypes from ``oracle/_build``): a plain-C
    restatement of the reference functions, each citing the reference
    file:line it follows (``/root/reference/pkg/src/pushrank/...``).
  * ``oracle/_ref`` (see ``refdriver.py``): the reference's *own* push kernel
    (``_kernels.pyx``) compiled from the reference tree by ``make ref``.

Parity pinning: tests/test_oracle_golden.py checks this oracle against the
golden vectors in tests/golden/, which tests/golden/make_golden.py produced
by importing and running the real reference package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

ROW_DTYPE = np.dtype([
    ("h_l1", "<f8"), ("alpha", "<f8"), ("active_mass", "<f8"), ("carry_mass", "<f8"),
    ("converged", "<i8"), ("work", "<i8"), ("push_ops", "<i8"), ("push_ops_dangling", "<i8"),
    ("digest", "<u8"),
])

_lib = None
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_rowp = np.ctypeslib.ndpointer(dtype=ROW_DTYPE, flags="C_CONTIGUOUS")
_I = ctypes.c_int64
_D = ctypes.c_double


def build() -> str:
    """Compile oracle.c (``make -C oracle``); returns the library path."""
    subprocess.run(["make", "-s", "-C", HERE, "_build/liboracle.so"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_from_edges.restype = _I
        L.orc_from_edges.argtypes = [_I, _i64p, _i64p, _I, _i64p, _i64p, _i64p, _i64p]
        L.orc_classify.restype = _I
        L.orc_classify.argtypes = [_I, _i64p, _i64p, _i64p, _i64p, _u8p, ctypes.POINTER(_I)]
        L.orc_dangling_target_counts.restype = None
        L.orc_dangling_target_counts.argtypes = [_I, _i64p, _i64p, _u8p, _i64p]
        L.orc_preprocess_ifp2.restype = _I
        L.orc_preprocess_ifp2.argtypes = [_I, _i64p, _i64p, _i64p, _i64p, _u8p,
                                          _i64p, _i64p, _i64p, _i64p, _i64p, _i64p]
        L.orc_sync_rounds.restype = _I
        L.orc_sync_rounds.argtypes = [ctypes.c_int, _I, _i64p, _i64p, _i64p, ctypes.c_void_p,
                                      _D, _D, _I, _f64p, _f64p, _rowp, _I, ctypes.POINTER(_I)]
        L.orc_sync_rounds_pull.restype = _I
        L.orc_sync_rounds_pull.argtypes = [ctypes.c_int, _I, _i64p, _i64p, _i64p, _i64p, ctypes.c_void_p,
                                           _D, _D, _I, ctypes.c_int, _f64p, _f64p, _rowp, _I,
                                           ctypes.POINTER(_I)]
        L.orc_rmat.restype = _I
        L.orc_rmat.argtypes = [ctypes.c_int, _I, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_settle.restype = _I
        L.orc_settle.argtypes = [_I, _i64p, _i64p, _i64p, _i64p, _D, _f64p, _f64p]
        L.orc_power.restype = _I
        L.orc_power.argtypes = [_I, _i64p, _i64p, _i64p, _D, _f64p, _I, _D, _f64p, _f64p, ctypes.c_int]
        L.orc_async_phase.restype = ctypes.c_int
        L.orc_async_phase.argtypes = [_I, _f64p, _f64p, _i64p, _i64p, _i64p, _i64p, _i64p,
                                      ctypes.c_int, _i64p, _I, ctypes.c_void_p, _D, _D,
                                      ctypes.POINTER(_I), ctypes.POINTER(_I)]
        _lib = L
    return _lib


# ---------------------------------------------------------------- graph core

def from_edges(n: int, src, dst) -> SimpleNamespace:
    """Restates graph.py:133-177 (dedup via sort, CSR, stable CSC)."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    if src.shape != dst.shape:
        raise ValueError("source and target arrays must have equal length")
    if n < 1:
        raise ValueError("graph must have at least one vertex")
    if src.size and (src.min() < 0 or dst.min() < 0 or max(src.max(), dst.max()) >= n):
        raise ValueError("vertex id out of range")
    m_raw = int(src.size)
    out_off = np.zeros(n + 1, np.int64)
    in_off = np.zeros(n + 1, np.int64)
    out_tgt = np.zeros(max(m_raw, 1), np.int64)
    in_src = np.zeros(max(m_raw, 1), np.int64)
    m = lib().orc_from_edges(n, src, dst, m_raw, out_off, out_tgt, in_off, in_src)
    return SimpleNamespace(
        n=n, m=int(m), out_offsets=out_off, out_targets=out_tgt[:m].copy(),
        out_degree=np.diff(out_off), in_offsets=in_off, in_sources=in_src[:m].copy(),
        in_degree=np.diff(in_off), raw_edge_count=m_raw)


def graph_arrays(g) -> SimpleNamespace:
    """Accept any object with the reference Graph's array attributes."""
    return SimpleNamespace(
        n=int(g.n), m=int(g.m),
        out_offsets=np.ascontiguousarray(g.out_offsets, np.int64),
        out_targets=np.ascontiguousarray(g.out_targets, np.int64),
        out_degree=np.ascontiguousarray(g.out_degree, np.int64),
        in_offsets=np.ascontiguousarray(g.in_offsets, np.int64),
        in_sources=np.ascontiguousarray(g.in_sources, np.int64),
        in_degree=np.ascontiguousarray(g.in_degree, np.int64))


def classify(g) -> SimpleNamespace:
    """Restates graph.py:274-318 (joint dangling/unreferenced peel)."""
    g = graph_arrays(g)
    flags = np.zeros(g.n, np.uint8)
    rounds = _I(0)
    m_d = lib().orc_classify(g.n, g.out_offsets, g.out_targets, g.in_offsets, g.in_sources,
                             flags, ctypes.byref(rounds))
    return SimpleNamespace(
        dangling=np.flatnonzero(flags & 1), unreferenced=np.flatnonzero(flags & 2),
        weak_dangling=np.flatnonzero(flags & 4), weak_unreferenced=np.flatnonzero(flags & 8),
        dangling_edge_count=int(m_d), peel_rounds=int(rounds.value))


def dangling_mask(n: int, dangling_ids) -> np.ndarray:
    mask = np.zeros(n, np.uint8)
    mask[np.asarray(dangling_ids, np.int64)] = 1
    return mask


def dangling_target_counts(g, dangling_ids) -> np.ndarray:
    """Restates graph.py:334-340."""
    g = graph_arrays(g)
    out = np.zeros(g.n, np.int64)
    lib().orc_dangling_target_counts(g.n, g.out_offsets, g.out_targets,
                                     dangling_mask(g.n, dangling_ids), out)
    return out


def preprocess_ifp2(g, dangling_ids) -> SimpleNamespace:
    """Restates graph.py:343-378 (live CSR + dangling-source CSR)."""
    g = graph_arrays(g)
    mask = dangling_mask(g.n, dangling_ids)
    n_d = int(mask.sum())
    live_off = np.zeros(g.n + 1, np.int64)
    live_tgt = np.zeros(max(g.m, 1), np.int64)
    live_deg = np.zeros(g.n, np.int64)
    d_ids = np.zeros(max(n_d, 1), np.int64)
    s_off = np.zeros(n_d + 1, np.int64)
    s_ids = np.zeros(max(g.m, 1), np.int64)
    live_m = lib().orc_preprocess_ifp2(g.n, g.out_offsets, g.out_targets, g.in_offsets,
                                       g.in_sources, mask, live_off, live_tgt, live_deg,
                                       d_ids, s_off, s_ids)
    return SimpleNamespace(
        live_offsets=live_off, live_targets=live_tgt[:live_m].copy(), live_degree=live_deg,
        dangling_ids=d_ids[:n_d].copy(), source_offsets=s_off,
        source_ids=s_ids[:int(s_off[-1])].copy(), dangling_edge_count=int(s_off[-1]))


def rmat_graph_edges(scale: int, edge_factor: int, seed: int = 0, threads: int = 0,
                     a: float = 0.57, b: float = 0.19, c: float = 0.19):
    """``(n, src, dst)``: the R-MAT samples of the BASELINE configs with
    self-loops dropped in sample order -- the same edge list as
    ``synthetic.rmat_graph`` (numpy) and the device generator
    (``pr_graph_rmat``), computed by threaded C (orc_rmat) so that C5's
    1.07 B samples reach the oracle without the device."""
    threads = threads or (os.cpu_count() or 1)
    S = float(1 << 32)
    ta, tb, tc = int(a * S), int((a + b) * S), int((a + b + c) * S)
    kept = lib().orc_rmat(scale, edge_factor, ta, tb, tc, seed, threads, None, None)
    src = np.empty(kept, np.int64)
    dst = np.empty(kept, np.int64)
    lib().orc_rmat(scale, edge_factor, ta, tb, tc, seed, threads, src.ctypes.data, dst.ctypes.data)
    return 1 << scale, src, dst


# ---------------------------------------------------------------- engines

VARIANTS = {"ifp1": 0, "ifp2": 1, "fp-full": 2}


def sync_simulate(g, variant: str = "ifp1", damping: float = 0.85, threshold: float = 1e-10,
                  max_iterations: int = 1_000_000, pg=None, threads: int = 0) -> SimpleNamespace:
    """Restates engines.py:349-485 (round-synchronous twin).

    ``rows`` is a structured array (ROW_DTYPE) with one row per state; an
    ifp2 run appends the post-settle row (engines.py:458-472).

    ``threads > 0`` runs the rounds as a CSC pull over that many threads
    (orc_sync_rounds_pull): the reserved/pending state is bit-identical to
    the sequential scatter form (tests/test_oracle_golden.py checks it), the
    trace's float sums are combined per thread.  For the full-size configs.
    """
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    g = graph_arrays(g)
    n = g.n
    dang = (g.out_degree == 0)
    if variant == "ifp2":
        if pg is None:
            pg = preprocess_ifp2(g, np.flatnonzero(dang))
        offsets, targets = pg.live_offsets, pg.live_targets
        dt = None
    else:
        offsets, targets = g.out_offsets, g.out_targets
        dt = dangling_target_counts(g, np.flatnonzero(dang))
    reserved = np.zeros(n, np.float64)
    h = np.zeros(n, np.float64)
    cap = 4096
    if threads > 0:
        row_len = np.ascontiguousarray(np.diff(offsets), np.int64)
        while True:
            rows = np.zeros(cap, ROW_DTYPE)
            nrows = _I(0)
            it = lib().orc_sync_rounds_pull(VARIANTS[variant], n, g.in_offsets,
                                            np.ascontiguousarray(g.in_sources if g.m else np.zeros(1, np.int64)),
                                            g.out_degree, row_len, dt.ctypes.data if dt is not None else None,
                                            damping, threshold, max_iterations, int(threads), reserved, h,
                                            rows, cap, ctypes.byref(nrows))
            if it != -2:
                break
            cap *= 4
    while threads <= 0:
        rows = np.zeros(cap, ROW_DTYPE)
        nrows = _I(0)
        targets_c = np.ascontiguousarray(targets if targets.size else np.zeros(1, np.int64))
        it = lib().orc_sync_rounds(VARIANTS[variant], n, offsets, targets_c, g.out_degree,
                                   dt.ctypes.data if dt is not None else None,
                                   damping, threshold, max_iterations, reserved, h, rows, cap,
                                   ctypes.byref(nrows))
        if it != -2:
            break
        cap *= 4
    if it == -1:
        raise RuntimeError(f"sync simulation did not settle in {max_iterations} iterations")
    rows = rows[: nrows.value].copy()
    reserved_pre, h_pre = reserved.copy(), h.copy()
    if variant == "ifp2":
        settled = settle(pg, g.out_degree, damping, reserved, h)
        above = h > threshold
        above_mass = float(h[above].sum())
        l1 = float(h.sum())
        extra = np.zeros(1, ROW_DTYPE)
        extra["h_l1"] = l1
        extra["converged"] = int(np.count_nonzero(~above))
        extra["alpha"] = 1.0 if above_mass == 0.0 else float(h[above & ~dang].sum()) / above_mass
        extra["work"] = 0
        extra["push_ops"] = rows["push_ops"][-1] + settled
        extra["push_ops_dangling"] = rows["push_ops_dangling"][-1] + settled
        extra["active_mass"] = above_mass
        extra["carry_mass"] = l1 - above_mass
        rows = np.concatenate([rows, extra])
        values = reserved.copy()
    elif variant == "ifp1":
        values = reserved + h
    else:
        values = reserved.copy()
    total = float(values.sum())
    return SimpleNamespace(values=values / total, reserved=reserved, h=h, rows=rows,
                           iterations=int(it), mass_total=total,
                           reserved_pre_settle=reserved_pre, h_pre_settle=h_pre)


def settle(pg, out_degree, damping: float, reserved: np.ndarray, h: np.ndarray) -> int:
    """Restates engines.py:269-289 in sequential ascending-source order."""
    d_ids = np.ascontiguousarray(pg.dangling_ids, np.int64)
    if d_ids.size == 0:
        return 0
    return int(lib().orc_settle(d_ids.size, d_ids,
                                np.ascontiguousarray(pg.source_offsets, np.int64),
                                np.ascontiguousarray(pg.source_ids, np.int64),
                                np.ascontiguousarray(out_degree, np.int64), damping, reserved, h))


def power_method(g, damping: float = 0.85, iterations: int = 210, tolerance: float = 0.0,
                 personalization=None, workers: int = 1) -> SimpleNamespace:
    """Restates solvers.py:186-243 (pull SpMV + rank-one dangling restart);
    ``workers`` threads split the multiply by destination range (identical
    result, solvers.py:124-183)."""
    g = graph_arrays(g)
    p = (np.full(g.n, 1.0 / g.n) if personalization is None
         else np.ascontiguousarray(personalization, np.float64))
    pi = np.zeros(g.n, np.float64)
    deltas = np.zeros(max(iterations, 1), np.float64)
    src = g.in_sources if g.in_sources.size else np.zeros(1, np.int64)
    k = lib().orc_power(g.n, g.in_offsets, np.ascontiguousarray(src), g.out_degree, damping, p,
                        iterations, tolerance, pi, deltas, int(workers))
    if iterations == 0:
        pi = p.copy()
    return SimpleNamespace(values=pi, deltas=deltas[:k].copy(), iterations=int(k))


def split(ids: np.ndarray, weights: np.ndarray, workers: int, strategy: str) -> list:
    """Restates engines.py:76-89 (worker vertex sets)."""
    if strategy == "contiguous":
        parts = np.array_split(ids, workers)
    elif strategy == "strided":
        parts = [ids[j::workers] for j in range(workers)]
    elif strategy == "degree-balanced":
        order = np.lexsort((ids, -weights))
        parts = [ids[order[j::workers]] for j in range(workers)]
    else:
        raise ValueError(f"unknown partition strategy {strategy!r}")
    return [np.sort(p).astype(np.int64) for p in parts]


def async_run(g, algorithm: str = "ifp1", damping: float = 0.85, threshold: float = 1e-10,
              workers: int = 1, strategy: str = "degree-balanced", pg=None) -> SimpleNamespace:
    """Port of ifp1_run / ifp2_run (engines.py:225-343) on pthreads, restating
    the compiled worker loop and quiescence probe (_kernels.pyx:66-137)."""
    g = graph_arrays(g)
    n = g.n
    dang = g.out_degree == 0
    universe = np.flatnonzero(~dang)
    sets = split(universe, g.out_degree[universe] + 1, workers, strategy)
    verts = np.concatenate(sets) if sets else np.zeros(0, np.int64)
    set_off = np.zeros(len(sets) + 1, np.int64)
    set_off[1:] = np.cumsum([s.size for s in sets])
    h = np.ones(n, np.float64)
    reserved = np.zeros(n, np.float64)
    if algorithm == "ifp1":
        offsets, targets = g.out_offsets, g.out_targets
        dt = dangling_target_counts(g, np.flatnonzero(dang))
    elif algorithm == "ifp2":
        if pg is None:
            pg = preprocess_ifp2(g, np.flatnonzero(dang))
        offsets, targets = pg.live_offsets, pg.live_targets
        dt = None
    else:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    po, pd = _I(0), _I(0)
    tg = np.ascontiguousarray(targets if targets.size else np.zeros(1, np.int64))
    vv = verts if verts.size else np.zeros(1, np.int64)
    sc = universe if universe.size else np.zeros(1, np.int64)
    lib().orc_async_phase(n, h, reserved, offsets, tg, g.out_degree, vv, set_off, len(sets),
                          sc, universe.size, dt.ctypes.data if dt is not None else None,
                          threshold, damping, ctypes.byref(po), ctypes.byref(pd))
    push_ops, push_dang = int(po.value), int(pd.value)
    if algorithm == "ifp2":
        settled = settle(pg, g.out_degree, damping, reserved, h)
        push_ops += settled
        push_dang += settled
        values = reserved.copy()
    else:
        values = reserved + h
    total = float(values.sum())
    return SimpleNamespace(values=values / total, reserved=reserved, h=h, push_ops=push_ops,
                           push_ops_dangling=push_dang, mass_total=total)


def dense_pagerank(g, damping: float = 0.85) -> np.ndarray:
    """Restates dense_oracle (solvers.py:95-121) for tiny graphs."""
    g = graph_arrays(g)
    n = g.n
    if n > 2000:
        raise ValueError("dense oracle refused: n exceeds the 2000-vertex guard")
    p = np.full(n, 1.0 / n)
    w = np.zeros((n, n))
    for v in range(n):
        lo, hi = g.out_offsets[v], g.out_offsets[v + 1]
        if hi > lo:
            w[g.out_targets[lo:hi], v] += 1.0 / g.out_degree[v]
        else:
            w[:, v] = p
    x = np.linalg.solve(np.eye(n) - damping * w, (1.0 - damping) * p)
    return x / x.sum()
