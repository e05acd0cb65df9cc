"""IFP1 / IFP2 engines on the B200 (drop-in for ``engines.py`` of the reference).

Entry points keep the reference signatures (``engines.py:225-233``,
``292-299``, ``349-356``, ``488-494``) and outputs:

* ``ifp1_run``  -- values = (reserved + pending) / total  (engines.py:259-265)
* ``ifp2_run``  -- phase 1 on live edges, one dangling settle, values =
  reserved / total; the trace ends with [phase-1 final, post-settle] rows
  (engines.py:326-342)
* ``sync_simulate`` -- the round-synchronous twin, bit-exact reserved /
  pending state (``mode="exact"``)
* ``ifp2_full_run`` -- classify + preprocess timed separately

The CPU engines' K free-running worker threads become device rounds: each
round drains every active vertex of the current state at once (Jacobi), as
one CSC-pull launch in dense rounds or a frontier scatter in the sparse
tail, with the whole loop captured in one CUDA graph.  ``workers`` and
``strategy`` are validated and recorded for parity (they select CPU worker
sets in the reference, engines.py:76-117) but do not change the device
schedule.  ``mode`` selects the round policy: "auto" (default), "pull",
"push" or "exact" (env ``PUSHRANK_CUDA_MODE``).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._backend import resolve_backend
from .graph import IFP2Graph, VertexClassification, classify, device_graph, preprocess_ifp2
from .solvers import PageRankVector, SolverConfig
from .trace import RunTrace, samples_from_rows

PARTITION_STRATEGIES = ("contiguous", "strided", "degree-balanced")
SYNC_VARIANTS = ("ifp1", "ifp2", "fp-full")
DEFAULT_MAX_ROUNDS = 1_000_000


def _check_workers(workers: int, strategy: str) -> None:
    if workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    if strategy not in PARTITION_STRATEGIES:
        raise ValueError(f"unknown partition strategy {strategy!r}")


def _mode(mode: str | None) -> str:
    mode = (mode or os.environ.get("PUSHRANK_CUDA_MODE", "auto")).lower()
    if mode not in _lib.MODE:
        raise ValueError(f"unknown mode {mode!r} (expected one of {sorted(_lib.MODE)})")
    return mode


@dataclass
class MassState:
    """Reserved and pending mass per vertex (engines.py:44-54): a fresh
    state reserves nothing and holds one raw unit of pending mass on every
    vertex.  The device engines keep this state in HBM (``h`` / ``reserved``
    of the run workspace, initialised by ``k_init``); the host class stays
    for callers that build or inspect states themselves."""

    reserved: np.ndarray
    pushing: np.ndarray

    @classmethod
    def fresh(cls, n: int) -> "MassState":
        return cls(reserved=np.zeros(n, dtype=np.float64), pushing=np.ones(n, dtype=np.float64))


@dataclass
class Partition:
    """Vertex-to-worker assignment (engines.py:57-73): disjoint ascending id
    sets per CPU worker over the scan universe, plus the dangling side for
    the two-phase settle.  The device engines schedule by degree bins
    instead (csrc/sched.cu); ``workers`` / ``strategy`` of the entry points
    are validated through the same rules and recorded in ``trace.meta``."""

    strategy: str
    worker_vertices: list
    worker_dangling: list | None = None

    @property
    def workers(self) -> int:
        return len(self.worker_vertices)


def _assign(ids: np.ndarray, weights: np.ndarray, workers: int, strategy: str) -> list:
    """One worker set per worker, each sorted ascending (engines.py:76-89):
    contiguous blocks (np.array_split sizes), every workers-th id, or
    heaviest-first round-robin (weight descending, ties by id)."""
    if strategy == "contiguous":
        sets = np.array_split(ids, workers)
    elif strategy == "strided":
        sets = [ids[k::workers] for k in range(workers)]
    elif strategy == "degree-balanced":
        by_weight = np.lexsort((ids, -weights))
        sets = [ids[by_weight[k::workers]] for k in range(workers)]
    else:
        raise ValueError(f"unknown partition strategy {strategy!r}")
    return [np.sort(np.asarray(s)).astype(np.int64) for s in sets]


def partition_vertices(g, workers: int, strategy: str = "degree-balanced",
                       cls: VertexClassification | None = None) -> Partition:
    """Split the vertices among CPU workers (engines.py:92-117).

    With ``cls``: the non-dangling vertices (weight out-degree + 1) and,
    separately, the dangling ones (weight in-degree + 1).  Without it: all
    vertices by out-degree + 1."""
    if workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    out_deg = np.asarray(g.out_degree, np.int64)
    if cls is None:
        every = np.arange(g.n, dtype=np.int64)
        return Partition(strategy, _assign(every, out_deg + 1, workers, strategy))
    dang = cls.dangling_mask(g.n)
    live = np.flatnonzero(~dang)
    dead = np.flatnonzero(dang)
    in_deg = np.asarray(g.in_degree, np.int64)
    return Partition(strategy, _assign(live, out_deg[live] + 1, workers, strategy),
                     _assign(dead, in_deg[dead] + 1, workers, strategy))


def _sample_period(n: int, sample_every: float | None) -> float:
    """The reference's default trace period: 10 ms up to 1e5 vertices,
    250 ms above (engines.py:219-222)."""
    if sample_every is not None:
        return sample_every
    return 0.01 if n <= 100_000 else 0.25


def _keep_rows(rows, sample_every, n):
    """Time-based trace sampling as in _run_phase (engines.py:199-215): the
    device writes one row per round with its device timestamp (wall_ms);
    keep a row whenever ``period`` seconds have passed since the last kept
    one (the first row always), and always the final row.  ``inf`` keeps
    only the final row, 0 every round."""
    period = _sample_period(n, sample_every)
    if len(rows) == 0:
        return rows
    if math.isinf(period):
        return rows[-1:]
    keep, last = [], -math.inf
    wall_s = np.asarray(rows["wall_ms"], np.float64) * 1e-3
    for i in range(len(rows) - 1):
        if wall_s[i] - last >= period:
            keep.append(i)
            last = wall_s[i]
    keep.append(len(rows) - 1)
    return rows[np.asarray(keep)]


def ifp1_run(g, cls: VertexClassification | None, cfg: SolverConfig, workers: int = 1,
             strategy: str = "degree-balanced", backend: str | None = None, sample_every: float | None = None,
             mode: str | None = None) -> tuple[PageRankVector, RunTrace]:
    """One-phase push over the non-dangling vertices (engines.py:225-266).

    Every vertex starts with one unit of pending mass; each round drains all
    non-dangling vertices above ``cfg.threshold`` (100% reservation) and
    pushes ``damping*h/out_degree`` along every out-edge, dangling targets
    included.  Dangling accumulation and sub-threshold residue count.
    """
    cfg.validate(g.n)
    _check_workers(workers, strategy)
    kern = resolve_backend(backend)
    mode = _mode(mode)
    dev = device_graph(g)
    start = time.perf_counter()
    values, rows, res, _, _ = dev.run("ifp1", mode, cfg.damping, cfg.threshold, DEFAULT_MAX_ROUNDS,
                                      _lib.CONV_SCAN)
    wall = time.perf_counter() - start
    trace = RunTrace(samples=samples_from_rows(_keep_rows(rows, sample_every, g.n)),
                     meta={"algorithm": "ifp1", "threshold": cfg.threshold, "workers": workers,
                           "strategy": strategy, "backend": kern.NAME, "mode": mode, "rounds": int(res.rounds),
                           "pull_rounds": int(res.pull_rounds), "push_rounds": int(res.push_rounds),
                           "device_ms": float(res.push_ms), "wall_s": wall})
    vec = PageRankVector(values=values, algorithm="ifp1", damping=cfg.damping, threshold=cfg.threshold,
                         iterations=len(trace.samples), mass_total=float(res.mass_total), workers=workers)
    return vec, trace


def ifp2_run(pg: IFP2Graph, cfg: SolverConfig, workers: int = 1, strategy: str = "degree-balanced",
             backend: str | None = None, sample_every: float | None = None,
             mode: str | None = None) -> tuple[PageRankVector, RunTrace]:
    """Two-phase push (engines.py:292-343): phase 1 restricted to live
    (non-dangling) targets with weights 1/original out-degree, then one fused
    settle of every dangling vertex (K7) and normalisation."""
    g = pg.base
    cfg.validate(g.n)
    _check_workers(workers, strategy)
    kern = resolve_backend(backend)
    mode = _mode(mode)
    dev = device_graph(pg)
    dev.preprocess_ifp2()
    start = time.perf_counter()
    values, rows, res, _, _ = dev.run("ifp2", mode, cfg.damping, cfg.threshold, DEFAULT_MAX_ROUNDS,
                                      _lib.CONV_SCAN)
    wall = time.perf_counter() - start
    phase1, settle_row = rows[:-1], rows[-1:]
    kept = np.concatenate([_keep_rows(phase1, sample_every, g.n), settle_row])
    trace = RunTrace(samples=samples_from_rows(kept),
                     meta={"algorithm": "ifp2", "threshold": cfg.threshold, "workers": workers,
                           "strategy": strategy, "backend": kern.NAME, "mode": mode, "rounds": int(res.rounds),
                           "pull_rounds": int(res.pull_rounds), "push_rounds": int(res.push_rounds),
                           "settled": int(res.settled), "device_ms": float(res.push_ms), "wall_s": wall})
    vec = PageRankVector(values=values, algorithm="ifp2", damping=cfg.damping, threshold=cfg.threshold,
                         iterations=len(trace.samples), mass_total=float(res.mass_total), workers=workers)
    return vec, trace


def sync_simulate(subject, cfg: SolverConfig, variant: str = "ifp1", cls: VertexClassification | None = None,
                  max_iterations: int = DEFAULT_MAX_ROUNDS, on_iteration=None,
                  mode: str = "exact") -> tuple[PageRankVector, RunTrace]:
    """Deterministic round-synchronous twin (engines.py:349-485).

    ``mode="exact"`` (default) sums every destination's inflow sequentially
    in ascending source order, so reserved/pending states are bit-identical
    to the reference's ``np.bincount`` accumulation; one trace row per state
    including the terminal one.  ``on_iteration(t, reserved, pushing)`` is
    called after each round with read-only host views.
    """
    if variant not in SYNC_VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if isinstance(subject, IFP2Graph):
        pg, g = subject, subject.base
    else:
        pg, g = None, subject
    cfg.validate(g.n)
    mode = _mode(mode)
    dev = device_graph(g)
    if variant == "ifp2":
        if pg is None:
            pg = preprocess_ifp2(g, cls if cls is not None else classify(g))
        dev.preprocess_ifp2()
    start = time.perf_counter()
    values, rows, res, _, _ = dev.run(variant, mode, cfg.damping, cfg.threshold, max_iterations, _lib.CONV_ALL,
                                      on_round=on_iteration)
    trace = RunTrace(samples=samples_from_rows(rows),
                     meta={"algorithm": f"sync-{variant}", "threshold": cfg.threshold, "workers": 1,
                           "backend": "sync-cuda", "mode": mode, "device_ms": float(res.push_ms)})
    trace.meta["wall_s"] = time.perf_counter() - start
    trace.meta["iterations"] = int(res.rounds)
    vec = PageRankVector(values=values, algorithm=f"sync-{variant}", damping=cfg.damping, threshold=cfg.threshold,
                         iterations=int(res.rounds), mass_total=float(res.mass_total), workers=1)
    return vec, trace


def ifp2_full_run(g, cfg: SolverConfig, workers: int = 1, strategy: str = "degree-balanced",
                  backend: str | None = None, mode: str | None = None) -> tuple[PageRankVector, RunTrace, float]:
    """Classify + preprocess (timed as ``preprocess_s``) + ifp2_run (engines.py:488-507)."""
    t0 = time.perf_counter()
    cls = classify(g)
    pg = preprocess_ifp2(g, cls)
    preprocess_s = time.perf_counter() - t0
    vec, trace = ifp2_run(pg, cfg, workers=workers, strategy=strategy, backend=backend, mode=mode)
    trace.meta["preprocess_s"] = preprocess_s
    return vec, trace, preprocess_s
