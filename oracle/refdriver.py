"""Drive the reference's own compiled push kernel (oracle/_ref).

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py ``--impl reference`` and the
``cpu_baseline`` leg).  ``oracle/_ref/_kernels*.so`` is the reference's
``_kernels.pyx`` (``/root/reference/pkg/src/pushrank/_kernels.pyx:66-137``)
compiled unmodified by ``make -C oracle ref``.  The orchestration around it
restates ``engines._run_phase`` (engines.py:185-216): K Python threads run
``worker_loop`` with the GIL released while the calling thread polls
``probe``; ``sample_every=inf`` semantics (no intermediate samples), exactly
how the reference's harness times it (bench.py:162-170).
"""

from __future__ import annotations

import glob
import importlib.util
import os
import threading
import time
from types import SimpleNamespace

import numpy as np

from . import dangling_target_counts, graph_arrays, preprocess_ifp2, settle, split

HERE = os.path.dirname(os.path.abspath(__file__))
_mod = None


def available() -> bool:
    return bool(glob.glob(os.path.join(HERE, "_ref", "_kernels*.so")))


def kernels():
    global _mod
    if _mod is None:
        paths = glob.glob(os.path.join(HERE, "_ref", "_kernels*.so"))
        if not paths:
            raise ImportError("oracle/_ref not built (make -C oracle ref)")
        spec = importlib.util.spec_from_file_location("_kernels", paths[0])
        _mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(_mod)
    return _mod


def run(g, algorithm: str = "ifp1", damping: float = 0.85, threshold: float = 1e-10,
        workers: int = 1, strategy: str = "degree-balanced", pg=None, budget_s: float | None = None,
        dt=None) -> SimpleNamespace:
    """ifp1_run / ifp2_run on the reference's compiled kernel; returns the
    normalised vector, push counters and the push-phase wall time.

    ``budget_s`` bounds the sample (bench.py at C5, where one CPU solve
    takes many minutes): the monitor raises the stop flag after that many
    seconds, as the reference's own stop path does (engines.py:205-216), and
    the result has ``complete=False``, the pushes done and the elapsed time
    (no settle, no vector).  ``dt`` passes precomputed dangling target
    counts (IFP1)."""
    K = kernels()
    g = graph_arrays(g)
    n = g.n
    dang = g.out_degree == 0
    universe = np.flatnonzero(~dang)
    sets = split(universe, g.out_degree[universe] + 1, workers, strategy)
    h = np.ones(n, np.float64)
    reserved = np.zeros(n, np.float64)
    if algorithm == "ifp1":
        offsets, targets = g.out_offsets, g.out_targets
        if dt is None:
            dt = dangling_target_counts(g, np.flatnonzero(dang))
    else:
        if pg is None:
            pg = preprocess_ifp2(g, np.flatnonzero(dang))
        offsets = np.ascontiguousarray(pg.live_offsets, np.int64)
        targets = np.ascontiguousarray(pg.live_targets, np.int64)
        dt = np.zeros(n, np.int64)
    ctrl = np.zeros(1, np.int64)
    wstate = np.zeros(8 * max(1, len(sets)), np.int64)
    start = time.perf_counter()
    threads = [threading.Thread(target=K.worker_loop,
                                args=(h, reserved, offsets, targets, g.out_degree, s, threshold,
                                      damping, ctrl, wstate, j, dt, None), daemon=True)
               for j, s in enumerate(sets)]
    for t in threads:
        t.start()
    pause = 0.0005 if universe.size > 100_000 else 0.0
    complete = True
    try:
        while not K.probe(h, universe, threshold, wstate, len(threads), None):
            if budget_s is not None and time.perf_counter() - start >= budget_s:
                complete = False
                break
            time.sleep(pause)
    finally:
        ctrl[0] = 1
        for t in threads:
            t.join()
    push_ops = int(wstate[2::8].sum())
    push_dang = int(wstate[3::8].sum())
    if not complete:
        wall = time.perf_counter() - start
        return SimpleNamespace(values=None, push_ops=push_ops, push_ops_dangling=push_dang, wall_s=wall,
                               mass_total=None, complete=False)
    if algorithm == "ifp2":
        settled = settle(pg, g.out_degree, damping, reserved, h)
        push_ops += settled
        push_dang += settled
        values = reserved.copy()
    else:
        values = reserved + h
    wall = time.perf_counter() - start
    total = float(values.sum())
    return SimpleNamespace(values=values / total, push_ops=push_ops, push_ops_dangling=push_dang,
                           wall_s=wall, mass_total=total, complete=True)
