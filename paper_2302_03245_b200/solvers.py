"""Solver configuration, result vector and the Power-method baseline.

``SolverConfig`` / ``PageRankVector`` keep the reference's fields, defaults
and ``ValueError`` texts (``solvers.py:30-88``).  ``power_method`` keeps the
reference signature (``solvers.py:186-192``) and runs K8 on the device:
the degree-binned CSC gather of the dense push round plus a fused
normalise / L1-delta / dangling-restart epilogue, iterated inside one CUDA
graph.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from .graph import device_graph
from .trace import RunTrace, TraceSample

REFERENCE_ITERATIONS = 210


@dataclass
class SolverConfig:
    damping: float = 0.85
    personalization: np.ndarray | None = None
    threshold: float = 1e-10
    max_iterations: int = REFERENCE_ITERATIONS

    def validate(self, n: int) -> None:
        if not 0.0 < self.damping < 1.0:
            raise ValueError(f"damping must be in (0,1), got {self.damping}")
        if not self.threshold > 0.0:
            raise ValueError(f"threshold must be positive, got {self.threshold}")
        if self.max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        if self.personalization is not None:
            p = np.asarray(self.personalization, dtype=np.float64)
            if p.shape != (n,):
                raise ValueError("personalization length must equal vertex count")
            if np.any(p < 0) or abs(p.sum() - 1.0) > 1e-9:
                raise ValueError("personalization must be a probability distribution")

    def restart_vector(self, n: int) -> np.ndarray:
        if self.personalization is None:
            return np.full(n, 1.0 / n, dtype=np.float64)
        return np.asarray(self.personalization, dtype=np.float64).copy()

    def with_threshold(self, threshold: float) -> "SolverConfig":
        return replace(self, threshold=threshold)


@dataclass
class PageRankVector:
    values: np.ndarray
    algorithm: str
    damping: float
    threshold: float | None = None
    iterations: int | None = None
    mass_total: float | None = None
    workers: int | None = None

    def normalized(self) -> "PageRankVector":
        total = float(self.values.sum())
        if total <= 0:
            raise ValueError("cannot normalize a vector with non-positive total")
        return replace(self, values=self.values / total, mass_total=total)


def power_method(g, cfg: SolverConfig, workers: int = 1, tolerance: float = 0.0,
                 on_iterate=None) -> tuple[PageRankVector, RunTrace]:
    """Damped power iteration with the dangling mass folded in as a rank-one
    restart (solvers.py:186-243), on the device.  ``workers`` is accepted
    for signature parity (the reference proves the result is independent of
    it, test_solvers.py:84-87); ``on_iterate(k, pi)`` switches to
    host-observed iterations and may stop early by returning truthy."""
    cfg.validate(g.n)
    dev = device_graph(g)
    start = time.perf_counter()
    pi, deltas, conv, res = dev.power(cfg.damping, cfg.max_iterations, tolerance, cfg.threshold,
                                      cfg.personalization, on_iterate)
    wall = time.perf_counter() - start
    trace = RunTrace(meta={"algorithm": "power", "workers": workers, "damping": cfg.damping,
                           "tolerance": tolerance, "backend": "cuda", "device_ms": res.push_ms})
    m, n = dev.m, dev.n
    per = res.push_ms / max(len(deltas), 1)
    for k, (d, c) in enumerate(zip(deltas, conv)):
        trace.samples.append(TraceSample(t=k, h_l1=float(d), converged=int(c), alpha=1.0, work=m + n,
                                         push_ops=(k + 1) * m, push_ops_dangling=0, wall_ms=per * (k + 1)))
    trace.meta["iterations"] = len(deltas)
    trace.meta["wall_s"] = wall
    if cfg.max_iterations == 0:
        pi = cfg.restart_vector(n)
    vec = PageRankVector(values=pi, algorithm="power", damping=cfg.damping, iterations=len(deltas),
                         workers=workers, mass_total=float(pi.sum()))
    return vec, trace
