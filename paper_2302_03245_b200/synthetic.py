"""Seeded synthetic workloads C1-C5 (BASELINE.json ``configs``).

None of the reference's datasets are in the image (``pkg/data/MANIFEST.csv``
lists them by URL only) and the reference's own generator
(``pkg/src/pushrank/synth.py:17-111``) cannot produce R-MAT / Zipf-DAG
shapes, so these seeded generators stand in for them.  Every generator
returns ``(n, src, dst)`` as int64 edge arrays *before* ``from_edges``
(which de-duplicates, ``graph.py:151-152``); self-loops are removed here
because the BASELINE configs say "duplicates and self-loops removed".

R-MAT uses a counter-based hash (splitmix64 of (seed, edge, level)) so the
same edge list can be produced by numpy here and by the device generator
``pr_rmat_generate`` in the CUDA library (C5 is too large for the host).
"""

from __future__ import annotations

import numpy as np

U64 = np.uint64
_GOLDEN = U64(0x9E3779B97F4A7C15)
_M1 = U64(0xBF58476D1CE4E5B9)
_M2 = U64(0x94D049BB133111EB)

RMAT_ABC = (0.57, 0.19, 0.19)


def mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = (x ^ (x >> U64(30))) * _M1
        x = (x ^ (x >> U64(27))) * _M2
        return x ^ (x >> U64(31))


def rmat_thresholds(a: float, b: float, c: float) -> tuple[int, int, int]:
    """Cumulative quadrant thresholds on the 32-bit scale."""
    scale = float(1 << 32)
    ta = int(a * scale)
    tb = int((a + b) * scale)
    tc = int((a + b + c) * scale)
    return ta, tb, tc


def rmat_edges(scale: int, edge_factor: int, a: float = RMAT_ABC[0], b: float = RMAT_ABC[1],
               c: float = RMAT_ABC[2], seed: int = 0, first: int = 0,
               count: int | None = None) -> tuple[int, np.ndarray, np.ndarray]:
    """Raw R-MAT samples ``first .. first+count`` (self-loops kept).

    Sample ``i`` at level ``l`` (MSB first) draws ``u = mix64(key0 + (i*64+l)*golden) >> 32``
    and picks quadrant a/b/c/d by the cumulative thresholds: a=(0,0),
    b=(0,1), c=(1,0), d=(1,1) for (src bit, dst bit).
    """
    n = 1 << scale
    total = edge_factor * n
    if count is None:
        count = total - first
    ta, tb, tc = (U64(t) for t in rmat_thresholds(a, b, c))
    key0 = mix64(np.array([seed], dtype=U64))[0]
    idx = np.arange(first, first + count, dtype=U64)
    src = np.zeros(count, dtype=U64)
    dst = np.zeros(count, dtype=U64)
    with np.errstate(over="ignore"):
        base = key0 + idx * U64(64) * _GOLDEN
        for level in range(scale):
            u = mix64(base + U64(level) * _GOLDEN) >> U64(32)
            sbit = (u >= tb).astype(U64)
            dbit = (((u >= ta) & (u < tb)) | (u >= tc)).astype(U64)
            src = (src << U64(1)) | sbit
            dst = (dst << U64(1)) | dbit
    return n, src.astype(np.int64), dst.astype(np.int64)


def _drop_self_loops(src: np.ndarray, dst: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    keep = src != dst
    return src[keep], dst[keep]


def poisson_graph(n: int = 10_000, mean_degree: float = 8.0, dangling_frac: float = 0.10,
                  unreferenced_frac: float = 0.05, seed: int = 0):
    """C1: out-degree ~ Poisson(mean) with distinct uniform targets, no self-loops.

    A seeded permutation picks disjoint forced-dangling (first
    ``dangling_frac*n``) and forced-unreferenced (next ``unreferenced_frac*n``)
    sets; unreferenced vertices are removed from the target pool.
    """
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    n_d = int(round(n * dangling_frac))
    n_u = int(round(n * unreferenced_frac))
    dangling = np.zeros(n, dtype=bool)
    dangling[perm[:n_d]] = True
    unref = np.zeros(n, dtype=bool)
    unref[perm[n_d:n_d + n_u]] = True
    pool = np.flatnonzero(~unref)
    pos_in_pool = np.full(n, -1, dtype=np.int64)
    pos_in_pool[pool] = np.arange(pool.size)
    degrees = rng.poisson(mean_degree, size=n)
    srcs, dsts = [], []
    for v in np.flatnonzero(~dangling):
        p = pos_in_pool[v]
        avail = pool.size - (1 if p >= 0 else 0)
        d = int(min(degrees[v], avail))
        if d == 0:
            continue
        pick = rng.choice(avail, size=d, replace=False)
        if p >= 0:
            pick = pick + (pick >= p)   # skip the vertex itself
        srcs.append(np.full(d, v, dtype=np.int64))
        dsts.append(pool[pick])
    src = np.concatenate(srcs) if srcs else np.zeros(0, dtype=np.int64)
    dst = np.concatenate(dsts) if dsts else np.zeros(0, dtype=np.int64)
    return n, src, dst


def rmat_graph(scale: int, edge_factor: int, seed: int = 0, drop_out_frac: float = 0.0):
    """C2/C3/C5 shape: R-MAT samples, self-loops removed, optional seeded
    out-edge drop for ``drop_out_frac`` of the vertices (C3: 20%)."""
    n, src, dst = rmat_edges(scale, edge_factor, seed=seed)
    src, dst = _drop_self_loops(src, dst)
    if drop_out_frac > 0.0:
        rng = np.random.default_rng(seed + 0x5EED)
        victims = np.zeros(n, dtype=bool)
        victims[rng.permutation(n)[: int(n * drop_out_frac)]] = True
        keep = ~victims[src]
        src, dst = src[keep], dst[keep]
    return n, src, dst


def layered_dag(n: int = 2_000_000, layers: int = 50, zipf_s: float = 2.0, max_degree: int = 200,
                back_frac: float = 0.02, seed: int = 0):
    """C4: ``layers`` equal layers; out-degree ~ Zipf(s) truncated at
    ``max_degree`` (rejection), targets uniform over strictly later layers
    (last layer dangling), plus ``back_frac * m`` back-edges from layers
    1..L-2 to uniformly chosen earlier-layer vertices."""
    rng = np.random.default_rng(seed)
    width = n // layers
    n = width * layers
    fwd = np.arange(width * (layers - 1), dtype=np.int64)
    deg = rng.zipf(zipf_s, size=fwd.size)
    bad = deg > max_degree
    while bad.any():
        deg[bad] = rng.zipf(zipf_s, size=int(bad.sum()))
        bad = deg > max_degree
    src = np.repeat(fwd, deg)
    lo = (src // width + 1) * width
    dst = lo + (rng.random(src.size) * (n - lo)).astype(np.int64)
    n_back = int(round(back_frac * src.size))
    bsrc = rng.integers(width, width * (layers - 1), size=n_back)
    bdst = (rng.random(n_back) * ((bsrc // width) * width)).astype(np.int64)
    src = np.concatenate([src, bsrc])
    dst = np.concatenate([dst, bdst])
    return n, src, dst


CONFIGS = {
    "c1": "poisson n=10000 deg~Poisson(8) 10% dangling 5% unreferenced",
    "c2": "rmat scale=20 ef=5 (.57,.19,.19,.05)",
    "c3": "rmat scale=22 ef=16 (.57,.19,.19,.05), 20% out-edges dropped",
    "c4": "layered DAG n=2e6 50 layers Zipf(2)<=200 + 2% back-edges",
    "c5": "rmat scale=26 ef=16 (.57,.19,.19,.05)",
}


def make(config: str, seed: int = 0):
    """``(n, src, dst)`` for a BASELINE config name (c1..c4 on the host)."""
    config = config.lower()
    if config == "c1":
        return poisson_graph(seed=seed)
    if config == "c2":
        return rmat_graph(20, 5, seed=seed)
    if config == "c3":
        return rmat_graph(22, 16, seed=seed, drop_out_frac=0.2)
    if config == "c4":
        return layered_dag(seed=seed)
    if config == "c5":
        raise ValueError("c5 is generated on the device (pr_rmat_generate); 1.07B samples")
    raise ValueError(f"unknown config {config!r}")
