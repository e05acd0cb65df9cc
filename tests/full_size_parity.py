"""Full-size parity of the CUDA path against the CPU oracle, any BASELINE
config (C1-C5) or a forced-C5-path R-MAT, as a script (C5 takes minutes of
host CPU) and as the body of the ``-m gpu`` tests in test_gpu_parity.py.

    python tests/full_size_parity.py c5 [--algos ifp2,ifp1] [--modes auto,pull,push]
                                        [--xi 1e-10] [--out profiles/r02_parity_c5.json]

What it checks (BASELINE.json north_star):
  * integer preprocessing bit-exact: the device graph's CSR/CSC, classify's
    four id sets + m_d, and preprocess_ifp2's six arrays against the oracle's
    restatement (graph.py:133-177, 274-318, 343-378) built from an
    independently generated edge list (C5: orc_rmat on the host vs the
    device generator pr_graph_rmat);
  * the fast engines (IFP1 and IFP2, each mode) against the oracle's
    round-synchronous twin (engines.py:349-485; at full size its threaded
    CSC-pull form, bit-identical to the sequential restatement --
    tests/test_oracle_golden.py): L1 <= 1e-9 and identical top-100 under
    (-score, id) (serialize.py:16), push_ops_dangling == m_d for IFP2, mass 1.

The chain to the reference: the oracle is pinned bit-exact against outputs
of the real reference package (tests/golden/, made by make_golden.py) on 50
corpus graphs, C1 and the acceptance graph.

TEST INFRASTRUCTURE: imports ``oracle`` as the checker only.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

INT_KEYS = ("out_offsets", "out_targets", "in_offsets", "in_sources")
CLS_KEYS = ("dangling", "unreferenced", "weak_dangling", "weak_unreferenced")
IFP2_KEYS = ("live_offsets", "live_targets", "live_degree", "dangling_ids", "source_offsets", "source_ids")


def top100(values):
    return np.lexsort((np.arange(values.size), -values))[:100]


def _host_edges(config: str, scale: int | None):
    import oracle
    from paper_2302_03245_b200 import synthetic
    if config == "c5":
        return oracle.rmat_graph_edges(26, 16, seed=0)
    if config == "rmat":
        return oracle.rmat_graph_edges(scale, 16, seed=0)
    return synthetic.make(config, seed=0)


def _device_graph(config: str, scale: int | None, n, src, dst):
    import paper_2302_03245_b200 as P
    if config in ("c5", "rmat"):
        s = 26 if config == "c5" else scale
        dev = P.graph.DeviceGraph.rmat(s, 16, seed=0)      # generated, de-duplicated and built on the device
        return P.graph.Graph(dev, raw_edge_count=16 << s, name=config)
    return P.from_edges(n, src, dst, name=config)


def run(config: str, algos=("ifp2", "ifp1"), modes=("auto", "pull", "push"), xi: float = 1e-10,
        threads: int = 0, scale: int | None = None, log=print) -> dict:
    """Runs every check; returns a JSON-able verdict (raises nothing: the
    caller asserts on ``verdict['ok']``)."""
    import oracle
    import paper_2302_03245_b200 as P
    threads = threads or (os.cpu_count() or 1)
    out = {"config": config if config != "rmat" else f"rmat scale={scale} ef=16 (forced C5 code path)",
           "xi": xi, "threads": threads, "checks": [], "ok": True}

    def check(name, ok, **kw):
        out["checks"].append(dict(name=name, ok=bool(ok), **kw))
        out["ok"] = out["ok"] and bool(ok)
        log(f"[parity {config}] {name}: {'ok' if ok else 'FAIL'} {kw if kw else ''}")

    t0 = time.perf_counter()
    n, src, dst = _host_edges(config, scale)
    out["edges_raw"] = int(src.size)
    g = _device_graph(config, scale, n, src, dst)
    ref = oracle.from_edges(n, src, dst)
    del src, dst
    out["n"], out["m"] = int(ref.n), int(ref.m)
    log(f"[parity {config}] n={ref.n} m={ref.m} built in {time.perf_counter() - t0:.1f}s")
    check("graph n/m", g.n == ref.n and g.m == ref.m, device=[int(g.n), int(g.m)], oracle=[int(ref.n), int(ref.m)])
    for k in INT_KEYS:
        check(f"from_edges {k} bit-exact", np.array_equal(getattr(g, k), getattr(ref, k)))
    cls = P.classify(g)
    rc = oracle.classify(ref)
    for k in CLS_KEYS:
        check(f"classify {k} bit-exact", np.array_equal(getattr(cls, k), getattr(rc, k)), count=int(len(getattr(rc, k))))
    check("classify m_d", cls.dangling_edge_count == rc.dangling_edge_count, m_d=int(rc.dangling_edge_count))
    check("dangling_target_counts bit-exact",
          np.array_equal(P.dangling_target_counts(g, cls), oracle.dangling_target_counts(ref, rc.dangling)))
    pg = P.preprocess_ifp2(g, cls)
    rp = oracle.preprocess_ifp2(ref, rc.dangling)
    for k in IFP2_KEYS:
        check(f"preprocess_ifp2 {k} bit-exact", np.array_equal(getattr(pg, k), getattr(rp, k)))
    # drop the device graph's host exports before the long oracle runs
    for obj in (g, pg):
        obj._arrays = None
    cfg = P.SolverConfig(threshold=xi)
    for algo in algos:
        t1 = time.perf_counter()
        o = oracle.sync_simulate(ref, algo, threshold=xi, threads=threads, pg=rp if algo == "ifp2" else None)
        log(f"[parity {config}] oracle {algo}: {o.iterations} rounds in {time.perf_counter() - t1:.1f}s")
        for mode in modes:
            t2 = time.perf_counter()
            if algo == "ifp2":
                vec, tr = P.ifp2_run(pg, cfg, mode=mode)
            else:
                vec, tr = P.ifp1_run(g, cls, cfg, mode=mode)
            wall = time.perf_counter() - t2
            l1 = float(np.abs(vec.values - o.values).sum())
            same_top = bool(np.array_equal(top100(vec.values), top100(o.values)))
            kw = dict(l1=l1, top100_identical=same_top, rounds=int(tr.meta.get("rounds", -1)),
                      oracle_rounds=int(o.iterations), mass=float(vec.values.sum()), wall_s=round(wall, 3))
            ok = l1 <= 1e-9 and same_top and abs(vec.values.sum() - 1.0) <= 1e-12
            if algo == "ifp2":
                kw["push_ops_dangling"] = int(tr.final.push_ops_dangling)
                ok = ok and tr.final.push_ops_dangling == rc.dangling_edge_count
            else:
                ok = ok and tr.final.push_ops_dangling >= rc.dangling_edge_count
            check(f"{algo} {mode} vs oracle sync twin", ok, **kw)
        del o
    out["wall_s"] = round(time.perf_counter() - t0, 1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--scale", type=int, default=None, help="config 'rmat': R-MAT scale (ef 16)")
    ap.add_argument("--algos", default="ifp2,ifp1")
    ap.add_argument("--modes", default="auto,pull,push")
    ap.add_argument("--xi", type=float, default=1e-10)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    v = run(a.config, tuple(a.algos.split(",")), tuple(a.modes.split(",")), a.xi, a.threads, a.scale)
    s = json.dumps(v, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")
    print(json.dumps({"config": v["config"], "ok": v["ok"], "wall_s": v["wall_s"]}))
    sys.exit(0 if v["ok"] else 1)


if __name__ == "__main__":
    main()
