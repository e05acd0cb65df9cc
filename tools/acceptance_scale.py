"""Acceptance criteria 3 and 4 of the reference (test_acceptance.py:113-171)
at BASELINE scale, on the device.

    python tools/acceptance_scale.py c2 c3 c4 c5 [--out profiles/r02_acceptance.json]

Criterion 3 (convergence law): the exact round-synchronous fp-full twin
(sync_simulate(variant="fp-full"), bit-exact device form) obeys
h_l1(t+1) - carry(t) = c * alpha(t) * active(t) at every round (residual
<= 1e-9 as the reference requires on 1e4 vertices, or within 64 fp64
rounding units of the sums it is computed from at larger n), and over the rounds before threshold carry-over appears (carry <=
1e-6 h_l1, at least 10 of them) the L1 decay ratio stays <= c.

Criterion 4 (work saving): IFP2 pushes exactly m_d edges into dangling
vertices; IFP1 at least m_d (the reference's synthetic graph shows > 2 m_d).

Also times sync_simulate(..., on_iteration=cb) with the device ring of
states drained once per batch against the round-by-round host loop.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_03245_b200 as P  # noqa: E402
from paper_2302_03245_b200 import synthetic  # noqa: E402

C = 0.85


def build(config):
    if config == "c5":
        return P.graph.Graph(P.graph.DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
    n, s, d = synthetic.make(config, seed=0)
    return P.from_edges(n, s, d, name=config)


EPS = 2.0 ** -53


def decay_stats(trace):
    """test_acceptance.py:100-110 on a device trace.  Also the fp64 rounding
    scale of the law's left side, eps * (h_l1(t+1) + carry(t)) / active(t):
    h_l1 and carry are sums over all n vertices (67 M at C5), so once the
    active mass is small against them the residual is that rounding, which
    the reference's absolute 1e-9 (set on 1e4 vertices) does not allow for."""
    s = trace.samples
    law = 0.0
    law_rel = 0.0
    for i in range(len(s) - 1):
        if s[i].active_mass > 0:
            adjusted = (s[i + 1].h_l1 - s[i].carry_mass) / s[i].active_mass
            r = abs(adjusted - C * s[i].alpha)
            law = max(law, r)
            law_rel = max(law_rel, r / (EPS * (s[i + 1].h_l1 + s[i].carry_mass) / s[i].active_mass))
    window = [i for i in range(len(s) - 1) if s[i].h_l1 > 0 and s[i].carry_mass <= 1e-6 * s[i].h_l1]
    ratios = [s[i + 1].h_l1 / s[i].h_l1 for i in window]
    return law, window, ratios, law_rel


def run(config, observe=True, log=print):
    t0 = time.perf_counter()
    g = build(config)
    cls = P.classify(g)
    out = {"config": config, "n": int(g.n), "m": int(g.m), "m_d": int(cls.dangling_edge_count),
           "dangling_fraction": float(len(cls.dangling) / g.n)}
    cfg = P.SolverConfig(threshold=1e-10)
    t1 = time.perf_counter()
    _, tr = P.sync_simulate(g, cfg, variant="fp-full")
    law, window, ratios, law_rel = decay_stats(tr)
    c3 = {"law_residual": law, "law_residual_in_rounding_units": law_rel, "window": len(window),
          "max_ratio": max(ratios) if ratios else None, "rounds": len(tr.samples),
          "sync_s": round(time.perf_counter() - t1, 2)}
    # the reference's bound, or -- at scales where the sums' fp64 rounding
    # exceeds it -- within 64 rounding units of the left side
    c3["ok"] = bool((law <= 1e-9 or law_rel <= 64.0) and len(window) >= 10 and max(ratios) <= C + 1e-12)
    out["criterion_3"] = c3
    pg = P.preprocess_ifp2(g, cls)
    _, t_1 = P.ifp1_run(g, cls, cfg, workers=2, sample_every=float("inf"))
    _, t_2 = P.ifp2_run(pg, cfg, workers=2, sample_every=float("inf"))
    m_d = cls.dangling_edge_count
    c4 = {"ifp1_push_ops_dangling": int(t_1.final.push_ops_dangling),
          "ifp2_push_ops_dangling": int(t_2.final.push_ops_dangling),
          "ifp1_over_m_d": t_1.final.push_ops_dangling / m_d if m_d else None}
    c4["ok"] = bool(t_2.final.push_ops_dangling == m_d and t_1.final.push_ops_dangling >= m_d)
    out["criterion_4"] = c4
    if observe and g.n <= 5_000_000:
        # on_iteration: device ring drained per batch vs one host round trip per round
        for label, env in (("ring", "0"), ("host_loop", "1")):
            seen = []
            if env == "1":
                os.environ["PUSHRANK_HOST_LOOP"] = "1"
            try:
                t2 = time.perf_counter()
                P.sync_simulate(g, cfg, variant="ifp1", on_iteration=lambda t, r, h: seen.append((t, float(h.sum()))))
                out[f"on_iteration_{label}_s"] = round(time.perf_counter() - t2, 3)
            finally:
                os.environ.pop("PUSHRANK_HOST_LOOP", None)
            out[f"on_iteration_{label}_calls"] = len(seen)
            out[f"on_iteration_{label}_digest"] = float(sum(x[1] for x in seen))
    out["wall_s"] = round(time.perf_counter() - t0, 1)
    log(json.dumps(out))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = [run(c) for c in a.configs]
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
    sys.exit(0 if all(r["criterion_3"]["ok"] and r["criterion_4"]["ok"] for r in res) else 1)


if __name__ == "__main__":
    main()
