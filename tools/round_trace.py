"""Per-round trace of one solve (C5 built on the device): pushed edges,
drained vertices and device time per round, to see how much of each dense
sweep gathers shares of inactive sources.  Usage: tools/round_trace.py [c5|c3|...] [ifp2|ifp1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2302_03245_b200 as P  # noqa: E402
from paper_2302_03245_b200 import _lib  # noqa: E402
from paper_2302_03245_b200.graph import DeviceGraph  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
algo = sys.argv[2] if len(sys.argv) > 2 else "ifp2"
if cfg == "c5":
    g = P.graph.Graph(DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
else:
    n, s, d = bench.make_host_graph(cfg)
    g = P.from_edges(n, s, d, name=cfg)
P.preprocess_ifp2(g, P.classify(g))
dev = g.dev
for rep in range(2):
    _, rows, res, _, _ = dev.run(algo, "auto", 0.85, 1e-10, 1_000_000, _lib.CONV_SCAN, row_cap=1 << 16)
m_live = int(dev.preprocess_ifp2().live_edges) if algo == "ifp2" else g.m
print(f"{cfg} {algo}: rounds {res.rounds} (pull {res.pull_rounds}, push {res.push_rounds}), push_ops {res.push_ops}, "
      f"solve {res.push_ms:.1f} ms, live edges {m_live}")
po = rows["push_ops"].astype(np.int64)
wk = rows["work"].astype(np.int64)
ms = rows["wall_ms"]
print("round  pushed_edges  frac_of_live  work  dt_ms")
for t in range(1, len(rows)):
    dp = po[t] - po[t - 1]
    print(f"{t:5d} {dp:13d} {dp / max(m_live, 1):12.3f} {wk[t]:10d} {ms[t] - ms[t - 1]:7.3f}")
