"""Phase timing of bench.py's e2e step at any config (C5 built on the device):
pinned int64 host graph -> preprocess_ifp2 (upload) -> ifp2_run -> vector.
Run with PUSHRANK_TIMING=1 for the library's own phase marks.
Usage: python tools/e2e_phases.py [c5|c2|...] [steps]"""
import os
import sys
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2302_03245_b200 as P  # noqa: E402
from paper_2302_03245_b200.graph import DeviceGraph  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if cfg_name == "c5":
    g = P.graph.Graph(DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
else:
    n, src, dst = bench.make_host_graph(cfg_name)
    g = P.from_edges(n, src, dst, name=cfg_name)
host = bench.host_graph(g)
del g
torch.cuda.synchronize()
base = {k: getattr(host, k) for k in ("n", "m", "out_offsets", "out_targets", "in_offsets", "in_sources")}
cfg = P.SolverConfig(threshold=1e-10)
for i in range(steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    obj = SimpleNamespace(**base)
    pg = P.preprocess_ifp2(obj, None)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    vec, tr = P.ifp2_run(pg, cfg, mode="auto", sample_every=float("inf"))
    t2 = time.perf_counter()
    del obj, pg, vec
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"step {i}: preprocess_ifp2(upload) {1e3*(t1-t0):.1f} ms, ifp2_run {1e3*(t2-t1):.1f} "
          f"(device solve {tr.meta.get('device_ms', float('nan')):.1f}), free {1e3*(t3-t2):.1f}, "
          f"total {1e3*(t3-t0):.1f}", flush=True)
