"""Wall-clock breakdown of bench.py's e2e step (pinned host graph -> ifp2_run)."""
import os
import sys, time
from types import SimpleNamespace
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_03245_b200 as P
from paper_2302_03245_b200 import synthetic, _lib
from paper_2302_03245_b200.graph import device_graph

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, src, dst = synthetic.make(cfg_name)
g = P.from_edges(n, src, dst)
arrays = {k: torch.from_numpy(np.ascontiguousarray(getattr(g, k))).pin_memory().numpy()
          for k in ("out_offsets", "out_targets", "in_offsets", "in_sources")}
cfg = P.SolverConfig(threshold=1e-10)
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    obj = SimpleNamespace(n=g.n, m=g.m, **arrays)
    pg = P.preprocess_ifp2(obj, None)
    t1 = time.perf_counter()
    vec, tr = P.ifp2_run(pg, cfg, mode="auto", sample_every=float("inf"))
    t2 = time.perf_counter()
    dev_ms = tr.meta["device_ms"]
    del obj, pg
    t3 = time.perf_counter()
    print(f"step {i}: upload+counts {1e3*(t1-t0):.2f} ms, ifp2_run {1e3*(t2-t1):.2f} (device {dev_ms:.2f}), "
          f"free {1e3*(t3-t2):.2f}, total {1e3*(t3-t0):.2f}")
