"""Phase timing of the e2e path (host graph -> upload -> preprocess -> solve -> D2H)."""
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_03245_b200 as P
from paper_2302_03245_b200 import _lib, synthetic
from paper_2302_03245_b200.graph import DeviceGraph


def t():
    _lib.context().synchronize()
    return time.perf_counter()


cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, src, dst = synthetic.make(cfg)
g = P.from_edges(n, src, dst)
import torch
host = SimpleNamespace(n=g.n, m=g.m, **{k: torch.from_numpy(np.ascontiguousarray(getattr(g, k))).pin_memory().numpy()
                                        for k in ("out_offsets", "out_targets", "in_offsets", "in_sources")})
for it in range(4):
    t0 = t()
    dev = DeviceGraph.upload(host)
    t1 = t()
    dev.preprocess_ifp2()
    t2 = t()
    vals, rows, res, _, _ = dev.run("ifp2", "auto", 0.85, 1e-10, 1_000_000, 0, row_cap=1)
    t3 = t()
    vals, rows, res, _, _ = dev.run("ifp2", "auto", 0.85, 1e-10, 1_000_000, 0, row_cap=1)
    t4 = t()
    del dev
    t5 = t()
    print(f"iter {it}: upload {1e3*(t1-t0):.1f} ms, preprocess_ifp2 {1e3*(t2-t1):.1f}, first run "
          f"{1e3*(t3-t2):.1f} (device {res.push_ms:.1f}), second run {1e3*(t4-t3):.1f}, free {1e3*(t5-t4):.1f}")
