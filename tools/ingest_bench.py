"""Edge-list ingest timing: device load_edge_list vs the host path the
reference takes (pandas parse + numpy first-appearance remap), on C2 as text."""
import os
import sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_03245_b200 as P
from paper_2302_03245_b200 import synthetic, _lib
from paper_2302_03245_b200.ingest import _host_parse

n, src, dst = synthetic.make(sys.argv[1] if len(sys.argv) > 1 else "c2")
rng = np.random.default_rng(1)
ids = rng.integers(0, 1 << 40, size=n)
lines = np.char.add(np.char.add(ids[src].astype(str), " "), ids[dst].astype(str))
text = ("\n".join(lines.tolist()) + "\n").encode()
print(f"text {len(text)/1e6:.1f} MB, {src.size} edges")
ts = []
for i in range(4):
    _lib.context().synchronize()
    t0 = time.perf_counter()
    g = P.load_edge_list(text)
    _lib.context().synchronize()
    ts.append(time.perf_counter() - t0)
    del g
print(f"device load_edge_list: {1e3*min(ts[1:]):.1f} ms (first call {1e3*ts[0]:.1f} ms)")
t0 = time.perf_counter()
s, d = _host_parse(text)
t1 = time.perf_counter()
flat = np.empty(s.size * 2, np.int64); flat[0::2] = s; flat[1::2] = d
u, first = np.unique(flat, return_index=True)
app = np.argsort(first, kind="stable")
rank = np.empty(u.size, np.int64); rank[app] = np.arange(u.size)
dense = rank[np.searchsorted(u, flat)]
t2 = time.perf_counter()
print(f"host path (reference's ingest steps): parse {1e3*(t1-t0):.0f} ms + remap {1e3*(t2-t1):.0f} ms")
