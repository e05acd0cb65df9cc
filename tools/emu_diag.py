"""Diagnostic: emulated P-rank solve at C5 -- residual decay per round and the
result against the single-GPU engine.  python tools/emu_diag.py PARTS"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_03245_b200 as P
from paper_2302_03245_b200 import distributed as D

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
if cfg == "c5":
    g = P.graph.Graph(P.graph.DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
else:
    from paper_2302_03245_b200 import synthetic
    n, s, d = synthetic.make(cfg, seed=0)
    g = P.from_edges(n, s, d)
plist = [D.partition_device(g, parts, r, "ifp2", 0.85, 1e-10) for r in range(parts)]
steps = [D.CudaLocalStep(p, 0.85, 1e-10, "ifp2", device=0, fast=True) for p in plist]
print("bounds", plist[0].bounds.tolist(), "sections", [s.launches_per_round() for s in steps])
dev = torch.device("cuda", 0)
stats = torch.zeros((parts, 9), dtype=torch.float64, device=dev)
ptrs = [q for r, st in enumerate(steps) for q in st.share_buffers(parts, r)]
for r, st in enumerate(steps):
    st.set_peer_ptrs(parts, r, ptrs)
    st.init_fused(stats[r])
rounds, trace = 0, []
while True:
    torch.cuda.synchronize()
    h = stats.cpu().numpy()
    trace.append((h[:, 0].sum(), h[:, 1].sum(), int(h[:, 3].sum())))
    if h[:, 3].sum() == 0:
        break
    for r, st in enumerate(steps):
        st.round_fused(rounds, stats[r])
    rounds += 1
print("rounds", rounds)
n_d = None
for t in range(0, len(trace), max(1, len(trace) // 25)):
    l1, above, nact = trace[t]
    print(f"t={t:4d} h_l1={l1:.6e} active_mass={above:.6e} nact={nact}")
S = plist[0].slot
x = torch.zeros(S * parts, dtype=torch.float64, device=dev)
for r, st in enumerate(steps):
    st.settle_shares(x[r * S:(r + 1) * S])
for st in steps:
    st.settle(x)
total = sum(st.local_total() for st in steps)
vals = np.concatenate([st.values(total) for st in steps])   # run-layout order
pg = P.preprocess_ifp2(g, P.classify(g))
vec, tr = P.ifp2_run(pg, P.SolverConfig(threshold=1e-10))
perm = np.asarray(g.dev.run_perm()) if hasattr(g.dev, "run_perm") else None
ref = vec.values
if perm is None:
    # run order from the degrees (distributed.run_order)
    order = D.run_order(np.diff(np.asarray(g.out_offsets)), np.diff(np.asarray(g.in_offsets)))
    full = np.empty(g.n); full[order] = vals
else:
    full = np.empty(g.n); full[perm] = vals
print("mass", full.sum(), "L1 vs engine", np.abs(full - ref).sum(), "engine rounds", tr.meta.get("rounds"))
