"""Share-gather locality of a config's IFP2 pull sweep (diagnostic).

    python tools/hot_sources.py [c5|c3|c2]

For the run layout (class, then descending in-degree), prints the fraction
of the dense sweep's edges whose source id is below H, per degree bin
(hub > 4096 in-edges, warp > 64, thread rows), for H = 2^10 .. 2^24.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_03245_b200 as P  # noqa: E402
from paper_2302_03245_b200 import distributed as D, synthetic  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    if cfg == "c5":
        g = P.graph.Graph(P.graph.DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
    else:
        n, s, d = synthetic.make(cfg, seed=0)
        g = P.from_edges(n, s, d)
    in_off = np.asarray(g.in_offsets)
    out_deg = np.diff(np.asarray(g.out_offsets))
    in_deg = np.diff(in_off)
    order = D.run_order(out_deg, in_deg)
    n = order.size
    dev = torch.device("cuda")
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    rank[torch.from_numpy(order).to(dev)] = torch.arange(n, device=dev)
    src = torch.from_numpy(np.asarray(g.in_sources)).to(dev)
    indeg = torch.from_numpy(in_deg).to(dev)
    tgt = torch.repeat_interleave(torch.arange(n, device=dev), indeg)
    cls0 = (torch.from_numpy(out_deg).to(dev) > 0) & (indeg > 0)
    keep = cls0[tgt]
    s_run = rank[src[keep]]
    d_t = indeg[tgt[keep]]
    del src, tgt
    bins = {"hub": d_t > 4096, "warp": (d_t > 64) & (d_t <= 4096), "thread": d_t <= 64}
    tot = s_run.numel()
    print(f"{cfg}: n={n} sweep edges={tot} class0 rows={int(cls0.sum())}")
    lg = torch.floor(torch.log2(s_run.double() + 1)).long()
    hdr = "H      " + "  ".join(f"{k:>14s}" for k in ["all"] + list(bins))
    print(hdr)
    cums = {}
    for k, m in [("all", None)] + list(bins.items()):
        h = torch.bincount(lg if m is None else lg[m], minlength=40).double()
        cums[k] = (torch.cumsum(h, 0) / max(h.sum().item(), 1)).cpu().numpy(), int(h.sum().item())
    for b in range(10, 25):
        row = [f"{cums[k][0][b - 1]:.3f} ({cums[k][1] / 1e6:6.0f}M)" for k in ["all"] + list(bins)]
        print(f"2^{b:<4d} " + "  ".join(f"{r:>14s}" for r in row))


if __name__ == "__main__":
    main()
