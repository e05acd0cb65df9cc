"""Share-exchange volume of the partitioned rounds (diagnostic).

    python tools/exchange_volume.py c5 2 4 8

For each rank count P, builds the P device partitions one after another on
this GPU (pr_part_from_graph) and sums their sparse-exchange entries: shares
stored per dense round with the masks (own replica included), against the
dense fused exchange (every rank stores every owned share into all P
replicas: P * n) and the NCCL all-gather ((P-1) * n received in total).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_03245_b200 as P  # noqa: E402
from paper_2302_03245_b200 import distributed as D, synthetic  # noqa: E402


def main():
    cfg = sys.argv[1]
    counts = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
    if cfg == "c5":
        g = P.graph.Graph(P.graph.DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
    else:
        n, s, d = synthetic.make(cfg, seed=0)
        g = P.from_edges(n, s, d)
    n = int(g.n)
    out = []
    for parts in counts:
        total = 0
        for r in range(parts):
            part = D.partition_device(g, parts, r, "ifp2", 0.85, 1e-10)
            step = D.CudaLocalStep(part, 0.85, 1e-10, "ifp2", device=0, fast=True)
            total += step.exchange_entries()
            del step
        row = {"config": cfg, "parts": parts, "n": n, "sparse_entries": total,
               "sparse_remote_lower_bound": total - n, "dense_fused_entries": parts * n,
               "allgather_entries": (parts - 1) * n,
               "sparse_vs_allgather": round((total - n) / max((parts - 1) * n, 1), 3)}
        print(json.dumps(row), flush=True)
        out.append(row)


if __name__ == "__main__":
    main()
