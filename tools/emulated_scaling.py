"""Rounds and per-rank kernel time of the partitioned path at P = 1, 2, 4, 8
with the ranks EMULATED on one GPU (distributed.run_emulated's loop: every
rank's round is its own launch on the shared stream, in rank order; no kernel
waits on another).  Not a multi-GPU measurement: it gives what one GPU can
give -- the round count of rank-local Gauss-Seidel sections at each P (the
algorithmic part of scaling) and each rank's own kernel time per round (its
partition's sweep with the fused stores landing in local HBM instead of
crossing NVLink) -- and a modelled solve time  sum over rounds of the slowest
rank's kernel + a fixed per-round cost for the statistics all-reduce.

    python tools/emulated_scaling.py c5 1 2 4 8
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2302_03245_b200 as P  # noqa: E402
from paper_2302_03245_b200 import distributed as D, synthetic  # noqa: E402

ALLREDUCE_US = 30.0   # assumed cost of the 9-double all-reduce + launch gap per round (not measured)


def solve(g, parts, algorithm="ifp2", damping=0.85, threshold=1e-10):
    plist = [D.partition_device(g, parts, r, algorithm, damping, threshold) for r in range(parts)]
    steps = [D.CudaLocalStep(p, damping, threshold, algorithm, device=0, fast=True) for p in plist]
    dev = torch.device("cuda", 0)
    stats = torch.zeros((parts, 9), dtype=torch.float64, device=dev)
    ptrs = [q for r, st in enumerate(steps) for q in st.share_buffers(parts, r)]
    for r, st in enumerate(steps):
        st.set_peer_ptrs(parts, r, ptrs)
    stream = steps[0].stream
    per_round = []
    out = None
    for rep in range(2):   # the second solve is the timed one (schedules built, rows sorted)
        for r, st in enumerate(steps):
            st.init_fused(stats[r])
        rounds, per_round, push_ops = 0, [], 0
        while True:
            torch.cuda.synchronize()
            host = stats.cpu().numpy()
            push_ops += int(host[:, 5].sum())
            if host[:, 3].sum() == 0:
                break
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(parts + 1)]
            ev[0].record(stream)
            for r, st in enumerate(steps):
                st.round_fused(rounds, stats[r])
                ev[r + 1].record(stream)
            torch.cuda.synchronize()
            per_round.append([ev[r].elapsed_time(ev[r + 1]) for r in range(parts)])
            rounds += 1
        t = np.array(per_round)
        out = {"parts": parts, "rounds": rounds, "push_ops": push_ops,
               "sections": [int(st.launches_per_round()) for st in steps],
               "owned": [int(p.owned) for p in plist],
               "rank_kernel_ms_total": [round(float(x), 2) for x in t.sum(axis=0)],
               "sum_over_rounds_of_slowest_rank_ms": round(float(t.max(axis=1).sum()), 2),
               "mean_round_slowest_rank_us": round(1e3 * float(t.max(axis=1).mean()), 1),
               "exchange_entries": int(sum(st.exchange_entries() for st in steps))}
    out["modelled_solve_ms"] = round(out["sum_over_rounds_of_slowest_rank_ms"] + out["rounds"] * ALLREDUCE_US / 1e3, 2)
    del steps, plist
    torch.cuda.empty_cache()
    return out


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    counts = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    if cfg == "c5":
        g = P.graph.Graph(P.graph.DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
    else:
        n, s, d = synthetic.make(cfg, seed=0)
        g = P.from_edges(n, s, d)
    base = None
    for parts in counts:
        row = solve(g, parts)
        row["config"] = cfg
        if base is None:
            base = row
        row["modelled_speedup_vs_first"] = round(base["modelled_solve_ms"] / row["modelled_solve_ms"], 2)
        row["modelled_gteps"] = round(row["push_ops"] / row["modelled_solve_ms"] / 1e6, 1)
        row["modelled_gteps_efficiency"] = round(row["modelled_gteps"] / (base["modelled_gteps"] * parts / base["parts"]), 3)
        row["note"] = (f"ranks emulated on one GPU; kernel times are each rank's own launch; {ALLREDUCE_US:.0f} us per round "
                       f"assumed for the all-reduce; NVLink store latency not modelled")
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
