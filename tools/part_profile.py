"""Where the partitioned path's time goes at one rank (diagnostic).

    PUSHRANK_DEVICE=0 python tools/part_profile.py c2 [--fused 0|1] [--batch 16]

One NCCL rank (world size 1), the device-built partition of the config, a
few solves of run_partitioned_queued under torch.profiler (CUPTI kernel
records, no nsys needed): per-kernel device time, the solve's span and the
device-idle share, against the single-GPU engine's solve time.
"""
import argparse
import collections
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_03245_b200 as P  # noqa: E402
from paper_2302_03245_b200 import distributed as D, synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--algo", default="ifp2")
    a = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    torch.cuda.set_device(0)
    if a.config == "c5":
        g = P.graph.Graph(P.graph.DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
    else:
        n, s, d = synthetic.make(a.config, seed=0)
        g = P.from_edges(n, s, d)
    part = D.partition_device(g, 1, 0, a.algo, 0.85, 1e-10)
    step = D.CudaLocalStep(part, 0.85, 1e-10, a.algo, device=0, fast=True)
    comm = D.Comm(device=torch.device("cuda", 0))
    fused = bool(a.fused) and step.setup_fused(comm)

    def solve():
        return D.run_partitioned_queued(step, comm, part, a.algo, 0.85, 1e-10, batch=a.batch, host_values=False,
                                        fused=fused)

    for _ in range(3):
        solve()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        _, _, info = solve()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 3
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        solve()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        agg[e.name[:70]][0] += 1
        agg[e.name[:70]][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    busy = sum(v[1] for v in agg.values())
    print(f"{a.config} {a.algo} fused={fused} batch={a.batch}: solve wall {wall * 1e3:.3f} ms, rounds {info['rounds']}, "
          f"device kernel time {busy / 1e3:.3f} ms")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
        print(f"  {k:70s} {c:5d} {t / 1e3:9.3f} ms")
    dev = g.dev
    from paper_2302_03245_b200 import _lib
    for _ in range(2):
        dev.run(a.algo, "auto", 0.85, 1e-10, 1_000_000, _lib.CONV_SCAN)
    _, _, res, _, _ = dev.run(a.algo, "auto", 0.85, 1e-10, 1_000_000, _lib.CONV_SCAN)
    print(f"  engine: {res.push_ms:.3f} ms device, {res.rounds} rounds")
    if fused:
        step.close_fused(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
