"""Partitioned path with the CUDA local step (csrc/part.cu) on one GPU.

Two ranks over gloo, both on cuda:0.  Their kernels never wait on each
other: the ranks meet only in host-side collectives.  The result must equal
the single-process round-synchronous twin bit-for-bit, as the CPU test
requires (tests/test_distributed.py).
"""

import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, algorithm, q):
    import torch.distributed as dist
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, src, dst = synthetic.make("c1", seed=0)
        g = oracle.from_edges(n, src, dst)
        part = D.partition_graph(g, world, rank, algorithm)
        step = D.CudaLocalStep(part, 0.85, 1e-10, algorithm, device=0)
        vals, rows, info = D.run_partitioned(step, D.Comm(), part, algorithm, 0.85, 1e-10, conv_scope_all=True)
        r, h = step.export()
        q.put((rank, r, h, vals, rows, info))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algorithm", ["ifp1", "ifp2"])
def test_cuda_partitions_match_sync_twin(algorithm):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, algorithm, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make("c1", seed=0)
    o = oracle.sync_simulate(oracle.from_edges(n, src, dst), algorithm, threshold=1e-10)
    assert np.array_equal(np.concatenate([x[1] for x in res]), o.reserved)
    assert np.array_equal(np.concatenate([x[2] for x in res]), o.h)
    assert [r["push_ops"] for r in res[0][4]] == o.rows["push_ops"].tolist()
    np.testing.assert_allclose(np.concatenate([x[3] for x in res]), o.values, rtol=1e-13, atol=0)
