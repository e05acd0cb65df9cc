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


def _worker(rank, world, port, algorithm, q, fast=False):
    import torch.distributed as dist
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, src, dst = synthetic.make("c1", seed=0)
        g = oracle.from_edges(n, src, dst)
        # the fast form partitions the run layout, as bench.py does
        order = D.run_order(np.diff(g.out_offsets), np.diff(g.in_offsets)) if fast else None
        part = D.partition_graph(g, world, rank, algorithm, order=order)
        step = D.CudaLocalStep(part, 0.85, 1e-10, algorithm, device=0, fast=fast)
        if fast:
            vals, rows, info = D.run_partitioned_queued(step, D.Comm(), part, algorithm, 0.85, 1e-10,
                                                        conv_scope_all=True, batch=5)
        else:
            vals, rows, info = D.run_partitioned(step, D.Comm(), part, algorithm, 0.85, 1e-10,
                                                 conv_scope_all=True)
        r, h = step.export()
        if fast:
            # back to original ids: this rank owns new ids [lo, hi) = order[lo:hi]
            q.put((rank, r, h, vals, rows, info, order[part.lo:part.hi]))
        else:
            q.put((rank, r, h, vals, rows, info))
    finally:
        dist.destroy_process_group()


def _run(algorithm, fast):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, algorithm, q, fast)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("algorithm", ["ifp1", "ifp2"])
def test_cuda_partitions_match_sync_twin(algorithm):
    res = _run(algorithm, False)
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make("c1", seed=0)
    o = oracle.sync_simulate(oracle.from_edges(n, src, dst), algorithm, threshold=1e-10)
    assert np.array_equal(np.concatenate([x[1] for x in res]), o.reserved)
    assert np.array_equal(np.concatenate([x[2] for x in res]), o.h)
    assert [r["push_ops"] for r in res[0][4]] == o.rows["push_ops"].tolist()
    np.testing.assert_allclose(np.concatenate([x[3] for x in res]), o.values, rtol=1e-13, atol=0)


@pytest.mark.parametrize("algorithm", ["ifp1", "ifp2"])
def test_fast_partitions_queued(algorithm):
    """The fast local step (binned dense-round gather over each partition's
    receiving rows, csrc/part.cu k_part_pull) with rounds queued in batches:
    the same fixed point as the sync twin (L1 <= 1e-9, identical top-100),
    mass 1, and run-to-run identical vectors."""
    res = _run(algorithm, True)
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make("c1", seed=0)
    o = oracle.sync_simulate(oracle.from_edges(n, src, dst), algorithm, threshold=1e-10)
    vals = np.empty(n)
    vals[np.concatenate([x[6] for x in res])] = np.concatenate([x[3] for x in res])
    assert np.abs(vals - o.values).sum() <= 1e-9
    top = lambda v: np.lexsort((np.arange(v.size), -v))[:100]   # noqa: E731
    assert np.array_equal(top(vals), top(o.values))
    assert abs(vals.sum() - 1.0) <= 1e-12
    assert abs(res[0][5]["rounds"] - o.iterations) <= 1
    res2 = _run(algorithm, True)
    again = np.empty(n)
    again[np.concatenate([x[6] for x in res2])] = np.concatenate([x[3] for x in res2])
    assert np.array_equal(again, vals)


def _emulate(algorithm, parts, fused, config="c1"):
    """distributed.run_emulated on a BASELINE config (ranks in one process)."""
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make(config, seed=0)
    g = oracle.from_edges(n, src, dst)
    vals, rounds = D.run_emulated(g, parts, algorithm, fused=fused)
    return vals, rounds, g


@pytest.mark.parametrize("algorithm", ["ifp1", "ifp2"])
def test_fused_exchange_emulated(algorithm):
    """Fused exchange (round kernels storing shares into every rank's
    replica) with 3 ranks emulated on one device: bit-identical to the
    all-gather form, and the sync twin's fixed point (L1 <= 1e-9, identical
    top-100)."""
    fused, r1, g = _emulate(algorithm, 3, True)
    gathered, r2, _ = _emulate(algorithm, 3, False)
    assert np.array_equal(fused, gathered)
    assert r1 == r2
    o = oracle.sync_simulate(g, algorithm, threshold=1e-10)
    assert np.abs(fused - o.values).sum() <= 1e-9
    top = lambda v: np.lexsort((np.arange(v.size), -v))[:100]   # noqa: E731
    assert np.array_equal(top(fused), top(o.values))
    assert abs(r1 - o.iterations) <= 1


@pytest.mark.parametrize("algorithm", ["ifp2", "ifp1"])
@pytest.mark.parametrize("sections", [2, 3])
def test_rank_local_gauss_seidel_emulated(sections, algorithm, monkeypatch):
    """Rank-local Gauss-Seidel sections in the partitioned local step
    (run-layout partitions; PUSHRANK_GS_SECTIONS forces them at C2; IFP1 by
    the id bound of earlier sections' class-0 sources): 2 ranks emulated on
    one device, fused exchange bit-identical to the all-gather form, the sync
    twin's fixed point (L1 <= 1e-9, identical top-100), and fewer rounds than
    Jacobi."""
    monkeypatch.setenv("PUSHRANK_GS_SECTIONS", str(sections))
    fused, r1, g = _emulate(algorithm, 2, True, config="c2")
    gathered, r2, _ = _emulate(algorithm, 2, False, config="c2")
    assert np.array_equal(fused, gathered)
    assert r1 == r2
    o = oracle.sync_simulate(g, algorithm, threshold=1e-10)
    assert np.abs(fused - o.values).sum() <= 1e-9
    top = lambda v: np.lexsort((np.arange(v.size), -v))[:100]   # noqa: E731
    assert np.array_equal(top(fused), top(o.values))
    assert abs(fused.sum() - 1.0) <= 1e-12
    assert r1 < o.iterations, (r1, o.iterations)
