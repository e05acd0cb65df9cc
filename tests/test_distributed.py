"""Multi-rank host path (vertex-range partitioning + per-round exchange) on CPU.

World size 2 over gloo on 127.0.0.1, with the numpy local step.  The
partitioned bulk-synchronous rounds must reproduce the single-process
round-synchronous twin bit-for-bit: the same reserved/pending state, the
same integer trace columns and the same round count.  Both sum each
destination's inflow in ascending source order, as engines.py:446 does.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2302_03245_b200 import distributed as D
from paper_2302_03245_b200 import synthetic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, config, algorithm, out_q, queued=False, relabel=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, src, dst = synthetic.make(config, seed=0)
        g = oracle.from_edges(n, src, dst)
        order = D.run_order(np.diff(g.out_offsets), np.diff(g.in_offsets)) if relabel else None
        part = D.partition_graph(g, world, rank, algorithm, order=order)
        step = D.NumpyLocalStep(part, 0.85, 1e-10, algorithm)
        comm = D.Comm()
        if queued:
            # rounds queued in batches of 5 (partial last batch, no-op rounds past the end)
            vals, rows, info = D.run_partitioned_queued(step, comm, part, algorithm, 0.85, 1e-10,
                                                        conv_scope_all=True, batch=5)
        else:
            vals, rows, info = D.run_partitioned(step, comm, part, algorithm, 0.85, 1e-10, conv_scope_all=True)
        out_q.put((rank, part.lo, part.hi, step.reserved, step.h, vals, rows, info))
    finally:
        dist.destroy_process_group()


def _run(world, config, algorithm, queued=False, relabel=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, config, algorithm, q, queued, relabel)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def test_edge_balanced_ranges():
    deg = np.array([100, 0, 0, 0, 50, 50, 1, 1, 1, 1], np.int64)
    b = D.edge_balanced_ranges(deg, 2)
    assert b[0] == 0 and b[-1] == deg.size and np.all(np.diff(b) >= 0)
    w = deg + D.ROW_COST
    loads = [w[b[i]:b[i + 1]].sum() for i in range(2)]
    assert max(loads) - min(loads) <= w.max()
    with pytest.raises(ValueError):
        D.edge_balanced_ranges(deg, 0)
    # only receiving rows weigh: the in-degree-0 tail and (IFP2) the dangling
    # receivers cost a rank nothing after rounds 0-1
    outd = np.array([3, 2, 0, 1, 0, 4, 1, 0, 2, 2], np.int64)
    for algo in ("ifp1", "ifp2"):
        rec = D.receiving_rows(deg, outd, algo)
        assert rec.tolist() == [bool(d > 0 and (algo == "ifp1" or o > 0)) for d, o in zip(deg, outd)]
        b = D.edge_balanced_ranges(deg, 3, rec)
        assert b[0] == 0 and b[-1] == deg.size and np.all(np.diff(b) >= 0)
        w = np.where(rec, deg + D.ROW_COST, 0)
        loads = [w[b[i]:b[i + 1]].sum() for i in range(3)]
        assert sum(loads) == w.sum() and max(loads) - min(loads) <= 2 * w.max()


def test_partition_covers_graph():
    n, src, dst = synthetic.make("c1", seed=0)
    g = oracle.from_edges(n, src, dst)
    parts = [D.partition_graph(g, 3, r, "ifp1") for r in range(3)]
    assert sum(p.owned for p in parts) == n
    assert sum(p.in_sources.size for p in parts) == g.m
    # padded ids invert to the original sources, in the original row order
    p = parts[1]
    S = p.slot
    back = p.bounds[p.in_sources // S] + p.in_sources % S
    assert np.array_equal(back, g.in_sources[g.in_offsets[p.lo]:g.in_offsets[p.hi]])


@pytest.mark.parametrize("queued", [False, True])
@pytest.mark.parametrize("algorithm", ["ifp1", "ifp2"])
def test_two_ranks_match_sync_twin_bit_exact(algorithm, queued):
    """Host-synchronised rounds and rounds queued in batches (statistics read
    back every 5 rounds) give the same state, trace and round count."""
    res = _run(2, "c1", algorithm, queued)
    n, src, dst = synthetic.make("c1", seed=0)
    g = oracle.from_edges(n, src, dst)
    o = oracle.sync_simulate(g, algorithm, threshold=1e-10)
    reserved = np.concatenate([r[3] for r in res])
    h = np.concatenate([r[4] for r in res])
    assert np.array_equal(reserved, o.reserved)
    assert np.array_equal(h, o.h)
    rows = res[0][6]
    for col in ("converged", "work", "push_ops", "push_ops_dangling"):
        assert [r[col] for r in rows] == o.rows[col].tolist(), col
    np.testing.assert_allclose([r["h_l1"] for r in rows], o.rows["h_l1"], rtol=1e-12)
    assert res[0][7]["rounds"] == o.iterations
    vals = np.concatenate([r[5] for r in res])
    np.testing.assert_allclose(vals, o.values, rtol=1e-13, atol=0)
    if algorithm == "ifp2":
        assert res[0][7]["settled"] == int((g.out_degree == 0)[g.out_targets].sum())


def test_run_order_partitions_bit_exact():
    """Partitions of the run layout (vertices renumbered as the engines do,
    csrc/graph.cu k_relabel_keys): each row keeps its sources' original
    order, so the sequential sums -- and the state, trace and values, once
    un-permuted -- still equal the sync twin bit for bit."""
    n, src, dst = synthetic.make("c1", seed=0)
    g = oracle.from_edges(n, src, dst)
    order = D.run_order(np.diff(g.out_offsets), np.diff(g.in_offsets))
    assert np.array_equal(np.sort(order), np.arange(n))
    indeg = np.diff(g.in_offsets)[order]
    outdeg = np.diff(g.out_offsets)[order]
    cls = np.where(outdeg > 0, np.where(indeg > 0, 0, 1), np.where(indeg > 0, 2, 3))
    assert np.all(np.diff(cls) >= 0)
    first = cls == 0
    assert np.all(np.diff(indeg[first]) <= 0)
    for algorithm in ("ifp1", "ifp2"):
        res = _run(2, "c1", algorithm, queued=True, relabel=True)
        o = oracle.sync_simulate(g, algorithm, threshold=1e-10)
        reserved = np.empty(n)
        reserved[order] = np.concatenate([r[3] for r in res])
        assert np.array_equal(reserved, o.reserved)
        vals = np.empty(n)
        vals[order] = np.concatenate([r[5] for r in res])
        np.testing.assert_allclose(vals, o.values, rtol=1e-13, atol=0)
        assert [r["push_ops"] for r in res[0][6]] == o.rows["push_ops"].tolist()
