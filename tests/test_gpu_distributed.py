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


def _worker_ipc(rank, world, port, algorithm, fused, q):
    """One rank of a real multi-process run on cuda:0: the partition built on
    the device from the rank's own device graph (pr_part_from_graph), the
    shares exchanged through CUDA IPC peer mappings of the other process's
    replicas (pr_part_share_buffers / pr_part_set_peers ->
    cudaIpcOpenMemHandle) or the all-gather; gloo collectives."""
    import torch.distributed as dist
    import paper_2302_03245_b200 as P
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, src, dst = synthetic.make("c2", seed=0)
        g = P.from_edges(n, src, dst)
        part = D.partition_device(g, world, rank, algorithm, 0.85, 1e-10)
        step = D.CudaLocalStep(part, 0.85, 1e-10, algorithm, device=0, fast=True)
        comm = D.Comm()
        ok = step.setup_fused(comm) if fused else False
        vals, rows, info = D.run_partitioned_queued(step, comm, part, algorithm, 0.85, 1e-10, batch=6, fused=ok)
        if ok:
            step.close_fused(comm)
        q.put((rank, ok, part.bounds.tolist(), part.lo, part.hi, vals, info["rounds"]))
    finally:
        dist.destroy_process_group()


def _run_ipc(algorithm, fused):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_ipc, args=(r, 2, port, algorithm, fused, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("algorithm", ["ifp2", "ifp1"])
def test_two_process_ipc_fused_exchange(algorithm):
    """Two processes, one device, C2: partitions built on the device (bounds
    identical to the host rule over the run layout), the fused exchange over
    CUDA IPC mappings between the processes bit-identical to the all-gather
    form, and the sync twin's fixed point (L1 <= 1e-9, identical top-100)."""
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    fused = _run_ipc(algorithm, True)
    assert all(r[1] for r in fused), "CUDA IPC mapping refused"
    gathered = _run_ipc(algorithm, False)
    n, src, dst = synthetic.make("c2", seed=0)
    g = oracle.from_edges(n, src, dst)
    order = D.run_order(np.diff(g.out_offsets), np.diff(g.in_offsets))
    ind, outd = np.diff(g.in_offsets)[order], np.diff(g.out_offsets)[order]
    host_bounds = D.edge_balanced_ranges(ind, 2, D.receiving_rows(ind, outd, algorithm))
    assert fused[0][2] == host_bounds.tolist()
    vals = {}
    for name, res in (("fused", fused), ("gathered", gathered)):
        v = np.empty(n)
        for r in res:
            v[order[r[3]:r[4]]] = r[5]
        vals[name] = v
    assert np.array_equal(vals["fused"], vals["gathered"])
    o = oracle.sync_simulate(g, algorithm, threshold=1e-10)
    assert np.abs(vals["fused"] - o.values).sum() <= 1e-9
    top = lambda v: np.lexsort((np.arange(v.size), -v))[:100]   # noqa: E731
    assert np.array_equal(top(vals["fused"]), top(o.values))


@pytest.mark.parametrize("algorithm", ["ifp2", "ifp1"])
def test_device_partitions_emulated(algorithm):
    """Partitions built on the device (pr_part_from_graph) against the host
    builder, 3 emulated ranks at C2: the same fixed point (L1 <= 1e-9 between
    the two, identical top-100) and round count."""
    import paper_2302_03245_b200 as P
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make("c2", seed=0)
    g = P.from_edges(n, src, dst)
    vd, rd = D.run_emulated(g, 3, algorithm, build="device")
    vh, rh = D.run_emulated(g, 3, algorithm, build="host")
    assert np.abs(vd - vh).sum() <= 1e-9 and rd == rh
    # device partitions carry the sparse exchange masks: the fused stores
    # reach only the replicas that read a share, and the result is still
    # bit-identical to the all-gather form
    vg, rg = D.run_emulated(g, 3, algorithm, build="device", fused=False)
    assert np.array_equal(vd, vg) and rd == rg
    part = D.partition_device(g, 3, 1, algorithm, 0.85, 1e-10)
    step = D.CudaLocalStep(part, 0.85, 1e-10, algorithm, device=0, fast=True)
    assert 0 < step.exchange_entries() < 3 * part.owned
    top = lambda v: np.lexsort((np.arange(v.size), -v))[:100]   # noqa: E731
    assert np.array_equal(top(vd), top(vh))


def _worker_nccl(port, algorithm, fused, q):
    """One NCCL rank with the collectives forced on (PUSHRANK_SOLO_COLLECTIVES):
    the in-place all-gather and the statistics all-reduce are real NCCL calls
    on the library stream, and the steady-state batch is captured into a CUDA
    graph with them inside -- the code path bench.py --gpus N runs, on the
    one GPU this box has.  Two solves on the same step: the second replays
    the captured graph from its second batch on."""
    import torch
    import torch.distributed as dist
    import paper_2302_03245_b200 as P
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["PUSHRANK_SOLO_COLLECTIVES"] = "1"
    os.environ["PUSHRANK_GS_SECTIONS"] = "2"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, src, dst = synthetic.make("c2", seed=0)
        g = P.from_edges(n, src, dst)
        part = D.partition_device(g, 1, 0, algorithm, 0.85, 1e-10)
        step = D.CudaLocalStep(part, 0.85, 1e-10, algorithm, device=0, fast=True)
        comm = D.Comm(device=torch.device("cuda", 0))
        assert not comm.solo
        ok = step.setup_fused(comm) if fused else False
        out = []
        for _ in range(2):
            vals, rows, info = D.run_partitioned_queued(step, comm, part, algorithm, 0.85, 1e-10, batch=6, fused=ok)
            out.append((vals.copy(), info["rounds"]))
        captured = step._queued["graph"] is not None
        if ok:
            step.close_fused(comm)
        q.put((ok, captured, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
def test_nccl_collectives_in_captured_batches(fused):
    """NCCL at one rank with every collective issued: the batch graphs carry
    the all-gather / all-reduce nodes, the replayed solve is bit-identical to
    the first one, and both match the sync twin."""
    import torch.multiprocessing as mp
    from paper_2302_03245_b200 import distributed as D
    from paper_2302_03245_b200 import synthetic
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker_nccl, args=(_port(), "ifp2", fused, q))
    p.start()
    ok, captured, out = q.get(timeout=900)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert captured, "the steady-state batch was not captured into a CUDA graph"
    assert ok == fused
    (v1, r1), (v2, r2) = out
    assert np.array_equal(v1, v2) and r1 == r2
    n, src, dst = synthetic.make("c2", seed=0)
    g = oracle.from_edges(n, src, dst)
    order = D.run_order(np.diff(g.out_offsets), np.diff(g.in_offsets))
    vals = np.empty(n)
    vals[order] = v1
    o = oracle.sync_simulate(g, "ifp2", threshold=1e-10)
    assert np.abs(vals - o.values).sum() <= 1e-9
    top = lambda v: np.lexsort((np.arange(v.size), -v))[:100]   # noqa: E731
    assert np.array_equal(top(vals), top(o.values))
