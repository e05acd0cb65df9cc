"""Vertex-range partitioned IFP rounds across GPUs.

The round is sharded by destination: rank p owns a contiguous vertex range
[lo_p, hi_p), with edge-balanced boundaries, and holds the in-edge rows of
its owned vertices.  One bulk-synchronous round (Jacobi, engines.py:420-454):

  1. local pull: h(t+1)_v = h_drained(t)_v + sum_{u in in(v)} s(t)_u for owned v,
     then the drain of state t+1 (reservation, share (c*h)/deg, statistics);
  2. exchange: all-gather of the owners' new shares into the full s(t+1);
  3. all-reduce of the round statistics -> global trace row and termination.

IFP2 settles each owned dangling vertex from an all-gather of c*reserved/deg
(engines.py:269-289), then all-reduces the mass total.  Vertex ids live in a
padded space (rank p's vertices at [p*S, p*S + hi_p - lo_p)), so every
exchange is one equal-sized ``all_gather_into_tensor`` (in place, NCCL over
NVLink on the GPU; gloo in the CPU tests).  The local step is pluggable:
``CudaLocalStep`` (libpushrank_cuda ``pr_part_*``) in production, a numpy step
in tests/test_distributed.py.  ``run_partitioned`` synchronises with the host
every round (any backend); ``run_partitioned_queued`` keeps the rounds, their
all-gathers and statistics all-reduces on the device and reads the
statistics back every few rounds (NCCL).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import os

import numpy as np

STAT_INTS = ("nact", "work", "push_ops", "push_dang", "conv_all", "conv_scan")
STAT_FLOATS = ("l1", "above", "nd_above")
# per-row weight of a receiving vertex in edge units (the device rule reads the same variable: csrc/part.cu)
ROW_COST = int(os.environ.get("PUSHRANK_PART_ROW_COST", "8"))


def receiving_rows(in_degree: np.ndarray, out_degree: np.ndarray, algorithm: str) -> np.ndarray:
    """The vertices a round gathers into: in-degree > 0 and, for IFP2, also
    out-degree > 0 (its dangling receivers are settled once, after the
    rounds).  Every other vertex is drained in rounds 0-1 only and costs a
    rank nothing afterwards."""
    rec = np.asarray(in_degree) > 0
    if algorithm == "ifp2":
        rec &= np.asarray(out_degree) > 0
    return rec


def edge_balanced_ranges(in_degree: np.ndarray, parts: int, receives: np.ndarray | None = None) -> np.ndarray:
    """Boundaries b[0..parts] (b[0]=0, b[parts]=n): contiguous ranges of equal
    weight in-degree + ROW_COST (pull work of a destination).  ``receives``
    (bool per vertex, ``receiving_rows``): vertices outside it weigh nothing
    -- without it the 40 M in-degree-0 / dangling vertices of C5 count 8
    units each and the ranks that own them idle (measured with emulated ranks
    at P = 8: 8-35 ms of kernel time per solve against 150-176 ms)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    n = int(in_degree.size)
    w = np.asarray(in_degree, np.int64) + ROW_COST
    if receives is not None:
        w = np.where(np.asarray(receives, bool), w, 0)
    cum = np.concatenate(([0], np.cumsum(w)))
    targets = (cum[-1] * np.arange(parts + 1)) // parts
    b = np.searchsorted(cum, targets, side="left").astype(np.int64)
    b[0], b[-1] = 0, n
    return np.maximum.accumulate(b)


@dataclass
class Partition:
    """One rank's share of the graph, in padded ids."""

    rank: int
    parts: int
    n: int                      # global vertices
    bounds: np.ndarray          # original-id boundaries [parts+1]
    slot: int                   # S: padded slice size
    lo: int
    hi: int
    in_offsets: np.ndarray      # local CSC rows of owned vertices [hi-lo+1]
    in_sources: np.ndarray      # padded source ids
    out_degree: np.ndarray      # owned out-degree (push weight denominator)
    row_len: np.ndarray         # owned push-row length (out or live degree)
    dtc: np.ndarray             # owned dangling-target counts (IFP1) or zeros
    dangling: np.ndarray        # owned dangling flags
    receives: np.ndarray        # owned rows pulled in phase 1 (IFP2: non-dangling)

    @property
    def owned(self) -> int:
        return self.hi - self.lo

    def padded(self, ids: np.ndarray) -> np.ndarray:
        """Original ids -> padded ids."""
        r = np.searchsorted(self.bounds, ids, side="right") - 1
        return r * self.slot + (ids - self.bounds[r])


def run_order(out_deg: np.ndarray, in_deg: np.ndarray) -> np.ndarray:
    """The engines' run layout (csrc/graph.cu k_relabel_keys): vertices by
    class (in>0 & out>0 | out>0 & in=0 | out=0 & in>0 | isolated), then by
    descending in-degree inside the receiving classes, ties by id.  Returns
    order[new id] = original id."""
    cls = np.where(out_deg > 0, np.where(in_deg > 0, 0, 1), np.where(in_deg > 0, 2, 3))
    key = np.where((cls == 0) | (cls == 2), -np.minimum(in_deg, 0x3FFFFFFF), 0)
    return np.lexsort((np.arange(out_deg.size), key, cls)).astype(np.int64)


def partition_graph(g, parts: int, rank: int, algorithm: str = "ifp1", order: np.ndarray | None = None) -> Partition:
    """Rank `rank`'s partition of a graph with the reference arrays
    (out_offsets/out_targets/in_offsets/in_sources, int64).

    ``order`` (order[new id] = original id, e.g. ``run_order``) partitions
    the renumbered graph instead: vertex ids, ranges and source ids are the
    new ones (what the fast local step wants: hot sources at low ids), and a
    row's sources keep their original CSC order.  Only this rank's rows are
    gathered."""
    n = int(g.n)
    out_off = np.asarray(g.out_offsets, np.int64)
    out_tgt = np.asarray(g.out_targets, np.int64)
    in_off = np.asarray(g.in_offsets, np.int64)
    in_src = np.asarray(g.in_sources, np.int64)
    out_deg = np.diff(out_off)
    dang = out_deg == 0
    # per-vertex push-row data in original ids
    if algorithm == "ifp2":
        # live push row length: out-edges into non-dangling targets (graph.py:353-356)
        kept = np.concatenate(([0], np.cumsum((~dang[out_tgt]).astype(np.int64))))
        row_len_all = kept[out_off[1:]] - kept[out_off[:-1]]
        dtc_all = None
    else:
        cum = np.concatenate(([0], np.cumsum(dang[out_tgt].astype(np.int64))))
        dtc_all = cum[out_off[1:]] - cum[out_off[:-1]]
        row_len_all = out_deg
    if order is None:
        order = None
        rank_of = None
        in_deg = np.diff(in_off)
        out_deg_o = out_deg
    else:
        order = np.asarray(order, np.int64)
        rank_of = np.empty(n, np.int64)
        rank_of[order] = np.arange(n, dtype=np.int64)
        in_deg = np.diff(in_off)[order]
        out_deg_o = out_deg[order]
    bounds = edge_balanced_ranges(in_deg, parts, receiving_rows(in_deg, out_deg_o, algorithm))
    slot = int(np.max(np.diff(bounds))) if parts else n
    slot = max(slot, 1)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    if order is None:
        verts = np.arange(lo, hi, dtype=np.int64)
        rows = in_off[lo:hi + 1] - in_off[lo]
        src = in_src[in_off[lo]:in_off[hi]]
    else:
        verts = order[lo:hi]
        d = in_deg[lo:hi]
        rows = np.concatenate(([0], np.cumsum(d)))
        starts = np.repeat(in_off[verts] - rows[:-1], d)
        src = rank_of[in_src[starts + np.arange(rows[-1], dtype=np.int64)]]
    r = np.searchsorted(bounds, src, side="right") - 1
    src_pad = r * slot + (src - bounds[r])
    row_len = row_len_all[verts]
    if algorithm == "ifp2":
        dtc = np.zeros(hi - lo, np.int64)
        receives = ~dang[verts]
    else:
        dtc = dtc_all[verts]
        receives = np.ones(hi - lo, bool)
    return Partition(rank=rank, parts=parts, n=n, bounds=bounds, slot=slot, lo=lo, hi=hi,
                     in_offsets=rows, in_sources=src_pad, out_degree=out_deg[verts].copy(),
                     row_len=row_len, dtc=dtc, dangling=dang[verts].copy(), receives=receives)


@dataclass
class DevicePartition:
    """A rank's partition built on the device (``pr_part_from_graph``): the
    metadata of ``Partition`` without the host arrays, and the library
    handle of the device-resident rows (CudaLocalStep takes it over)."""

    rank: int
    parts: int
    n: int
    bounds: np.ndarray          # run-layout boundaries [parts+1]
    slot: int
    lo: int
    hi: int
    algorithm: str
    damping: float
    threshold: float
    handle: object = None

    @property
    def owned(self) -> int:
        return self.hi - self.lo

    def to_host(self) -> Partition:
        """The rows as a host ``Partition`` (pr_part_export_rows), e.g. to
        upload them again through pr_part_create or to compare with
        partition_graph.  Needs the handle (before a CudaLocalStep takes it)."""
        import ctypes

        from . import _lib
        L = _lib.load()
        e = ctypes.c_int64()
        _lib.check(L.pr_part_sizes(self.handle, None, None, ctypes.byref(e)), "pr_part_sizes")
        k, m = self.owned, int(e.value)
        arr = {"off": np.empty(k + 1, np.int64), "src": np.empty(max(m, 1), np.int64),
               "deg": np.empty(max(k, 1), np.int64), "len": np.empty(max(k, 1), np.int64),
               "dtc": np.empty(max(k, 1), np.int64), "dang": np.empty(max(k, 1), np.uint8),
               "recv": np.empty(max(k, 1), np.uint8)}
        _lib.check(L.pr_part_export_rows(self.handle, *[_lib.ptr(arr[x]) for x in
                                                        ("off", "src", "deg", "len", "dtc", "dang", "recv")]),
                   "pr_part_export_rows")
        return Partition(rank=self.rank, parts=self.parts, n=self.n, bounds=self.bounds, slot=self.slot, lo=self.lo,
                         hi=self.hi, in_offsets=arr["off"], in_sources=arr["src"][:m], out_degree=arr["deg"][:k],
                         row_len=arr["len"][:k], dtc=arr["dtc"][:k], dangling=arr["dang"][:k].astype(bool),
                         receives=arr["recv"][:k].astype(bool))

    def release(self) -> None:
        """Destroy the device rows if no local step took them."""
        if self.handle is not None:
            from . import _lib
            _lib.load().pr_part_destroy(self.handle)
            self.handle = None


def partition_device(g, parts: int, rank: int, algorithm: str, damping: float, threshold: float) -> DevicePartition:
    """``partition_graph(g, parts, rank, algorithm, order=run_order(...))``
    built on the graph's device from its run layout (csrc/part.cu
    part_from_graph): no host export of the graph -- what every rank of the
    C5 bench does with its own copy of the graph."""
    import ctypes

    from . import _lib
    from .graph import device_graph
    dev = device_graph(g)
    bounds = np.zeros(parts + 1, np.int64)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().pr_part_from_graph(dev.handle, int(parts), int(rank), _lib.ALGO[algorithm],
                                              float(damping), float(threshold), _lib.ptr(bounds), ctypes.byref(h)),
               "pr_part_from_graph")
    slot = max(int(np.max(np.diff(bounds))), 1)
    return DevicePartition(rank=rank, parts=parts, n=int(g.n), bounds=bounds, slot=slot, lo=int(bounds[rank]),
                           hi=int(bounds[rank + 1]), algorithm=algorithm, damping=float(damping),
                           threshold=float(threshold), handle=h)


@dataclass
class RoundRow:
    ints: dict
    floats: dict
    push_ops: int = 0
    push_ops_dangling: int = 0
    rows: list = field(default_factory=list)


class Comm:
    """Exchange + reductions over torch.distributed (any backend)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.device = device
        # one rank: every collective is the identity (all-gather of the own
        # slice into itself, sum over one rank) -- issue none, unless
        # PUSHRANK_SOLO_COLLECTIVES=1 asks for them (tests: the NCCL calls and
        # their capture into the batch graphs, exercised on a one-GPU box)
        self.solo = dist.get_world_size() == 1 and os.environ.get("PUSHRANK_SOLO_COLLECTIVES", "0") != "1"

    def _staged(self, t) -> bool:
        # gloo has no CUDA all-gather: device tensors go through host copies
        return t.is_cuda and self.dist.get_backend() == "gloo"

    def allgather_slots(self, full, mine_view) -> None:
        # `mine_view` aliases this rank's slice of `full`: in-place all-gather
        if self.solo:
            return
        if self._staged(full):
            host = full.cpu()
            self.dist.all_gather_into_tensor(host, mine_view.cpu())
            full.copy_(host)
            return
        self.dist.all_gather_into_tensor(full, mine_view.clone() if full.device.type == "cpu" else mine_view)

    def allreduce_row(self, row) -> None:
        """In-place sum of a statistics row (device or host tensor)."""
        if self.solo:
            return
        if self._staged(row):
            host = row.cpu()
            self.dist.all_reduce(host)
            row.copy_(host)
            return
        self.dist.all_reduce(row)

    def allreduce_stats(self, ints: np.ndarray, floats: np.ndarray):
        # one all-reduce per round: the integer counters ride in a float64
        # tensor (exact below 2**53) after the float statistics
        t = self.torch
        buf = np.concatenate([np.asarray(floats, np.float64), np.asarray(ints, np.float64)])
        tb = t.tensor(buf, dtype=t.float64, device=self.device)
        self.dist.all_reduce(tb)
        out = tb.cpu().numpy()
        k = len(floats)
        return np.rint(out[k:]).astype(np.int64), out[:k]


def run_partitioned(step, comm, part: Partition, algorithm: str, damping: float, threshold: float,
                    max_rounds: int = 1_000_000, conv_scope_all: bool = False):
    """Drive the bulk-synchronous rounds; returns (values_owned, rows, info).

    ``step`` implements init(s_mine) / round(t, s_in, s_mine) / settle_shares(x_mine) /
    settle(x_full) / local_total() / values(total); each fills the rank's
    slice in place and returns (ints[6], floats[3]) statistics where relevant.
    """
    torch = comm.torch
    S, P = part.slot, part.parts
    full = [torch.zeros(S * P, dtype=torch.float64, device=comm.device) for _ in range(2)]
    mine = [f[part.rank * S:(part.rank + 1) * S] for f in full]
    rows = []
    push_ops = push_dang = 0

    def record(ints, floats):
        nonlocal push_ops, push_dang
        gi, gf = comm.allreduce_stats(ints, floats)
        nact, work, pops, pdang, conv_all, conv_scan = (int(x) for x in gi)
        l1, above, nd_above = (float(x) for x in gf)
        rows.append({"h_l1": l1, "converged": conv_all if conv_scope_all else conv_scan,
                     "alpha": nd_above / above if above > 0 else 1.0, "work": work, "push_ops": push_ops,
                     "push_ops_dangling": push_dang, "active_mass": above, "carry_mass": l1 - above})
        push_ops += pops
        push_dang += pdang
        return nact

    ints, floats = step.init(mine[0])
    comm.allgather_slots(full[0], mine[0])
    nact = record(ints, floats)
    t = 0
    while nact > 0:
        if t >= max_rounds:
            raise RuntimeError(f"sync simulation did not settle in {max_rounds} iterations")
        src, dst = full[t & 1], full[(t + 1) & 1]
        ints, floats = step.round(t, src, mine[(t + 1) & 1])
        comm.allgather_slots(dst, mine[(t + 1) & 1])
        nact = record(ints, floats)
        t += 1
    settled = 0
    if algorithm == "ifp2":
        step.settle_shares(mine[0])
        comm.allgather_slots(full[0], mine[0])
        settled, ints, floats = step.settle(full[0])
        gi, gf = comm.allreduce_stats(np.array([settled, 0, 0, 0, ints[4], ints[5]], np.int64), floats)
        settled = int(gi[0])
        push_ops += settled
        push_dang += settled
        rows.append({"h_l1": float(gf[0]), "converged": int(gi[4] if conv_scope_all else gi[5]),
                     "alpha": float(gf[2] / gf[1]) if gf[1] > 0 else 1.0, "work": 0, "push_ops": push_ops,
                     "push_ops_dangling": push_dang, "active_mass": float(gf[1]),
                     "carry_mass": float(gf[0] - gf[1])})
    total_local = step.local_total()
    _, gt = comm.allreduce_stats(np.zeros(6, np.int64), np.array([total_local, 0.0, 0.0]))
    total = float(gt[0])
    return step.values(total), rows, {"rounds": t, "mass_total": total, "push_ops": push_ops,
                                      "push_ops_dangling": push_dang, "settled": settled}


def run_partitioned_queued(step, comm, part: Partition, algorithm: str, damping: float, threshold: float,
                           max_rounds: int = 1_000_000, conv_scope_all: bool = False, batch: int = 8,
                           graph: bool | None = None, host_values: bool = True, fused: bool = False):
    """``run_partitioned`` with the rounds queued on the device: each round
    is the local step, the all-gather of its shares and an in-place
    all-reduce of its 9 statistics (a row of a device buffer), all issued on
    the library stream without host synchronisation; the host reads the
    statistics of ``batch`` rounds at a time and stops at the first state
    with no active vertex.  Rounds queued past that state are no-ops (no
    vertex above the threshold: zero shares, unchanged mass), so the result
    and the trace equal run_partitioned's.  Needs a step with
    ``init_device`` / ``round_device`` (CudaLocalStep, whose ``stream`` the
    collectives are ordered on; NumpyLocalStep for the CPU tests).

    ``graph`` (default: on with NCCL): a batch of rounds -- the local
    kernels and the NCCL collectives -- is captured once into a CUDA graph
    on the library stream and replayed for every later batch (and solve), so
    a round costs no host launches.  Batches start at even rounds, so the
    share-buffer parities of a replay are those of the capture.

    ``fused=True`` (CudaLocalStep after ``setup_fused``): no all-gather --
    the round kernel stores its shares into every rank's replica through
    peer memory, and the statistics all-reduce is the round's barrier
    (no rank starts round t+1, which overwrites the replicas round t reads,
    before every rank has finished round t).

    ``host_values=False`` leaves the owned result on the device (the step's
    reserved/pending buffers) and returns None for it: the timed solve of
    bench.py, like the single-GPU engine's device time, excludes the D2H."""
    import contextlib
    torch = comm.torch
    S, P = part.slot, part.parts
    dev = getattr(step, "dev", None) or comm.device or torch.device("cpu")
    stream = getattr(step, "stream", None)
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    if graph is None:
        graph = stream is not None and comm.dist.get_backend() == "nccl"
    batch += batch & 1
    rows = []
    push_ops = push_dang = 0

    drained = 0   # vertices drained over the solve (the roofline's 40 B per active vertex)

    def record(r):
        nonlocal push_ops, push_dang, drained
        l1, above, nd_above = float(r[0]), float(r[1]), float(r[2])
        nact, work, pops, pdang, conv_all, conv_scan = (int(round(x)) for x in r[3:9])
        rows.append({"h_l1": l1, "converged": conv_all if conv_scope_all else conv_scan,
                     "alpha": nd_above / above if above > 0 else 1.0, "work": work, "push_ops": push_ops,
                     "push_ops_dangling": push_dang, "active_mass": above, "carry_mass": l1 - above})
        push_ops += pops
        push_dang += pdang
        drained += nact
        return nact

    with ctx:
        cache = getattr(step, "_queued", None) if graph else None
        if cache is None or cache["batch"] != batch or cache["fused"] != fused:
            full = [torch.zeros(S * P, dtype=torch.float64, device=dev) for _ in range(2)]
            cache = {"batch": batch, "fused": fused, "full": full, "mine": [f[part.rank * S:(part.rank + 1) * S] for f in full],
                     "stats": torch.zeros((batch, 9), dtype=torch.float64, device=dev), "graph": None}
            if graph:
                step._queued = cache
        full, mine, stats = cache["full"], cache["mine"], cache["stats"]

        skip = getattr(step, "skip_if_done", None)

        def queue_batch(nb, t0):
            for j in range(nb):
                tt = t0 + j
                # a round queued past termination skips its sweep on the device
                # (the previous round's all-reduced row shows no active vertex)
                if skip is not None and (j > 0 or t0 > 0):
                    skip(stats[j - 1] if j > 0 else stats[batch - 1])
                if fused:
                    step.round_fused(tt, stats[j])
                else:
                    step.round_device(full[tt & 1], mine[(tt + 1) & 1], stats[j], tt)
                    comm.allgather_slots(full[(tt + 1) & 1], mine[(tt + 1) & 1])
                comm.allreduce_row(stats[j])

        def run_batch(t0):
            if not graph:
                nb = max(1, min(batch, max_rounds - t0))
                queue_batch(nb, t0)
                return nb
            if t0 == 0:
                # the first batch of every solve runs eagerly: it holds the
                # Jacobi and transition sweeps (sweep_kind 0 and 1), which the
                # captured steady-state batch does not
                queue_batch(batch, t0)
                return batch
            if cache["graph"] is None:
                # capture once the schedule exists (built by the first, eager
                # batch); every later batch (t0 > 0) has the same parities and
                # sweep kinds (Gauss-Seidel from round 2 on) as this one
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    queue_batch(batch, t0)
                cache["graph"] = g
            cache["graph"].replay()
            return batch

        if fused:
            step.init_fused(stats[0])
        else:
            step.init_device(mine[0], stats[0])
            comm.allgather_slots(full[0], mine[0])
        comm.allreduce_row(stats[0])
        nact = record(stats[0].cpu().numpy())
        t = 0
        queued = 0   # rounds launched, including those queued past termination (no-ops)
        while nact > 0:
            if t >= max_rounds:
                raise RuntimeError(f"sync simulation did not settle in {max_rounds} iterations")
            nb = run_batch(t)
            queued += nb
            host = stats[:nb].cpu().numpy()
            for j in range(nb):
                nact = record(host[j])
                t += 1
                if nact == 0:
                    break
        settled = 0
        if algorithm == "ifp2":
            step.settle_shares(mine[0])
            comm.allgather_slots(full[0], mine[0])
            settled, ints, floats = step.settle(full[0])
            gi, gf = comm.allreduce_stats(np.array([settled, 0, 0, 0, ints[4], ints[5]], np.int64), floats)
            settled = int(gi[0])
            push_ops += settled
            push_dang += settled
            rows.append({"h_l1": float(gf[0]), "converged": int(gi[4] if conv_scope_all else gi[5]),
                         "alpha": float(gf[2] / gf[1]) if gf[1] > 0 else 1.0, "work": 0, "push_ops": push_ops,
                         "push_ops_dangling": push_dang, "active_mass": float(gf[1]),
                         "carry_mass": float(gf[0] - gf[1])})
        total_local = step.local_total()
        _, gt = comm.allreduce_stats(np.zeros(6, np.int64), np.array([total_local, 0.0, 0.0]))
        total = float(gt[0])
        values = step.values(total) if host_values else None
    return values, rows, {"rounds": t, "mass_total": total, "push_ops": push_ops,
                          "push_ops_dangling": push_dang, "settled": settled, "drained": drained,
                          "queued_rounds": queued}


def sweep_kind(t: int) -> int:
    """Kind of round t (0-based, after the state-0 drain) for rank-local
    Gauss-Seidel sections (csrc/part.cu, bins.cuh Src): 0 Jacobi (every share
    owed to every target), 1 transition, 2 Gauss-Seidel."""
    return 0 if t == 0 else 1 if t == 1 else 2


def _stats_row(row, ints, floats) -> None:
    import torch
    row.copy_(torch.from_numpy(np.concatenate([np.asarray(floats, np.float64), np.asarray(ints, np.float64)])))


class NumpyLocalStep:
    """CPU local step (reference semantics, sequential ascending-source sums in
    bincount order).  Test double for tests/test_distributed.py; never used by
    the GPU path."""

    def __init__(self, part: Partition, damping: float, threshold: float, algorithm: str):
        self.p, self.c, self.xi, self.algo = part, damping, threshold, algorithm
        k = part.owned
        self.h = np.ones(k)
        self.reserved = np.zeros(k)
        self.scan = ~part.dangling
        self.act = np.zeros(k, bool)

    def _drain(self, s_mine):
        p, h = self.p, self.h
        above = h > self.xi
        act = above & self.scan
        self.act = act
        ints = np.array([act.sum(), (p.out_degree[act] + 1).sum(), p.row_len[act].sum(), p.dtc[act].sum(),
                         (~above).sum(), (~above & self.scan).sum()], np.int64)
        floats = np.array([h.sum(), h[above].sum(), h[above & ~p.dangling].sum()])
        share = np.zeros(p.slot)
        links = act & (p.row_len > 0)
        share[:p.owned][links] = self.c * h[links] / p.out_degree[links]
        self.reserved[act] += h[act]
        s_mine.copy_(__import__("torch").from_numpy(share))
        return ints, floats

    def init(self, s_mine):
        return self._drain(s_mine)

    def round(self, t, s_in, s_mine):
        p = self.p
        s = s_in.numpy()
        inflow = np.zeros(p.owned)
        for v in range(p.owned):
            if not p.receives[v]:
                continue
            acc = 0.0
            for e in range(p.in_offsets[v], p.in_offsets[v + 1]):
                acc += s[p.in_sources[e]]
            inflow[v] = acc
        self.h = np.where(self.act, 0.0, self.h) + inflow
        return self._drain(s_mine)

    # queued form (run_partitioned_queued)
    def init_device(self, s_mine, stats_row):
        _stats_row(stats_row, *self.init(s_mine))

    def round_device(self, s_in, s_mine, stats_row, t: int = 0):
        _stats_row(stats_row, *self.round(t, s_in, s_mine))

    def settle_shares(self, x_mine):
        p = self.p
        x = np.zeros(p.slot)
        nz = p.out_degree > 0
        x[:p.owned][nz] = self.c * self.reserved[nz] / p.out_degree[nz]
        x_mine.copy_(__import__("torch").from_numpy(x))

    def settle(self, x_full):
        p = self.p
        x = x_full.numpy()
        settled = 0
        for v in np.flatnonzero(p.dangling):
            acc = 0.0
            for e in range(p.in_offsets[v], p.in_offsets[v + 1]):
                acc += x[p.in_sources[e]]
                settled += 1
            self.reserved[v] = self.h[v] + acc
            self.h[v] = 0.0
        h = self.h
        above = h > self.xi
        ints = np.array([0, 0, 0, 0, (~above).sum(), (~above & self.scan).sum()], np.int64)
        floats = np.array([h.sum(), h[above].sum(), h[above & ~p.dangling].sum()])
        return settled, ints, floats

    def local_total(self):
        return float((self.reserved + self.h).sum() if self.algo == "ifp1" else self.reserved.sum())

    def values(self, total):
        x = self.reserved + self.h if self.algo == "ifp1" else self.reserved
        return x / total


class CudaLocalStep:
    """Production local step: libpushrank_cuda ``pr_part_*`` (csrc/part.cu).

    Exchange tensors may live on the GPU (NCCL; used directly) or on the CPU
    (gloo; staged through device buffers).  Library calls return with their
    stream synchronised; torch's stream is synchronised before each call that
    reads torch-written data.
    """

    def __init__(self, part: Partition, damping: float, threshold: float, algorithm: str, device=None,
                 fast: bool = False):
        import ctypes

        import torch

        from . import _lib
        self._lib, self._ct, self.torch = _lib, ctypes, torch
        self.part, self.algo = part, algorithm
        # fast: the binned dense-round gather (run_partitioned_queued); else the
        # exact ascending-source sums (bit-identical to sync_simulate)
        self.fast = bool(fast)
        ctx = _lib.context(device)
        self.dev = torch.device("cuda", ctx.device)
        L = _lib.load()
        self.L = L
        k = part.owned
        if isinstance(part, DevicePartition):
            # built on the device (pr_part_from_graph): take the handle over
            if part.handle is None:
                raise ValueError("device partition already taken by another local step")
            if (part.algorithm, part.damping, part.threshold) != (algorithm, float(damping), float(threshold)):
                raise ValueError("device partition was built for another algorithm / damping / threshold")
            self.h, part.handle = part.handle, None
            self.s_full = torch.zeros(part.slot * part.parts, dtype=torch.float64, device=self.dev)
            self.s_mine = torch.zeros(part.slot, dtype=torch.float64, device=self.dev)
            return
        arr = {
            "off": np.ascontiguousarray(part.in_offsets, np.int64),
            "src": np.ascontiguousarray(part.in_sources if part.in_sources.size else np.zeros(1), np.int64),
            "deg": np.ascontiguousarray(part.out_degree if k else np.zeros(1), np.int64),
            "len": np.ascontiguousarray(part.row_len if k else np.zeros(1), np.int64),
            "dtc": np.ascontiguousarray(part.dtc if k else np.zeros(1), np.int64),
            "dang": np.ascontiguousarray(part.dangling if k else np.zeros(1), np.uint8),
            "recv": np.ascontiguousarray(part.receives if k else np.zeros(1), np.uint8),
        }
        h = ctypes.c_void_p()
        _lib.check(L.pr_part_create(ctx.handle, k, part.slot, *[_lib.ptr(arr[x]) for x in ("off", "src")],
                                    int(part.in_sources.size), *[_lib.ptr(arr[x]) for x in
                                                                 ("deg", "len", "dtc", "dang", "recv")],
                                    _lib.ALGO[algorithm], float(damping), float(threshold), ctypes.byref(h)),
                   "pr_part_create")
        self.h = h
        _lib.check(L.pr_part_set_rank(h, int(part.parts), int(part.rank)), "pr_part_set_rank")
        self.s_full = torch.zeros(part.slot * part.parts, dtype=torch.float64, device=self.dev)
        self.s_mine = torch.zeros(part.slot, dtype=torch.float64, device=self.dev)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.L.pr_part_destroy(h)
            self.h = None

    def _sync(self):
        self.torch.cuda.current_stream(self.dev).synchronize()

    def _stats(self):
        return np.zeros(6, np.int64), np.zeros(3, np.float64)

    def _out(self, t):
        return t if t.is_cuda else self.s_mine

    def _back(self, t):
        if not t.is_cuda:
            t.copy_(self.s_mine.cpu())

    def init(self, s_mine):
        ints, floats = self._stats()
        out = self._out(s_mine)
        self._sync()
        self._lib.check(self.L.pr_part_init(self.h, self._ct.c_void_p(out.data_ptr()), self._lib.ptr(ints),
                                            self._lib.ptr(floats)), "pr_part_init")
        self._back(s_mine)
        return ints, floats

    def round(self, t, s_in, s_mine):
        ints, floats = self._stats()
        if s_in.is_cuda:
            src = s_in
        else:
            self.s_full.copy_(s_in)
            src = self.s_full
        out = self._out(s_mine)
        self._sync()
        self._lib.check(self.L.pr_part_round(self.h, self._ct.c_void_p(src.data_ptr()),
                                             self._ct.c_void_p(out.data_ptr()), self._lib.ptr(ints),
                                             self._lib.ptr(floats)), "pr_part_round")
        self._back(s_mine)
        return ints, floats

    # -- queued form (run_partitioned_queued): device tensors, no host sync
    @property
    def stream(self):
        p = self._ct.c_void_p()
        self._lib.check(self.L.pr_part_stream(self.h, self._ct.byref(p)), "pr_part_stream")
        return self.torch.cuda.ExternalStream(p.value or 0, device=self.dev)

    def init_device(self, s_mine, stats_row):
        self._lib.check(self.L.pr_part_init_device(self.h, self._ct.c_void_p(s_mine.data_ptr()),
                                                   self._ct.c_void_p(stats_row.data_ptr())), "pr_part_init_device")

    def round_device(self, s_in, s_mine, stats_row, t: int = 0):
        self._lib.check(self.L.pr_part_round_device(self.h, self._ct.c_void_p(s_in.data_ptr()),
                                                    self._ct.c_void_p(s_mine.data_ptr()), int(self.fast),
                                                    sweep_kind(t), self._ct.c_void_p(stats_row.data_ptr())),
                        "pr_part_round_device")

    # -- fused exchange (run_partitioned_queued(fused=True)): replicas of the
    # full share vector in peer memory, written by the round kernel itself
    def share_buffers(self, parts: int, rank: int, ipc=None):
        full = (self._ct.c_void_p * 2)()
        self._lib.check(self.L.pr_part_share_buffers(self.h, int(parts), int(rank), full, ipc),
                        "pr_part_share_buffers")
        return full[0], full[1]

    def setup_fused(self, comm) -> bool:
        """Allocate this rank's replicas and map every other rank's (CUDA IPC
        handles exchanged over the process group).  Collective: every rank
        calls it, and it returns True on all ranks or False on all (then the
        caller keeps the all-gather form)."""
        parts, rank = self.part.parts, self.part.rank
        ipc = self._ct.create_string_buffer(128)
        try:
            self.share_buffers(parts, rank, ipc)
            mine = ipc.raw
        except Exception:   # noqa: BLE001 -- reported through the collective decision
            mine = None
        handles = [None] * parts
        comm.dist.all_gather_object(handles, mine)
        ok = all(h is not None for h in handles)
        if ok:
            blob = self._ct.create_string_buffer(b"".join(handles), 128 * parts)
            ok = self.L.pr_part_set_peers(self.h, blob) == self._lib.PR_OK
        flag = self.torch.tensor([1.0 if ok else 0.0], dtype=self.torch.float64,
                                 device=self.dev if comm.dist.get_backend() == "nccl" else "cpu")
        comm.dist.all_reduce(flag, op=comm.dist.ReduceOp.MIN)
        return bool(flag.item() > 0.5)

    def close_fused(self, comm) -> None:
        """Collective: unmap the other ranks' replicas, then a barrier, so
        that no rank frees a replica (at destruction) that another still maps.
        The captured batch graph holds the unmapped peer addresses: drop it."""
        self._queued = None
        self._lib.check(self.L.pr_part_close_peers(self.h), "pr_part_close_peers")
        comm.dist.barrier()

    def set_peer_ptrs(self, parts: int, rank: int, ptrs) -> None:
        arr = (self._ct.c_void_p * len(ptrs))(*ptrs)
        self._lib.check(self.L.pr_part_set_peer_ptrs(self.h, int(parts), int(rank), arr), "pr_part_set_peer_ptrs")

    def launches_per_round(self) -> int:
        v = self._ct.c_int32(0)
        self._lib.check(self.L.pr_part_launches_per_round(self.h, self._ct.byref(v)), "pr_part_launches_per_round")
        return int(v.value)

    def init_fused(self, stats_row):
        self._lib.check(self.L.pr_part_init_fused(self.h, self._ct.c_void_p(stats_row.data_ptr())),
                        "pr_part_init_fused")

    def exchange_entries(self) -> int:
        """Shares the fused exchange stores per dense round at most (the sparse
        boundary exchange of a device-built partition; owned * parts when
        every replica receives every share)."""
        e = self._ct.c_int64()
        self._lib.check(self.L.pr_part_exchange_entries(self.h, self._ct.byref(e)), "pr_part_exchange_entries")
        return int(e.value)

    def skip_if_done(self, prev_row):
        """The next fast round skips its sweep if ``prev_row`` (the previous
        round's all-reduced statistics, device memory) has no active vertex."""
        if self.fast:
            self._lib.check(self.L.pr_part_skip_if_done(self.h, self._ct.c_void_p(prev_row.data_ptr())),
                            "pr_part_skip_if_done")

    def round_fused(self, t: int, stats_row):
        self._lib.check(self.L.pr_part_round_fused(self.h, int(t) & 1, sweep_kind(t),
                                                   self._ct.c_void_p(stats_row.data_ptr())), "pr_part_round_fused")

    def settle_shares(self, x_mine):
        out = self._out(x_mine)
        self._sync()
        self._lib.check(self.L.pr_part_settle_shares(self.h, self._ct.c_void_p(out.data_ptr())), "settle_shares")
        self._back(x_mine)

    def settle(self, x_full):
        ints, floats = self._stats()
        if x_full.is_cuda:
            src = x_full
        else:
            self.s_full.copy_(x_full)
            src = self.s_full
        settled = self._ct.c_int64(0)
        self._sync()
        self._lib.check(self.L.pr_part_settle(self.h, self._ct.c_void_p(src.data_ptr()), self._ct.byref(settled),
                                              self._lib.ptr(ints), self._lib.ptr(floats)), "pr_part_settle")
        return int(settled.value), ints, floats

    def local_total(self):
        tot = self._ct.c_double(0.0)
        self._lib.check(self.L.pr_part_total(self.h, 1 if self.algo == "ifp1" else 0, self._ct.byref(tot)),
                        "pr_part_total")
        return float(tot.value)

    def export(self):
        k = self.part.owned
        r, h = np.zeros(max(k, 1)), np.zeros(max(k, 1))
        self._lib.check(self.L.pr_part_export(self.h, self._lib.ptr(r), self._lib.ptr(h)), "pr_part_export")
        return r[:k], h[:k]

    def values(self, total):
        r, h = self.export()
        x = r + h if self.algo == "ifp1" else r
        return x / total


def run_emulated(g, parts: int, algorithm: str, damping: float = 0.85, threshold: float = 1e-10,
                 fused: bool = True, device: int = 0, max_rounds: int = 1_000_000, build: str = "host"):
    """The partitioned fast path with ``parts`` ranks emulated in one process
    on one device (B200_PROFILING.md: ranks sharing a GPU must not wait on
    each other): every rank's round is its own launch on the shared library
    stream, in rank order, and a round starts once every rank finished the
    previous one.  ``fused``: shares stored into every rank's replica by the
    round kernel (pr_part_set_peer_ptrs); else each rank's slot of one shared
    full vector (what the all-gather produces).  Returns (values in original
    ids, rounds).  ``build="device"``: partitions built on the device from
    the graph's run layout (pr_part_from_graph) instead of on the host.  For
    tests and smoke checks on a single GPU."""
    import torch
    n = int(g.n)
    order = run_order(np.diff(np.asarray(g.out_offsets)), np.diff(np.asarray(g.in_offsets)))
    if build == "device":
        plist = [partition_device(g, parts, r, algorithm, damping, threshold) for r in range(parts)]
    else:
        plist = [partition_graph(g, parts, r, algorithm, order=order) for r in range(parts)]
    steps = [CudaLocalStep(p, damping, threshold, algorithm, device=device, fast=True) for p in plist]
    S = plist[0].slot
    dev = torch.device("cuda", device)
    stats = torch.zeros((parts, 9), dtype=torch.float64, device=dev)
    full = [torch.zeros(S * parts, dtype=torch.float64, device=dev) for _ in range(2)]
    if fused:
        ptrs = [q for r, st in enumerate(steps) for q in st.share_buffers(parts, r)]
        for r, st in enumerate(steps):
            st.set_peer_ptrs(parts, r, ptrs)
            st.init_fused(stats[r])
    else:
        for r, st in enumerate(steps):
            st.init_device(full[0][r * S:(r + 1) * S], stats[r])
    rounds = 0
    while True:
        torch.cuda.synchronize()
        if stats[:, 3].sum().item() == 0:
            break
        if rounds >= max_rounds:
            raise RuntimeError(f"sync simulation did not settle in {max_rounds} iterations")
        for r, st in enumerate(steps):
            if fused:
                st.round_fused(rounds, stats[r])
            else:
                st.round_device(full[rounds & 1], full[(rounds + 1) & 1][r * S:(r + 1) * S], stats[r], rounds)
        rounds += 1
    torch.cuda.synchronize()
    if algorithm == "ifp2":
        x = torch.zeros(S * parts, dtype=torch.float64, device=dev)
        for r, st in enumerate(steps):
            st.settle_shares(x[r * S:(r + 1) * S])
        for st in steps:
            st.settle(x)
    total = sum(st.local_total() for st in steps)
    values = np.empty(n)
    for p, st in zip(plist, steps):
        values[order[p.lo:p.hi]] = st.values(total)
    return values, rounds
