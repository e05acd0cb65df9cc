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
in tests/test_distributed.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

STAT_INTS = ("nact", "work", "push_ops", "push_dang", "conv_all", "conv_scan")
STAT_FLOATS = ("l1", "above", "nd_above")
ROW_COST = 8


def edge_balanced_ranges(in_degree: np.ndarray, parts: int) -> np.ndarray:
    """Boundaries b[0..parts] (b[0]=0, b[parts]=n): contiguous ranges of equal
    weight in-degree + ROW_COST (pull work of a destination)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    n = int(in_degree.size)
    w = np.asarray(in_degree, np.int64) + ROW_COST
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


def partition_graph(g, parts: int, rank: int, algorithm: str = "ifp1") -> Partition:
    """Rank `rank`'s partition of a graph with the reference arrays
    (out_offsets/out_targets/in_offsets/in_sources, int64)."""
    n = int(g.n)
    out_off = np.asarray(g.out_offsets, np.int64)
    out_tgt = np.asarray(g.out_targets, np.int64)
    in_off = np.asarray(g.in_offsets, np.int64)
    in_src = np.asarray(g.in_sources, np.int64)
    out_deg = np.diff(out_off)
    in_deg = np.diff(in_off)
    dang = out_deg == 0
    bounds = edge_balanced_ranges(in_deg, parts)
    slot = int(np.max(np.diff(bounds))) if parts else n
    slot = max(slot, 1)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    rows = in_off[lo:hi + 1] - in_off[lo]
    src = in_src[in_off[lo]:in_off[hi]]
    r = np.searchsorted(bounds, src, side="right") - 1
    src_pad = r * slot + (src - bounds[r])
    if algorithm == "ifp2":
        # live push row length: out-edges into non-dangling targets (graph.py:353-356)
        keep = ~dang[out_tgt]
        kept = np.concatenate(([0], np.cumsum(keep.astype(np.int64))))
        row_len = (kept[out_off[1:]] - kept[out_off[:-1]])[lo:hi]
        dtc = np.zeros(hi - lo, np.int64)
        receives = ~dang[lo:hi]
    else:
        isd = dang[out_tgt].astype(np.int64)
        cum = np.concatenate(([0], np.cumsum(isd)))
        dtc = (cum[out_off[1:]] - cum[out_off[:-1]])[lo:hi]
        row_len = out_deg[lo:hi].copy()
        receives = np.ones(hi - lo, bool)
    return Partition(rank=rank, parts=parts, n=n, bounds=bounds, slot=slot, lo=lo, hi=hi,
                     in_offsets=rows, in_sources=src_pad, out_degree=out_deg[lo:hi].copy(),
                     row_len=row_len, dtc=dtc, dangling=dang[lo:hi].copy(), receives=receives)


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

    def allgather_slots(self, full, mine_view) -> None:
        # `mine_view` aliases this rank's slice of `full`: in-place all-gather
        self.dist.all_gather_into_tensor(full, mine_view.clone() if full.device.type == "cpu" else mine_view)

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

    def __init__(self, part: Partition, damping: float, threshold: float, algorithm: str, device=None):
        import ctypes

        import torch

        from . import _lib
        self._lib, self._ct, self.torch = _lib, ctypes, torch
        self.part, self.algo = part, algorithm
        ctx = _lib.context(device)
        self.dev = torch.device("cuda", ctx.device)
        L = _lib.load()
        self.L = L
        k = part.owned
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
