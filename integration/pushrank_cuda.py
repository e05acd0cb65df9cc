"""pushrank/_cuda.py -- the reference-side binding of libpushrank_cuda.so.

This is the file a pushrank maintainer adds to
run the push phases of ``ifp1_run`` / ``ifp2_run`` (engines.py:225-343) on
the B200 through the C-ABI (include/pushrank_cuda.h), plus three small
edits to the reference:

  _backend.py  resolve_backend("cuda") returns this module;
  engines.py   _run_phase(...) gains ``graph=None, algorithm=None`` and, as
               its first statement,
                   if backend.NAME == "cuda":
                       return backend.run_phase(graph, algorithm, h, reserved, xi, damping,
                                                scan_ids, dangling_mask, degree, trace, start_time)
               and ifp1_run / ifp2_run pass ``graph=g, algorithm="ifp1"`` /
               ``graph=pg, algorithm="ifp2"``.

Everything else in ifp1_run / ifp2_run stays as it is -- including
``_settle_dangling`` (engines.py:269-289, called at engines.py:330) and the
settle trace row: ``run_phase`` hands back the phase-1 state *before* the
settle.  The device run (pr_run) settles the dangling vertices itself, so
this binding restores their pre-settle values on the host copy -- pending
1.0 and reserved 0.0, which is what every dangling vertex holds when phase
1 ends (IFP2 never scans them and never pushes into them, engines.py:
317-330) -- and subtracts the settle's m_d pushes from the counters.  The
reference then settles exactly once, in its own summation order.

Only plain ctypes and numpy: no torch, no import of the B200 package.
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np

NAME = "cuda"
NEEDS_LOCK = False
ABI = 3


class _Params(ctypes.Structure):          # pr_run_params
    _fields_ = [("algorithm", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("damping", ctypes.c_double), ("threshold", ctypes.c_double),
                ("max_rounds", ctypes.c_int64), ("push_switch", ctypes.c_double),
                ("converged_scope", ctypes.c_int32), ("host_loop", ctypes.c_int32),
                ("on_round", ctypes.c_void_p), ("user", ctypes.c_void_p)]


class _Result(ctypes.Structure):          # pr_run_result (PR_ABI_VERSION 3)
    _fields_ = [(k, ctypes.c_int64) for k in ("rounds", "rows", "push_ops", "push_ops_dangling",
                                              "settled", "pull_rounds", "push_rounds")] + \
               [(k, ctypes.c_double) for k in ("mass_total", "push_ms", "round_ms", "bytes_moved",
                                               "pull_ms", "pull_bytes", "sparse_ms")] + \
               [("launches", ctypes.c_int64)]


class _Ifp2Counts(ctypes.Structure):      # pr_ifp2_counts
    _fields_ = [("live_edges", ctypes.c_int64), ("dangling", ctypes.c_int64), ("source_edges", ctypes.c_int64)]


_state = {}


def _lib():
    """libpushrank_cuda.so (PUSHRANK_CUDA_LIB, else next to this file) and
    one device context."""
    if "L" not in _state:
        path = os.environ.get("PUSHRANK_CUDA_LIB",
                              os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpushrank_cuda.so"))
        L = ctypes.CDLL(path)
        L.pr_last_error.restype = ctypes.c_char_p
        if L.pr_abi_version() != ABI:
            raise RuntimeError(f"libpushrank_cuda ABI {L.pr_abi_version()}, binding expects {ABI}")
        ctx = ctypes.c_void_p()
        if L.pr_ctx_create(int(os.environ.get("PUSHRANK_DEVICE", "0")), ctypes.byref(ctx)):
            raise RuntimeError(L.pr_last_error().decode())
        _state.update(L=L, ctx=ctx)
    return _state["L"], _state["ctx"]


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(L, rc, what):
    if rc:
        raise RuntimeError(f"{what}: {L.pr_last_error().decode()}")


def worker_loop(*args, **kwargs):
    raise RuntimeError("the cuda backend runs whole phases on the device (run_phase), not CPU workers")


def probe(*args, **kwargs):
    raise RuntimeError("the cuda backend runs whole phases on the device (run_phase), not CPU workers")


class Phase:
    """What _run_phase's callers read from the phase (engines.py:125-140)."""

    def __init__(self, push_ops: int, push_ops_dangling: int):
        self.push_ops = int(push_ops)
        self.push_ops_dangling = int(push_ops_dangling)


def run_phase(graph, algorithm, h, reserved, xi, damping, scan_ids, dangling_mask, degree, trace, start_time):
    """One push phase on the device; fills ``h`` / ``reserved`` (the caller's
    MassState arrays) with the phase-final state, appends the final trace
    sample like _run_phase (engines.py:185-216), returns the counters."""
    from .engines import _sample          # the reference's own row builder

    L, ctx = _lib()
    g = graph.base if algorithm == "ifp2" else graph
    arrs = [np.ascontiguousarray(a, np.int64) for a in (g.out_offsets, g.out_targets, g.in_offsets, g.in_sources)]
    handle = ctypes.c_void_p()
    _check(L, L.pr_graph_upload(ctx, ctypes.c_int64(g.n), ctypes.c_int64(g.m), _ptr(arrs[0]), _ptr(arrs[1]),
                                _ptr(arrs[2]), _ptr(arrs[3]), ctypes.byref(handle)), "pr_graph_upload")
    try:
        if algorithm == "ifp2":
            counts = _Ifp2Counts()
            _check(L, L.pr_preprocess_ifp2(handle, ctypes.byref(counts)), "pr_preprocess_ifp2")
        prm = _Params(algorithm={"ifp1": 0, "ifp2": 1}[algorithm], mode=0, damping=damping, threshold=xi,
                      max_rounds=1_000_000)
        res = _Result()
        out_r, out_h = np.empty(g.n), np.empty(g.n)
        _check(L, L.pr_run(handle, ctypes.byref(prm), None, _ptr(out_r), _ptr(out_h), None, ctypes.c_int64(0),
                           ctypes.byref(res)), "pr_run")
    finally:
        L.pr_graph_destroy(handle)
    push_ops, push_dang = res.push_ops, res.push_ops_dangling
    if algorithm == "ifp2":
        # undo the device settle: the reference settles once itself
        d = np.asarray(graph.dangling_ids, np.int64)
        out_r[d] = 0.0
        out_h[d] = 1.0
        push_ops -= res.settled
        push_dang -= res.settled
    reserved[:] = out_r
    h[:] = out_h
    trace.samples.append(_sample(len(trace.samples), h, scan_ids, dangling_mask, degree, xi, push_ops, push_dang,
                                 (time.perf_counter() - start_time) * 1e3))
    return Phase(push_ops, push_dang)
