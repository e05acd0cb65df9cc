"""ctypes binding of libpushrank_cuda.so (include/pushrank_cuda.h).

This is the only way the package reaches the device: there is no CPU
fallback.  If the shared library is missing, or no CUDA device is present,
every entry point raises ``RuntimeError`` ("fail loudly").
"""

from __future__ import annotations

import ctypes
import weakref
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PUSHRANK_LIB") or os.path.join(HERE, "lib", "libpushrank_cuda.so")

c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_i32 = ctypes.c_int32
c_vp = ctypes.c_void_p

PR_OK, PR_ERR_ARG, PR_ERR_CUDA, PR_ERR_STATE, PR_ERR_NOT_SETTLED, PR_ERR_NOMEM, PR_ERR_FORMAT = 0, -1, -2, -3, -4, -5, -6
ALGO = {"ifp1": 0, "ifp2": 1, "fp-full": 2}
MODE = {"auto": 0, "pull": 1, "push": 2, "exact": 3}
CONV_SCAN, CONV_ALL = 0, 1


class RoundStats(ctypes.Structure):
    """pr_round_stats -- one trace row (trace.py:12-38)."""
    _fields_ = [("h_l1", c_f64), ("alpha", c_f64), ("active_mass", c_f64), ("carry_mass", c_f64),
                ("converged", c_i64), ("work", c_i64), ("push_ops", c_i64),
                ("push_ops_dangling", c_i64), ("digest", ctypes.c_uint64), ("wall_ms", c_f64)]


ROUND_DTYPE = np.dtype([(name, "<u8" if name == "digest" else ("<f8" if t is c_f64 else "<i8"))
                        for name, t in RoundStats._fields_])

ROUND_CB = ctypes.CFUNCTYPE(None, c_vp, c_i64, ctypes.POINTER(c_f64), ctypes.POINTER(c_f64))
POWER_CB = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_i64, ctypes.POINTER(c_f64))


class RunParams(ctypes.Structure):
    _fields_ = [("algorithm", c_i32), ("mode", c_i32), ("damping", c_f64), ("threshold", c_f64),
                ("max_rounds", c_i64), ("push_switch", c_f64), ("converged_scope", c_i32),
                ("host_loop", c_i32), ("on_round", ROUND_CB), ("user", c_vp)]


class RunResult(ctypes.Structure):
    _fields_ = [("rounds", c_i64), ("rows", c_i64), ("push_ops", c_i64), ("push_ops_dangling", c_i64),
                ("settled", c_i64), ("pull_rounds", c_i64), ("push_rounds", c_i64),
                ("mass_total", c_f64), ("push_ms", c_f64), ("round_ms", c_f64), ("bytes_moved", c_f64),
                ("pull_ms", c_f64), ("pull_bytes", c_f64), ("sparse_ms", c_f64), ("launches", c_i64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class ClassCounts(ctypes.Structure):
    _fields_ = [("dangling", c_i64), ("unreferenced", c_i64), ("weak_dangling", c_i64),
                ("weak_unreferenced", c_i64), ("dangling_edge_count", c_i64), ("peel_rounds", c_i64)]


class Ifp2Counts(ctypes.Structure):
    _fields_ = [("live_edges", c_i64), ("dangling", c_i64), ("source_edges", c_i64)]


_PP = ctypes.POINTER(c_vp)
_PI64 = ctypes.POINTER(c_i64)
_PF64 = ctypes.POINTER(c_f64)

SIGNATURES = {
    "pr_abi_version": (ctypes.c_int, []),
    "pr_last_error": (ctypes.c_char_p, []),
    "pr_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "pr_ctx_create": (ctypes.c_int, [ctypes.c_int, _PP]),
    "pr_ctx_destroy": (ctypes.c_int, [c_vp]),
    "pr_ctx_synchronize": (ctypes.c_int, [c_vp]),
    "pr_graph_from_edges": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, _PP]),
    "pr_graph_from_device_edges": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, _PP]),
    "pr_graph_upload": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, _PP]),
    "pr_graph_attach_out_targets": (ctypes.c_int, [c_vp, c_vp]),
    "pr_host_alloc": (ctypes.c_int, [c_i64, _PP]),
    "pr_graph_load_edge_list": (ctypes.c_int, [c_vp, ctypes.c_char_p, c_i64, _PP, c_vp]),
    "pr_graph_from_raw_ids": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, _PP]),
    "pr_graph_original_ids": (ctypes.c_int, [c_vp, c_vp]),
    "pr_rank_order": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp]),
    "pr_write_ranking_csv": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, ctypes.c_char_p]),
    "pr_format_score": (ctypes.c_int, [ctypes.c_double, ctypes.c_char_p]),
    "pr_host_free": (ctypes.c_int, [c_vp]),
    "pr_graph_destroy": (ctypes.c_int, [c_vp]),
    "pr_graph_info": (ctypes.c_int, [c_vp, _PI64, _PI64]),
    "pr_graph_h2d_bytes": (ctypes.c_int, [c_vp, _PI64]),
    "pr_graph_export": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_classify": (ctypes.c_int, [c_vp, ctypes.POINTER(ClassCounts)]),
    "pr_classify_export": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_dangling_target_counts": (ctypes.c_int, [c_vp, c_vp]),
    "pr_preprocess_ifp2": (ctypes.c_int, [c_vp, ctypes.POINTER(Ifp2Counts)]),
    "pr_ifp2_export": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_run": (ctypes.c_int, [c_vp, ctypes.POINTER(RunParams), c_vp, c_vp, c_vp, c_vp, c_i64,
                              ctypes.POINTER(RunResult)]),
    "pr_run_device": (ctypes.c_int, [c_vp, ctypes.POINTER(RunParams), c_vp, c_vp, c_vp, c_vp, c_i64,
                                     ctypes.POINTER(RunResult)]),
    "pr_power": (ctypes.c_int, [c_vp, c_f64, c_i64, c_f64, c_f64, c_vp, c_vp, c_vp, c_vp,
                                ctypes.POINTER(RunResult)]),
    "pr_power_observed": (ctypes.c_int, [c_vp, c_f64, c_i64, c_f64, c_f64, c_vp, c_vp, c_vp, c_vp,
                                         POWER_CB, c_vp, ctypes.POINTER(RunResult)]),
    "pr_error_report": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, ctypes.POINTER(c_f64), ctypes.POINTER(c_f64),
                                       _PI64, _PI64]),
    "pr_power_to_target": (ctypes.c_int, [c_vp, c_f64, c_i64, c_vp, c_vp, c_f64, _PI64]),
    "pr_rmat_generate": (ctypes.c_int, [c_vp, ctypes.c_int, c_i64, c_f64, c_f64, c_f64,
                                        ctypes.c_uint64, c_i64, c_i64, c_vp, c_vp]),
    "pr_graph_rmat": (ctypes.c_int, [c_vp, ctypes.c_int, c_i64, c_f64, c_f64, c_f64, ctypes.c_uint64,
                                     _PP]),
    "pr_part_create": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_i32, c_f64, c_f64, _PP]),
    "pr_part_init": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pr_part_round": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_part_init_device": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "pr_part_round_device": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "pr_part_stream": (ctypes.c_int, [c_vp, _PP]),
    "pr_part_share_buffers": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp, c_vp]),
    "pr_part_set_peers": (ctypes.c_int, [c_vp, c_vp]),
    "pr_part_set_peer_ptrs": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp]),
    "pr_part_set_rank": (ctypes.c_int, [c_vp, c_i32, c_i32]),
    "pr_part_from_graph": (ctypes.c_int, [c_vp, c_i32, c_i32, c_i32, c_f64, c_f64, c_vp, _PP]),
    "pr_part_sizes": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pr_part_skip_if_done": (ctypes.c_int, [c_vp, c_vp]),
    "pr_part_exchange_entries": (ctypes.c_int, [c_vp, c_vp]),
    "pr_part_export_rows": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_part_launches_per_round": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i32)]),
    "pr_part_init_fused": (ctypes.c_int, [c_vp, c_vp]),
    "pr_part_close_peers": (ctypes.c_int, [c_vp]),
    "pr_part_round_fused": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp]),
    "pr_part_settle_shares": (ctypes.c_int, [c_vp, c_vp]),
    "pr_part_settle": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pr_part_total": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(c_f64)]),
    "pr_part_export": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "pr_part_destroy": (ctypes.c_int, [c_vp]),
    "pr_device_alloc": (ctypes.c_int, [c_vp, c_i64, _PP]),
    "pr_device_free": (ctypes.c_int, [c_vp, c_vp]),
    "pr_memcpy_h2d": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64]),
    "pr_memcpy_d2h": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64]),
}

_lib = None
_lock = threading.Lock()


class CudaBackendError(RuntimeError):
    """The CUDA library is missing or no usable device is present."""


def load():
    """Load libpushrank_cuda.so (no compute; safe without a GPU)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaBackendError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                # an A/B variant library (PUSHRANK_LIB) may predate newer entry points
                fn = getattr(L, name, None) if os.environ.get("PUSHRANK_LIB") else getattr(L, name)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    msg = load().pr_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == PR_OK:
        return
    msg = last_error()
    if rc == PR_ERR_ARG:
        raise ValueError(msg)
    if rc == PR_ERR_NOT_SETTLED:
        raise RuntimeError(msg)
    raise CudaBackendError(f"{what}: {msg} (code {rc})" if what else f"{msg} (code {rc})")


def ptr(a) -> c_vp | None:
    """Host pointer of a C-contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    return c_vp(a.ctypes.data)


def pinned_empty(n: int, dtype=np.float64) -> np.ndarray:
    """numpy array in a page-locked block from the library's cache
    (pr_host_alloc); the block returns to the cache when the array dies."""
    dt = np.dtype(dtype)
    nbytes = max(int(n), 1) * dt.itemsize
    p = c_vp()
    check(load().pr_host_alloc(nbytes, ctypes.byref(p)), "host_alloc")
    buf = (ctypes.c_char * nbytes).from_address(p.value)
    weakref.finalize(buf, _host_free, p.value)
    return np.frombuffer(buf, dtype=dt, count=int(n))


def _host_free(addr: int) -> None:
    try:
        load().pr_host_free(c_vp(addr))
    except Exception:
        pass


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = load().pr_device_count(ctypes.byref(n))
    return int(n.value) if rc == PR_OK else 0


class Context:
    """One device + stream + scratch workspace (pr_ctx)."""

    def __init__(self, device: int = 0):
        L = load()
        h = c_vp()
        rc = L.pr_ctx_create(int(device), ctypes.byref(h))
        if rc != PR_OK:
            raise CudaBackendError(f"no usable CUDA device {device}: {last_error()}")
        self.handle = h
        self.device = int(device)

    def synchronize(self) -> None:
        check(load().pr_ctx_synchronize(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            load().pr_ctx_destroy(self.handle)
            self.handle = None


_contexts: dict[int, Context] = {}


def default_device() -> int:
    for key in ("PUSHRANK_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0


def context(device: int | None = None) -> Context:
    dev = default_device() if device is None else int(device)
    with _lock:
        ctx = _contexts.get(dev)
    if ctx is None:
        ctx = Context(dev)
        with _lock:
            _contexts[dev] = ctx
    return ctx
