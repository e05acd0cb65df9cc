"""Backend seam (mirrors ``_backend.py:20-45`` of the reference).

The reference resolves a CPU kernel module ("c" / "python").  Here the
only backend is the sm_100a CUDA library; there is deliberately no CPU
fallback, so ``auto`` means ``cuda`` and a missing library or device raises.
"""

from __future__ import annotations

import os

from . import _lib


class _CudaBackend:
    NAME = "cuda"
    NEEDS_LOCK = False

    @staticmethod
    def library():
        return _lib.load()


CUDA = _CudaBackend()


def available_backends() -> list[str]:
    """``["cuda"]`` when the library loads and a device is visible, else ``[]``."""
    try:
        _lib.load()
    except _lib.CudaBackendError:
        return []
    return ["cuda"] if _lib.device_count() > 0 else []


def resolve_backend(name: str | None = None):
    if name is None:
        name = os.environ.get("PUSHRANK_BACKEND", "auto")
    name = name.lower()
    if name in ("cuda", "gpu", "auto"):
        return CUDA
    raise ValueError(f"unknown backend {name!r} (expected 'cuda' or 'auto'; this build has no CPU backend)")
