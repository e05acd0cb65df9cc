"""Per-round launch overhead of the round-loop structures (pr_debug_graph)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "PUSHRANK_LIB" not in os.environ:  # pr_debug_graph lives in tools/ubench.cu (variant library)
    import subprocess
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "var.py"), "ubench", "-DPR_UBENCH"], check=True,
                   env=dict(os.environ, VAR_EXTRA=os.path.join(ROOT, "tools", "ubench.cu")))
    os.environ["PUSHRANK_LIB"] = os.path.join(ROOT, "build", "var", "lib_ubench.so")
from paper_2302_03245_b200 import _lib  # noqa: E402

L = _lib.load()
L.pr_debug_graph.restype = ctypes.c_int
L.pr_debug_graph.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
ctx = _lib.context()
names = {0: "stream launches", 1: "WHILE{kernel}", 2: "WHILE{SWITCH{kernel}}", 3: "WHILE{kernel x4}", 4: "WHILE{kernel x8}", 5: "WHILE{coop kernel}", 6: "WHILE{k x8 PDL prog}", 7: "WHILE{k x8 PDL launch}"}
for blocks in (148, 592):
    for v in (0, 1, 2, 3, 4, 5, 6, 7):
        us = ctypes.c_double()
        rc = L.pr_debug_graph(ctx.handle, v, 2000, blocks, ctypes.byref(us))
        if rc:
            print(f"blocks={blocks:5d} {names[v]:24s} failed: {L.pr_last_error().decode()}")
            continue
        print(f"blocks={blocks:5d} {names[v]:24s} {us.value:7.2f} us/round")
