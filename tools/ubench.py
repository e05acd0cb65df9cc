"""Gather microbenchmarks on the C2 run layout (pr_debug_gather).

tools/ubench.cu is not part of the product library: this script builds a
variant library with it (tools/var.py, VAR_EXTRA) and loads that one."""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "PUSHRANK_LIB" not in os.environ:
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "var.py"), "ubench", "-DPR_UBENCH"], check=True,
                   env=dict(os.environ, VAR_EXTRA=os.path.join(ROOT, "tools", "ubench.cu")))
    os.environ["PUSHRANK_LIB"] = os.path.join(ROOT, "build", "var", "lib_ubench.so")
import paper_2302_03245_b200 as P
from paper_2302_03245_b200 import _lib, synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c5":
    g = P.graph.Graph(P.graph.DeviceGraph.rmat(26, 16, seed=0), raw_edge_count=16 << 26, name="c5")
else:
    n, s, d = synthetic.make(cfg)
    g = P.from_edges(n, s, d)
L = _lib.load()
L.pr_debug_gather.restype = ctypes.c_int
L.pr_debug_gather.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
names = {0: "gather8 thread-contig", 1: "gather16 thread-contig", 2: "gather lane-interleaved", 3: "index stream only",
         4: "lane-interleaved, 8-lane LDGs", 5: "uniform random gather", 6: "sequential gather",
         7: "cold only (id >= H)", 8: "hot only (id < H)", 9: "hot from smem, cold global"}
bps_list = [int(b) for b in os.environ.get("UB_BPS", "4,8").split(",")]
for v in [int(a) for a in (sys.argv[2].split(",") if len(sys.argv) > 2 else range(7))]:
    for bps in bps_list:
        ms = ctypes.c_double()
        _lib.check(L.pr_debug_gather(g.dev.handle, v, 20, bps, ctypes.byref(ms)))
        print(f"{cfg} H={os.environ.get('PR_UB_H', 16384)} {names[v]:26s} blocks/SM={bps:2d}: {ms.value*1e3:8.1f} us")
