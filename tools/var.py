"""Build a variant library with extra -D flags: tools/var.py NAME "-DX=1 -DY=2"
-> build/var/lib_NAME.so (used by tools/ab.sh through PUSHRANK_LIB)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_03245_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2].split()
# extra translation units (diagnostics that are not part of the product
# library, e.g. tools/ubench.cu): VAR_EXTRA="a.cu b.cu"
extra = [os.path.abspath(x) for x in os.environ.get("VAR_EXTRA", "").split()]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
odir = os.path.join(root, "build", "var", name)
os.makedirs(odir, exist_ok=True)
sources = B.SOURCES + extra
objs = [os.path.join(odir, os.path.basename(s)[:-3] + ".o") for s in sources]


def one(p):
    subprocess.run([B.nvcc(), *B.NVCC_FLAGS, "-I", os.path.join(B.HERE, "csrc"), *defs, "-c", "-o", p[1], p[0]],
                   check=True,
                   stderr=subprocess.DEVNULL)


with ThreadPoolExecutor(len(objs)) as ex:
    list(ex.map(one, zip(sources, objs)))
subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                os.path.join(root, "build", "var", f"lib_{name}.so"), *objs], check=True)
print("built", name)
