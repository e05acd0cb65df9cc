"""The pipelined index upload (csrc/hostio.cu): host-narrowed chunks and the
raw int64 tail must give the same device graph as a plain copy, for the
adaptive split and for every static split of the array between the two lanes, from page-locked and pageable
host memory, with chunk sizes that do not divide the array."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import os, sys
import numpy as np
sys.path.insert(0, os.environ["REPO"])
import torch
import paper_2302_03245_b200 as P
from paper_2302_03245_b200 import synthetic
from paper_2302_03245_b200.graph import DeviceGraph
from types import SimpleNamespace

n, src, dst = synthetic.make("c2", seed=3)
g = P.from_edges(n, src, dst)
ref = {k: np.ascontiguousarray(getattr(g, k)) for k in ("out_offsets", "out_targets", "in_offsets", "in_sources")}
pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in ref.items()}
m = int(g.m)
for host in (ref, pinned):
    for frac in (None, "0", "0.37", "0.77", "1"):
        # None: the adaptive split (both lanes claim chunks until they meet)
        if frac is None:
            os.environ.pop("PUSHRANK_UPLOAD_HOSTFRAC", None)
        else:
            os.environ["PUSHRANK_UPLOAD_HOSTFRAC"] = frac
        for lazy in (True, False):
            dev = DeviceGraph.upload(SimpleNamespace(n=g.n, m=m, **host), lazy_out_targets=lazy)
            out = dev.export()
            for k in ref:
                assert np.array_equal(out[k], ref[k]), (frac, lazy, k)
            # offsets always travel as int64; the index arrays as 4 or 8 bytes per element
            assert 16 * (n + 1) + 8 * m <= dev.h2d_bytes <= 16 * (n + 1) + 16 * m + 8 * m, dev.h2d_bytes
            del dev
    # the solve on an uploaded graph equals the solve on the built one
    os.environ["PUSHRANK_UPLOAD_HOSTFRAC"] = "0.5"
    dev_graph = SimpleNamespace(n=g.n, m=m, **host)
    v1, _ = P.ifp2_run(P.preprocess_ifp2(dev_graph, None), P.SolverConfig(threshold=1e-12), mode="pull")
    v2, _ = P.ifp2_run(P.preprocess_ifp2(g, None), P.SolverConfig(threshold=1e-12), mode="pull")
    assert np.array_equal(v1.values, v2.values)
print("ok")
"""


def test_pipelined_upload_bit_exact():
    env = dict(os.environ, REPO=REPO, PUSHRANK_UPLOAD_MIN="0", PUSHRANK_UPLOAD_CHUNK="99991",
               PUSHRANK_UPLOAD_THREADS="5")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
