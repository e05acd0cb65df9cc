"""The reference itself against the CUDA path, on the GPU box.

baseline/_ref holds the reference package as installed by ``pip install
--no-deps --target baseline/_ref`` from a scratch copy of /root/reference
(with its tests/ directory copied beside it); it is git-ignored but travels
to the GPU box, so these tests read nothing under /root/reference.  They
skip when it is absent.

* test_reference_suite_files: the reference's own test_engines.py,
  test_graph.py, test_solvers.py, test_metrics.py and test_acceptance.py run
  unmodified with every hot-path name bound to this package
  (tests/refgate_shim.py) and backend "cuda".
* test_reference_side_binding: integration/pushrank_cuda.py (INTEGRATION.md
  section B) dropped into a scratch copy of the reference as
  pushrank/_cuda.py, with the three documented edits applied; the
  reference's own unchanged ifp1_run / ifp2_run with backend="cuda" must
  match backend="c" (its compiled CPU kernel) -- in particular IFP2 settles
  exactly once (push_ops_dangling == m_d, mass of the dangling vertices).
"""

import json
import os
import shutil
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
LIB = os.path.join(REPO, "paper_2302_03245_b200", "lib", "libpushrank_cuda.so")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "pushrank")),
                                 reason="reference not installed in baseline/_ref")]

# reference test files run through the shim; test_backends.py (the CPU
# worker_loop / probe kernel protocol) and test_cli.py are outside the path
SUITE = ["test_engines.py", "test_graph.py", "test_solvers.py", "test_metrics.py", "test_acceptance.py"]
# reference tests that exercise something this package deliberately does not
# provide (reason); deselected, listed in DESIGN.md section 3
NOT_PROVIDED = {
    "test_metrics.py::test_sweep_cycle_all_algorithms_tiny_err":
        "sweeps algorithm 'fp', the serial forward_push_ppr test oracle (solvers.py:271-343), which is outside "
        "the push-round path; the harness raises ValueError for it",
}


def test_reference_suite_files():
    tests = os.path.join(REF, "tests")
    if not os.path.isdir(tests):
        pytest.skip("reference tests not staged in baseline/_ref/tests")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, REPO, os.path.join(REPO, "tests"), tests]))
    deselect = [a for t in NOT_PROVIDED for a in ("--deselect", t)]
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "refgate_shim", "-p", "no:cacheprovider",
                          "--rootdir", tests, *deselect, *SUITE],
                         cwd=tests, env=env, capture_output=True, text=True, timeout=1800)
    tail = "\n".join(out.stdout.splitlines()[-40:])
    assert out.returncode == 0, tail + out.stderr[-2000:]
    assert " passed" in tail, tail


SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import pushrank as R
from pushrank import synth
assert R.resolve_backend("cuda").NAME == "cuda"
out = []
graphs = [("chain3", R.from_edges(3, [0, 1], [1, 2])), ("fanin3", R.from_edges(3, [0, 1], [2, 2])),
          ("cycle2", R.from_edges(2, [0, 1], [1, 0])), ("empty3", R.from_edges(3, [], []))]
sys.path.insert(0, "/root/repo/tests")
graphs += [(f"rand{i}", g) for i, g in enumerate(__import__("corpus").random_corpus(12, seed=31))]
graphs.append(("synth42", synth.generate(10_000, 100_000, dangling_fraction=0.2, seed=42)))
cfg = R.SolverConfig(threshold=1e-10)
for name, g in graphs:
    cls = R.classify(g)
    pg = R.preprocess_ifp2(g, cls)
    row = {"name": name, "n": int(g.n), "m_d": int(cls.dangling_edge_count)}
    for algo in ("ifp1", "ifp2"):
        res = {}
        for be in ("c", "cuda"):
            if algo == "ifp1":
                v, t = R.ifp1_run(g, cls, cfg, workers=2, backend=be)
            else:
                v, t = R.ifp2_run(pg, cfg, workers=2, backend=be)
            res[be] = (v.values, t)
        a, b = res["c"][0], res["cuda"][0]
        top = lambda x: np.lexsort((np.arange(x.size), -x))[:100]
        row[algo] = {"l1": float(np.abs(a - b).sum()), "top100": bool(np.array_equal(top(a), top(b))),
                     "sum": float(b.sum()), "pod_cuda": int(res["cuda"][1].final.push_ops_dangling),
                     "pod_c": int(res["c"][1].final.push_ops_dangling),
                     "rows_cuda": len(res["cuda"][1].samples)}
    out.append(row)
print(json.dumps(out))
'''


def test_reference_side_binding(tmp_path):
    scratch = tmp_path / "ref"
    shutil.copytree(os.path.join(REF, "pushrank"), scratch / "pushrank")
    shutil.copy(os.path.join(REPO, "integration", "pushrank_cuda.py"), scratch / "pushrank" / "_cuda.py")
    shutil.copy(os.path.join(REF, "tests", "corpus.py"), tmp_path / "corpus.py") \
        if os.path.exists(os.path.join(REF, "tests", "corpus.py")) else None
    # the three edits INTEGRATION.md section B documents
    be = scratch / "pushrank" / "_backend.py"
    src = be.read_text()
    old = '    if name in ("python", "py", "pure"):'
    assert src.count(old) == 1
    be.write_text(src.replace(old, '    if name == "cuda":\n        from . import _cuda\n        return _cuda\n' + old))
    en = scratch / "pushrank" / "engines.py"
    src = en.read_text()
    edits = [
        ("               start_time, sample_every):\n",
         "               start_time, sample_every, graph=None, algorithm=None):\n"
         "    if backend.NAME == \"cuda\":\n"
         "        return backend.run_phase(graph, algorithm, h, reserved, xi, damping, scan_ids,\n"
         "                                 dangling_mask, degree, trace, start_time)\n"),
        ("               _auto_sample_every(g.n, sample_every))\n    trace.meta[\"wall_s\"]",
         "               _auto_sample_every(g.n, sample_every), graph=g, algorithm=\"ifp1\")\n"
         "    trace.meta[\"wall_s\"]"),
        ("                       _auto_sample_every(g.n, sample_every))\n    settled",
         "                       _auto_sample_every(g.n, sample_every), graph=pg, algorithm=\"ifp2\")\n"
         "    settled"),
    ]
    for old, new in edits:
        assert src.count(old) == 1, old
        src = src.replace(old, new)
    en.write_text(src)
    env = dict(os.environ, PUSHRANK_CUDA_LIB=LIB)
    script = SCRIPT.replace("/root/repo/tests", str(tmp_path))
    out = subprocess.run([sys.executable, "-c", script, str(scratch)], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    rows = json.loads(out.stdout.strip().splitlines()[-1])
    bad = []
    for r in rows:
        for algo in ("ifp1", "ifp2"):
            x = r[algo]
            # top-100 under (-score, id) is compared on the acceptance graph;
            # the tiny graphs are tie-heavy (cycle2: [0.5, 0.5]), where 1e-12
            # differences legitimately reorder equal scores
            if not (x["l1"] <= 1e-9 and abs(x["sum"] - 1.0) <= 1e-12 and (x["top100"] or r["n"] < 1000)):
                bad.append((r["name"], algo, x))
        # single settle: every dangling in-edge pushed exactly once
        if not (r["ifp2"]["pod_cuda"] == r["m_d"] == r["ifp2"]["pod_c"] and r["ifp1"]["pod_cuda"] >= r["m_d"]):
            bad.append((r["name"], "push_ops_dangling", r))
    assert not bad, bad
    assert any(r["name"] == "synth42" for r in rows)
