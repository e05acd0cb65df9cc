"""pytest plugin (``-p refgate_shim``) that runs the reference's own test
files against this package under the ``pushrank`` name (SURVEY.md section 7
step 3).

Loaded before the reference's conftest and test modules are imported, it
imports the installed reference package (baseline/_ref, on PYTHONPATH) and
rebinds every hot-path name -- graph core, engines, sync twin, power method,
types, the ERR harness -- to this package's CUDA implementation, in the
package namespace and in the submodules the tests import from
(pushrank.graph, pushrank.engines, pushrank.solvers, pushrank.bench).
``available_backends()`` reports only "cuda", so the suite's ``backend``
fixture (tests/conftest.py:38-40 in the reference) runs every engine test on
the device.  Names off the push-round path stay the reference's own:
dense_oracle / series_pagerank / forward_push_ppr (test oracles), synth,
cli.  TEST INFRASTRUCTURE only.
"""

import paper_2302_03245_b200 as P
import pushrank
import pushrank._backend
import pushrank.bench
import pushrank.engines
import pushrank.graph
import pushrank.solvers
from paper_2302_03245_b200 import graph as PG
from paper_2302_03245_b200 import harness as PH

OURS = {
    "from_edges": P.from_edges, "classify": P.classify, "preprocess_ifp2": P.preprocess_ifp2,
    "dangling_target_counts": PG.dangling_target_counts, "load_edge_list": P.load_edge_list,
    "GraphFormatError": P.GraphFormatError, "stats": P.stats, "StatsRow": P.StatsRow,
    "ifp1_run": P.ifp1_run, "ifp2_run": P.ifp2_run, "ifp2_full_run": P.ifp2_full_run,
    "sync_simulate": P.sync_simulate, "power_method": P.power_method,
    "partition_vertices": P.partition_vertices, "MassState": P.MassState, "Partition": P.Partition,
    "SolverConfig": P.SolverConfig, "PageRankVector": P.PageRankVector,
    "RunTrace": P.RunTrace, "TraceSample": P.TraceSample,
    "resolve_backend": P.resolve_backend,
}
HARNESS = [n for n in dir(PH) if not n.startswith("__") and hasattr(pushrank.bench, n)
           and n not in ("np", "os", "time", "math", "json", "hashlib", "dataclass", "annotations")]


def _cuda_only():
    return ["cuda"]


for mod in (pushrank, pushrank.graph, pushrank.engines, pushrank.solvers, pushrank.bench):
    for name, obj in OURS.items():
        if hasattr(mod, name):
            setattr(mod, name, obj)
for name in HARNESS:
    setattr(pushrank.bench, name, getattr(PH, name))
pushrank.available_backends = _cuda_only
pushrank._backend.available_backends = _cuda_only
