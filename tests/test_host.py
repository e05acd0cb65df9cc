"""CPU-only checks of the host layer and the C-ABI library (no compute)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2302_03245_b200 as P
from paper_2302_03245_b200 import _lib, synthetic

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    names = []
    for fn in os.listdir(os.path.join(REPO, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(REPO, "include", fn)).read()
            names += re.findall(r"^\s*(?:int|const char \*|void)\s*\**\s*(pr_\w+)\s*\(", text, re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)
    assert L.pr_abi_version() == 3


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.RoundStats) == 80
    assert _lib.ROUND_DTYPE.itemsize == 80
    assert ctypes.sizeof(_lib.RunResult) == 15 * 8


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_no_cpu_fallback_without_device():
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    assert P.available_backends() == []
    with pytest.raises(RuntimeError):
        P.from_edges(3, [0, 1], [1, 2])


def test_solver_config_validation_messages():
    with pytest.raises(ValueError, match="damping"):
        P.SolverConfig(damping=1.0).validate(3)
    with pytest.raises(ValueError, match="threshold"):
        P.SolverConfig(threshold=-1).validate(3)
    with pytest.raises(ValueError, match="personalization"):
        P.SolverConfig(personalization=np.ones(2)).validate(3)
    with pytest.raises(ValueError, match="non-negative"):
        P.SolverConfig(max_iterations=-1).validate(3)
    P.SolverConfig().validate(3)
    assert P.SolverConfig().restart_vector(4).tolist() == [0.25] * 4


def test_backend_resolution():
    assert P.resolve_backend("cuda").NAME == "cuda"
    assert P.resolve_backend("auto").NAME == "cuda"
    with pytest.raises(ValueError, match="backend"):
        P.resolve_backend("python")


def test_from_edges_argument_errors_before_device():
    with pytest.raises(ValueError, match="equal length"):
        P.from_edges(3, [0, 1], [1])
    with pytest.raises(ValueError, match="at least one"):
        P.from_edges(0, [], [])
    with pytest.raises(ValueError, match="range"):
        P.from_edges(2, [0], [2])


def test_trace_csv(tmp_path):
    tr = P.RunTrace(samples=[P.TraceSample(0, 1.5, 2, 1.0, 3, 4, 5, 6.0)])
    path = tmp_path / "t.csv"
    tr.write_csv(path)
    lines = path.read_text().splitlines()
    assert lines[0] == "t,h_l1,converged,alpha,work,push_ops,push_ops_dangling,wall_ms"
    assert lines[1] == "0,1.5,2,1.0,3,4,5,6.000"
    assert tr.final.push_ops == 4


def test_rmat_numpy_generator_is_deterministic_and_sane():
    n, s1, d1 = synthetic.rmat_edges(12, 4, seed=3)
    _, s2, d2 = synthetic.rmat_edges(12, 4, seed=3, first=100, count=50)
    assert np.array_equal(s1[100:150], s2) and np.array_equal(d1[100:150], d2)
    assert n == 4096 and s1.max() < n and d1.max() < n
    # quadrant a dominates: the low half of the id range holds ~76% of sources
    assert 0.70 < np.mean(s1 < n // 2) < 0.82


# ------------------------------------------------------------ edge-list ingest (host part)

def test_edge_list_host_parse_matches_reference_errors():
    """The host re-parse that load_edge_list falls back to for text the
    device parser refuses reports the reference's exceptions (graph.py:
    180-236); pinned by tests/golden/edge_lists.npz (made by the reference)."""
    import os
    from paper_2302_03245_b200.ingest import GraphFormatError, _host_parse
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "edge_lists.npz"))
    for i in range(int(d["n_bad"])):
        text = d[f"bad{i}_text"].tobytes()
        want_type, want_msg = str(d[f"bad{i}_type"]), str(d[f"bad{i}_msg"])
        try:
            src, dst = _host_parse(text)
        except Exception as exc:  # noqa: BLE001
            assert type(exc).__name__ == want_type, (i, exc)
            assert str(exc) == want_msg, (i, exc)
            continue
        # no exception: only the empty streams get here (load_edge_list raises)
        assert src.size == 0 and "empty graph" in want_msg, i
    for i in range(int(d["n_ok"])):
        src, dst = _host_parse(d[f"ok{i}_text"].tobytes())
        assert src.size == int(d[f"ok{i}_raw"]), i


def test_score_format_is_python_repr():
    """Ranking CSV scores are written natively as Python repr(float)
    (serialize.py:21): shortest round-trip digits, fixed notation for decimal
    exponents -4..15, scientific otherwise."""
    from paper_2302_03245_b200.serialize import format_score
    rng = np.random.default_rng(7)
    special = [0.0, -0.0, 1.0, -1.0, 0.1, 0.0001, 0.00001, 1e15, 1e16, 1.5e16, 123456789012345.0,
               1234567890123456.0, 12345678901234567.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
               1 / 3, 2 / 3, 0.15, 0.3, 1e-10, 9.999999999999999e-05, 0.00010000000000000009, 100.0, 1e22]
    vals = special + list(rng.random(2000)) + list(rng.random(1000) * 1e-12) \
        + list(10.0 ** rng.uniform(-300, 300, 2000)) + list(-(10.0 ** rng.uniform(-20, 20, 500)))
    for v in vals:
        assert format_score(v) == repr(float(v)), v
