"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's golden vectors.

Bars (BASELINE.json north_star): integer preprocessing bit-exact; exact
(sync) rounds bit-identical state; fast engines within L1 <= 1e-9 of the
reference vectors with identical top-100 under (-score, id).
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import corpus_graph

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2302_03245_b200")
from paper_2302_03245_b200 import synthetic  # noqa: E402

XI = 1e-12
INT_KEYS = ("out_offsets", "out_targets", "in_offsets", "in_sources")
CLS_KEYS = ("dangling", "unreferenced", "weak_dangling", "weak_unreferenced")
IFP2_KEYS = ("live_offsets", "live_targets", "live_degree", "dangling_ids", "source_offsets", "source_ids")
MODES = ("auto", "pull", "push")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def top100(values):
    order = np.lexsort((np.arange(values.size), -values))   # (-score, id), serialize.py:16
    return order[:100]


def cfg(xi=XI):
    return P.SolverConfig(threshold=xi)


# ------------------------------------------------------------ graph core

def test_corpus_preprocessing_bit_exact(golden_corpus):
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        g = P.from_edges(n, src, dst)
        for k in INT_KEYS:
            assert np.array_equal(getattr(g, k), golden_corpus[f"g{i}_{k}"]), (i, k)
        cls = P.classify(g)
        for k in CLS_KEYS:
            assert np.array_equal(getattr(cls, k), golden_corpus[f"g{i}_{k}"]), (i, k)
        assert cls.dangling_edge_count == int(golden_corpus[f"g{i}_m_d"])
        assert np.array_equal(P.dangling_target_counts(g, cls), golden_corpus[f"g{i}_dtc"])
        pg = P.preprocess_ifp2(g, cls)
        for k in IFP2_KEYS:
            assert np.array_equal(getattr(pg, k), golden_corpus[f"g{i}_{k}"]), (i, k)


@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c4"])
def test_config_preprocessing_bit_exact(config, golden_c1):
    n, src, dst = synthetic.make(config, seed=0)
    g = P.from_edges(n, src, dst)
    ref = oracle.from_edges(n, src, dst)
    for k in INT_KEYS:
        assert np.array_equal(getattr(g, k), getattr(ref, k)), k
    cls = P.classify(g)
    rc = oracle.classify(ref)
    for k in CLS_KEYS:
        assert np.array_equal(getattr(cls, k), getattr(rc, k)), k
    assert cls.dangling_edge_count == rc.dangling_edge_count
    pg = P.preprocess_ifp2(g, cls)
    rp = oracle.preprocess_ifp2(ref, rc.dangling)
    for k in IFP2_KEYS:
        assert np.array_equal(getattr(pg, k), getattr(rp, k)), k
    if config == "c1":
        for k in INT_KEYS + CLS_KEYS + IFP2_KEYS:
            gold = golden_c1[f"{k}_sha256"]
            obj = pg if k in IFP2_KEYS else (cls if k in CLS_KEYS else g)
            assert sha(getattr(obj, k)) == str(gold), k


def test_upload_roundtrip_and_errors():
    n, src, dst = synthetic.make("c1", seed=1)
    ref = oracle.from_edges(n, src, dst)
    dev = P.graph.DeviceGraph.upload(ref)
    out = dev.export()
    for k in INT_KEYS:
        assert np.array_equal(out[k], getattr(ref, k)), k
    with pytest.raises(ValueError, match="range"):
        P.from_edges(2, [0], [2])
    with pytest.raises(ValueError):
        P.from_edges(0, [], [])


def test_lazy_out_targets_upload():
    """CSC-only upload: the fast engines rebuild their out-adjacency on the
    device; calls that need the original out_targets attach them on demand,
    and the C-ABI refuses them loudly before that."""
    from paper_2302_03245_b200 import _lib
    import ctypes
    n, src, dst = synthetic.make("c1", seed=3)
    ref = oracle.from_edges(n, src, dst)
    lazy = P.graph.DeviceGraph.upload(ref)
    eager = P.graph.DeviceGraph.upload(ref, lazy_out_targets=False)
    assert lazy._pending_out_targets is not None
    assert lazy.h2d_bytes == eager.h2d_bytes - 8 * ref.m
    c = _lib.ClassCounts()
    assert _lib.load().pr_classify(lazy.handle, ctypes.byref(c)) == _lib.PR_ERR_STATE
    assert "out_targets" in _lib.load().pr_last_error().decode()
    for algo in ("ifp1", "ifp2"):
        lazy.preprocess_ifp2()
        eager.preprocess_ifp2()
        vl, _, rl, _, _ = lazy.run(algo, "auto", 0.85, 1e-10, 10_000, _lib.CONV_SCAN)
        ve, _, re, _, _ = eager.run(algo, "auto", 0.85, 1e-10, 10_000, _lib.CONV_SCAN)
        # push rounds add with atomics, so the two runs can differ in the last
        # bits (and, rarely, in a vertex sitting exactly at the threshold)
        assert abs(rl.push_ops - re.push_ops) <= 1e-3 * re.push_ops and abs(rl.rounds - re.rounds) <= 1, algo
        assert np.abs(vl - ve).sum() <= 1e-11, algo
    assert lazy._pending_out_targets is not None   # never needed by the fast engines
    assert np.array_equal(lazy.dangling_target_counts(), eager.dangling_target_counts())
    out = lazy.export()                            # attaches
    assert lazy._pending_out_targets is None
    assert np.array_equal(out["out_targets"], ref.out_targets)
    assert lazy.classify().dangling == eager.classify().dangling


def test_load_edge_list_matches_reference():
    """load_edge_list (graph.py:201-259) on the device: every array of the
    reference's Graph bit-exact (first-appearance remap, dedup, CSR/CSC),
    and the reference's exception for every malformed text."""
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "edge_lists.npz"))
    for i in range(int(d["n_ok"])):
        g = P.load_edge_list(d[f"ok{i}_text"].tobytes())
        assert g.n == int(d[f"ok{i}_n"]) and g.raw_edge_count == int(d[f"ok{i}_raw"]), i
        for k in ("original_ids", "out_offsets", "out_targets", "in_offsets", "in_sources"):
            assert np.array_equal(getattr(g, k), d[f"ok{i}_{k}"]), (i, k)
    for i in range(int(d["n_bad"])):
        with pytest.raises(Exception) as info:
            P.load_edge_list(d[f"bad{i}_text"].tobytes())
        assert type(info.value).__name__ == str(d[f"bad{i}_type"]), i
        assert str(info.value) == str(d[f"bad{i}_msg"]), i
    # path and stream sources, name inference (graph.py:211-219)
    import io, tempfile
    with tempfile.NamedTemporaryFile("wb", suffix=".txt", delete=False) as fh:
        fh.write(b"7 3\n3 1\n")
    try:
        g = P.load_edge_list(fh.name)
        assert g.name == os.path.splitext(os.path.basename(fh.name))[0]
        assert g.original_ids.tolist() == [7, 3, 1]
    finally:
        os.unlink(fh.name)
    g = P.load_edge_list(io.BytesIO(b"0\t1\n1\t0\n"), name="s")
    assert g.name == "s" and g.m == 2
    # the device parser took the valid texts: a graph built from it runs
    vec, _ = P.ifp2_run(P.preprocess_ifp2(g, P.classify(g)), cfg())
    assert vec.values == pytest.approx([0.5, 0.5], abs=1e-10)


def test_ranking_csv_matches_reference(tmp_path):
    """write_ranking_csv (serialize.py:14-21): device ordering (score desc,
    ties by original id) and native row writing, byte-identical to the
    reference's file; ranking_order equals np.lexsort((ids, -values))."""
    import os
    from types import SimpleNamespace
    from paper_2302_03245_b200 import serialize
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "serialize.npz"))
    for i in range(int(d["count"])):
        vals, ids = d[f"c{i}_values"], d[f"c{i}_ids"]
        g = SimpleNamespace(original_ids=ids)
        vec = P.PageRankVector(values=vals, algorithm="x", damping=0.85)
        path = tmp_path / f"r{i}.csv"
        serialize.write_ranking_csv(vec, g, path)
        assert path.read_bytes() == d[f"c{i}_csv"].tobytes(), i
        assert np.array_equal(serialize.ranking_order(vals, g), np.lexsort((ids, -vals))), i
        assert np.array_equal(serialize.ranking_order(vals, g, k=10), np.lexsort((ids, -vals))[:10]), i
    # binary vector round trip (serialize.py:24-38)
    vec = P.PageRankVector(values=d["c0_values"], algorithm="x", damping=0.85)
    serialize.write_vector_binary(vec, tmp_path / "v.bin")
    assert np.array_equal(serialize.read_vector_binary(tmp_path / "v.bin"), d["c0_values"])


def test_rmat_device_generator_matches_numpy():
    from paper_2302_03245_b200 import _lib
    import ctypes
    ctx = _lib.context()
    L = _lib.load()
    count = 200_000
    ps, pd = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(L.pr_device_alloc(ctx.handle, 8 * count, ctypes.byref(ps)))
    _lib.check(L.pr_device_alloc(ctx.handle, 8 * count, ctypes.byref(pd)))
    _lib.check(L.pr_rmat_generate(ctx.handle, 20, 5, 0.57, 0.19, 0.19, 7, 12345, count, ps, pd))
    hs, hd = np.empty(count, np.int64), np.empty(count, np.int64)
    _lib.check(L.pr_memcpy_d2h(ctx.handle, _lib.ptr(hs), ps, 8 * count))
    _lib.check(L.pr_memcpy_d2h(ctx.handle, _lib.ptr(hd), pd, 8 * count))
    L.pr_device_free(ctx.handle, ps)
    L.pr_device_free(ctx.handle, pd)
    _, s, d = synthetic.rmat_edges(20, 5, seed=7, first=12345, count=count)
    assert np.array_equal(hs, s) and np.array_equal(hd, d)


# ------------------------------------------------------------ exact (sync) rounds

def _sync_check(gold, key, vec, tr):
    for col in ("converged", "work", "push_ops", "push_ops_dangling"):
        assert np.array_equal(np.asarray(tr.column(col)), gold[key + col]), (key, col)
    scale = max(1.0, float(gold[key + "h_l1"][0]))
    for col in ("h_l1", "alpha", "active_mass", "carry_mass"):
        np.testing.assert_allclose(tr.column(col), gold[key + col], rtol=1e-12, atol=1e-14 * scale)
    np.testing.assert_allclose(vec.values, gold[key + "values"], rtol=1e-13, atol=1e-17)


def test_corpus_sync_exact_state_bit_identical(golden_corpus):
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        g = P.from_edges(n, src, dst)
        cls = P.classify(g)
        pg = P.preprocess_ifp2(g, cls)
        for variant in ("ifp1", "ifp2", "fp-full"):
            key = f"g{i}_sync_{variant.replace('-', '_')}_"
            last = {}

            def cb(t, r, h, last=last):
                last["r"], last["h"] = r.copy(), h.copy()

            subject = pg if variant == "ifp2" else g
            vec, tr = P.sync_simulate(subject, cfg(), variant=variant, cls=cls, on_iteration=cb)
            _sync_check(golden_corpus, key, vec, tr)
            if key + "reserved_pre_settle" in golden_corpus:
                assert np.array_equal(last["r"], golden_corpus[key + "reserved_pre_settle"]), key
                assert np.array_equal(last["h"], golden_corpus[key + "h_pre_settle"]), key


@pytest.mark.parametrize("config", ["c1", "c2"])
def test_sync_exact_per_round_digest_matches_oracle(config):
    """Every round's (reserved, pending) state bit-identical to the oracle's
    restatement of sync_simulate, via the per-row state digest (device graph
    loop, no host round trips)."""
    n, src, dst = synthetic.make(config, seed=0)
    g = P.from_edges(n, src, dst)
    ref = oracle.from_edges(n, src, dst)
    for variant in ("ifp1", "ifp2"):
        o = oracle.sync_simulate(ref, variant, threshold=1e-10)
        dev = P.graph.device_graph(g)
        if variant == "ifp2":
            dev.preprocess_ifp2()
        values, rows, res, reserved, pending = dev.run(variant, "exact", 0.85, 1e-10, 1_000_000,
                                                       1, want_state=True)
        k = len(o.rows) - (1 if variant == "ifp2" else 0)
        assert res.rounds == o.iterations
        assert np.array_equal(rows["digest"][:k], o.rows["digest"][:k]), variant
        for col in ("converged", "work", "push_ops", "push_ops_dangling"):
            assert np.array_equal(rows[col], o.rows[col]), (variant, col)
        if variant == "ifp1":
            assert np.array_equal(reserved, o.reserved) and np.array_equal(pending, o.h)
        np.testing.assert_allclose(values, o.values, rtol=1e-12, atol=0)


# ------------------------------------------------------------ fast engines vs reference

@pytest.mark.parametrize("mode", MODES)
def test_corpus_engines_match_reference(golden_corpus, mode):
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        g = P.from_edges(n, src, dst)
        cls = P.classify(g)
        pg = P.preprocess_ifp2(g, cls)
        v1, t1 = P.ifp1_run(g, cls, cfg(), workers=4, mode=mode)
        v2, t2 = P.ifp2_run(pg, cfg(), workers=4, mode=mode)
        tol = max(1e-10, 10 * XI * n)
        assert np.max(np.abs(v1.values - golden_corpus[f"g{i}_ifp1_values"])) <= tol, i
        assert np.max(np.abs(v2.values - golden_corpus[f"g{i}_ifp2_values"])) <= tol, i
        assert t2.final.push_ops_dangling == cls.dangling_edge_count
        assert t1.final.push_ops_dangling >= cls.dangling_edge_count
        if f"g{i}_dense_values" in golden_corpus:
            d = golden_corpus[f"g{i}_dense_values"]
            assert np.max(np.abs(v1.values - d) / d) <= max(1e-8, 10 * XI * n)


@pytest.mark.parametrize("mode", MODES)
def test_c1_engines_parity(golden_c1, mode):
    n, src, dst = synthetic.make("c1", seed=0)
    g = P.from_edges(n, src, dst)
    cls = P.classify(g)
    pg = P.preprocess_ifp2(g, cls)
    for algo, run in (("ifp1", lambda: P.ifp1_run(g, cls, cfg(), mode=mode)),
                      ("ifp2", lambda: P.ifp2_run(pg, cfg(), mode=mode))):
        vec, tr = run()
        ref = golden_c1[f"{algo}_values"]
        assert np.abs(vec.values - ref).sum() <= 1e-9, algo
        assert np.array_equal(top100(vec.values), top100(ref)), algo
        assert abs(vec.values.sum() - 1.0) <= 1e-12
    assert tr.final.push_ops_dangling == int(golden_c1["ifp2_push_ops_dangling"])
    # the phase-1 final row precedes the settle row (engines.py:331-335)
    assert tr.samples[-2].push_ops_dangling == 0


@pytest.mark.parametrize("xi", [1e-10, 1e-12])
def test_c2_full_size_parity(xi):
    """C2 at full size: fast engine vs the oracle sync twin (L1 <= 1e-9,
    identical top-100) and mass conservation."""
    n, src, dst = synthetic.make("c2", seed=0)
    g = P.from_edges(n, src, dst)
    ref = oracle.from_edges(n, src, dst)
    cls = P.classify(g)
    pg = P.preprocess_ifp2(g, cls)
    for algo in ("ifp1", "ifp2"):
        o = oracle.sync_simulate(ref, algo, threshold=xi)
        for mode in MODES:
            if algo == "ifp1":
                vec, tr = P.ifp1_run(g, cls, cfg(xi), mode=mode)
            else:
                vec, tr = P.ifp2_run(pg, cfg(xi), mode=mode)
            assert np.abs(vec.values - o.values).sum() <= 1e-9, (algo, mode)
            assert np.array_equal(top100(vec.values), top100(o.values)), (algo, mode)
            if algo == "ifp2":
                assert tr.final.push_ops_dangling == cls.dangling_edge_count


@pytest.mark.parametrize("sections", [2, 3, 8])
def test_gauss_seidel_sections_parity(sections, monkeypatch, golden_corpus):
    """IFP2 dense sweeps cut into Gauss-Seidel sections (big graphs use them
    by default; PUSHRANK_GS_SECTIONS forces them here): same fixed point as
    the round-synchronous oracle (L1 <= 1e-9, identical top-100), mass 1,
    every dangling in-edge settled, and fewer rounds than Jacobi."""
    monkeypatch.setenv("PUSHRANK_GS_SECTIONS", str(sections))
    n, src, dst = synthetic.make("c2", seed=0)
    g = P.from_edges(n, src, dst)
    ref = oracle.from_edges(n, src, dst)
    cls = P.classify(g)
    pg = P.preprocess_ifp2(g, cls)
    o = oracle.sync_simulate(ref, "ifp2", threshold=XI)
    for mode in MODES:
        vec, tr = P.ifp2_run(pg, cfg(), mode=mode)
        assert np.abs(vec.values - o.values).sum() <= 1e-9, mode
        assert np.array_equal(top100(vec.values), top100(o.values)), mode
        assert abs(vec.values.sum() - 1.0) <= 1e-12
        assert tr.final.push_ops_dangling == cls.dangling_edge_count
        if mode == "pull":
            assert tr.meta["rounds"] < o.iterations, (tr.meta["rounds"], o.iterations)
    # and on every corpus graph (tiny ones have a single section)
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        pg = P.preprocess_ifp2(P.from_edges(n, src, dst), None)
        v2, _ = P.ifp2_run(pg, cfg(), mode="auto")
        assert np.max(np.abs(v2.values - golden_corpus[f"g{i}_ifp2_values"])) <= max(1e-10, 10 * XI * n), i


@pytest.mark.parametrize("sections", [2, 3, 8])
def test_gauss_seidel_sections_ifp1(sections, monkeypatch):
    """IFP1 sweeps in Gauss-Seidel sections: the IFP1 schedule interleaves
    class-0 rows and dangling receivers by degree, so earlier sections'
    sources are found by an id bound (class-0 ids stay in row order) and the
    push filter by each vertex's row section.  Same fixed point as the
    oracle's IFP1 twin (L1 <= 1e-9, identical top-100), mass 1, fewer rounds
    in pull mode, and bit-identical pull-mode runs (the round-0 seeds are
    gathered by the first dense round in fixed order, not scattered)."""
    monkeypatch.setenv("PUSHRANK_GS_SECTIONS", str(sections))
    n, src, dst = synthetic.make("c2", seed=0)
    g = P.from_edges(n, src, dst)
    cls = P.classify(g)
    o = oracle.sync_simulate(oracle.from_edges(n, src, dst), "ifp1", threshold=XI)
    for mode in MODES:
        vec, tr = P.ifp1_run(g, cls, cfg(), mode=mode)
        assert np.abs(vec.values - o.values).sum() <= 1e-9, mode
        assert np.array_equal(top100(vec.values), top100(o.values)), mode
        assert abs(vec.values.sum() - 1.0) <= 1e-12
        if mode == "pull":
            assert tr.meta["rounds"] < o.iterations, (tr.meta["rounds"], o.iterations)
            again, _ = P.ifp1_run(g, cls, cfg(), mode=mode)
            assert np.array_equal(again.values, vec.values)


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_config_engines_parity(config):
    """C3 (52 M edges, 2 Gauss-Seidel sections) and C4 (the DAG that
    exercises IFP1 peeling and dangling convergence): integer preprocessing
    bit-exact, then IFP1 and IFP2 in auto, pull and push modes against the
    oracle's round-synchronous twin -- L1 <= 1e-9, identical top-100, mass 1,
    push_ops_dangling == m_d (IFP2) -- via tests/full_size_parity.py."""
    import full_size_parity as F
    v = F.run(config, xi=1e-10)
    bad = [c for c in v["checks"] if not c["ok"]]
    assert not bad, bad


def test_forced_c5_code_path_parity(monkeypatch):
    """C5's code path at a size the oracle finishes in about a minute: R-MAT
    scale 23 (134 M edges) with 6 Gauss-Seidel sections, source-sorted CSC
    rows and the streamed (evict-first) k_pull forced as at C5.  Device vs
    host edge generators, integer preprocessing bit-exact, IFP2 and IFP1
    (auto + pull) against the oracle twin.  The full C5 run of the same
    script is profiles/r02_parity_c5.json."""
    import full_size_parity as F
    monkeypatch.setenv("PUSHRANK_GS_SECTIONS", "6")
    monkeypatch.setenv("PUSHRANK_SORT_ROWS", "1")
    monkeypatch.setenv("PUSHRANK_PREFETCH", "0")
    v = F.run("rmat", scale=23, modes=("auto", "pull"), xi=1e-10)
    bad = [c for c in v["checks"] if not c["ok"]]
    assert not bad, bad


def test_c5_full_size_properties():
    """C5 (R-MAT scale 26, 1.06 B edges; too large for the oracle): size-
    independent properties of the fast IFP2 engine (6 Gauss-Seidel sections):
    mass 1, m_d dangling pushes, agreement with 210 power iterations (L1 and
    top-100), and the ranking order against numpy."""
    from paper_2302_03245_b200 import serialize
    dev = P.graph.DeviceGraph.rmat(26, 16, seed=0)
    g = P.graph.Graph(dev, raw_edge_count=16 << 26, name="c5")
    cls = P.classify(g)
    vec, tr = P.ifp2_run(P.preprocess_ifp2(g, cls), cfg())
    assert abs(vec.values.sum() - 1.0) <= 1e-12
    assert tr.final.push_ops_dangling == cls.dangling_edge_count
    pw, _ = P.power_method(g, P.SolverConfig(max_iterations=210))
    assert np.abs(vec.values - pw.values).sum() <= 1e-8
    assert np.array_equal(top100(vec.values), top100(pw.values))
    order = serialize.ranking_order(vec.values, None, k=1000)
    assert np.array_equal(order, np.lexsort((np.arange(g.n), -vec.values))[:1000])


# ------------------------------------------------------------ known answers (reference tests)

def test_known_answers():
    c = P.SolverConfig()
    chain = P.from_edges(3, [0, 1], [1, 2])
    exact = np.array([1.0, 1.85, 2.5725]) / 5.4225                  # test_solvers.py:16-18
    v, _ = P.ifp1_run(chain, P.classify(chain), cfg())
    assert np.max(np.abs(v.values - exact)) <= 1e-10
    pv, _ = P.power_method(chain, c)
    assert np.max(np.abs(pv.values - exact)) < 1e-12               # test_solvers.py:58-61
    fanin = P.from_edges(3, [0, 1], [2, 2])
    cls = P.classify(fanin)
    v2, t2 = P.ifp2_run(P.preprocess_ifp2(fanin, cls), cfg(), workers=2)
    assert np.max(np.abs(v2.values - np.array([1.0, 1.0, 2.7]) / 4.7)) <= 1e-12  # test_engines.py:246-257
    assert t2.samples[-2].push_ops == 0
    cyc = P.from_edges(2, [0, 1], [1, 0])
    v, _ = P.ifp1_run(cyc, P.classify(cyc), cfg())
    assert v.values == pytest.approx([0.5, 0.5], abs=1e-10)
    empty = P.from_edges(3, [], [])
    ce = P.classify(empty)
    v, _ = P.ifp1_run(empty, ce, cfg(), workers=2)
    assert v.values == pytest.approx([1 / 3] * 3, abs=1e-12)       # test_engines.py:278-286
    v, _ = P.ifp2_run(P.preprocess_ifp2(empty, ce), cfg(), workers=2)
    assert v.values == pytest.approx([1 / 3] * 3, abs=1e-12)
    chain_cls = P.classify(chain)
    assert chain_cls.weak_dangling.tolist() == [1] and chain_cls.weak_unreferenced.tolist() == [1]
    single = P.from_edges(1, [], [])
    v, _ = P.ifp1_run(single, P.classify(single), cfg())
    assert v.values.tolist() == [1.0]
    # star4, fp-full sync: a quarter of the mass on the only scanned vertex,
    # first decay 0.85 * 0.25 (test_engines.py:192-197)
    star = P.from_edges(4, [0, 0, 0], [1, 2, 3])
    _, ts = P.sync_simulate(star, cfg(), variant="fp-full")
    assert ts.samples[0].alpha == 0.25
    assert ts.samples[1].h_l1 / ts.samples[0].h_l1 == pytest.approx(0.85 * 0.25, abs=1e-12)


def test_power_matches_reference(golden_corpus, golden_c1):
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        g = P.from_edges(n, src, dst)
        vec, tr = P.power_method(g, P.SolverConfig(max_iterations=210))
        np.testing.assert_allclose(vec.values, golden_corpus[f"g{i}_power_values"], rtol=0, atol=1e-14)
        np.testing.assert_allclose(tr.column("h_l1"), golden_corpus[f"g{i}_power_deltas"], rtol=1e-9, atol=1e-15)
    n, src, dst = synthetic.make("c1", seed=0)
    vec, _ = P.power_method(P.from_edges(n, src, dst), P.SolverConfig(max_iterations=210))
    np.testing.assert_allclose(vec.values, golden_c1["power_values"], rtol=1e-12, atol=0)
    sums = []
    P.power_method(P.from_edges(n, src, dst), P.SolverConfig(max_iterations=20),
                   on_iterate=lambda k, pi: sums.append(float(pi.sum())))
    assert len(sums) == 20 and all(abs(s - 1.0) <= 1e-12 for s in sums)


def test_validation_errors():
    chain = P.from_edges(3, [0, 1], [1, 2])
    cls = P.classify(chain)
    with pytest.raises(ValueError, match="damping"):
        P.ifp1_run(chain, cls, P.SolverConfig(damping=1.5))
    with pytest.raises(ValueError, match="threshold"):
        P.ifp1_run(chain, cls, P.SolverConfig(threshold=0.0))
    with pytest.raises(ValueError, match=">= 1"):
        P.ifp1_run(chain, cls, cfg(), workers=0)
    with pytest.raises(ValueError, match="strategy"):
        P.ifp1_run(chain, cls, cfg(), strategy="zigzag")
    with pytest.raises(ValueError, match="variant"):
        P.sync_simulate(chain, cfg(), variant="both")
    with pytest.raises(ValueError, match="backend"):
        P.ifp1_run(chain, cls, cfg(), backend="fortran")
    cyc = P.from_edges(2, [0, 1], [1, 0])
    with pytest.raises(RuntimeError, match="settle"):
        P.sync_simulate(cyc, cfg(), variant="ifp1", max_iterations=3)
