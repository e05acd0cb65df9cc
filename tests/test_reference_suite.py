"""The reference's own test files, restated against this package (SURVEY.md
section 7 step 3): every case of pkg/tests/test_engines.py, test_graph.py and
test_solvers.py that exercises the hot path, with ``backend`` left to the
package default ("cuda").  The GPU box has no /root/reference, so the seeded
corpora those tests draw (corpus.random_corpus(count, seed)), the reference's
dense oracle on them and its partition_vertices outputs come from
tests/golden/suite.npz, written by tests/golden/make_golden.py --only suite
from the real reference package.

Not restated (outside the push-round path, SURVEY.md section 2 / DESIGN.md
section 8): the dense/series/forward-push test oracles themselves
(test_solvers.py:21-45, 89-203 except the power and validation cases) and
the web-Stanford table (dataset absent; test_graph.py:176-188).  Where a
reference test checks an engine against ``dense_oracle``, the reference's
dense values from suite.npz stand in.

Each test names the reference test it restates (file:line).
"""

from __future__ import annotations

import io
import os
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2302_03245_b200 as P
from paper_2302_03245_b200.engines import PARTITION_STRATEGIES

from conftest import GOLDEN

XI = 1e-12
CHAIN3_EXACT = np.array([1.0, 1.85, 2.5725]) / 5.4225      # test_solvers.py:16-18


@pytest.fixture(scope="module")
def suite():
    return dict(np.load(os.path.join(GOLDEN, "suite.npz")))


def _cfg(xi=XI):
    return P.SolverConfig(threshold=xi)


def _edges(suite, seed, i):
    pre = f"s{seed}_{i}_"
    return int(suite[pre + "n"]), suite[pre + "src"], suite[pre + "dst"], suite[pre + "dense"]


def _count(suite, seed):
    return sum(1 for k in suite if k.startswith(f"s{seed}_") and k.endswith("_n"))


def _corpus(suite, seed, count=None):
    """(graph, reference dense values) of corpus.random_corpus(count, seed)."""
    count = count if count is not None else _count(suite, seed)
    out = []
    for i in range(count):
        n, src, dst, dense = _edges(suite, seed, i)
        out.append((P.from_edges(n, src, dst, name=f"rand{i}-n{n}"), dense))
    return out


def _host_graph(n, src, dst):
    """Degree arrays of an edge set after the reference's dedup (graph.py:137)."""
    key = np.unique(np.asarray(src, np.int64) * n + np.asarray(dst, np.int64))
    s, d = key // n, key % n
    return SimpleNamespace(n=n, out_degree=np.bincount(s, minlength=n).astype(np.int64),
                           in_degree=np.bincount(d, minlength=n).astype(np.int64))


def _host_cls(g):
    return SimpleNamespace(dangling=np.flatnonzero(g.out_degree == 0),
                           dangling_mask=lambda n: g.out_degree == 0)


def chain3():
    return P.from_edges(3, [0, 1], [1, 2], name="chain3")


def cycle2():
    return P.from_edges(2, [0, 1], [1, 0], name="cycle2")


def star4():
    return P.from_edges(4, [0, 0, 0], [1, 2, 3], name="star4")


def fanin3():
    return P.from_edges(3, [0, 1], [2, 2], name="fanin3")


def single_vertex():
    return P.from_edges(1, [], [], name="single")


def handcrafted():
    return [chain3(), cycle2(), star4(), fanin3(), single_vertex(), P.from_edges(2, [0, 0], [0, 1], name="selfloop2")]


# ------------------------------------------------------------------ host side (no GPU)

def test_mass_state_initialization():
    # test_engines.py:29-32
    state = P.MassState.fresh(5)
    assert np.array_equal(state.reserved, np.zeros(5))
    assert np.array_equal(state.pushing, np.ones(5))


def test_partition_chain_contiguous():
    # test_engines.py:35-39, 42-45 (chain3: 0 -> 1 -> 2, dangling {2})
    g = _host_graph(3, [0, 1], [1, 2])
    part = P.partition_vertices(g, 2, "contiguous", _host_cls(g))
    assert [s.tolist() for s in part.worker_vertices] == [[0], [1]]
    assert [s.tolist() for s in part.worker_dangling] == [[2], []]
    assert P.partition_vertices(g, 1, "contiguous", _host_cls(g)).worker_vertices[0].tolist() == [0, 1]
    assert part.workers == 2


def test_partition_strided_example():
    # test_engines.py:48-52
    g = _host_graph(10, list(range(9)), list(range(1, 10)))
    part = P.partition_vertices(g, 3, "strided")
    assert [s.tolist() for s in part.worker_vertices] == [[0, 3, 6, 9], [1, 4, 7], [2, 5, 8]]


def test_partition_rejects_bad_input():
    # test_engines.py:55-59
    g = _host_graph(3, [0, 1], [1, 2])
    with pytest.raises(ValueError, match=">= 1"):
        P.partition_vertices(g, 0)
    with pytest.raises(ValueError, match="strategy"):
        P.partition_vertices(g, 2, "zigzag")


@pytest.mark.parametrize("strategy", PARTITION_STRATEGIES)
def test_partition_matches_reference(suite, strategy):
    # test_engines.py:62-77 (cover, disjoint, deterministic, ascending) and
    # the reference's own worker sets, element for element
    for i in range(_count(suite, 23)):
        n, src, dst, _ = _edges(suite, 23, i)
        g = _host_graph(n, src, dst)
        cls = _host_cls(g)
        part = P.partition_vertices(g, 3, strategy, cls)
        pre = f"s23_{i}_part_{strategy}_"
        assert [s.size for s in part.worker_vertices] == suite[pre + "vlen"].tolist()
        assert np.array_equal(np.concatenate(part.worker_vertices), suite[pre + "v"])
        assert [s.size for s in part.worker_dangling] == suite[pre + "dlen"].tolist()
        assert np.array_equal(np.concatenate(part.worker_dangling), suite[pre + "d"])
        universe = np.setdiff1d(np.arange(n), cls.dangling)
        assert np.array_equal(np.sort(np.concatenate(part.worker_vertices)), universe)
        for s in part.worker_vertices:
            assert s.size <= 1 or np.all(np.diff(s) > 0)


def test_partition_degree_balance_bound(suite):
    # test_engines.py:80-94, plus the reference's worker sets
    for k in range(5):
        g = _host_graph(400, suite[f"bal{k}_src"], suite[f"bal{k}_dst"])
        part = P.partition_vertices(g, 4, "degree-balanced")
        assert np.array_equal(np.concatenate(part.worker_vertices), suite[f"bal{k}_v"])
        assert [s.size for s in part.worker_vertices] == suite[f"bal{k}_vlen"].tolist()
        weights = g.out_degree + 1
        loads = np.array([int(weights[s].sum()) for s in part.worker_vertices])
        if weights.max() <= loads.mean():
            assert loads.max() <= 2 * loads.mean()
        assert all(s.size > 0 for s in part.worker_vertices)


# ------------------------------------------------------------------ engines (test_engines.py)

@pytest.mark.gpu
def test_ifp1_cycle():
    # test_engines.py:97-100
    g = cycle2()
    vec, _ = P.ifp1_run(g, P.classify(g), _cfg(), workers=1)
    assert vec.values == pytest.approx([0.5, 0.5], abs=1e-10)


@pytest.mark.gpu
def test_ifp1_chain_matches_oracle_all_k():
    # test_engines.py:103-114
    g = chain3()
    cls = P.classify(g)
    results = {}
    for workers in (1, 2, 4):
        vec, _ = P.ifp1_run(g, cls, _cfg(), workers=workers)
        assert np.max(np.abs(vec.values - CHAIN3_EXACT) / CHAIN3_EXACT) <= 1e-8
        results[workers] = vec.values
    for workers in (2, 4):
        assert np.max(np.abs(results[workers] - results[1])) <= 1e-10


@pytest.mark.gpu
def test_ifp1_counts_dangling_pushes():
    # test_engines.py:117-120
    g = chain3()
    cls = P.classify(g)
    _, trace = P.ifp1_run(g, cls, _cfg(), workers=1)
    assert trace.final.push_ops_dangling >= cls.dangling_edge_count


@pytest.mark.gpu
def test_ifp2_chain_matches_ifp1():
    # test_engines.py:123-128
    g = chain3()
    cls = P.classify(g)
    v1, _ = P.ifp1_run(g, cls, _cfg(), workers=2)
    v2, t2 = P.ifp2_run(P.preprocess_ifp2(g, cls), _cfg(), workers=2)
    assert np.max(np.abs(v1.values - v2.values)) <= 1e-8
    assert t2.final.push_ops_dangling == 1


@pytest.mark.gpu
def test_ifp2_cycle_settle_is_noop():
    # test_engines.py:131-137
    g = cycle2()
    cls = P.classify(g)
    v1, _ = P.ifp1_run(g, cls, _cfg(), workers=2)
    v2, t2 = P.ifp2_run(P.preprocess_ifp2(g, cls), _cfg(), workers=2)
    assert np.max(np.abs(v1.values - v2.values)) <= 1e-10
    assert t2.final.push_ops_dangling == 0


@pytest.mark.gpu
def test_ifp2_fanin_exact():
    # test_engines.py:140-152
    g = fanin3()
    cls = P.classify(g)
    vec, trace = P.ifp2_run(P.preprocess_ifp2(g, cls), _cfg(), workers=2)
    expected = np.array([1.0, 1.0, 2.7]) / 4.7
    assert np.max(np.abs(vec.values - expected)) <= 1e-12
    assert trace.samples[-2].push_ops == 0


@pytest.mark.gpu
def test_ifp2_full_run_reports_preprocess():
    # test_engines.py:155-159
    vec, trace, preprocess_s = P.ifp2_full_run(chain3(), _cfg(), workers=1)
    assert preprocess_s >= 0.0
    assert trace.meta["preprocess_s"] == preprocess_s
    assert vec.values.sum() == pytest.approx(1.0, abs=1e-12)


@pytest.mark.gpu
def test_engines_match_oracle_on_corpus(suite):
    # test_engines.py:162-174 (corpus seed 31, reference dense oracle)
    for g, dense in _corpus(suite, 31):
        cfg = _cfg()
        cls = P.classify(g)
        v1, t1 = P.ifp1_run(g, cls, cfg, workers=4)
        v2, t2 = P.ifp2_run(P.preprocess_ifp2(g, cls), cfg, workers=4)
        tol = max(1e-8, 10 * cfg.threshold * g.n)
        for vec in (v1, v2):
            assert np.max(np.abs(vec.values - dense) / dense) <= tol
        assert t2.final.push_ops_dangling == cls.dangling_edge_count
        assert t1.final.push_ops_dangling >= cls.dangling_edge_count


@pytest.mark.gpu
def test_engine_repeat_runs_agree(suite):
    # test_engines.py:177-184 (corpus seed 41)
    (g, _), = _corpus(suite, 41)
    cls = P.classify(g)
    base, _ = P.ifp1_run(g, cls, _cfg(), workers=8)
    for _ in range(4):
        vec, _ = P.ifp1_run(g, cls, _cfg(), workers=8)
        assert np.max(np.abs(vec.values - base.values)) <= 5 * XI


@pytest.mark.gpu
def test_sync_cycle_ratio_is_damping():
    # test_engines.py:187-194
    _, trace = P.sync_simulate(cycle2(), _cfg(), variant="ifp1")
    s = trace.samples
    for i in range(len(s) - 1):
        if s[i].carry_mass == 0.0 and s[i + 1].h_l1 > 0:
            assert s[i + 1].h_l1 / s[i].h_l1 == pytest.approx(0.85, abs=1e-12)
            assert s[i].alpha == 1.0


@pytest.mark.gpu
def test_sync_star_first_ratio():
    # test_engines.py:197-202
    _, trace = P.sync_simulate(star4(), _cfg(), variant="fp-full")
    s = trace.samples
    assert s[0].alpha == pytest.approx(0.25, abs=0)
    assert s[1].h_l1 / s[0].h_l1 == pytest.approx(0.85 * 0.25, abs=1e-12)


@pytest.mark.gpu
def test_sync_variants_match_oracle():
    # test_engines.py:205-210 (dense values of the three small graphs, exact)
    cases = [(chain3(), CHAIN3_EXACT), (fanin3(), np.array([1.0, 1.0, 2.7]) / 4.7), (cycle2(), np.array([0.5, 0.5]))]
    for g, dense in cases:
        for variant in ("ifp1", "ifp2", "fp-full"):
            vec, _ = P.sync_simulate(g, _cfg(), variant=variant)
            assert np.max(np.abs(vec.values - dense) / dense) <= 1e-8


@pytest.mark.gpu
def test_sync_bit_identical_across_runs(suite):
    # test_engines.py:213-219 (corpus seed 55)
    (g, _), = _corpus(suite, 55)
    a_vec, a_tr = P.sync_simulate(g, _cfg(), variant="ifp1")
    b_vec, b_tr = P.sync_simulate(g, _cfg(), variant="ifp1")
    assert np.array_equal(a_vec.values, b_vec.values)
    assert a_tr.column("h_l1") == b_tr.column("h_l1")
    assert a_tr.column("push_ops") == b_tr.column("push_ops")


@pytest.mark.gpu
def test_sync_trace_invariants(suite):
    # test_engines.py:222-230 (corpus seed 61)
    for g, _ in _corpus(suite, 61):
        for variant in ("ifp1", "fp-full"):
            _, trace = P.sync_simulate(g, _cfg(), variant=variant)
            h = trace.column("h_l1")
            assert all(b <= a + 1e-12 for a, b in zip(h, h[1:]))
            assert all(0.0 <= s.alpha <= 1.0 for s in trace.samples)
            assert all(s.work >= 0 for s in trace.samples)


@pytest.mark.gpu
def test_sync_decay_slope_bounded_by_damping(suite):
    # test_engines.py:233-244 (corpus seed 71)
    for g, _ in _corpus(suite, 71):
        _, trace = P.sync_simulate(g, _cfg(), variant="fp-full")
        s = [x for x in trace.samples if x.carry_mass <= 1e-9 * max(x.h_l1, 1e-300)]
        masses = [x.h_l1 for x in s if x.h_l1 > 0]
        if len(masses) < 4:
            continue
        slope = np.polyfit(np.arange(len(masses)), np.log(masses), 1)[0]
        assert slope <= np.log(0.85) + 1e-9


@pytest.mark.gpu
def test_sync_exact_decay_law(suite):
    # test_engines.py:247-254 (corpus seed 77)
    (g, _), = _corpus(suite, 77)
    _, trace = P.sync_simulate(g, _cfg(), variant="fp-full")
    s = trace.samples
    for i in range(len(s) - 1):
        if s[i].active_mass > 0:
            adjusted = (s[i + 1].h_l1 - s[i].carry_mass) / s[i].active_mass
            assert abs(adjusted - 0.85 * s[i].alpha) <= 1e-9


@pytest.mark.gpu
def test_sync_reserved_monotone(suite):
    # test_engines.py:257-267 (corpus seed 83)
    (g, _), = _corpus(suite, 83)
    last = {"r": np.zeros(g.n)}
    calls = []

    def watch(t, reserved, pushing):
        assert np.all(reserved >= last["r"] - 1e-15)
        assert np.all(pushing >= 0.0)
        last["r"] = reserved.copy()
        calls.append(t)

    P.sync_simulate(g, _cfg(), variant="ifp1", on_iteration=watch)
    assert calls


@pytest.mark.gpu
def test_sync_work_savings_vs_two_phase(suite):
    # test_engines.py:270-278 (corpus seed 91)
    for g, _ in _corpus(suite, 91):
        cls = P.classify(g)
        _, t1 = P.sync_simulate(g, _cfg(), variant="ifp1", cls=cls)
        _, t2 = P.sync_simulate(g, _cfg(), variant="ifp2", cls=cls)
        assert t2.final.push_ops_dangling == cls.dangling_edge_count
        assert t1.final.push_ops_dangling >= t2.final.push_ops_dangling


@pytest.mark.gpu
def test_sync_rejects_unknown_variant():
    # test_engines.py:281-283
    with pytest.raises(ValueError, match="variant"):
        P.sync_simulate(chain3(), _cfg(), variant="both")


@pytest.mark.gpu
def test_all_dangling_graph_is_uniform():
    # test_engines.py:286-295
    g = P.from_edges(3, [], [])
    cls = P.classify(g)
    vec, _ = P.ifp1_run(g, cls, _cfg(), workers=2)
    assert vec.values == pytest.approx([1 / 3] * 3, abs=1e-12)
    vec2, _ = P.ifp2_run(P.preprocess_ifp2(g, cls), _cfg(), workers=2)
    assert vec2.values == pytest.approx([1 / 3] * 3, abs=1e-12)


@pytest.mark.gpu
def test_trace_sampling_is_time_based():
    # engines.py:199-222: rows every sample_every seconds plus the final one;
    # 0 keeps every round, inf only the final sample
    g = chain3()
    cls = P.classify(g)
    _, every = P.ifp1_run(g, cls, _cfg(), sample_every=0.0)
    _, last = P.ifp1_run(g, cls, _cfg(), sample_every=float("inf"))
    _, auto = P.ifp1_run(g, cls, _cfg())
    assert len(every.samples) == every.meta["rounds"] + 1
    assert len(last.samples) == 1 and last.samples[0].push_ops == every.samples[-1].push_ops
    assert 1 <= len(auto.samples) <= len(every.samples)
    assert [s.t for s in every.samples] == list(range(len(every.samples)))


# ------------------------------------------------------------------ graph core (test_graph.py)

@pytest.mark.gpu
def test_load_edge_list_cases():
    # test_graph.py:20-68
    g = P.load_edge_list(b"0 1\n1 2\n")
    assert g.n == 3 and g.m == 2 and g.edge_set() == {(0, 1), (1, 2)}
    g = P.load_edge_list(b"# c\n5 9\n5 9\n")
    assert g.n == 2 and g.m == 1 and g.edge_set() == {(0, 1)}
    assert g.original_ids.tolist() == [5, 9] and g.raw_edge_count == 2
    g = P.load_edge_list(b"7 3\n3 1\n")
    assert g.original_ids.tolist() == [7, 3, 1] and g.edge_set() == {(0, 1), (1, 2)}
    assert P.load_edge_list(io.BytesIO(b"0\t1\n1\t0\n")).m == 2
    with pytest.raises(P.GraphFormatError, match="line 2"):
        P.load_edge_list(b"0 1\nx 2\n")
    with pytest.raises(P.GraphFormatError, match="line 3"):
        P.load_edge_list(b"# head\n0 1\n4\n")
    for empty in (b"", b"# only comments\n"):
        with pytest.raises(P.GraphFormatError, match="empty"):
            P.load_edge_list(empty)
    with pytest.raises(P.GraphFormatError):
        P.load_edge_list(b"0 1\n-2 1\n")
    g = P.load_edge_list(b"0 0\n0 1\n0 1\n")
    assert g.m == 2 and g.edge_set() == {(0, 0), (0, 1)} and g.out_degree[0] == 2


@pytest.mark.gpu
def test_from_edges_id_range_checked():
    # test_graph.py:71-75
    with pytest.raises(ValueError):
        P.from_edges(2, [0], [2])
    with pytest.raises(ValueError):
        P.from_edges(0, [], [])


@pytest.mark.gpu
def test_graph_invariants_on_corpus(suite):
    # test_graph.py:78-83 (handcrafted + random_corpus(20))
    for g in handcrafted() + [x for x, _ in _corpus(suite, 20260811, 20)]:
        g.validate()
        assert g.out_offsets[-1] == g.m
        assert np.array_equal(np.diff(g.out_offsets), g.out_degree)
        assert int(g.in_degree.sum()) == g.m


@pytest.mark.gpu
def test_classify_chain_cycle():
    # test_graph.py:86-101
    cls = P.classify(chain3())
    assert (cls.dangling.tolist(), cls.unreferenced.tolist()) == ([2], [0])
    assert (cls.weak_dangling.tolist(), cls.weak_unreferenced.tolist()) == ([1], [1])
    assert cls.dangling_edge_count == 1
    cls = P.classify(cycle2())
    assert cls.dangling.size == cls.unreferenced.size == cls.weak_dangling.size == cls.weak_unreferenced.size == 0
    assert cls.dangling_edge_count == 0


@pytest.mark.gpu
def test_classify_deterministic_and_weak_disjoint(suite):
    # test_graph.py:104-113 (random_corpus(15))
    for g, _ in _corpus(suite, 20260811, 15):
        a, b = P.classify(g), P.classify(g)
        for field in ("dangling", "unreferenced", "weak_dangling", "weak_unreferenced"):
            assert np.array_equal(getattr(a, field), getattr(b, field))
        assert not np.intersect1d(a.dangling, a.weak_dangling).size
        assert not np.intersect1d(a.unreferenced, a.weak_unreferenced).size
        assert 0 <= a.dangling_edge_count <= g.m


@pytest.mark.gpu
def test_stats_chain_and_isolated():
    # test_graph.py:116-125
    g = chain3()
    row = P.stats(g, P.classify(g))
    assert (row.n, row.m, row.dangling_vertices, row.dangling_edges) == (3, 2, 1, 1)
    assert row.avg_degree == pytest.approx(2 / 3, abs=1e-12)
    lone = single_vertex()
    row = P.stats(lone, P.classify(lone))
    assert (row.n, row.m, row.dangling_vertices, row.dangling_edges) == (1, 0, 1, 0)
    assert row.avg_degree == 0.0
    assert row.as_csv_row() == ["single", 1, 0, 1, 0, "0"]


@pytest.mark.gpu
def test_preprocess_small_graphs():
    # test_graph.py:128-153
    g = chain3()
    pg = P.preprocess_ifp2(g, P.classify(g))
    assert pg.live_targets[pg.live_offsets[0]:pg.live_offsets[1]].tolist() == [1]
    assert pg.live_degree.tolist() == [1, 0, 0]
    assert pg.dangling_ids.tolist() == [2] and pg.source_ids.tolist() == [1]
    assert pg.dangling_edge_count == 1
    g = cycle2()
    pg = P.preprocess_ifp2(g, P.classify(g))
    assert np.array_equal(pg.live_targets, g.out_targets) and np.array_equal(pg.live_offsets, g.out_offsets)
    assert pg.dangling_ids.size == 0 and pg.source_ids.size == 0
    g = fanin3()
    pg = P.preprocess_ifp2(g, P.classify(g))
    assert pg.live_targets.size == 0 and pg.source_ids.tolist() == [0, 1]


@pytest.mark.gpu
def test_preprocess_roundtrip_and_degree_split(suite):
    # test_graph.py:156-176 (handcrafted + random_corpus(20))
    for g in handcrafted() + [x for x, _ in _corpus(suite, 20260811, 20)]:
        cls = P.classify(g)
        pg = P.preprocess_ifp2(g, cls)
        dt = P.dangling_target_counts(g, cls)
        assert np.array_equal(pg.live_degree + dt, g.out_degree)
        live_src = np.repeat(np.arange(g.n), pg.live_degree)
        live_edges = set(zip(live_src.tolist(), pg.live_targets.tolist()))
        dang_edges = set()
        for i, v in enumerate(pg.dangling_ids.tolist()):
            for u in pg.source_ids[pg.source_offsets[i]:pg.source_offsets[i + 1]].tolist():
                dang_edges.add((u, v))
        assert live_edges | dang_edges == g.edge_set()
        assert len(live_edges) + len(dang_edges) == g.m
        assert pg.source_ids.size == cls.dangling_edge_count
        assert np.array_equal(pg.base.out_degree, g.out_degree)


# ------------------------------------------------------------------ power method (test_solvers.py)

@pytest.mark.gpu
def test_power_cases():
    # test_solvers.py:48-61, 80-84, 87-90
    g = chain3()
    vec, trace = P.power_method(g, P.SolverConfig(max_iterations=0))
    assert vec.values == pytest.approx([1 / 3] * 3, abs=0)
    assert trace.samples == []
    vec, _ = P.power_method(cycle2(), P.SolverConfig())
    assert vec.values == pytest.approx([0.5, 0.5], abs=1e-14)
    vec, _ = P.power_method(g, P.SolverConfig())
    assert np.max(np.abs(vec.values - CHAIN3_EXACT)) < 1e-12
    v1, _ = P.power_method(g, P.SolverConfig(), workers=1)
    v4, _ = P.power_method(g, P.SolverConfig(), workers=4)
    assert np.array_equal(v1.values, v4.values)
    _, trace = P.power_method(cycle2(), P.SolverConfig(max_iterations=210), tolerance=1e-6)
    assert len(trace.samples) < 210


@pytest.mark.gpu
def test_power_iterates_are_distributions(suite):
    # test_solvers.py:64-69 (corpus seed 5)
    (g, _), = _corpus(suite, 5)
    sums = []
    P.power_method(g, P.SolverConfig(max_iterations=50), on_iterate=lambda k, pi: sums.append(float(pi.sum())))
    assert sums and all(abs(s - 1.0) <= 1e-12 for s in sums)


@pytest.mark.gpu
def test_power_contraction(suite):
    # test_solvers.py:72-78 (corpus seed 3)
    for g, _ in _corpus(suite, 3):
        _, trace = P.power_method(g, P.SolverConfig(max_iterations=40))
        deltas = trace.column("h_l1")
        for a, b in zip(deltas, deltas[1:]):
            if a <= 1e-14:
                break
            assert b <= 0.85 * a + 1e-13


@pytest.mark.gpu
def test_reference_route_equivalence_small_corpus(suite):
    # test_solvers.py:180-192 (corpus seed 17): the power route and the push
    # engines against the reference's dense oracle
    for g, dense in _corpus(suite, 17):
        cfg = P.SolverConfig(threshold=1e-12)
        cls = P.classify(g)
        routes = [P.power_method(g, cfg)[0].values, P.ifp1_run(g, cls, cfg)[0].values,
                  P.ifp2_run(P.preprocess_ifp2(g, cls), cfg)[0].values]
        for values in routes:
            assert np.max(np.abs(values - dense) / dense) < 1e-8


@pytest.mark.gpu
def test_config_validation():
    # test_solvers.py:195-203, through the entry points that validate
    g = cycle2()
    with pytest.raises(ValueError, match="damping"):
        P.power_method(g, P.SolverConfig(damping=1.0))
    with pytest.raises(ValueError, match="threshold"):
        P.ifp1_run(g, P.classify(g), P.SolverConfig(threshold=0.0))
    with pytest.raises(ValueError, match="personalization"):
        P.power_method(g, P.SolverConfig(personalization=np.array([0.7, 0.7])))
    with pytest.raises(ValueError, match="personalization"):
        P.power_method(g, P.SolverConfig(personalization=np.array([1.0])))
