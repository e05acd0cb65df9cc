"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The golden fixtures were produced by running the real reference package
(tests/golden/make_golden.py).  Integer preprocessing and the synchronous
round state must match bit-for-bit; asynchronous engines within the
reference's own cross-backend bound (test_backends.py:36-56: 5*xi).
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import corpus_graph

XI = 1e-12
INT_KEYS = ("out_offsets", "out_targets", "in_offsets", "in_sources", "dangling", "unreferenced",
            "weak_dangling", "weak_unreferenced", "dtc", "live_offsets", "live_targets",
            "live_degree", "dangling_ids", "source_offsets", "source_ids")


def oracle_ints(g):
    cls = oracle.classify(g)
    pg = oracle.preprocess_ifp2(g, cls.dangling)
    return {
        "out_offsets": g.out_offsets, "out_targets": g.out_targets,
        "in_offsets": g.in_offsets, "in_sources": g.in_sources,
        "dangling": cls.dangling, "unreferenced": cls.unreferenced,
        "weak_dangling": cls.weak_dangling, "weak_unreferenced": cls.weak_unreferenced,
        "dtc": oracle.dangling_target_counts(g, cls.dangling),
        "live_offsets": pg.live_offsets, "live_targets": pg.live_targets,
        "live_degree": pg.live_degree, "dangling_ids": pg.dangling_ids,
        "source_offsets": pg.source_offsets, "source_ids": pg.source_ids,
    }, cls


def check_sync(gold, prefix, g, threads=0):
    for variant in ("ifp1", "ifp2", "fp-full"):
        key = f"{prefix}sync_{variant.replace('-', '_')}_"
        r = oracle.sync_simulate(g, variant, threshold=XI, threads=threads)
        rows = r.rows
        for col in ("converged", "work", "push_ops", "push_ops_dangling"):
            assert np.array_equal(rows[col], gold[key + col]), (key, col)
        for col in ("h_l1", "alpha", "active_mass", "carry_mass"):
            # fp sums: numpy pairwise vs sequential; carry = l1 - above cancels
            scale = max(1.0, float(gold[key + "h_l1"][0]))
            np.testing.assert_allclose(rows[col], gold[key + col], rtol=1e-12, atol=1e-14 * scale)
        assert r.iterations == int(gold[key + "iterations"])
        if key + "reserved_pre_settle" in gold:      # absent when no round ran
            assert np.array_equal(r.reserved_pre_settle, gold[key + "reserved_pre_settle"])
            assert np.array_equal(r.h_pre_settle, gold[key + "h_pre_settle"])
        if variant == "ifp1":
            assert np.array_equal(r.values, gold[key + "values"])
        else:
            np.testing.assert_allclose(r.values, gold[key + "values"], rtol=1e-13, atol=1e-16)


def test_corpus_integer_preprocessing_bit_exact(golden_corpus):
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        g = oracle.from_edges(n, src, dst)
        ints, cls = oracle_ints(g)
        for k in INT_KEYS:
            assert np.array_equal(ints[k], golden_corpus[f"g{i}_{k}"]), (i, k)
        assert cls.dangling_edge_count == int(golden_corpus[f"g{i}_m_d"])


@pytest.mark.parametrize("threads", [0, 3])
def test_corpus_sync_rounds_bit_exact(golden_corpus, threads):
    """threads=0: the sequential scatter restatement; threads=3: the threaded
    CSC pull form used at full size (C3-C5) -- same state, bit for bit."""
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        check_sync(golden_corpus, f"g{i}_", oracle.from_edges(n, src, dst), threads=threads)


def test_corpus_async_port_and_power(golden_corpus):
    for i in range(int(golden_corpus["count"])):
        n, src, dst = corpus_graph(golden_corpus, i)
        g = oracle.from_edges(n, src, dst)
        for algo in ("ifp1", "ifp2"):
            r = oracle.async_run(g, algo, threshold=XI, workers=4)
            ref = golden_corpus[f"g{i}_{algo}_values"]
            assert np.max(np.abs(r.values - ref)) <= 5 * XI * max(1, n / 10)
        r2 = oracle.async_run(g, "ifp2", threshold=XI, workers=2)
        assert r2.push_ops_dangling == int(golden_corpus[f"g{i}_ifp2_push_ops_dangling"])
        pw = oracle.power_method(g, iterations=210)
        np.testing.assert_allclose(pw.values, golden_corpus[f"g{i}_power_values"], rtol=0, atol=1e-14)
        np.testing.assert_allclose(pw.deltas, golden_corpus[f"g{i}_power_deltas"], rtol=1e-9, atol=1e-15)
        if f"g{i}_dense_values" in golden_corpus:
            np.testing.assert_allclose(oracle.dense_pagerank(g), golden_corpus[f"g{i}_dense_values"],
                                       rtol=1e-12, atol=0)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def test_c1_oracle_matches_reference(golden_c1):
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make("c1", seed=0)
    assert _sha(np.stack([src, dst])) == str(golden_c1["edges_sha256"])
    g = oracle.from_edges(n, src, dst)
    ints, cls = oracle_ints(g)
    for k in INT_KEYS:
        assert _sha(ints[k]) == str(golden_c1[f"{k}_sha256"]), k
    check_sync(golden_c1, "", g)
    check_sync(golden_c1, "", g, threads=4)
    r1 = oracle.async_run(g, "ifp1", threshold=XI, workers=4)
    assert np.abs(r1.values - golden_c1["ifp1_values"]).sum() <= 1e-9
    pw = oracle.power_method(g, iterations=210)
    np.testing.assert_allclose(pw.values, golden_c1["power_values"], rtol=1e-12, atol=0)


def test_synth42_oracle_matches_reference(golden_synth42):
    gold = golden_synth42
    g = oracle.from_edges(int(gold["n_in"]), gold["src"].astype(np.int64), gold["dst"].astype(np.int64))
    ints, _ = oracle_ints(g)
    for k in INT_KEYS:
        assert _sha(ints[k]) == str(gold[f"{k}_sha256"]), k
    check_sync(gold, "", g)
    check_sync(gold, "", g, threads=4)


@pytest.mark.skipif(not __import__("oracle.refdriver").refdriver.available(),
                    reason="oracle/_ref not built")
def test_reference_kernel_driver_matches_golden(golden_c1):
    from oracle import refdriver
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make("c1", seed=0)
    g = oracle.from_edges(n, src, dst)
    for algo in ("ifp1", "ifp2"):
        r = refdriver.run(g, algo, threshold=XI, workers=4)
        assert np.abs(r.values - golden_c1[f"{algo}_values"]).sum() <= 1e-9
    assert r.push_ops_dangling == int(golden_c1["ifp2_push_ops_dangling"])


def test_oracle_rmat_matches_synthetic():
    """orc_rmat (threaded C, used to bring C5's edge list to the oracle) is
    the repo's seeded R-MAT definition, self-loops dropped in sample order."""
    from paper_2302_03245_b200 import synthetic
    for scale, ef, seed, threads in ((12, 16, 0, 1), (14, 5, 7, 3), (16, 8, 3, 8)):
        n, s, d = synthetic.rmat_graph(scale, ef, seed=seed)
        n2, s2, d2 = oracle.rmat_graph_edges(scale, ef, seed=seed, threads=threads)
        assert n == n2 and np.array_equal(s, s2) and np.array_equal(d, d2)
