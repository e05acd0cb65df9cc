"""Generate golden fixtures by running the REAL reference package.

Run here (the container that has /root/reference), never on the GPU box:

    python tests/golden/make_golden.py [--ref-src /tmp/refpkg/src]

The reference is built from a scratch copy (``/root/reference`` is
read-only): ``cp -r /root/reference/pkg /tmp/refpkg && cd /tmp/refpkg &&
python setup.py build_ext --inplace``; this script does that when the copy
is missing.  Only the reference's *outputs* are written, into
tests/golden/*.npz: no reference source is copied into the repo.

Fixtures
  corpus.npz  handcrafted graphs (tests/corpus.py:16-41 in the reference)
              plus seeded random corpora (corpus.py:44-69, seeds used by the
              reference's own tests) -- full arrays: graph build, classify,
              IFP2 split, sync_simulate (ifp1/ifp2/fp-full) final state and
              trace, ifp1_run/ifp2_run vectors, power vectors, dense oracle.
  c1.npz      BASELINE config C1 (paper_2302_03245_b200.synthetic seed 0):
              sha256 digests of the integer arrays, full float vectors.
  synth42.npz the reference acceptance graph synth.generate(10_000, 100_000,
              0.2, seed=42) (test_acceptance.py:41-45): edges + outputs.
  edge_lists.npz  load_edge_list (graph.py:201-259) on edge-list texts: the
              cases of test_graph.py:20-68 plus tabs, CRLF, inline comments,
              blank lines, '+' signs, 43-bit ids, no trailing newline, a
              seeded 20k-edge list; and malformed texts with the exception
              class and message.  ``--only edge_lists`` regenerates just this.
  harness.npz the ERR harness (bench.py:90-329) on C1 and the acceptance
              graph: the 210-iteration reference vector, ERR reports of
              fixed estimates, _power_iterations_to_target hits, sweep_xi
              errors of the deterministic engines, compare_algorithms
              settings, and formatted CSV rows.  ``--only harness``.
  suite.npz   the seeded corpora of the reference's test_engines.py /
              test_graph.py / test_solvers.py (edges + dense oracle) and its
              partition_vertices outputs.  ``--only suite``.
  serialize.npz  write_ranking_csv (serialize.py:14-21) output bytes for
              reference vectors on edge-list graphs with sparse original ids,
              a uniform vector (all ties) and the C1 power vector.
              ``--only serialize``.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
XI = 1e-12


def ensure_reference(ref_src: str) -> None:
    if not os.path.isdir(ref_src):
        root = os.path.dirname(ref_src)
        shutil.copytree("/root/reference/pkg", root)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=root,
                       check=True, stdout=subprocess.DEVNULL)
    sys.path.insert(0, ref_src)
    sys.path.insert(0, "/root/reference/pkg/tests")   # read-only import of corpus.py


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def reference_outputs(P, g, prefix: str, out: dict, full_ints: bool, dense: bool) -> None:
    cls = P.classify(g)
    pg = P.preprocess_ifp2(g, cls)
    from pushrank.graph import dangling_target_counts
    dtc = dangling_target_counts(g, cls)
    ints = {
        "out_offsets": g.out_offsets, "out_targets": g.out_targets,
        "in_offsets": g.in_offsets, "in_sources": g.in_sources,
        "dangling": cls.dangling, "unreferenced": cls.unreferenced,
        "weak_dangling": cls.weak_dangling, "weak_unreferenced": cls.weak_unreferenced,
        "dtc": dtc, "live_offsets": pg.live_offsets, "live_targets": pg.live_targets,
        "live_degree": pg.live_degree, "dangling_ids": pg.dangling_ids,
        "source_offsets": pg.source_offsets, "source_ids": pg.source_ids,
    }
    for k, v in ints.items():
        if full_ints:
            out[f"{prefix}{k}"] = np.asarray(v, np.int64)
        else:
            out[f"{prefix}{k}_sha256"] = np.array(digest(v))
    out[f"{prefix}n"] = np.int64(g.n)
    out[f"{prefix}m"] = np.int64(g.m)
    out[f"{prefix}m_d"] = np.int64(cls.dangling_edge_count)
    cfg = P.SolverConfig(threshold=XI)
    for variant in ("ifp1", "ifp2", "fp-full"):
        last = {}

        def cb(t, reserved, pushing, last=last):
            last["r"] = reserved.copy()
            last["h"] = pushing.copy()

        subject = pg if variant == "ifp2" else g
        vec, tr = P.sync_simulate(subject, cfg, variant=variant, cls=cls, on_iteration=cb)
        key = f"{prefix}sync_{variant.replace('-', '_')}_"
        out[key + "values"] = vec.values
        if last:
            out[key + "reserved_pre_settle"] = last["r"]
            out[key + "h_pre_settle"] = last["h"]
        for col in ("h_l1", "converged", "alpha", "work", "push_ops", "push_ops_dangling",
                    "active_mass", "carry_mass"):
            out[key + col] = np.asarray(tr.column(col))
        out[key + "iterations"] = np.int64(tr.meta["iterations"])
    v1, t1 = P.ifp1_run(g, cls, cfg, workers=4, backend="c")
    v2, t2 = P.ifp2_run(pg, cfg, workers=4, backend="c")
    out[f"{prefix}ifp1_values"] = v1.values
    out[f"{prefix}ifp1_push_ops_dangling"] = np.int64(t1.final.push_ops_dangling)
    out[f"{prefix}ifp2_values"] = v2.values
    out[f"{prefix}ifp2_push_ops_dangling"] = np.int64(t2.final.push_ops_dangling)
    out[f"{prefix}ifp2_phase1_push_ops"] = np.int64(t2.samples[-2].push_ops)
    pv, ptr = P.power_method(g, P.SolverConfig(max_iterations=210))
    out[f"{prefix}power_values"] = pv.values
    out[f"{prefix}power_deltas"] = np.asarray(ptr.column("h_l1"))
    if dense:
        out[f"{prefix}dense_values"] = P.dense_oracle(g, P.SolverConfig()).values


def edge_list_texts() -> tuple[list[bytes], list[bytes]]:
    ok = [b"0 1\n1 2\n", b"# c\n5 9\n5 9\n", b"7 3\n3 1\n", b"0\t1\n1\t0\n",
          b"10 20\r\n20 30\r\n30 10\r\n", b"1 2 # note\n2 3\n", b"\n  4   5\n\n5 4\n   \n",
          b"9000000000000 1\n1 42\n42 9000000000000\n", b"0 0\n0 1\n0 1\n", b"+1 2\n2 +3\n",
          b"1 2\n2 3", b"3 3\n"]
    rng = np.random.default_rng(20261019)
    ids = rng.integers(0, 1 << 40, size=3000)
    e = rng.integers(0, ids.size, size=(20000, 2))
    lines = [f"{ids[a]} {ids[b]}" for a, b in e]
    for k in range(0, len(lines), 997):
        lines.insert(k, "# block")
    ok.append(("\n".join(lines) + "\n").encode())
    bad = [b"0 1\nx 2\n", b"# head\n0 1\n4\n", b"", b"# only comments\n", b"0 1\n-2 1\n", b"0 1 2\n",
           b"0 1\n1 2 3\n", b"5#c 6\n", b"1 99999999999999999999\n", b"0 1\n\xff 2\n"]
    return ok, bad


def edge_lists(P) -> None:
    ok, bad = edge_list_texts()
    out = {"n_ok": np.int64(len(ok)), "n_bad": np.int64(len(bad))}
    for i, t in enumerate(ok):
        g = P.load_edge_list(t)
        out[f"ok{i}_text"] = np.frombuffer(t, np.uint8)
        out[f"ok{i}_n"] = np.int64(g.n)
        out[f"ok{i}_raw"] = np.int64(g.raw_edge_count)
        for k in ("original_ids", "out_offsets", "out_targets", "in_offsets", "in_sources"):
            out[f"ok{i}_{k}"] = np.asarray(getattr(g, k), np.int64)
    for i, t in enumerate(bad):
        out[f"bad{i}_text"] = np.frombuffer(t, np.uint8)
        try:
            P.load_edge_list(t)
            raise SystemExit(f"bad case {i} did not raise")
        except Exception as exc:  # noqa: BLE001 -- record whatever the reference raises
            out[f"bad{i}_type"] = np.array(type(exc).__name__)
            out[f"bad{i}_msg"] = np.array(str(exc))
    np.savez_compressed(os.path.join(HERE, "edge_lists.npz"), **out)
    print("edge_lists.npz:", len(ok), "ok,", len(bad), "malformed")


def serialize_cases(P) -> None:
    import tempfile
    from pushrank.serialize import write_ranking_csv
    ok, _ = edge_list_texts()
    cases = []
    g = P.load_edge_list(ok[-1])                       # 3000 vertices, 40-bit ids
    cfg = P.SolverConfig(threshold=1e-12)
    cases.append((g, P.ifp1_run(g, P.classify(g), cfg)[0]))
    cases.append((g, P.PageRankVector(values=np.full(g.n, 1.0 / g.n), algorithm="uniform", damping=0.85)))
    g2 = P.load_edge_list(b"7 3\n3 1\n1 7\n9 9\n")
    cases.append((g2, P.power_method(g2, cfg)[0]))
    sys.path.insert(0, REPO)
    from paper_2302_03245_b200 import synthetic
    n, src, dst = synthetic.make("c1", seed=0)
    g3 = P.from_edges(n, src, dst)
    cases.append((g3, P.power_method(g3, P.SolverConfig(max_iterations=210))[0]))
    out = {"count": np.int64(len(cases))}
    for i, (graph, vec) in enumerate(cases):
        with tempfile.NamedTemporaryFile(suffix=".csv", delete=False) as fh:
            path = fh.name
        write_ranking_csv(vec, graph, path)
        with open(path, "rb") as fh:
            out[f"c{i}_csv"] = np.frombuffer(fh.read(), np.uint8)
        os.unlink(path)
        out[f"c{i}_values"] = np.asarray(vec.values, np.float64)
        out[f"c{i}_ids"] = np.asarray(graph.original_ids, np.int64)
    np.savez_compressed(os.path.join(HERE, "serialize.npz"), **out)
    print("serialize.npz:", len(cases), "cases")


HARNESS_TARGETS = (1e-2, 1e-3, 1e-4, 1e-6, 1e-8, 1e-10, 1e-13)
HARNESS_XIS = (1e-4, 1e-6, 1e-8)


def harness_cases(P) -> None:
    from pushrank import bench as B
    sys.path.insert(0, REPO)
    from paper_2302_03245_b200 import synthetic

    out = {}
    n, src, dst = synthetic.make("c1", seed=0)
    graphs = [("c1", P.from_edges(n, src, dst, name="c1"))]
    from pushrank import synth
    graphs.append(("synth42", synth.generate(10_000, 100_000, dangling_fraction=0.2, seed=42)))
    for name, g in graphs:
        pre = f"{name}_"
        cfg = P.SolverConfig()
        ref = B.reference_vector(g, cfg)
        out[pre + "ref"] = ref.values
        if name == "synth42":
            out[pre + "src"] = np.repeat(np.arange(g.n), np.diff(g.out_offsets)).astype(np.int32)
            out[pre + "dst"] = np.asarray(g.out_targets, np.int32)
            out[pre + "n"] = np.int64(g.n)
        # ERR of fixed estimates (the reference's own ifp1 / spi-20 vectors)
        cls = P.classify(g)
        est1, _ = P.ifp1_run(g, cls, cfg.with_threshold(1e-6), sample_every=float("inf"))
        est2, _ = P.power_method(g, P.SolverConfig(max_iterations=20))
        for k, est in (("ifp1", est1), ("spi20", est2)):
            r = B.max_relative_error(est, ref)
            out[pre + k + "_est"] = est.values
            out[pre + k + "_err"] = np.array([r.max_relative_error, r.l1_error])
            out[pre + k + "_worst"] = np.int64(r.worst_vertex)
        hits = [B._power_iterations_to_target(g, cfg, ref, t) for t in HARNESS_TARGETS]
        out[pre + "targets"] = np.array(HARNESS_TARGETS)
        out[pre + "hits"] = np.array([-1 if h is None else h for h in hits], np.int64)
        rows = B.sweep_xi(g, ["sync-ifp1", "sync-ifp2", "spi"], HARNESS_XIS, workers=1, reps=1)
        out[pre + "sweep_err"] = np.array([r.err for r in rows])
        out[pre + "sweep_samples"] = np.array([r.samples for r in rows], np.int64)
        cmp_rows = B.compare_algorithms(g, 1e-4, workers=2, reps=1,
                                        algorithms=("spi", "mpi", "sync-ifp1", "sync-ifp2"))
        out[pre + "compare_setting"] = np.array([r.setting for r in cmp_rows])
        out[pre + "compare_qualified"] = np.array([r.qualified for r in cmp_rows])
    row = B.SweepRow("d", "ifp2", 1e-6, 4, 1.2345678901234567e-05, 0.1234567, 0.5, 12, True)
    crow = B.ComparisonRow("d", "spi", 1e-4, 3.3e-05, 0.25, 0.125, "iterations=42", True, 2)
    urow = B.ComparisonRow("d", "ifp1", 1e-4, float("nan"), float("nan"), 0.1, "unreached", False)
    out["csv_rows"] = np.array([repr(row.as_csv_row()), repr(crow.as_csv_row()), repr(urow.as_csv_row())])
    out["slope"] = np.float64(B.fit_loglog_slope([1e-4, 1e-6, 1e-8], [0.01, 0.1, 0.9]))
    np.savez_compressed(os.path.join(HERE, "harness.npz"), **out)
    print("harness.npz")


# seeded corpora the reference's own test files draw (tests/test_engines.py,
# test_graph.py, test_solvers.py): (seed, count)
SUITE_CORPORA = ((23, 10), (31, 12), (41, 1), (55, 1), (61, 8), (71, 5), (77, 1), (83, 1), (91, 8),
                 (20260811, 20), (3, 8), (5, 1), (9, 1), (17, 10))


def suite_cases(P, corpus) -> None:
    """suite.npz: the graphs of the reference test suite's seeded corpora
    (edges), the reference's dense oracle on each, and the reference's
    partition_vertices outputs (engines.py:92-117) for the partition tests
    (test_engines.py:35-96), so tests/test_reference_suite.py restates those
    tests against this package without the reference installed."""
    out = {}
    for seed, count in SUITE_CORPORA:
        for i, g in enumerate(corpus.random_corpus(count, seed=seed)):
            pre = f"s{seed}_{i}_"
            out[pre + "n"] = np.int64(g.n)
            out[pre + "src"] = np.repeat(np.arange(g.n), np.diff(g.out_offsets)).astype(np.int64)
            out[pre + "dst"] = np.asarray(g.out_targets, np.int64)
            out[pre + "dense"] = P.dense_oracle(g, P.SolverConfig()).values
            if seed == 23:
                cls = P.classify(g)
                for strat in ("contiguous", "strided", "degree-balanced"):
                    part = P.partition_vertices(g, 3, strat, cls)
                    out[pre + f"part_{strat}_v"] = np.concatenate(part.worker_vertices)
                    out[pre + f"part_{strat}_vlen"] = np.array([x.size for x in part.worker_vertices], np.int64)
                    out[pre + f"part_{strat}_d"] = np.concatenate(part.worker_dangling)
                    out[pre + f"part_{strat}_dlen"] = np.array([x.size for x in part.worker_dangling], np.int64)
    rng = np.random.default_rng(4)
    for k in range(5):
        n = 400
        src = rng.integers(0, n, size=4000)
        dst = rng.integers(0, n, size=4000)
        g = P.from_edges(n, src, dst)
        part = P.partition_vertices(g, 4, "degree-balanced")
        out[f"bal{k}_src"] = src.astype(np.int64)
        out[f"bal{k}_dst"] = dst.astype(np.int64)
        out[f"bal{k}_v"] = np.concatenate(part.worker_vertices)
        out[f"bal{k}_vlen"] = np.array([x.size for x in part.worker_vertices], np.int64)
    np.savez_compressed(os.path.join(HERE, "suite.npz"), **out)
    print("suite.npz:", sum(c for _, c in SUITE_CORPORA), "graphs")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-src", default="/tmp/refpkg/src")
    ap.add_argument("--only", default=None, choices=["edge_lists", "serialize", "harness", "suite"])
    args = ap.parse_args()
    ensure_reference(args.ref_src)
    import pushrank as P
    import corpus
    from pushrank import synth

    if args.only == "edge_lists":
        edge_lists(P)
        return
    if args.only == "serialize":
        serialize_cases(P)
        return
    if args.only == "harness":
        harness_cases(P)
        return
    if args.only == "suite":
        suite_cases(P, corpus)
        return
    edge_lists(P)
    suite_cases(P, corpus)
    serialize_cases(P)
    harness_cases(P)

    sys.path.insert(0, REPO)
    from paper_2302_03245_b200 import synthetic

    meta = {"numpy": np.__version__, "reference_version": P.__version__, "xi": XI}

    # --- corpus (full arrays)
    graphs = corpus.handcrafted()
    for seed, count in ((20260811, 20), (31, 12), (101, 10), (55, 1), (83, 1)):
        graphs += corpus.random_corpus(count, seed=seed)
    out = {"count": np.int64(len(graphs))}
    for i, g in enumerate(graphs):
        src = np.repeat(np.arange(g.n), np.diff(g.out_offsets))
        out[f"g{i}_src"] = src.astype(np.int64)
        out[f"g{i}_dst"] = np.asarray(g.out_targets, np.int64)
        out[f"g{i}_name"] = np.array(g.name)
        reference_outputs(P, g, f"g{i}_", out, full_ints=True, dense=g.n <= 2000)
    out["meta"] = np.array(repr(meta))
    np.savez_compressed(os.path.join(HERE, "corpus.npz"), **out)
    print("corpus.npz:", len(graphs), "graphs")

    # --- C1 (digests + vectors)
    n, src, dst = synthetic.make("c1", seed=0)
    g = P.from_edges(n, src, dst, name="c1")
    out = {"edges_sha256": np.array(digest(np.stack([src, dst])))}
    reference_outputs(P, g, "", out, full_ints=False, dense=False)
    out["meta"] = np.array(repr(meta))
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)
    print("c1.npz: n", g.n, "m", g.m)

    # --- acceptance synthetic (edges stored)
    g = synth.generate(10_000, 100_000, dangling_fraction=0.2, seed=42)
    src = np.repeat(np.arange(g.n), np.diff(g.out_offsets))
    out = {"n_in": np.int64(g.n), "src": src.astype(np.int32),
           "dst": np.asarray(g.out_targets, np.int32)}
    reference_outputs(P, g, "", out, full_ints=False, dense=False)
    out["meta"] = np.array(repr(meta))
    np.savez_compressed(os.path.join(HERE, "synth42.npz"), **out)
    print("synth42.npz: n", g.n, "m", g.m)


if __name__ == "__main__":
    main()
