"""Benchmark: IFP2 (default) push rounds on BASELINE config C5 on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--algo ifp2|ifp1] [--mode auto|pull|push]

One "step" = one full solve of the hot path on the resident graph: every
push round until no vertex holds pending mass above xi = 1e-10 (the L1 <
1e-10 stopping rule), plus the IFP2 dangling settle and the
normalised output.  Metric: GTEPS = edges pushed (the reference's push_ops,
engines.py:155-157) / device seconds of the push phase.  Prints ONE JSON
line (rank 0).

--impl reference times the reference's own compiled CPU push kernel
(oracle/_ref, /root/reference/pkg/src/pushrank/_kernels.pyx) driven like
ifp2_run / ifp1_run with all host threads, on the same graph and metric.
At C5 (1.06 B edges) one CPU solve takes many minutes, so every reference
step is a bounded sample: the asynchronous push phase run for a fixed wall
budget from the initial state, GTEPS = pushes / elapsed (the line says so).
The C5 graph for the CPU legs is built on the GPU and exported as the
reference's int64 CSR/CSC (that build is bit-exact
against the oracle: profiles/r02_parity_c5.json).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

XI = 1e-10
DAMPING = 0.85


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--algo", default="ifp2", choices=["ifp1", "ifp2"])
    ap.add_argument("--mode", default="auto", choices=["auto", "pull", "push"])
    ap.add_argument("--cpu-sample-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=0.0,
                    help="seconds per bounded CPU sample (0: full solves below C5, 6 s at C5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-full", action="store_true",
                    help="also run one complete CPU solve (all host threads) at C5 for the time-to-solution and "
                         "pushes-per-solve comparison (minutes of CPU)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--push-switch", type=float, default=0.0,
                    help="AUTO policy: push when the next round's work < this fraction of (E_D+|D|) (0 = library default)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_desc(args, n, m):
    return {"workload": f"{args.config}: {__import__('paper_2302_03245_b200.synthetic', fromlist=['x']).CONFIGS[args.config]}",
            "algorithm": args.algo, "mode": args.mode, "n": int(n), "m": int(m), "seed": 0,
            "threshold": XI, "damping": DAMPING,
            "l2": "flushed between steps (256 MiB write)"}


def make_host_graph(config):
    from paper_2302_03245_b200 import synthetic
    return synthetic.make(config, seed=0)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                return
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_graph(g):
    """The reference's int64 CSR/CSC of a device graph, in page-locked host
    memory (the e2e leg uploads from it; the CPU legs read it)."""
    from types import SimpleNamespace
    from paper_2302_03245_b200 import _lib
    n, m = int(g.n), int(g.m)
    out = {"out_offsets": _lib.pinned_empty(n + 1, np.int64), "out_targets": _lib.pinned_empty(max(m, 1), np.int64),
           "in_offsets": _lib.pinned_empty(n + 1, np.int64), "in_sources": _lib.pinned_empty(max(m, 1), np.int64)}
    dev = g.dev
    dev.need_out_targets()
    _lib.check(_lib.load().pr_graph_export(dev.handle, *[_lib.ptr(out[k]) for k in
                                                         ("out_offsets", "out_targets", "in_offsets", "in_sources")]),
               "export")
    out["out_targets"] = out["out_targets"][:m]
    out["in_sources"] = out["in_sources"][:m]
    return SimpleNamespace(n=n, m=m, out_degree=np.diff(out["out_offsets"]), in_degree=np.diff(out["in_offsets"]),
                           **out)


def _ref_solve(g_host, algo, threads, pg, dt, budget):
    """One run of the reference's compiled worker loop (oracle/_ref) or, if
    it is missing, the oracle's pthread port; budget=None: a full solve."""
    import oracle
    from oracle import refdriver
    if refdriver.available():
        r = refdriver.run(g_host, algo, DAMPING, XI, workers=threads, pg=pg, budget_s=budget, dt=dt)
        return r.push_ops, r.wall_s, r.complete, "reference"
    t0 = time.perf_counter()
    r = oracle.async_run(g_host, algo, DAMPING, XI, workers=threads, pg=pg)
    return r.push_ops, time.perf_counter() - t0, True, "port"


def cpu_plan(g_host, config, budget, reps=3):
    """BASELINE.md section 3's CPU baseline on this host: the reference's
    ifp1/ifp2 push phase at workers = os.cpu_count() and 1, power iteration
    as spi (1 worker) and mpi (cpu_count workers), classify + preprocess_ifp2
    timed apart (bench.py:192-206's Table-2 style), median of ``reps`` as in
    _median_timed (bench.py:151-159).  With ``budget`` (C5) every engine run
    is a bounded sample (GTEPS over the first ``budget`` seconds of the
    solve) and the power method runs a few iterations (per-iteration time x
    210 is reported); the engines are the reference's compiled kernel
    (oracle/_ref), classify / preprocess / power are the oracle's C port."""
    import oracle
    cores = os.cpu_count() or 1
    plan = {"host": cpu_model(), "cpu_count": cores, "bounded_s": budget}
    t0 = time.perf_counter()
    cls = oracle.classify(g_host)
    t1 = time.perf_counter()
    pg = oracle.preprocess_ifp2(g_host, cls.dangling)
    t2 = time.perf_counter()
    dt = oracle.dangling_target_counts(g_host, cls.dangling)
    plan["classify_s"] = t1 - t0
    plan["preprocess_ifp2_s"] = t2 - t1
    plan["preprocess_kind"] = "port (oracle.c)"
    head = None
    for algo in ("ifp2", "ifp1"):
        for k in (cores, 1):
            runs = []
            for _ in range(1 if (budget or k == 1) else reps):
                runs.append(_ref_solve(g_host, algo, k, pg if algo == "ifp2" else None,
                                       dt if algo == "ifp1" else None,
                                       (budget if k > 1 else budget / 2) if budget else None))
            walls = [r[1] for r in runs]
            med = statistics.median(walls)
            ops = runs[-1][0]
            key = f"{algo}_k{k}"
            plan[key] = {"gteps": ops / med / 1e9, "wall_s": med, "push_ops": int(ops),
                         "complete_solve": bool(runs[-1][2]), "kind": runs[-1][3], "workers": k,
                         "samples": len(runs)}
            if head is None:
                head = plan[key]
    iters = 2 if budget else 210
    for name, k in (("spi", 1), ("mpi", cores)):
        t0 = time.perf_counter()
        pw = oracle.power_method(g_host, DAMPING, iterations=(1 if (budget and k == 1) else iters), workers=k)
        dt_s = time.perf_counter() - t0
        per_it = dt_s / max(pw.iterations, 1)
        plan[name] = {"iterations_run": int(pw.iterations), "s_per_iteration": per_it,
                      "s_for_210": per_it * 210, "workers": k, "kind": "port (oracle.c orc_power)"}
    return head, plan


def recorded_cpu_full(config):
    """The committed complete CPU solve of the same workload (bench.py
    --cpu-full on a B200 box's host, profiles/r02_bench_c5_cpufull.json): the
    default run only times a bounded CPU sample, so the pushes a full
    asynchronous CPU solve needs are quoted from that file, marked as
    recorded, when its config equals this line's."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_bench_c5_cpufull.json")
    try:
        with open(path) as f:
            rec = json.loads(f.read().strip().splitlines()[-1])
        same = all(rec["config"].get(k) == config.get(k) for k in ("workload", "algorithm", "n", "m", "threshold"))
        full = next(v for k, v in rec["cpu_baseline"]["plan"].items() if k.endswith("_full_solve"))
        if same and full["complete_solve"]:
            return {"push_ops": full["push_ops"], "wall_s": full["wall_s"], "kind": full["kind"],
                    "source": "profiles/r02_bench_c5_cpufull.json"}
    except Exception:
        pass
    return None


def run_reference(args):
    """--impl reference: the reference's compiled push kernel (oracle/_ref)
    on this host's cores, on the same graph, metric and config as our arm.
    Below C5 every step is a full solve; at C5 a bounded sample (see the
    module docstring)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import oracle.refdriver as rd
    threads = os.cpu_count() or 1
    build_note = "oracle.from_edges (C restatement of graph.py:133-177) on the host"
    t0 = time.perf_counter()
    if args.config == "c5":
        os.environ.setdefault("PUSHRANK_DEVICE", "0")
        import paper_2302_03245_b200 as P
        dev = P.graph.DeviceGraph.rmat(26, 16, seed=0)
        g = host_graph(P.graph.Graph(dev, raw_edge_count=16 << 26, name="c5"))
        del dev
        build_note = ("built on the GPU (pr_graph_rmat + from_edges kernels) and exported as the reference's "
                      "int64 CSR/CSC, per BASELINE.md section 3; bit-exact vs the oracle: profiles/r02_parity_c5.json")
    else:
        n, src, dst = make_host_graph(args.config)
        g = oracle.from_edges(n, src, dst)
    build_s = time.perf_counter() - t0
    dang = np.flatnonzero(g.out_degree == 0)
    pg = oracle.preprocess_ifp2(g, dang) if args.algo == "ifp2" else None
    dt = oracle.dangling_target_counts(g, dang) if args.algo == "ifp1" else None
    bounded = args.config == "c5"
    budget = None
    if bounded:
        # the whole --steps K --warmup W run within a few minutes
        budget = args.cpu_budget or max(3.0, min(12.0, 120.0 / max(args.steps, 1)))
    for _ in range(args.warmup):
        _ref_solve(g, args.algo, threads, pg, dt, 1.0 if bounded else None)
    walls, ops_list, kind, complete = [], [], "reference", True
    for _ in range(args.steps):
        ops, wall, comp, kind = _ref_solve(g, args.algo, threads, pg, dt, budget)
        walls.append(wall)
        ops_list.append(ops)
        complete = complete and comp
    total = sum(walls)
    value = sum(ops_list) / total / 1e9
    sample = (f"{args.steps} bounded samples of the {args.algo} push phase on {args.config}: each runs the reference "
              f"kernel with {threads} workers for {budget:.1f} s from the initial state (xi={XI}); GTEPS = pushes / "
              f"elapsed" if bounded else
              f"{args.steps} full {args.algo} solves of {args.config} (xi={XI}), mean")
    line = {"impl": "reference", "metric": "GTEPS", "value": value, "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(walls),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_desc(args, g.n, g.m),
            "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": threads, "kind": kind,
                             "sample": sample, "model": cpu_model()},
            "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "push_ops_per_step": int(statistics.median(ops_list)), "complete_solves": complete,
            "time_to_l1_ms": (1e3 * total / len(walls)) if complete else None,
            "graph_build": build_note, "graph_build_s": build_s,
            "driver": "oracle/refdriver.py: K Python threads run the compiled worker_loop with the GIL released "
                      "while the caller polls probe (engines.py:185-216); the final _sample is skipped"}
    print(json.dumps(line), flush=True)


def run_ours(args):
    rank, world, local = dist_env()
    os.environ.setdefault("PUSHRANK_DEVICE", str(local))
    import torch
    import paper_2302_03245_b200 as P
    from paper_2302_03245_b200 import _lib
    from paper_2302_03245_b200.graph import DeviceGraph

    # PUSHRANK_DIST_BACKEND=gloo (functional check of the N > 1 path on a
    # single-GPU box: host collectives, every rank on device 0); nccl otherwise
    backend = os.environ.get("PUSHRANK_DIST_BACKEND", "nccl")
    if world > 1 and backend == "gloo":
        local = local % max(torch.cuda.device_count(), 1)
        os.environ["PUSHRANK_DEVICE"] = str(local)
    # PUSHRANK_PARTITIONED=1 (under torchrun) runs the partitioned path even
    # at one rank: the cost of the partitioned rounds against the engine
    partitioned = world > 1 or os.environ.get("PUSHRANK_PARTITIONED", "0") == "1"
    if partitioned:
        import torch.distributed as dist
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    t0 = time.perf_counter()
    if args.config == "c5":
        # 1.07B R-MAT samples: generated, de-duplicated and built on the device
        dev0 = DeviceGraph.rmat(26, 16, seed=0)
        g = P.graph.Graph(dev0, raw_edge_count=16 << 26, name="c5")
    else:
        n, src, dst = make_host_graph(args.config)
        t0 = time.perf_counter()
        g = P.from_edges(n, src, dst, name=args.config)
    cls = P.classify(g)
    pg = P.preprocess_ifp2(g, cls)
    preprocess_s = time.perf_counter() - t0
    if partitioned:
        return run_partitioned_bench(args, g, rank, world, local, preprocess_s)
    dev = g.dev
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        flush.zero_()
        torch.cuda.synchronize()
        _, _, res, _, _ = dev.run(args.algo, args.mode, DAMPING, XI, 1_000_000, _lib.CONV_SCAN,
                                  push_switch=args.push_switch, row_cap=1)
        return res

    for _ in range(args.warmup):
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    results = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            results.append(step())
    torch.cuda.synchronize()
    dev_ms = [r.push_ms for r in results]
    loop_ms = [r.round_ms for r in results]
    ops = [r.push_ops for r in results]
    total_ms = sum(dev_ms)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * sum(ops) / (total_ms * 1e-3) / 1e9
    r0 = results[-1]
    # roofline over the round loop (k_pull dominant): algorithmic bytes / loop time
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # dominant kernel = k_pull: its algorithmic bytes over its own device time
    # (globaltimer first-block start .. last-block finalise, summed over the
    # pull rounds of the timed steps; CUDA events cannot sit inside the
    # conditional graph that runs the rounds)
    pull_ms = sum(r.pull_ms for r in results)
    pull_bytes = sum(r.pull_bytes for r in results)
    n_pull = sum(r.pull_rounds for r in results)
    achieved = pull_bytes / (pull_ms * 1e-3) / 1e9 if pull_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}_{args.algo}")
        except Exception:
            traffic = None
    # device-counted by the library (every solve kernel counts its own launch,
    # including unrolled graph slots that exit at once), over the timed steps
    launches = sum(r.launches for r in results)
    line = {"metric": "GTEPS", "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_desc(args, g.n, g.m),
            "time_to_l1_ms": statistics.median(dev_ms), "round_loop_ms": statistics.median(loop_ms),
            "rounds": int(r0.rounds), "pull_rounds": int(r0.pull_rounds), "push_rounds": int(r0.push_rounds),
            "push_ops_per_step": int(r0.push_ops), "preprocess_s": preprocess_s,
            "split_ms": {"pull_kernels": statistics.median(r.pull_ms for r in results),
                         "sparse_kernels": statistics.median(r.sparse_ms for r in results),
                         "loop_other": statistics.median(r.round_ms - r.pull_ms - r.sparse_ms for r in results),
                         "outside_loop": statistics.median(r.push_ms - r.round_ms for r in results)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_pull (algorithmic bytes 12*E_pushed + 40*V_active + 8*n_scan per round)",
                         "kernel_avg_us": 1e3 * pull_ms / max(n_pull, 1),
                         "bytes_per_launch": pull_bytes / max(n_pull, 1),
                         "kernel_share_of_step": pull_ms / max(sum(dev_ms), 1e-9),
                         "loop_achieved": r0.bytes_moved / (r0.round_ms * 1e-3) / 1e9,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650"},
            "gpu_launches": int(launches), "clocks": clocks.summary()}
    if args.algo == "ifp2":
        line["l1_crossing"] = l1_crossing(args, dev, r0)
    host = None
    if not args.no_e2e or (rank == 0 and world == 1 and not args.no_cpu_baseline):
        t0 = time.perf_counter()
        host = host_graph(g)
        line["host_export_s"] = time.perf_counter() - t0
    if not args.no_e2e:
        line["e2e"] = e2e_measure(args, host)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            budget = args.cpu_budget or (6.0 if args.config == "c5" else None)
            head, plan = cpu_plan(host, args.config, budget)
            line["cpu_baseline"] = {
                "value": head["gteps"], "unit": "GTEPS", "cores": head["workers"], "kind": head["kind"],
                "model": plan["host"],
                "sample": (f"{args.algo} push phase, reference kernel, {head['workers']} workers: "
                           + (f"bounded sample, first {budget:.0f} s of the solve from the initial state"
                              if budget else f"median of {head['samples']} full solves")),
                "plan": plan}
            # time-based context beside GTEPS (the engines push different edge counts)
            full = head if head["complete_solve"] else None
            if full is None and args.cpu_full:
                # refdriver builds the IFP2 split / dangling-target counts itself
                ops, wall, comp, kind = _ref_solve(host, args.algo, os.cpu_count() or 1, None, None, None)
                full = {"wall_s": wall, "push_ops": int(ops), "complete_solve": bool(comp), "kind": kind}
                plan[f"{args.algo}_k{os.cpu_count() or 1}_full_solve"] = full
            if full is not None and full["complete_solve"]:
                line["vs_cpu_time_to_solution"] = full["wall_s"] * 1e3 / line["time_to_l1_ms"]
            line["pushes_per_solve"] = {"ours": int(r0.push_ops),
                                        "cpu_reference": full["push_ops"] if full else None}
            if full is None:
                rec = recorded_cpu_full(line["config"])
                if rec:
                    line["pushes_per_solve"]["cpu_reference_recorded"] = rec
        except Exception as e:  # baseline failure must not hide the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "GTEPS", "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"failed: {e!r}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_partitioned_bench(args, g, rank, world, local, preprocess_s):
    """N > 1: vertex-range partitions, one per rank, NCCL all-gather of shares
    per round (paper_2302_03245_b200/distributed.py, csrc/part.cu).  Each rank
    holds the same global graph here (built on its own GPU) and keeps only its
    partition for the run.  Time = max over ranks of the solve, measured with
    CUDA-synchronised barriers on both sides."""
    import torch
    import torch.distributed as dist
    from paper_2302_03245_b200 import distributed as D
    # this rank's partition of the engines' run layout (hot sources at low
    # ids), built on its own GPU from its device graph: no host export of the
    # graph (pr_part_from_graph); the host copy of the rows is what the e2e
    # leg uploads every step
    part = D.partition_device(g, world, rank, args.algo, DAMPING, XI)
    host_part = part.to_host()
    comm = D.Comm(device=torch.device("cpu") if dist.get_backend() == "gloo" else torch.device("cuda", local))
    # the partition is uploaded once (inputs resident in HBM for `value`);
    # pr_part_init resets the round state of every solve.  Fast local step
    # (binned gather) with the rounds, all-gathers and statistics all-reduces
    # queued on the library stream (statistics read back every 8 rounds)
    step = D.CudaLocalStep(part, DAMPING, XI, args.algo, device=local, fast=True)
    # fused exchange (shares stored into every rank's replica by the round
    # kernel, peer memory over NVLink) unless PUSHRANK_FUSED=0 or the peer
    # mapping fails on any rank (then the NCCL all-gather form)
    want_fused = dist.get_backend() == "nccl" and os.environ.get("PUSHRANK_FUSED", "1") != "0"
    fused = want_fused and step.setup_fused(comm)

    def solve(s, host_values=False, fused=fused):
        vals, rows, info = D.run_partitioned_queued(s, comm, part, args.algo, DAMPING, XI, batch=16,
                                                    host_values=host_values, fused=fused)
        return vals, info

    for _ in range(args.warmup):
        solve(step)
    # device time per rank: CUDA events on the library stream, where the
    # rounds and their collectives are queued; max over ranks
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    lib_stream = step.stream
    info = None
    with ClockSampler(local) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(lib_stream)
        for _ in range(args.steps):
            vals, info = solve(step)
        ev1.record(lib_stream)
        torch.cuda.synchronize()
        dist.barrier()
    red_dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([ev0.elapsed_time(ev1) * 1e-3], dtype=torch.float64, device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_s = float(t.item())
    value = info["push_ops"] * args.steps / total_s / 1e9
    # e2e: partition upload + solve + owned values back, every step
    dist.barrier()
    t0 = time.perf_counter()
    e2e_fused = False
    for _ in range(2):
        # a fresh partition per step, replicas and peer mappings included
        # (cudaMalloc + IPC open, tens of ms): still far cheaper than the
        # all-gather form, whose every round moves P x slot shares per rank
        # (the slot is the largest rank's vertex count, 59 M at P = 8 since the
        # bounds stopped weighing vertices no round gathers into)
        s2 = D.CudaLocalStep(host_part, DAMPING, XI, args.algo, device=local, fast=True)
        e2e_fused = bool(want_fused and s2.setup_fused(comm))
        solve(s2, host_values=True, fused=e2e_fused)
        if e2e_fused:
            s2.close_fused(comm)
        del s2
    torch.cuda.synchronize()
    te = torch.tensor([(time.perf_counter() - t0) / 2], dtype=torch.float64, device=red_dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    # roofline of the partitioned round loop: the algorithmic bytes of the
    # rounds (12 B per pushed edge, 40 B per drained vertex,
    # 8 B per scanned vertex and round; the IFP2 settle's pushes counted as
    # edges) over the whole solve's device time, per GPU, against the HBM peak
    peak = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)) \
        if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    n_scan = float(g.n - int(g.dev.classify().dangling))
    bytes_solve = 12.0 * info["push_ops"] + 40.0 * info.get("drained", 0) + 8.0 * n_scan * (info["rounds"] + 1)
    achieved = bytes_solve * args.steps / total_s / world / 1e9
    if rank == 0:
        line = {"metric": "GTEPS", "value": value, "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(config_desc(args, g.n, g.m), parallelism=f"vertex-range x{world}"),
                "rounds": info["rounds"], "push_ops_per_step": info["push_ops"], "preprocess_s": preprocess_s,
                "e2e": {"value": info["push_ops"] / e2e_s / 1e9, "unit": "GTEPS",
                        # bytes pr_part_create copies: int64 offsets, int32 sources / degrees /
                        # row lengths / dangling-target counts, uint8 flags
                        "h2d_bytes_per_step": int(8 * (host_part.owned + 1) + 4 * host_part.in_sources.size
                                                  + 12 * host_part.owned + 2 * host_part.owned),
                        "d2h_bytes_per_step": int(8 * part.owned), "ms_per_step": 1e3 * e2e_s,
                        "path": "per step: partition upload (pr_part_create) + replicas and peer mappings + rounds ("
                                + ("fused" if e2e_fused else "all-gather") + " exchange) + owned values D2H"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": None,
                             "kernel": "partitioned round loop per GPU (k_part_pull + exchange + statistics), "
                                       "algorithmic bytes 12*E_pushed + 40*V_drained + 8*n_scan per round",
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
                # per queued round (rounds queued past termination launch too): one
                # k_part_pull per section (the last also reduces the statistics);
                # init (2) and settle/total (4)
                "gpu_launches": int((step.launches_per_round() * info.get("queued_rounds", info["rounds"]) + 6)
                                    * args.steps),
                "clocks": clocks.summary(),
                "exchange": ("fused: the round kernel stores each share into the replicas of the ranks that read "
                             "it (peer memory; sparse boundary exchange)" if fused
                             else "NCCL all-gather of shares per round"),
                "exchange_entries_per_round": {"sparse": step.exchange_entries(),
                                               "dense": int(part.owned) * world},
                "partition_build": "on each rank's GPU from its device graph's run layout (pr_part_from_graph)",
                "note": ("partitioned rounds queued on the device and graph-captured (statistics read back "
                         "every 16 rounds; rounds queued past termination skip their sweep); local step = binned dense-round gather (k_part_pull); "
                         "all-reduce of 9 statistics per round (the round barrier)")}
        print(json.dumps(line), flush=True)
    if fused:
        step.close_fused(comm)
    dist.destroy_process_group()


def l1_crossing(args, dev, res_timed):
    """the first round whose non-dangling residual
    L1_p = sum_{v non-dangling} h_v / n is below 1e-10, from one extra traced
    solve (untimed).  IFP2 keeps exactly 1.0 pending on every dangling vertex
    until the settle, so the non-dangling residual is h_l1 - n_dangling.
    `ms` is that row's device timestamp (globaltimer, from the solve start)
    plus the settle/normalise time of the timed solves."""
    from paper_2302_03245_b200 import _lib
    n_d = int(dev.preprocess_ifp2().dangling)
    _, rows, res, _, _ = dev.run(args.algo, args.mode, DAMPING, XI, 1_000_000, _lib.CONV_SCAN,
                                 push_switch=args.push_switch, row_cap=1 << 16)
    l1p = (rows["h_l1"] - n_d) / dev.n
    hit = np.nonzero(l1p < 1e-10)[0]
    if not hit.size:
        return None
    r = int(hit[0])
    return {"round": r, "rounds_total": int(res.rows) - 1, "l1_p": float(max(l1p[r], 0.0)),
            "ms": float(rows["wall_ms"][r] + (res_timed.push_ms - res_timed.round_ms))}


def e2e_measure(args, host):
    """Same metric through the public API from HOST buffers: each step uploads
    the reference-layout graph from page-locked int64 arrays (the upload
    copies what the fast engine needs -- in-adjacency + out_offsets -- and
    defers out_targets), builds the run layout and IFP2 split on the device,
    solves, and copies the vector back.  h2d_bytes_per_step counts the bytes
    actually copied."""
    from paper_2302_03245_b200.graph import device_graph
    import torch
    import paper_2302_03245_b200 as P
    from types import SimpleNamespace
    base = {k: getattr(host, k) for k in ("n", "m", "out_offsets", "out_targets", "in_offsets", "in_sources")}
    cfg = P.SolverConfig(threshold=XI)
    times, ops, h2d = [], 0, 0
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        obj = SimpleNamespace(**base)
        if args.algo == "ifp2":
            pg = P.preprocess_ifp2(obj, None)
            vec, tr = P.ifp2_run(pg, cfg, mode=args.mode, sample_every=float("inf"))
        else:
            vec, tr = P.ifp1_run(obj, None, cfg, mode=args.mode, sample_every=float("inf"))
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            ops = tr.final.push_ops
            h2d = device_graph(obj).h2d_bytes
        # release this step's graph before the next upload (a user would not
        # keep two copies alive); the freed pool blocks are then reused at the
        # same addresses, which also lets the next solve reuse its executable
        # graph
        if args.algo == "ifp2":
            del pg
        del obj, vec
    mean = sum(times) / len(times)
    return {"value": ops / mean / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(8 * host.n), "ms_per_step": 1e3 * mean,
            "path": f"{args.algo}_run() on a host-array graph (page-locked int64 CSR/CSC): upload + device "
                    f"preprocess + solve + D2H of the vector"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
