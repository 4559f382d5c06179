#!/usr/bin/env python
"""Benchmark of the BC hot path: BC TEPS = sources x edges / second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--gpu-mode source-sharded|graph-partitioned] [--workload ...]

Workload at N = 1: BASELINE.json configs[1] -- R-MAT scale-20, edge factor 16,
1024 sampled sources (``sorted(random.Random(0).sample(range(n), 1024))``, the
reference's sampling rule, engine.py:82-84), one B200.  A *step* is one full
BC computation over that source list.

``--gpus N`` with N > 1 and no torchrun environment re-launches this file
under ``python -m torch.distributed.run`` with N ranks (one per GPU, NCCL,
rendezvous on 127.0.0.1); under torchrun it joins the job it was launched in.
  source-sharded     graph replicated, every rank adds 1024 more sources (weak
                     scaling), ONE all-reduce of the BC vector, inside the timed
                     region
  graph-partitioned  one part per rank, all ranks work on the same sources
                     (strong scaling); ``--forward hybir`` = the paper's
                     border-matrix forward phase, ``bsp`` = level-synchronous

Printed JSON (one line, rank 0):
  value     whole-job TEPS, graph resident in HBM, timed with CUDA events on
            the stream the kernels run on, max over ranks
  e2e       same metric through the public call ``run_bc(g, cfg)`` with host
            buffers: CSR + sources host->device, BC vector device->host, inside
            the timed region (wall clock bracketed by device synchronisation)
  roofline  the dense level kernel: bytes of the BATCHED byte model (DESIGN.md
            section 5: adjacency word + mask probe once per group, one fp64 per
            (DAG arc, lane) gathered, per-vertex reads / writes) over the
            kernel's own CUDA-event time, against the measured HBM copy
            bandwidth; ``dram_frac`` = DRAM bytes of the committed ncu capture
            over the same time; ``per_source_model`` = SURVEY.md 8(d)'s
            unbatched figure for comparison
  cpu_baseline  the C/OpenMP oracle port of the reference's sequential Brandes
            on the box's host cores, a STRIDED source sample (every j-th source
            of the sorted list, so isolated sources are as frequent as in the
            full list); plus the pure-Python reference's own time on config 1
            as measured in the build container (profiles/)
  partitioned   (N = 1) the paper's partitioned algorithm on one GPU: config 1
            in hybir / bsp-baseline mode and road-like 2048^2 in 8 strips
  extra     (N = 1) the north-star target R-MAT scale-22 x 4096 sources, with
            an oracle parity sample
``--impl reference`` times the CPU port alone on the same strided sample rule
and prints the same line shape with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import random
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "bc_teps"
UNIT = "TEPS (sources*edges/s)"


def workload(name: str):
    from paper_2008_05718_b200 import generators as G
    if name == "rmat20":
        g = G.rmat(20, 16, 1)
        label = "R-MAT scale-20 edge-factor-16 (a,b,c)=(.57,.19,.19) seed 1, undirected unweighted"
    elif name == "rmat22":
        g = G.rmat(22, 16, 1)
        label = "R-MAT scale-22 edge-factor-16 (a,b,c)=(.57,.19,.19) seed 1, undirected unweighted"
    elif name == "rmat24":
        g = G.rmat(24, 16, 1)
        label = "R-MAT scale-24 edge-factor-16 (a,b,c)=(.57,.19,.19) seed 1, undirected unweighted"
    elif name == "rmat16":
        g = G.rmat(16, 16, 1)
        label = "R-MAT scale-16 edge-factor-16 (smoke-size)"
    elif name == "rmat12":
        g = G.rmat(12, 8, 1)
        label = "R-MAT scale-12 edge-factor-8 (BASELINE config 1)"
    elif name == "road2048":
        g = G.road_like(2048, 2048, keep=0.2, seed=1)
        label = "road-like 2048x2048 (random spanning tree of the grid + 20% of the other grid edges)"
    elif name == "road512":
        g = G.road_like(512, 512, keep=0.2, seed=1)
        label = "road-like 512x512 (smoke-size)"
    elif name == "er22":
        g = G.erdos_renyi(1 << 22, 1 << 26, 1)
        label = "Erdos-Renyi n=2^22, 2^26 random pairs (avg degree 32)"
    else:
        raise SystemExit("unknown workload %r" % name)
    return g, label


def pick_sources(n: int, k: int, seed: int = 0):
    return sorted(random.Random(seed).sample(range(n), min(k, n)))


def strided_sample(sources, k: int):
    """k sources spread evenly over the (sorted) list.  A prefix of the sorted list is biased on
    R-MAT graphs: low ids are the high-degree vertices and are almost never isolated."""
    k = max(1, min(k, len(sources)))
    idx = (np.arange(k, dtype=np.int64) * len(sources)) // k
    return [sources[i] for i in idx]


def isolated_fraction(g, sources) -> float:
    if not len(sources):
        return 0.0
    s = np.asarray(sources, dtype=np.int64)
    return float(np.mean(g.offsets[s + 1] == g.offsets[s]))


def measured_peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.proc = None
        self.path = None
        self.index = device_index

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
            os.unlink(self.path)
        except Exception:
            return out
        sm, reasons = [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                out["sm_max_mhz"] = float(r[2])
            except ValueError:
                continue
            for name, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if sm:
            # "under load" = the upper half of the samples (idle clocks sit low)
            sm.sort()
            out["sm_mhz"] = statistics.median(sm[len(sm) // 2:])
            out["samples"] = len(sm)
        out["reasons"] = sorted(reasons)
        return out


def ncu_traffic(workload_name: str):
    """DRAM bytes the dense level kernel moved per launch (mean over exactly the launches of one
    step), from the newest committed ncu `--set full` capture (profiles/r*_traffic.json, written
    by tools/summarize_profiles.py; null when no capture matches the workload)."""
    for rnd in ("r2", "r1"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd + "_traffic.json")) as fh:
                rec = json.load(fh)
            if rec.get(workload_name):
                return rec[workload_name], "profiles/%s_traffic.json" % rnd
        except Exception:
            continue
    return None, None


def per_source_bytes(st: dict, n: int):
    """SURVEY.md 8(d), every source counted on its own: forward 8*A_r + 16*T + 28*n_r,
    backward 8*A_r + 16*T + 44*n_r, initialisation 20*n per source."""
    fwd = 8 * st["arcs_reached"] + 16 * st["dag_arcs"] + 28 * st["reached"]
    bwd = 8 * st["arcs_reached"] + 16 * st["dag_arcs"] + 44 * st["reached"]
    init = 20 * n * st["sources"]
    return fwd, bwd, init


def python_reference_record():
    """The pure-Python reference's own timing on config 1, measured in the build container
    (the reference cannot travel to the GPU box): tools/time_python_reference.py."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_python_reference_c1.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


def cpu_sample(g, sources, seconds_target=15.0):
    """Time the oracle port on a bounded, strided sample of the source list."""
    import oracle as O
    threads = O.host_threads()
    k = min(len(sources), 2 * threads)
    sample = strided_sample(sources, k)
    t0 = time.perf_counter()
    O.brandes_bc(g, sample, threads=threads)
    dt = time.perf_counter() - t0
    # one refinement so the sample lands near the target duration
    if dt < seconds_target / 3 and k < len(sources):
        k2 = min(len(sources), int(k * min(64.0, seconds_target / max(dt, 1e-3))))
        k2 = max(threads, (k2 // threads) * threads)
        if k2 > k:
            k = k2
            sample = strided_sample(sources, k)
            t0 = time.perf_counter()
            O.brandes_bc(g, sample, threads=threads)
            dt = time.perf_counter() - t0
    rec = {"value": g.num_edges * k / dt, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": "%d of the %d sources (every %.1f-th of the sorted list), %.1f s on %d OpenMP threads "
                     "(oracle/brandes_oracle.c)" % (k, len(sources), len(sources) / k, dt, threads),
           "isolated_fraction_sample": isolated_fraction(g, sample),
           "isolated_fraction_all": isolated_fraction(g, sources)}
    return rec, k, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    g, label = workload(args.workload)
    sources = pick_sources(g.num_vertices, args.sources)
    import oracle as O
    threads = O.host_threads()
    # bounded sample per step: sized from one probe so W + K steps end within minutes
    probe, k, dt = cpu_sample(g, sources, seconds_target=8.0)
    per_source = dt / k
    budget = 150.0 / max(1, args.steps + args.warmup)
    k_step = int(min(len(sources), max(threads, budget / per_source)))
    k_step = max(threads, (k_step // threads) * threads)
    sample = strided_sample(sources, k_step)
    k_step = len(sample)
    for _ in range(args.warmup):
        O.brandes_bc(g, sample, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.brandes_bc(g, sample, threads=threads)
    dt = time.perf_counter() - t0
    value = g.num_edges * k_step * args.steps / dt
    iso_s, iso_a = isolated_fraction(g, sample), isolated_fraction(g, sources)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": label, "n": g.num_vertices, "m": g.num_edges,
                   "sources": len(sources), "sources_per_step": k_step,
                   "isolated_fraction_sample": iso_s, "isolated_fraction_all": iso_a},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "%d of the %d sources per step (every %.1f-th of the sorted list; isolated "
                                   "sources %.1f %% of the sample, %.1f %% of the list) on %d OpenMP threads; "
                                   "the reference is pure Python (1 core), this is its bit-identical C restatement"
                                   % (k_step, len(sources), len(sources) / k_step, 100 * iso_s, 100 * iso_a,
                                      threads),
                         "python_reference": python_reference_record()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------------
# the paper's partitioned algorithm on ONE GPU (k parts in one address space) and the
# north-star target: extra records of the N = 1 line
# ---------------------------------------------------------------------------------------------

def rel_err(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-9))) if len(a) else 0.0


def partitioned_block(budget_s: float = 120.0):
    """Config 1 in the reference's two partitioned modes and road-like 2048^2 in 8 strips, one GPU."""
    import oracle as O
    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200 import generators as G
    from paper_2008_05718_b200._capi import Engine, MODE_DIRECT, MODE_HYBIR
    t_start = time.perf_counter()
    out = {}
    g = G.rmat(12, 8, 1)
    srcs = list(range(g.num_vertices))
    obc, _ = O.brandes_bc(g, srcs)
    for mode in ("hybir", "bsp-baseline"):
        cfg = P.RunConfig(sources=srcs, mode=mode, num_partitions=2, per_source_reports=False)
        P.run_bc(g, cfg)
        res = P.run_bc(g, cfg)
        st = res.stats
        out["config1_" + mode] = {
            "workload": "R-MAT s12 ef8, all 4096 sources, 2 parts (reference partitioner)",
            "borders": [int(x) for x in res.borders.counts()], "ms": st["ms_total"], "ms_border": st["ms_border"],
            "iterations": int(st["iterations"]), "teps": g.num_edges * len(srcs) / max(st["ms_total"], 1e-9) * 1e3,
            "bc_rel_vs_oracle": rel_err(res.bc, obc), "parity": bool(rel_err(res.bc, obc) <= 1e-9)}
    if time.perf_counter() - t_start < budget_s:
        side, k, nsrc = 2048, 8, 512
        g = G.road_like(side, side, keep=0.2, seed=1)
        srcs = pick_sources(g.num_vertices, nsrc)
        part = P.strip_partition(side, side, k)
        with Engine(g) as e:
            e.set_option("groups", 16)
            e.set_option("reports", 0)
            e.set_partition(k, part.assignment)
            counts = [int(x) for x in e.border_counts(k)]
            t0 = time.perf_counter()
            e.run(srcs[:32], MODE_HYBIR)             # builds the border tables
            t_tables = time.perf_counter() - t0
            bc, st = e.run(srcs, MODE_HYBIR)
            bcd, std = e.run(srcs, MODE_DIRECT)
        out["road2048_hybir_8_strips"] = {
            "workload": "road-like 2048x2048, 512 sources, 8 row strips in one address space (config 3's algorithm)",
            "borders": counts, "ms": st["ms_total"], "ms_border": st["ms_border"], "ms_forward": st["ms_forward"],
            "ms_backward": st["ms_backward"], "iterations": int(st["iterations"]), "levels": int(st["max_levels"]),
            "tables_and_first_batch_s": t_tables, "teps": g.num_edges * nsrc / st["ms_total"] * 1e3,
            "direct_ms": std["ms_total"], "bc_rel_vs_direct": rel_err(bc, bcd),
            "parity": bool(rel_err(bc, bcd) <= 1e-9)}
    return out


def north_star_block(check: int = 8):
    """R-MAT scale-22 EF-16, 4096 sources on one GPU (the north-star target), parity on a strided sample."""
    import oracle as O
    from paper_2008_05718_b200._capi import Engine
    from paper_2008_05718_b200.engine import default_groups
    t0 = time.perf_counter()
    g, label = workload("rmat22")
    t_build = time.perf_counter() - t0
    srcs = pick_sources(g.num_vertices, 4096)
    sample = strided_sample(srcs, check)
    groups = default_groups(g, len(srcs))
    with Engine(g) as e:
        e.set_option("groups", groups)
        e.set_option("model_counters", 1)
        _, model = e.run(srcs)                      # untimed: warm-up + byte-model counters
        e.set_option("model_counters", 0)
        bc, st = e.run(srcs)
        bcs, _ = e.run(sample)
    obc, info = O.brandes_bc(g, sample)
    err = rel_err(bcs, obc)
    return {"workload": label, "n": g.num_vertices, "m": g.num_edges, "sources": len(srcs), "groups": groups,
            "ms": st["ms_total"], "teps": g.num_edges * len(srcs) / st["ms_total"] * 1e3,
            "levels": int(st["max_levels"]), "launches": int(st["launches"]), "graph_build_s": t_build,
            "level_kernel_ms": st["ms_level"], "level_model_bytes": int(model["level_model_bytes"]),
            "level_kernel_model_gbs": model["level_model_bytes"] / max(st["ms_level"], 1e-9) / 1e6,
            "parity_sources": len(sample), "bc_rel_vs_oracle": err, "parity": bool(err <= 1e-9),
            "oracle_sigma_max": info["sigma_max"]}


def weighted_block(side: int = 1024, n_sources: int = 128, wmax: int = 100000, check: int = 4):
    """General arc weights (csrc/bc_sssp.cuh): a road-like side x side grid with
    DIMACS-style weights, BC of n_sources sources on the GPU, the oracle's heap Dijkstra on a
    strided sample of them on one host core beside it, and BC parity on that sample."""
    import numpy as np
    import oracle as O
    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200 import generators as G
    from paper_2008_05718_b200._capi import Engine
    base = G.road_like(side, side, seed=1)
    src, dst = base.arc_src, base.arc_dst
    keep = src < dst
    w = np.random.default_rng(5).integers(1, wmax + 1, size=int(keep.sum()))
    g = P.from_edge_arrays(base.num_vertices, src[keep], dst[keep], w)
    srcs = pick_sources(g.num_vertices, n_sources)
    sample = strided_sample(srcs, check)
    with Engine(g) as e:
        e.set_option("groups", max(1, min(16, n_sources // 32)))
        e.run(srcs[:32])                            # untimed: allocation, page-in
        bc, st = e.run(srcs)
        bcs, _ = e.run(sample)
    t0 = time.perf_counter()
    obc, info = O.brandes_bc(g, sample, threads=1)
    t_cpu = time.perf_counter() - t0
    err = rel_err(bcs, obc)
    return {"workload": "road-like %dx%d grid, integer weights 1..%d (general-weight sweeps, mode direct)" % (side, side, wmax),
            "n": g.num_vertices, "m": g.num_edges, "sources": len(srcs), "ms": st["ms_total"],
            "teps": g.num_edges * len(srcs) / st["ms_total"] * 1e3, "dag_depth_arcs": int(st["max_levels"]),
            "launches": int(st["launches"]),
            "cpu_oracle_teps_1core": g.num_edges * len(sample) / t_cpu, "cpu_sample_sources": len(sample),
            "bc_rel_vs_oracle": err, "parity": bool(err <= 1e-9)}


# ---------------------------------------------------------------------------------------------
# graph-partitioned multi-GPU mode
# ---------------------------------------------------------------------------------------------

def run_partitioned(args):
    """--gpu-mode graph-partitioned: one part per rank, strong scaling (all ranks work on the same
    sources).  Forward phase per --forward: hybir = border matrices (two all-reduces per batch),
    bsp = one border exchange per level; the backward phase exchanges border values only at the
    levels the batch's cross-part dependencies name (planned once per batch, no host round trip
    per level)."""
    import torch
    import torch.distributed as dist

    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200.multigpu import init_process_group
    from paper_2008_05718_b200.partitioned import PartitionedRunner

    rank, world = init_process_group("nccl")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    g, label = workload(args.workload)
    n, m = g.num_vertices, g.num_edges
    sources = pick_sources(n, args.sources)
    if args.workload.startswith("road"):
        side = int(args.workload[4:])
        part = P.strip_partition(side, side, world)
    elif args.partitioner == "grow":
        part = P.grow_partition(g, world, seed=0)
    elif args.partitioner == "refine":
        part = P.refine_partition(g, P.grow_partition(g, world, seed=0))
    else:
        part = P.block_partition(g, world)
    # the border-matrix forward phase needs every part's b_p x b_p table on every rank: above the
    # budget (R-MAT: ~57 % of the vertices are borders) the run takes the level-synchronous forward
    # phase, as run_bc does
    forward = args.forward
    if forward == "hybir":
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            if P.choose_mode("hybir", P.identify_borders(g, part), 64e9) != "hybir":
                forward = "bsp"
    runner = PartitionedRunner(g, part, dev, args.groups or 4, forward)
    for _ in range(args.warmup):
        runner.run(sources)
    runner.reset_counters()
    sampler = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize(dev)
    if rank == 0:
        sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        bc = runner.run(sources)
    ev1.record()
    dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = sampler.stop() if rank == 0 else {}
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_total = float(ms.item())
    counters = runner.counters()
    # ---- end to end through the public call: host CSR in, host BC vector out on every rank
    runner.close()
    cfg = P.RunConfig(sources=sources, mode="hybir" if forward == "hybir" else "bsp-baseline",
                      num_gpus=world, gpu_mode="graph-partitioned", partition=part, device=local,
                      groups=args.groups or 4, per_source_reports=False)
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    res = P.run_bc(g, cfg)
    torch.cuda.synchronize(dev)
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    own = int(np.sum(np.asarray(part.assignment) == rank))
    rows = int(g.offsets[-1] * own / max(n, 1))
    level_bytes = torch.tensor([counters["level_model_bytes"], counters["ms_level"] * 1e6], dtype=torch.float64,
                               device=dev)
    dist.all_reduce(level_bytes, op=dist.ReduceOp.SUM)
    dist.barrier()
    dist.destroy_process_group()
    if rank != 0:
        return 0
    peak, peak_src = measured_peak_gbs()
    lb, lms = float(level_bytes[0].item()), float(level_bytes[1].item()) / 1e6
    achieved = lb / max(lms, 1e-9) / 1e6 if lms > 0 else None   # GB/s per GPU: sum of bytes over sum of kernel time
    cpu = None
    if not args.no_cpu:
        cpu, _, _ = cpu_sample(g, sources)
    steps_all = max(1, args.steps)
    line = {
        "metric": METRIC, "value": m * len(sources) * args.steps / (ms_total / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "n": n, "m": m, "sources": len(sources), "mode": "graph-partitioned",
                   "forward": forward, "forward_requested": args.forward, "partitioner": "strips" if args.workload.startswith("road") else args.partitioner,
                   "borders": runner.border_counts, "levels": runner.levels,
                   "state_vertices_per_rank": runner.local_n, "owned_vertices_rank0": own,
                   "forward_exchanges_per_step": counters["forward_exchanges"] / steps_all,
                   "backward_exchanges_per_step": counters["backward_exchanges"] / steps_all,
                   "backward_levels_per_step": counters["backward_levels"] / steps_all,
                   "exchanged_bytes_per_step": counters["exchanged_bytes"] / steps_all,
                   "l2": "per-batch state far above the 126 MB L2, no flush needed"},
        "e2e": {"value": m * len(sources) / float(e2e_s.item()), "unit": UNIT,
                "h2d_bytes_per_step": 8 * (own + 1) + 4 * rows + 8 * len(sources), "d2h_bytes_per_step": 8 * n,
                "steps": 1, "call": "run_bc(g, RunConfig(num_gpus=N, gpu_mode='graph-partitioned', ...))"},
        "gpu_launches": int(counters["launches"]),
        "clocks": clocks,
        "roofline": {"bound": "hbm", "kernel": "level_kernel<forward | backward> (per rank, own rows)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": None, "peak_source": peak_src,
                     "model": "batched byte model, DESIGN.md section 5; bytes and kernel time summed over ranks"},
        "cpu_baseline": cpu,
        "bc_sum": float(bc.sum().item()), "bc_sum_e2e": float(res.bc.sum()),
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------------
# the default line: batched Brandes on one GPU / source-sharded over N
# ---------------------------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2008_05718_b200 as P
    from paper_2008_05718_b200._capi import Engine, MODE_DIRECT
    from paper_2008_05718_b200.engine import default_groups

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # launched by torchrun (even with one rank): join the NCCL job, so the N = 1 line of a scaling
    # run goes through the same collectives as N > 1
    use_dist = world > 1 or ("RANK" in os.environ and "MASTER_ADDR" in os.environ)
    if use_dist:
        from paper_2008_05718_b200.multigpu import init_process_group
        init_process_group("nccl")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the engine has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    g, label = workload(args.workload)
    g.pin()                                    # e2e copies the CSR from pinned host memory
    n, m = g.num_vertices, g.num_edges
    all_sources = pick_sources(n, args.sources * world)
    mine = all_sources[rank::world]            # 1024 per rank: weak scaling
    groups = args.groups or default_groups(g, len(mine))

    eng = Engine(g, local)
    eng.set_option("groups", groups)
    if args.item_arcs:
        eng.set_option("item_arcs", args.item_arcs)
    if args.relabel >= 0:
        eng.set_option("relabel", args.relabel)
    bc_dev = torch.zeros(n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        bc_dev.zero_()
        st = eng.run_device(mine, bc_dev.data_ptr(), stream.cuda_stream, MODE_DIRECT)
        if use_dist:
            dist.all_reduce(bc_dev, op=dist.ReduceOp.SUM)
        return st

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        st = step()
    # one untimed step with the byte-model counters on (the forward pulls then count the arcs they
    # scan: one more atomic per work item, so the timed steps run without it)
    eng.set_option("model_counters", 1)
    model = step()
    eng.set_option("model_counters", 0)
    sampler = ClockSampler(local)
    barrier()
    if rank == 0:
        sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    keys = ("ms_forward", "ms_backward", "launches", "launches_forward", "launches_backward", "launches_level",
            "ms_level", "launches_level_timed")
    acc = {k: 0.0 for k in keys}
    ev0.record(stream)
    for _ in range(args.steps):
        st = step()
        for key in acc:
            acc[key] += st[key]
    ev1.record(stream)
    barrier()
    clocks = sampler.stop() if rank == 0 else {}
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_total = float(ms.item())
    value = m * len(all_sources) * args.steps / (ms_total / 1e3)

    # ---- end to end through the public API: host CSR in, host BC vector out
    eng.close()
    if use_dist:
        # the public multi-GPU call: every rank sweeps its shard of the sources, the BC vector is
        # all-reduced on the device and comes back to each host once
        from paper_2008_05718_b200.multigpu import run_bc_multi
        cfg = P.RunConfig(sources=all_sources, mode="direct", device=local, groups=groups, num_gpus=world,
                          gpu_mode="source-sharded", item_arcs=args.item_arcs or None, per_source_reports=False)
        e2e_call = lambda: run_bc_multi(g, cfg)
    else:
        cfg = P.RunConfig(sources=mine, mode="direct", device=local, groups=groups,
                          item_arcs=args.item_arcs or None, per_source_reports=False)
        e2e_call = lambda: P.run_bc(g, cfg)
    e2e_steps = max(1, min(args.steps, 3))
    e2e_call()                             # warm-up (allocator, page-in)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = e2e_call()
    barrier()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = m * len(all_sources) * e2e_steps / float(e2e_s.item())
    h2d = g.offsets.nbytes + g.col_idx.nbytes + 8 * len(mine)
    d2h = 8 * n + 64

    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    peak, peak_src = measured_peak_gbs()
    steps = args.steps
    # ---- roofline of the dominant kernel (dense level kernel + its hub pass): batched byte model
    # over the kernel's own CUDA-event time (bc_stats.ms_level)
    traffic, traffic_src = ncu_traffic(args.workload)
    lvl_ms = acc["ms_level"] / steps
    lvl_n = acc["launches_level_timed"] / steps
    lvl_avg = lvl_ms / max(lvl_n, 1)
    model_per_launch = model["level_model_bytes"] / max(model["launches_level"], 1)
    achieved = model_per_launch / max(lvl_avg, 1e-9) / 1e6
    fwd_b, bwd_b, init_b = per_source_bytes(st, n)
    roofline = {
        "bound": "hbm", "kernel": "level_kernel<forward | backward> + hub_kernel (dense pull levels; the child-driven tail levels of the backward sweep, bwd_child_init / bwd_push / bwd_child_apply, count as one level launch each)",
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
        "model": "batched byte model (DESIGN.md section 5): per launch, 8 B per arc scanned per group (col_idx word + "
                 "level-mask probe), 8 B per (DAG arc, lane) gathered, 8 B per (vertex, lane) value read or written, "
                 "4 B per dense mask word swept, 16 B of BC partial per backward entry, 8 B of row offsets per vertex",
        "bytes_per_launch": model_per_launch, "avg_launch_ms": lvl_avg, "launches_per_step": lvl_n,
        "ms_per_step": lvl_ms, "share_of_step": lvl_ms / (ms_total / steps),
        "components_per_step": {k: model[k] for k in ("level_scan_arcs", "level_pairs", "level_vertex_lanes",
                                                       "level_dense_words", "level_entries")},
        "dram_bytes_per_launch": traffic,
        "dram_achieved": (traffic / (lvl_avg / 1e3) / 1e9) if traffic and lvl_avg > 0 else None,
        "dram_frac": (traffic / (lvl_avg / 1e3) / 1e9 / peak) if traffic and lvl_avg > 0 else None,
        "dram_note": "DRAM bytes per launch from the committed ncu --set full capture over the live average launch "
                     "time: what the kernel really pulls from HBM (L2 serves the rest of the model's bytes)",
        "per_source_model": {
            "note": "SURVEY.md 8(d) counts every source on its own; 32 sources share each adjacency read here, "
                    "so this figure is not a bound for the batched kernel (it exceeds the peak)",
            "algorithmic_bytes_per_step": fwd_b + bwd_b + init_b,
            "achieved": (fwd_b + bwd_b + init_b) / (ms_total / steps / 1e3) / 1e9,
            "frac": (fwd_b + bwd_b + init_b) / (ms_total / steps / 1e3) / 1e9 / peak},
        "sweeps": {"forward_ms_per_step": acc["ms_forward"] / steps, "backward_ms_per_step": acc["ms_backward"] / steps,
                   "forward_launches_per_step": acc["launches_forward"] / steps,
                   "backward_launches_per_step": acc["launches_backward"] / steps},
    }
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu, _, _ = cpu_sample(g, all_sources)
        cpu["python_reference"] = python_reference_record()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "n": n, "m": m, "sources": len(all_sources),
                   "sources_per_gpu": len(mine), "mode": "source-sharded" if world > 1 else "single-gpu",
                   "groups": groups, "max_levels": st["max_levels"],
                   "isolated_fraction_sources": isolated_fraction(g, all_sources),
                   "renumbering": {-1: "engine default: vertices renumbered by descending degree once the handle has swept 2048 sources (warm-up)",
                                   0: "off", 1: "forced from the first step"}[args.relabel],
                   "l2": "per-batch state %.1f GB >> 126 MB L2, no flush needed"
                         % (groups * n * 560 / 1e9)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps,
                "call": ("run_bc(g, RunConfig(sources=..., mode='direct', num_gpus=N, gpu_mode='source-sharded'))"
                         if use_dist else "run_bc(g, RunConfig(sources=..., mode='direct'))")},
        "gpu_launches": int(acc["launches"]),
        "clocks": clocks,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "traversal": {k: st[k] for k in ("reached", "arcs_reached", "dag_arcs")},
    }
    if world == 1 and not args.no_extra and args.workload == "rmat20":
        from paper_2008_05718_b200._capi import release_cached_memory
        del g
        release_cached_memory()        # the extra records size their own state: start from an empty block cache
        try:
            line["partitioned"] = partitioned_block()
        except Exception as exc:   # an extra record must not cost the headline line
            line["partitioned"] = {"error": "%s: %s" % (type(exc).__name__, exc)}
        release_cached_memory()
        try:
            line["extra"] = {"north_star_rmat22_x4096": north_star_block()}
        except Exception as exc:
            line["extra"] = {"error": "%s: %s" % (type(exc).__name__, exc)}
        release_cached_memory()
        try:
            line["extra"]["weighted_road1024"] = weighted_block()
        except Exception as exc:
            line["extra"]["weighted_road1024"] = {"error": "%s: %s" % (type(exc).__name__, exc)}
    print(json.dumps(line))
    return 0


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args) -> int:
    """``python bench.py --gpus N`` outside torchrun: start N ranks of this file (one per GPU)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the log shows the transport (NVLS / P2P) NCCL picked
    log = os.path.join(tempfile.gettempdir(), "bench_nccl_%d.log" % os.getpid())
    env.setdefault("NCCL_DEBUG_FILE", log + ".%h.%p")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="rmat20")
    ap.add_argument("--sources", type=int, default=1024, help="sources per GPU (source-sharded) / in total (graph-partitioned)")
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--item-arcs", type=int, default=0)
    ap.add_argument("--relabel", type=int, default=-1, choices=(-1, 0, 1),
                    help="degree-descending renumbering of the resident graph: -1 = the engine's rule (skewed graphs, "
                         "once a handle has swept 2048 sources: from the fourth step on here), 0 = never, 1 = from the first step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the partitioned / north-star extra records")
    ap.add_argument("--gpu-mode", default="source-sharded", choices=("source-sharded", "graph-partitioned"))
    ap.add_argument("--forward", default="hybir", choices=("hybir", "bsp"),
                    help="forward phase of the graph-partitioned mode")
    ap.add_argument("--partitioner", default="block", choices=("block", "grow", "refine"))
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "RANK" not in os.environ:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:     # one rank per GPU: never several ranks on one device
            print("bench.py: --gpus %d but %d CUDA device(s) visible" % (args.gpus, have), file=sys.stderr)
            return 2
        return relaunch_under_torchrun(args)
    if args.gpu_mode == "graph-partitioned":
        return run_partitioned(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
